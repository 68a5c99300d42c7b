"""GPU parity of head-sliced migration (dyna_kv_migrate_heads; TP resharding,
SURVEY §8f NEXT-3, reading R14) against oracle.migrate_heads, bit for
bit on whole pools, plus a full-size TP-1 -> TP-4 Llama-3-8B reshard checked on
sampled rows and by the scatter/gather round trip."""
import itertools

import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from paper_2504_09285_b200 import dist as dd
from gpu_util import dev_table, pool_filled, pool_from_host

pytestmark = pytest.mark.gpu


ENGINES = [dk.DYNA_ENGINE_AUTO, dk.DYNA_ENGINE_VEC]   # AUTO = the TMA tile kernel where the geometry fits
ENGINE_IDS = ["tiles", "rows"]


def _heads_parity(gs, gd, n_tok, tr, lr, c, heads, hd0, seed=1, flags=0, piece=0, with_host=True, engine=0):
    ts, td = kvgen.table_pair(seed + 100, n_tok, gs, gd)
    hs, hd = kvgen.fill_bytes(seed, gs.pool_bytes), kvgen.fill_bytes(seed + 1, gd.pool_bytes)
    want = hd.copy()
    oracle.migrate_heads(hs, gs, ts, want, gd, td, tr, lr, heads, hd0)
    src, dst = pool_from_host(gs, hs), pool_from_host(gd, hd)
    st, dt = dev_table(src, ts, with_host), dev_table(dst, td, with_host)
    if not with_host:
        flags |= dk.DYNA_MIGRATE_UNCHECKED
    x = dk.dyna_kv_migrate_heads(st, dt, tr, lr, heads, hd0, c, 0, dk.opts(flags=flags, piece_bytes=piece,
                                                                            engine=engine))
    info = dk.dyna_kv_xfer_info(x)
    if engine == dk.DYNA_ENGINE_AUTO and heads[1] - heads[0] not in (0, gs.num_kv_heads):
        assert dk.dyna_kv_xfer_plan(x)["engine"] == dk.DYNA_ENGINE_TILES, "AUTO head slices should run as TMA tiles"
    dk.dyna_kv_wait(x)
    got = dst.tensor.cpu().numpy()
    assert np.array_equal(src.tensor.cpu().numpy(), hs), "source pool modified"
    if not np.array_equal(got, want):
        diff = np.flatnonzero(got != want)
        pytest.fail(f"{len(diff)} bytes differ; first at {diff[0]}")
    return src, dst, info


G8 = Geom(3, 8, 64, 2, 16, 40)      # 8 heads of 128 B: a TP-1 shard
G4 = Geom(3, 4, 64, 2, 16, 48)      # TP-2 shard
G2 = Geom(3, 2, 64, 2, 8, 96)       # TP-4 shard, other block size
G1 = Geom(3, 1, 64, 2, 32, 24)      # TP-8 shard


@pytest.mark.parametrize("gs,gd,heads,hd0", [
    (G8, G4, (0, 4), 0), (G8, G4, (4, 8), 0), (G8, G2, (2, 4), 0), (G8, G1, (7, 8), 0),
    (G4, G8, (0, 4), 4), (G2, G8, (0, 2), 6), (G1, G8, (0, 1), 3), (G4, G2, (1, 3), 0),
    (G2, G4, (0, 2), 1), (G8, G8, (3, 6), 1), (G8, G8, (0, 8), 0), (G4, G4, (2, 3), 2),
])
@pytest.mark.parametrize("c", [7, 16, 64, 500])
@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_heads_parity(gs, gd, heads, hd0, c, engine):
    _heads_parity(gs, gd, 500, (0, 451), (0, 3), c, heads, hd0, engine=engine)


@pytest.mark.parametrize("tr,lr", [((13, 400), (0, 3)), ((0, 1), (1, 2)), ((31, 33), (2, 3)), ((0, 500), (0, 3))])
@pytest.mark.parametrize("piece", [0, 256, 1024, 65536])
@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_heads_subranges_and_pieces(tr, lr, piece, engine):
    _heads_parity(G8, G2, 500, tr, lr, 48, (5, 7), 0, piece=piece, engine=engine)


@pytest.mark.parametrize("bss,bsd", [(16, 32), (32, 16), (16, 24), (8, 16)])
@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_heads_reblocking(bss, bsd, engine):
    gs = G8.with_(block_size=bss, num_blocks=40 * 16 // bss)
    gd = G2.with_(block_size=bsd, num_blocks=96 * 8 // bsd + 8)
    _heads_parity(gs, gd, 500, (3, 467), (0, 3), 40, (4, 6), 0, engine=engine)


@pytest.mark.parametrize("L,lr", [(5, (0, 5)), (5, (1, 4)), (7, (2, 7)), (40, (0, 40)), (40, (3, 38))])
@pytest.mark.parametrize("slice_heads", [1, 3, 4])
@pytest.mark.parametrize("d", [64, 8], ids=["128B-heads", "16B-heads"])
def test_tiles_slab_groups(L, lr, slice_heads, d):
    """The tile kernel's boxes span lkb (layer, K|V) slabs, lkb a divisor of 2*lm: odd layer counts,
    layer sub-ranges, prime slab counts (2*lm = 6, 10, 70) and 1..4-head slices (box bytes from 2 KiB to
    48 KiB before the slab factor) against the oracle."""
    gs = Geom(L, 8, d, 2, 16, 24)
    gd = Geom(L, 4, d, 2, 16, 30)
    _heads_parity(gs, gd, 300, (5, 290), lr, 64, (1, 1 + slice_heads), 4 - slice_heads, seed=L + slice_heads)


@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_heads_signal_flags_and_host_tables(engine):
    src, dst, (epoch, nck, sender, first) = _heads_parity(G8, G4, 500, (0, 451), (0, 3), 64, (4, 8), 0,
                                                          flags=dk.DYNA_MIGRATE_SIGNAL, with_host=False,
                                                          engine=engine)
    assert nck == 8 and epoch > 0
    fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(dst.handle, sender, first, nck, fl.data_ptr(), 0)
    torch.cuda.synchronize()
    assert (fl.numpy() == epoch).all()
    ts, td = kvgen.table_pair(101, 500, G8, G4)
    st = dk.table(src, None, ts)              # host-resident tables (the library uploads them)
    dt = dk.table(dst, None, td)
    hd = dst.tensor.cpu().numpy()
    want = hd.copy()
    oracle.migrate_heads(src.tensor.cpu().numpy(), G8, ts, want, G4, td, (100, 300), (1, 3), (0, 2), 2)
    dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(st, dt, (100, 300), (1, 3), (0, 2), 2, 32, 0, dk.opts(engine=engine)))
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_heads_empty_and_errors():
    src, dst = pool_filled(G8, 1), pool_filled(G4, 2)
    ts, td = kvgen.table_pair(1, 200, G8, G4)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    for args in [((0, 0), (0, 3), (0, 4), 0), ((0, 100), (0, 3), (2, 2), 0), ((0, 100), (1, 1), (0, 4), 0)]:
        dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(st, dt, args[0], args[1], args[2], args[3], 32, 0))
    torch.cuda.synchronize()
    before = dst.tensor.clone()
    for heads, hd0 in [((0, 5), 0), ((3, 9), 0), ((0, 2), 3), ((0, 1), -1), ((2, 1), 0)]:
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_migrate_heads(st, dt, (0, 100), (0, 3), heads, hd0, 32, 0)
        assert e.value.status == dk.DYNA_ERANGE, (heads, hd0)
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_migrate_heads(st, dt, (0, 100), (0, 3), (0, 2), 0, 32, 0, dk.opts(variant=dk.DYNA_VARIANT_STAGED))
    assert e.value.status == dk.DYNA_ENOTSUP
    gw = Geom(3, 20, 64, 2, 16, 48)          # 2304-B slices: more than one 2-KiB box row, not a multiple of it
    wide_s, wide_d = pool_filled(gw, 4), pool_filled(gw, 5)
    tw = kvgen.table_pair(6, 200, gw, gw)
    with pytest.raises(dk.DynaKVError) as e:  # the BULK (tile) engine refuses a slice no tensor map can describe
        dk.dyna_kv_migrate_heads(dev_table(wide_s, tw[0]), dev_table(wide_d, tw[1]), (0, 100), (0, 3), (0, 18), 1, 32,
                                 0, dk.opts(engine=dk.DYNA_ENGINE_BULK))
    assert e.value.status == dk.DYNA_ENOTSUP
    other = pool_filled(Geom(2, 4, 64, 2, 16, 48), 3)
    with pytest.raises(dk.DynaKVError) as e:               # L differs
        dk.dyna_kv_migrate_heads(st, dev_table(other, td), (0, 100), (0, 2), (0, 2), 0, 32, 0)
    assert e.value.status == dk.DYNA_EGEOM
    torch.cuda.synchronize()
    assert torch.equal(dst.tensor, before)


@pytest.mark.parametrize("tp_s,tp_d", [(1, 4), (4, 1), (2, 4), (4, 2), (2, 8)])
@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_tp_reshard_round_trip_full_llama3_rows(tp_s, tp_d, engine):
    """Llama-3-8B rows (8 KV heads, d128, bf16): a request's KV sharded over tp_s source ranks is
    resharded onto tp_d destination ranks with dd.tp_reshard_plan (one dyna_kv_migrate_heads per
    overlapping rank pair, all on one GPU here), then gathered back into a TP-1 pool: the result
    equals one plain migration (oracle), byte for byte."""
    H, L, s = 8, 32, 1000
    g1 = kvgen.LLAMA3_8B.with_(num_blocks=80)
    gs = g1.with_(num_kv_heads=H // tp_s)
    gd = g1.with_(num_kv_heads=H // tp_d, block_size=32, num_blocks=40)
    full_s = pool_filled(g1, 11)
    t1s, _ = kvgen.table_pair(12, s, g1, g1)
    src_pools = [pool_filled(gs, 20 + r) for r in range(tp_s)]
    src_tabs = [kvgen.table_pair(30 + r, s, gs, gs)[1] for r in range(tp_s)]
    dst_pools = [pool_filled(gd, 40 + r) for r in range(tp_d)]
    dst_tabs = [kvgen.table_pair(50 + r, s, gd, gd)[1] for r in range(tp_d)]
    keep = []
    for r in range(tp_s):                    # build the TP-tp_s source shards from the TP-1 pool
        a = (dev_table(full_s, t1s), dev_table(src_pools[r], src_tabs[r]))
        keep.append(a)
        dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(*a, (0, s), (0, L), dd.tp_heads(H, tp_s, r), 0, 256, 0))
    xs = []
    for a, b, heads, hd0 in dd.tp_reshard_plan(H, tp_s, tp_d):     # the reshard under test
        t = (dev_table(src_pools[a], src_tabs[a]), dev_table(dst_pools[b], dst_tabs[b]))
        keep.append(t)
        xs.append(dk.dyna_kv_migrate_heads(*t, (0, s), (0, L), heads, hd0, 256, 0, dk.opts(engine=engine)))
    for x in xs:
        dk.dyna_kv_wait(x)
    back = pool_filled(g1, 60)
    _, t1d = kvgen.table_pair(61, s, g1, g1)
    for b in range(tp_d):
        t = (dev_table(dst_pools[b], dst_tabs[b]), dev_table(back, t1d))
        keep.append(t)
        h0, h1 = dd.tp_heads(H, tp_d, b)
        dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(*t, (0, s), (0, L), (0, h1 - h0), h0, 256, 0))
    torch.cuda.synchronize()
    want = kvgen.fill_bytes(60, g1.pool_bytes)
    oracle.migrate(full_s.tensor.cpu().numpy(), g1, t1s, want, g1, t1d, (0, s))
    assert np.array_equal(back.tensor.cpu().numpy(), want)


def test_full_size_qwen72b_tp4_to_tp8_sampled():
    """BASELINE.json configs[4] geometry (Qwen2-72B: 80 layers, 8 KV heads, d128, bf16, block 16,
    NB 6144 per pool) resharded from a TP-4 rank (2 heads) onto two TP-8 ranks (1 head each):
    sampled rows against the oracle's offsets (kvgen bytes), every row by a property check
    (destination head slice == source head slice through both tables), heads of other rows
    untouched."""
    H = 8
    gs = kvgen.QWEN2_72B.with_(num_kv_heads=2)
    gd = kvgen.QWEN2_72B.with_(num_kv_heads=1)
    s = 4096                                        # one 4096-token prompt (the 4' target shape)
    src = pool_filled(gs, 300)
    ts = kvgen.table_pair(301, s, gs, gs)[0]
    plan = [e for e in dd.tp_reshard_plan(H, 4, 8) if e[0] == 1]
    assert [(b, heads, hd0) for _, b, heads, hd0 in plan] == [(2, (0, 1), 0), (3, (1, 2), 0)]
    rng = np.random.default_rng(7)
    st = dev_table(src, ts)
    for _, b, heads, hd0 in plan:
        dst = pool_filled(gd, 310 + b)
        td = kvgen.table_pair(320 + b, s, gd, gd)[1]
        dt = dev_table(dst, td)
        dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(st, dt, (0, s), (0, 80), heads, hd0, 1024, 0))
        torch.cuda.synchronize()
        he = gs.head_dim * gs.elem_bytes
        bad = 0
        for _ in range(1500):                       # sampled: the oracle's offsets, kvgen's bytes
            l, kv, t = int(rng.integers(0, 80)), int(rng.integers(0, 2)), int(rng.integers(0, s))
            so = oracle.logical_off(gs, ts, l, kv, t, heads[0], 0)
            do = oracle.logical_off(gd, td, l, kv, t, hd0, 0)
            want = kvgen.bytes_at(300, so, (heads[1] - heads[0]) * he)
            bad += int(not np.array_equal(dst.tensor[do:do + len(want)].cpu().numpy(), want))
        assert bad == 0
        S = src.tensor.view(80, 2, gs.num_blocks, 16, 2, he)     # every row, property form
        D = dst.tensor.view(80, 2, gd.num_blocks, 16, 1, he)
        Ts = torch.as_tensor(ts.astype(np.int64), device="cuda")
        Td = torch.as_tensor(td.astype(np.int64), device="cuda")
        for a in range(0, s, 2048):
            t = torch.arange(a, min(a + 2048, s), device="cuda")
            assert torch.equal(D[:, :, Td[t // 16], t % 16, hd0:hd0 + 1], S[:, :, Ts[t // 16], t % 16, heads[0]:heads[1]])
        mask = torch.zeros(80, 2, gd.num_blocks, 16, dtype=torch.bool, device="cuda")
        t = torch.arange(0, s, device="cuda")
        mask[:, :, Td[t // 16], t % 16] = True
        ref = torch.empty_like(dst.tensor)
        dk.dyna_kv_debug_fill(ref.data_ptr(), ref.numel(), 310 + b, 0, torch.cuda.current_stream().cuda_stream)
        assert torch.equal(D[~mask], ref.view_as(D)[~mask])
        del dst, ref, D
        torch.cuda.empty_cache()


# ---------------------------------------------------------------- dyna_kv_reshard: the whole plan, one launch
@pytest.mark.parametrize("tp_s,tp_d", [(1, 8), (8, 1), (2, 4), (4, 2), (2, 8), (8, 2), (1, 2), (4, 4)])
@pytest.mark.parametrize("signal", [False, True])
@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_reshard_one_launch_matches_oracle(tp_s, tp_d, signal, engine):
    """Every rank pair of dd.tp_reshard_plan in ONE dyna_kv_reshard launch (interleaved items):
    every destination shard equals the oracle applying oracle.migrate_heads per pair; with
    signalling every entry's flags reach its own epoch."""
    H, L, s, c = 8, 3, 700, 128
    g = Geom(L, H, 64, 2, 16, 60)
    gs = g.with_(num_kv_heads=H // tp_s)
    gd = g.with_(num_kv_heads=H // tp_d, block_size=8, num_blocks=120)
    hs = [kvgen.fill_bytes(200 + r, gs.pool_bytes) for r in range(tp_s)]
    hd = [kvgen.fill_bytes(300 + r, gd.pool_bytes) for r in range(tp_d)]
    ts = [kvgen.table_pair(10 + r, s, gs, gs)[0] for r in range(tp_s)]
    td = [kvgen.table_pair(20 + r, s, gd, gd)[1] for r in range(tp_d)]
    plan = dd.tp_reshard_plan(H, tp_s, tp_d)
    want = [h.copy() for h in hd]
    for a, b, heads, hd0 in plan:
        oracle.migrate_heads(hs[a], gs, ts[a], want[b], gd, td[b], (0, s), (0, L), heads, hd0)
    src = [pool_from_host(gs, h, instance=a) for a, h in enumerate(hs)]
    dst = [pool_from_host(gd, h) for h in hd]
    st = [dev_table(p, t) for p, t in zip(src, ts)]
    dt = [dev_table(p, t) for p, t in zip(dst, td)]
    migs = [(st[a], dt[b], heads, hd0) for a, b, heads, hd0 in plan]
    n0 = dk.dyna_kv_launch_count()
    x = dk.dyna_kv_reshard(migs, (0, s), (0, L), c, 0, dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0,
                                                                engine=engine))
    if engine == dk.DYNA_ENGINE_AUTO and tp_s != tp_d:
        assert dk.dyna_kv_xfer_plan(x)["engine"] == dk.DYNA_ENGINE_TILES
    infos = [dk.dyna_kv_batch_info(x, i) for i in range(len(migs))] if signal else []
    dk.dyna_kv_wait(x)
    assert dk.dyna_kv_launch_count() - n0 == 1
    for b in range(tp_d):
        assert np.array_equal(dst[b].tensor.cpu().numpy(), want[b]), b
    for a in range(tp_s):
        assert np.array_equal(src[a].tensor.cpu().numpy(), hs[a])
    for (a, b, _, _), (epoch, first, nck, sender) in zip(plan, infos):
        fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
        dk.dyna_kv_copy_flags(dst[b].handle, sender, first, nck, fl.data_ptr(), 0)
        torch.cuda.synchronize()
        assert sender == a and nck == -(-s // c) and (fl.numpy() == epoch).all()


def test_reshard_head_aware_alias_checks():
    """Entries may write different heads of the same destination rows (a gather of TP ranks);
    overlapping heads of one row are refused (R7 per head), as are mismatched slice sizes."""
    H, L, s = 8, 2, 100
    g = Geom(L, H, 64, 2, 16, 40)
    g1 = g.with_(num_kv_heads=1)
    g2 = g.with_(num_kv_heads=2)
    src1 = [pool_filled(g1, 1 + r, instance=r) for r in range(2)]
    dst = pool_filled(g, 9)
    ts = kvgen.table_pair(3, s, g1, g1)[0]
    td = kvgen.table_pair(4, s, g, g)[1]
    st = [dev_table(p, ts) for p in src1]
    dt = dev_table(dst, td)
    dk.dyna_kv_wait(dk.dyna_kv_reshard([(st[0], dt, (0, 1), 0), (st[1], dt, (0, 1), 1)], (0, s), (0, L), 32))
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_reshard([(st[0], dt, (0, 1), 3), (st[1], dt, (0, 1), 3)], (0, s), (0, L), 32)
    assert e.value.status == dk.DYNA_EALIAS and "migration 1" in str(e.value)
    src2 = pool_filled(g2, 5)
    with pytest.raises(dk.DynaKVError) as e:          # 1-head and 2-head slices in one launch
        dk.dyna_kv_reshard([(st[0], dt, (0, 1), 0), (dev_table(src2, ts), dt, (0, 2), 2)], (0, s), (0, L), 32)
    assert e.value.status == dk.DYNA_EINVAL


@pytest.mark.parametrize("engine", ENGINES, ids=ENGINE_IDS)
def test_prepared_reshard_launch_and_graph_replay(engine):
    """dyna_kv_prepare_reshard: a TP 2 -> 8 reshard planned once; launches and CUDA-graph replays move
    the source rows as they are at that launch (the sources are rewritten in between), bit-exact."""
    H, L, s, c = 8, 3, 600, 128
    g = Geom(L, H, 64, 2, 16, 60)
    gs, gd = g.with_(num_kv_heads=4), g.with_(num_kv_heads=1, block_size=8, num_blocks=120)
    src = [pool_filled(gs, 200 + r, instance=r) for r in range(2)]
    dst = [pool_filled(gd, 300 + r) for r in range(8)]
    ts = [kvgen.table_pair(10 + r, s, gs, gs)[0] for r in range(2)]
    td = [kvgen.table_pair(20 + r, s, gd, gd)[1] for r in range(8)]
    plan = dd.tp_reshard_plan(H, 2, 8)
    st = [dev_table(p, t) for p, t in zip(src, ts)]
    dt = [dev_table(p, t) for p, t in zip(dst, td)]
    prep = dk.dyna_kv_prepare_reshard([(st[a], dt[b], heads, hd0) for a, b, heads, hd0 in plan], (0, s), (0, L), c,
                                      dk.opts(engine=engine))
    want = [kvgen.fill_bytes(300 + r, gd.pool_bytes) for r in range(8)]
    stream = torch.cuda.Stream()

    def expect(seed):
        for a, b, heads, hd0 in plan:
            oracle.migrate_heads(kvgen.fill_bytes(seed + a, gs.pool_bytes), gs, ts[a], want[b], gd, td[b], (0, s),
                                 (0, L), heads, hd0)
        for b in range(8):
            assert np.array_equal(dst[b].tensor.cpu().numpy(), want[b]), (seed, b)

    def refill(seed):
        for a in range(2):
            dk.dyna_kv_debug_fill(src[a].tensor.data_ptr(), src[a].tensor.numel(), seed + a, 0, 0)
        torch.cuda.synchronize()

    try:
        for seed in (400, 410):
            refill(seed)
            x = dk.dyna_kv_prepared_launch(prep, stream.cuda_stream)
            assert dk.dyna_kv_xfer_plan(x)["engine"] == (dk.DYNA_ENGINE_TILES if engine == 0 else dk.DYNA_ENGINE_VEC)
            dk.dyna_kv_wait(x)
            expect(seed)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            xg = dk.dyna_kv_prepared_launch(prep, stream.cuda_stream)
        dk.dyna_kv_wait(xg)
        refill(420)
        graph.replay()
        torch.cuda.synchronize()
        expect(420)
    finally:
        dk.dyna_kv_prepared_destroy(prep)
