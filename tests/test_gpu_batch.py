"""GPU parity of dyna_kv_migrate_batch (many requests, one launch) and of
host-resident block tables (uploaded by the library), against the oracle."""
import itertools

import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import (dev_table, mapped_mask, pool_filled, pool_from_host, sampled_rows_match, torch_rows_equal,
                      untouched_equal)

pytestmark = pytest.mark.gpu
ENGINES = [dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK, dk.DYNA_ENGINE_BULK_WS]


def host_table(pool, ids):
    return dk.table(pool, None, np.ascontiguousarray(ids, dtype=np.int32))


@pytest.mark.parametrize("variant,engine", list(itertools.product([1, 2], ENGINES)))
@pytest.mark.parametrize("which", ["src", "dst", "both"])
def test_host_resident_tables(variant, engine, which):
    g = Geom(3, 8, 128, 2, 16, 200)
    ts, td = kvgen.table_pair(4, 2000, g, g)
    hs, hd = kvgen.fill_bytes(1, g.pool_bytes), kvgen.fill_bytes(2, g.pool_bytes)
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (37, 1801))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    st = host_table(src, ts) if which in ("src", "both") else dev_table(src, ts)
    dt = host_table(dst, td) if which in ("dst", "both") else dev_table(dst, td)
    x = dk.migrate(st, dt, (37, 1801), (0, 3), 300, variant=variant, engine=engine)
    dk.dyna_kv_wait(x)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_upload_ring_wraps_many_calls():
    """Thousands of host-table calls cycle the 8 MiB upload ring several times."""
    g = Geom(1, 1, 8, 2, 16, 8192)          # row 16 B; tables of up to 8192 ids = 32 KiB each
    src, dst = pool_filled(g, 5), pool_filled(g, 6)
    rng = np.random.default_rng(0)
    ts, td = rng.permutation(8192).astype(np.int32), rng.permutation(8192).astype(np.int32)
    st, dt = host_table(src, ts), host_table(dst, td)
    xs = []
    for i in range(700):                    # 700 x 64 KiB of tables = 5.5 ring turns
        a = (i * 97) % (8192 * 16 - 200)
        xs.append(dk.migrate(st, dt, (a, 8192 * 16), (0, 1), 4096))
        if len(xs) > 64:
            dk.dyna_kv_wait(xs.pop(0))
    for x in xs:
        dk.dyna_kv_wait(x)
    assert torch_rows_equal(src, ts, dst, td, (0, 8192 * 16), (0, 1))


def test_upload_ring_mixed_sizes_behind_long_kernel():
    """Upload-ring reuse after misaligned wraps: host tables of mixed sizes
    (256 B .. 300 KB) and different contents per call, all queued behind a long kernel so no
    consumer has read its span when the ring wraps.  Every migration must read its own table:
    the destination equals the oracle applying the same migrations in stream order."""
    nb = 100_000
    g = Geom(1, 1, 8, 2, 1, nb)             # row 16 B, block size 1: one table id per token
    hs, hd = kvgen.fill_bytes(21, g.pool_bytes), kvgen.fill_bytes(22, g.pool_bytes)
    want = hd.copy()
    rng = np.random.default_rng(5)
    calls = []
    for i in range(90):
        n = int(rng.choice([64, 700, 5000, 30_000, 75_000]))
        ts = rng.choice(nb, n, replace=False).astype(np.int32)
        td = rng.choice(nb, n, replace=False).astype(np.int32)
        calls.append((ts, td, n))
        oracle.migrate(hs, g, ts, want, g, td, (0, n))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)           # ~0.1 s: every queued migration waits behind it
    xs = []
    for ts, td, n in calls:
        st, dt = host_table(src, ts), host_table(dst, td)
        xs.append((dk.migrate(st, dt, (0, n), (0, 1), max(1, n // 3)), st, dt))
    for x, _, _ in xs:
        dk.dyna_kv_wait(x)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("host_tables", [False, True])
def test_batch_matches_oracle(engine, host_tables):
    g = Geom(2, 8, 128, 2, 16, 1200)
    reqs = kvgen.migrating(kvgen.skewed_batch(7, 24))
    lens = [min(r.s, 600) for r in reqs]
    tabs = kvgen.batch_tables(8, [max(n, 1) + 40 for n in lens], g, g)
    hs, hd = kvgen.fill_bytes(11, g.pool_bytes), kvgen.fill_bytes(12, g.pool_bytes)
    want = hd.copy()
    rng = np.random.default_rng(1)
    ranges = []
    for n, (ts, td) in zip(lens, tabs):
        t0 = int(rng.integers(0, 30))
        ranges.append((t0, t0 + n))
        oracle.migrate(hs, g, ts, want, g, td, (t0, t0 + n))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    T = host_table if host_tables else dev_table
    migs = [(T(src, ts), T(dst, td), tr) for (ts, td), tr in zip(tabs, ranges)]
    migs.append((T(src, tabs[0][0]), T(dst, tabs[0][1]), (5, 5)))   # empty entry
    x = dk.migrate_batch(migs, (0, 2), 256, engine=engine)
    dk.dyna_kv_wait(x)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)
    assert np.array_equal(src.tensor.cpu().numpy(), hs)


def test_batch_mixed_destinations_and_reblocking():
    gs = Geom(2, 2, 64, 2, 16, 64)
    gd1, gd2 = gs.with_(block_size=32, num_blocks=40), gs.with_(block_size=8, num_blocks=140)
    hs = kvgen.fill_bytes(1, gs.pool_bytes)
    h1, h2 = kvgen.fill_bytes(2, gd1.pool_bytes), kvgen.fill_bytes(3, gd2.pool_bytes)
    ta, t1 = kvgen.table_pair(3, 300, gs, gd1)
    tb, t2 = kvgen.table_pair(4, 300, gs, gd2)
    tb = (tb + 20) % 64  # keep both sources valid; aliasing of sources is allowed
    w1, w2 = h1.copy(), h2.copy()
    oracle.migrate(hs, gs, ta, w1, gd1, t1, (0, 257))
    oracle.migrate(hs, gs, tb, w2, gd2, t2, (11, 300))
    src = pool_from_host(gs, hs)
    d1, d2 = pool_from_host(gd1, h1), pool_from_host(gd2, h2)
    x = dk.migrate_batch([(dev_table(src, ta), dev_table(d1, t1), (0, 257)),
                          (dev_table(src, tb), dev_table(d2, t2), (11, 300))], (0, 2), 64)
    dk.dyna_kv_wait(x)
    assert np.array_equal(d1.tensor.cpu().numpy(), w1)
    assert np.array_equal(d2.tensor.cpu().numpy(), w2)


def test_batch_errors_name_the_entry():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    bad = td.copy()
    bad[1] = bad[0]
    with pytest.raises(dk.DynaKVError) as e:
        dk.migrate_batch([(dev_table(src, ts), dev_table(dst, td), (0, 10)),
                          (dev_table(src, ts), dev_table(dst, bad), (0, 100))], (0, 2), 32)
    assert e.value.status == dk.DYNA_EALIAS and "migration 1" in str(e.value)


def test_config3_batch_full_size():
    """configs[2] (Llama-3-8B, 64 skewed requests) in ONE launch, full size, checked at any size."""
    g = kvgen.LLAMA3_8B
    reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
    tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
    src, dst = pool_filled(g, 31), pool_filled(g, 32)
    n0 = dk.dyna_kv_launch_count()
    x = dk.migrate_batch([(dev_table(src, ts), dev_table(dst, td), (0, r.s)) for r, (ts, td) in zip(reqs, tabs)],
                         (0, 32), 256)
    plan = dk.dyna_kv_xfer_plan(x)
    dk.dyna_kv_wait(x)
    assert dk.dyna_kv_launch_count() - n0 == 1
    assert (plan["variant"], plan["engine"]) == (dk.DYNA_VARIANT_FUSED, dk.DYNA_ENGINE_BULK)   # bench.py's kernel
    rng = np.random.default_rng(7)
    for r, (ts, td) in zip(reqs, tabs):
        assert torch_rows_equal(src, ts, dst, td, (0, r.s), (0, 32))
        # sampled rows against the oracle's offsets and the kvgen stream (independent of torch indexing)
        assert sampled_rows_match(31, g, ts, dst, g, td, (0, r.s), (0, 32), 8, rng) == 0
    assert untouched_equal(dst, 32, mapped_mask(g, [(td, (0, r.s)) for r, (ts, td) in zip(reqs, tabs)]))


def test_cuda_graph_capture_and_replay():
    """Many small migrations captured once in a CUDA graph, replayed: same bytes as the oracle."""
    g = kvgen.TOY
    hs, hd = kvgen.fill_bytes(1, g.pool_bytes), kvgen.fill_bytes(2, g.pool_bytes)
    tabs = kvgen.batch_tables(1, [256] * 4, g, g)
    want = hd.copy()
    for ts, td in tabs:
        oracle.migrate(hs, g, ts, want, g, td, (0, 100))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    T = [(dev_table(src, a), dev_table(dst, b)) for a, b in tabs]
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        xs = [dk.dyna_kv_migrate_ex(a, b, (0, 100), (0, 2), 32, stream.cuda_stream, None) for a, b in T]
        with pytest.raises(dk.DynaKVError) as e:   # host tables are refused under capture
            dk.dyna_kv_migrate_ex(dk.table(src, None, tabs[0][0]), T[0][1], (0, 100), (0, 2), 32,
                                  stream.cuda_stream, None)
        assert e.value.status == dk.DYNA_ENOTSUP
    for x in xs:
        dk.dyna_kv_wait(x)
    assert np.array_equal(dst.tensor.cpu().numpy(), hd)   # nothing ran yet
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(dst.tensor.cpu().numpy(), want)
    dst.tensor.copy_(torch.from_numpy(hd).cuda())
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_chunk_stream_prefill_then_decode():
    """Native chunk stream: prefill chunks + decoded tokens (s > P) pushed chunk by chunk in
    scheduler-sized steps; the last chunk is the partial one closed at the end; bytes match the oracle."""
    g = Geom(3, 8, 128, 2, 16, 200)
    hs, hd = kvgen.fill_bytes(91, g.pool_bytes), kvgen.fill_bytes(92, g.pool_bytes)
    ts, td = kvgen.table_pair(93, 1500, g, g)
    P, decoded = 1100, 37
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (0, P + decoded))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    cs = dk.dyna_kv_chunkstream_open(st, dt, 0, (0, 3), 256, torch.cuda.current_stream().cuda_stream, None)
    pushed = [dk.dyna_kv_chunkstream_produced(cs, n) for n in (256, 256, 256, 256, 76)]   # prefill of P = 1100
    pushed += [dk.dyna_kv_chunkstream_produced(cs, 1) for _ in range(decoded)]          # alpha decodes on
    assert sum(pushed) == 4
    assert dk.dyna_kv_chunkstream_close(cs) == 1                                        # [1024, 1137)
    info = dk.dyna_kv_chunkstream_info(cs)
    assert info["pushed_end"] == P + decoded and info["num_pushed"] == 5
    dk.dyna_kv_chunkstream_finish(cs)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


@pytest.mark.parametrize("engine", ENGINES + [dk.DYNA_ENGINE_AUTO])
def test_tp_sharded_rows(engine):
    """TP-8 shard of Qwen2-72B (1 KV head per rank: 256-B rows, 4-KiB segments) — SURVEY §8f NEXT-3."""
    g = Geom(8, 1, 128, 2, 16, 300)
    hs, hd = kvgen.fill_bytes(95, g.pool_bytes), kvgen.fill_bytes(96, g.pool_bytes)
    ts, td = kvgen.table_pair(97, 4000, g, g)
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (5, 3999))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    dk.dyna_kv_wait(dk.migrate(dev_table(src, ts), dev_table(dst, td), (5, 3999), (0, 8), 1024, engine=engine))
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_concurrent_host_threads():
    """Eight host threads migrate different requests at once, each on its own stream, mixing device
    tables, host-resident tables (upload ring), batches and signalling — bit-exact vs the oracle."""
    import threading
    g = Geom(2, 8, 128, 2, 16, 1600)
    hs, hd = kvgen.fill_bytes(201, g.pool_bytes), kvgen.fill_bytes(202, g.pool_bytes)
    lens = [700, 333, 1000, 64, 517, 1200, 90, 800]
    tabs = kvgen.batch_tables(203, lens, g, g)
    want = hd.copy()
    for n, (ts, td) in zip(lens, tabs):
        oracle.migrate(hs, g, ts, want, g, td, (0, n))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    torch.cuda.synchronize()
    errors = []

    def worker(i):
        try:
            n, (ts, td) = lens[i], tabs[i]
            stream = torch.cuda.Stream()
            kind = i % 4
            if kind == 1:
                st, dt = host_table(src, ts), host_table(dst, td)
            else:
                st, dt = dev_table(src, ts), dev_table(dst, td)
            torch.cuda.synchronize()
            for rep in range(5):
                if kind == 2:
                    x = dk.dyna_kv_migrate_batch([(st, dt, (0, n))], (0, 2), 128, stream.cuda_stream, None)
                else:
                    x = dk.dyna_kv_migrate_ex(st, dt, (0, n), (0, 2), 100 + 7 * i, stream.cuda_stream,
                                              dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL if kind == 3 else 0))
                dk.dyna_kv_wait(x)
        except Exception as e:  # noqa: BLE001 — reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


# ---------------------------------------------------------------- signalled batches (per-request chunk flags)
def _flags(pool, sender, first, n):
    fl = torch.zeros(max(n, 1), dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(pool.handle, sender, first, n, fl.data_ptr(), 0)
    torch.cuda.synchronize()
    return fl.numpy()[:n]


@pytest.mark.parametrize("engine", [0, dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK])
@pytest.mark.parametrize("host_tables", [False, True])
def test_signalled_batch_per_request_flags(host_tables, engine):
    """Each entry of a signalled batch gets its own epoch and slot range; every chunk flag of every
    request reaches its epoch, slot ranges of one (sender, destination) are disjoint, and the rows
    match the oracle.  Two destination pools, an empty entry, ragged starts."""
    gs = Geom(2, 8, 128, 2, 16, 1200)
    gd1, gd2 = gs.with_(num_blocks=700), gs.with_(block_size=32, num_blocks=400)
    reqs = kvgen.migrating(kvgen.skewed_batch(9, 20))
    lens = [min(r.s, 500) for r in reqs]
    hs = kvgen.fill_bytes(21, gs.pool_bytes)
    h1, h2 = kvgen.fill_bytes(22, gd1.pool_bytes), kvgen.fill_bytes(23, gd2.pool_bytes)
    w1, w2 = h1.copy(), h2.copy()
    rng = np.random.default_rng(3)
    free_s, free1, free2 = np.arange(gs.num_blocks), np.arange(gd1.num_blocks), np.arange(gd2.num_blocks)
    entries = []
    for i, n in enumerate(lens):
        t0 = int(rng.integers(0, 20))
        gd, free_d, want = (gd1, free1, w1) if i % 2 == 0 else (gd2, free2, w2)
        ts, free_s = kvgen.fragmented_table(rng, free_s, kvgen.blocks_needed(t0 + n, gs.block_size))
        td, free_d = kvgen.fragmented_table(rng, free_d, kvgen.blocks_needed(t0 + n, gd.block_size))
        if i % 2 == 0:
            free1 = free_d
        else:
            free2 = free_d
        oracle.migrate(hs, gs, ts, want, gd, td, (t0, t0 + n))
        entries.append((ts, td, (t0, t0 + n), i % 2))
    src = pool_from_host(gs, hs, instance=4)
    d1, d2 = pool_from_host(gd1, h1), pool_from_host(gd2, h2)
    T = host_table if host_tables else dev_table
    migs = [(T(src, ts), T(d1 if w == 0 else d2, td), tr) for ts, td, tr, w in entries]
    migs.insert(3, (T(src, entries[0][0]), T(d1, entries[0][1]), (7, 7)))     # empty entry
    c = 96
    x = dk.migrate_batch(migs, (0, 2), c, flags=dk.DYNA_MIGRATE_SIGNAL, engine=engine, piece_bytes=4096 if engine else 0)
    infos = [dk.dyna_kv_batch_info(x, i) for i in range(len(migs))]
    dk.dyna_kv_wait(x)
    assert infos[3][2] == 0
    used = {0: [], 1: []}
    epochs = {0: set(), 1: set()}
    for (ts, td, tr, w), info in zip(entries, infos[:3] + infos[4:]):
        epoch, first, nck, sender = info
        assert sender == 4 and nck == -(-(tr[1] - tr[0]) // c)
        fl = _flags(d1 if w == 0 else d2, sender, first, nck)
        assert (fl == epoch).all(), (info, fl)
        used[w] += list(range(first, first + nck))
        epochs[w].add(epoch)
    for w in (0, 1):
        assert len(used[w]) == len(set(used[w]))          # disjoint slot ranges per destination
        assert len(epochs[w]) == sum(1 for e in entries if e[3] == w)   # one epoch per request (per destination)
    assert np.array_equal(d1.tensor.cpu().numpy(), w1)
    assert np.array_equal(d2.tensor.cpu().numpy(), w2)


def test_signalled_batch_limits_and_errors():
    g = Geom(1, 2, 64, 2, 16, 4200)
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 65536, g, g)
    with pytest.raises(dk.DynaKVError) as e:        # 2 x 4096 chunks into one destination: slots would be shared
        dk.migrate_batch([(dev_table(src, ts), dev_table(dst, td), (0, 4096)),
                          (dev_table(src, ts), dev_table(dst, td), (4096, 8192))], (0, 1), 1,
                         flags=dk.DYNA_MIGRATE_SIGNAL)
    assert e.value.status == dk.DYNA_ERANGE
    # 2048 + 2048 one-token chunks fit: disjoint slot ranges, every flag raised (BULK ring, small pieces)
    x = dk.migrate_batch([(dev_table(src, ts), dev_table(dst, td), (0, 2048)),
                          (dev_table(src, ts), dev_table(dst, td), (4096, 6144))], (0, 1), 1,
                         flags=dk.DYNA_MIGRATE_SIGNAL, engine=dk.DYNA_ENGINE_BULK, piece_bytes=256)
    infos = [dk.dyna_kv_batch_info(x, i) for i in range(2)]
    dk.dyna_kv_wait(x)
    (e0, f0, n0, snd), (e1, f1, n1, _) = infos
    assert n0 == n1 == 2048 and (f0 + n0 <= f1 or f1 + n1 <= f0)
    assert (_flags(dst, snd, f0, n0) == e0).all() and (_flags(dst, snd, f1, n1) == e1).all()
    assert torch_rows_equal(src, ts, dst, td, (0, 2048), (0, 1))
    assert torch_rows_equal(src, ts, dst, td, (4096, 6144), (0, 1))
    x = dk.migrate_batch([(dev_table(src, ts), dev_table(dst, td), (0, 10))], (0, 1), 4)
    with pytest.raises(dk.DynaKVError) as e:         # not a signalled batch
        dk.dyna_kv_batch_info(x, 0)
    assert e.value.status == dk.DYNA_EINVAL
    dk.dyna_kv_wait(x)


# ---------------------------------------------------------------- native chunk streams
@pytest.mark.parametrize("signal", [False, True])
def test_native_chunkstream_prefill_then_decode(signal):
    """A 600-token prompt prefilled in 256-token steps, then 5 decoded tokens (s = 605 > P), pushed
    by the library's chunk stream: chunks close when full or at close(); every chunk's flag is in
    the stream's slots; the destination equals one plain migration of [begin, begin + 605)."""
    g = Geom(3, 8, 128, 2, 16, 200)
    begin, c = 7, 128
    ts, td = kvgen.table_pair(77, 800, g, g)
    hs, hd = kvgen.fill_bytes(61, g.pool_bytes), kvgen.fill_bytes(62, g.pool_bytes)
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (begin, begin + 605))
    src, dst = pool_from_host(g, hs, instance=3), pool_from_host(g, hd)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    o = dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0)
    s = dk.dyna_kv_chunkstream_open(st, dt, begin, (0, 3), c, 0, o)
    pushed = [dk.dyna_kv_chunkstream_produced(s, n) for n in (256, 256, 88, 1, 1, 1, 1, 1)]
    assert pushed == [2, 2, 0, 0, 0, 0, 0, 0]           # 4 full chunks; [512, 605) still open
    assert dk.dyna_kv_chunkstream_close(s) == 1
    info = dk.dyna_kv_chunkstream_info(s)
    assert info["num_pushed"] == 5 and info["pushed_end"] == begin + 605 and info["produced_end"] == begin + 605
    with pytest.raises(dk.DynaKVError):
        dk.dyna_kv_chunkstream_produced(s, 1)         # closed
    dk.dyna_kv_chunkstream_finish(s)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)
    if signal:
        fl = torch.zeros(5, dtype=torch.int64).pin_memory()
        dk.dyna_kv_copy_flags(dst.handle, info["sender"], info["first_slot"], 5, fl.data_ptr(), 0)
        torch.cuda.synchronize()
        assert (fl.numpy() == info["epoch"]).all()


def test_native_chunkstream_empty_and_errors():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    s = dk.dyna_kv_chunkstream_open(st, dt, 0, (0, 2), 32, 0, None)
    assert dk.dyna_kv_chunkstream_close(s) == 0         # s = 0: nothing to ship
    dk.dyna_kv_chunkstream_finish(s)
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_chunkstream_open(st, dt, 0, (0, 2), 32, 0, dk.opts(variant=dk.DYNA_VARIANT_STAGED))
    assert e.value.status == dk.DYNA_ENOTSUP
    s = dk.dyna_kv_chunkstream_open(st, dt, 0, (0, 2), 32, 0, None)
    with pytest.raises(dk.DynaKVError) as e:              # the chunk beyond the tables is refused
        dk.dyna_kv_chunkstream_produced(s, 300)
    assert e.value.status == dk.DYNA_ERANGE
    dk.dyna_kv_chunkstream_finish(s)


@pytest.mark.parametrize("signal", [False, True])
@pytest.mark.parametrize("host_tables", [False, True])
def test_batch_small_rows_as_tiles(signal, host_tables):
    """A batch of TP-8-shard migrations (256-B rows, 4-KiB blocks) between two source and two destination
    pools: AUTO runs it as ONE tile launch (one map set per (source, destination) pool pair, per-request
    chunk flags), equal to the oracle applying every request in order."""
    g = Geom(6, 1, 128, 2, 16, 400)
    reqs = kvgen.migrating(kvgen.skewed_batch(17, 16))
    lens = [min(r.s, 900) for r in reqs]
    hs = [kvgen.fill_bytes(40 + i, g.pool_bytes) for i in range(2)]
    hd = [kvgen.fill_bytes(50 + i, g.pool_bytes) for i in range(2)]
    tabs = [kvgen.batch_tables(60 + i, [n + 16 for n in lens[i::2]], g, g) for i in range(2)]
    want = [h.copy() for h in hd]
    src = [pool_from_host(g, h) for h in hs]
    dst = [pool_from_host(g, h) for h in hd]
    T = host_table if host_tables else dev_table
    migs, where = [], []
    rng = np.random.default_rng(3)
    for i in range(2):                       # pair (src i -> dst i) for even/odd requests
        for n, (ts, td) in zip(lens[i::2], tabs[i]):
            t0 = int(rng.integers(0, 16))
            oracle.migrate(hs[i], g, ts, want[i], g, td, (t0, t0 + n))
            migs.append((T(src[i], ts), T(dst[i], td), (t0, t0 + n)))
            where.append(i)
    x = dk.migrate_batch(migs, (0, 6), 128, flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0)
    assert dk.dyna_kv_xfer_plan(x)["engine"] == dk.DYNA_ENGINE_TILES
    infos = [dk.dyna_kv_batch_info(x, k) for k in range(len(migs))] if signal else []
    dk.dyna_kv_wait(x)
    for i in range(2):
        assert np.array_equal(dst[i].tensor.cpu().numpy(), want[i]), i
        assert np.array_equal(src[i].tensor.cpu().numpy(), hs[i]), i
    for (_, _, tr), i, (epoch, first, nck, sender) in zip(migs, where, infos):
        fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
        dk.dyna_kv_copy_flags(dst[i].handle, sender, first, nck, fl.data_ptr(), 0)
        torch.cuda.synchronize()
        assert nck == -(-(tr[1] - tr[0]) // 128) and (fl.numpy() == epoch).all()


def test_batch_tiles_need_one_run_grid():
    """Regression (seeded fuzzing): entries whose run grids differ (16- vs 8-token destination
    blocks) can still produce equal tile boxes (16 rows x 2 slabs = 8 rows x 4 slabs = 32 KiB of
    1-KiB rows); one tile launch takes its box geometry from its first plan, so such a batch must
    not be tiled.  It runs (on another engine) bit-exact."""
    gs = Geom(2, 8, 64, 2, 16, 300)                        # 1-KiB rows
    gd1, gd2 = gs.with_(block_size=16), gs.with_(block_size=8, num_blocks=600)
    hs = kvgen.fill_bytes(1, gs.pool_bytes)
    h1, h2 = kvgen.fill_bytes(2, gd1.pool_bytes), kvgen.fill_bytes(3, gd2.pool_bytes)
    (ta, t1), (tb, t2) = kvgen.table_pair(4, 700, gs, gd1), kvgen.table_pair(5, 700, gs, gd2)
    tb = (tb + 150) % 300
    w1, w2 = h1.copy(), h2.copy()
    oracle.migrate(hs, gs, ta, w1, gd1, t1, (0, 600))
    oracle.migrate(hs, gs, tb, w2, gd2, t2, (3, 650))
    src, d1, d2 = pool_from_host(gs, hs), pool_from_host(gd1, h1), pool_from_host(gd2, h2)
    x = dk.migrate_batch([(dev_table(src, ta), dev_table(d1, t1), (0, 600)),
                          (dev_table(src, tb), dev_table(d2, t2), (3, 650))], (0, 2), 128)
    dk.dyna_kv_wait(x)
    assert np.array_equal(d1.tensor.cpu().numpy(), w1)
    assert np.array_equal(d2.tensor.cpu().numpy(), w2)


# ---------------------------------------------------------------- prepared batches (plan once, launch many)
@pytest.mark.parametrize("rows", ["2KiB", "256B"])
def test_prepared_batch_launches_and_graph_replay(rows):
    """dyna_kv_prepare_batch plans and uploads a batch once; every dyna_kv_prepared_launch (and every
    replay of a CUDA graph that captured one) moves the rows as they are at that launch: the source
    is rewritten between launches and the destination must follow it, bit-exact vs the oracle.  Host
    tables are copied at prepare time (later edits of the host arrays do not matter)."""
    g = Geom(3, 8, 128, 2, 16, 600) if rows == "2KiB" else Geom(3, 1, 128, 2, 16, 600)
    reqs = kvgen.migrating(kvgen.skewed_batch(23, 12))
    lens = [min(r.s, 700) for r in reqs]
    tabs = kvgen.batch_tables(24, [n + 16 for n in lens], g, g)
    dst = pool_filled(g, 2)
    src = pool_filled(g, 1)
    migs = [(host_table(src, ts.copy()), dev_table(dst, td), (3, 3 + n)) for n, (ts, td) in zip(lens, tabs)]
    prep = dk.dyna_kv_prepare_batch(migs, (0, 3), 128)
    for m in migs:                                        # host arrays edited after prepare: irrelevant
        m[0]._keep[1][:] = 0                              # (the numpy array behind host_block_ids)
    s = torch.cuda.Stream()
    try:
        for seed in (31, 32):
            dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), seed, 0, 0)
            torch.cuda.synchronize()
            x = dk.dyna_kv_prepared_launch(prep, s.cuda_stream)
            plan = dk.dyna_kv_xfer_plan(x)
            dk.dyna_kv_wait(x)
            assert plan["launches"] == 1
            if rows == "256B":
                assert plan["engine"] == dk.DYNA_ENGINE_TILES
            want = kvgen.fill_bytes(2, g.pool_bytes) if seed == 31 else want
            for n, (ts, td) in zip(lens, tabs):
                oracle.migrate(kvgen.fill_bytes(seed, g.pool_bytes), g, ts, want, g, td, (3, 3 + n))
            assert np.array_equal(dst.tensor.cpu().numpy(), want), seed
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s):
            xg = dk.dyna_kv_prepared_launch(prep, s.cuda_stream)
        dk.dyna_kv_wait(xg)
        for seed in (33, 34):
            dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), seed, 0, 0)
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            for n, (ts, td) in zip(lens, tabs):
                oracle.migrate(kvgen.fill_bytes(seed, g.pool_bytes), g, ts, want, g, td, (3, 3 + n))
            assert np.array_equal(dst.tensor.cpu().numpy(), want), seed
    finally:
        dk.dyna_kv_prepared_destroy(prep)


def test_prepared_batch_errors_and_empty():
    g = Geom(2, 8, 128, 2, 16, 100)
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(3, 200, g, g)
    migs = [(dev_table(src, ts), dev_table(dst, td), (0, 100))]
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_prepare_batch(migs, (0, 2), 32, dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL))
    assert e.value.status == dk.DYNA_EINVAL
    with pytest.raises(dk.DynaKVError) as e:         # R7 is checked at prepare time
        dk.dyna_kv_prepare_batch(migs + [(dev_table(src, ts), dev_table(dst, td), (50, 60))], (0, 2), 32)
    assert e.value.status == dk.DYNA_EALIAS
    empty = dk.dyna_kv_prepare_batch([(dev_table(src, ts), dev_table(dst, td), (5, 5))], (0, 2), 32)
    dk.dyna_kv_wait(dk.dyna_kv_prepared_launch(empty, 0))
    dk.dyna_kv_prepared_destroy(empty)
