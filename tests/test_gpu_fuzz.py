"""Seeded differential fuzzing of the CUDA path against the oracle: random geometries (layers,
heads, head_dim, element size, block sizes on each side), random fragmented tables, random
token / layer / head ranges, chunk sizes, variants, engines and engine shapes, with and
without per-chunk flags.  Every case is compared byte for byte on the whole destination pool
(and the source pool is checked unchanged)."""
import os

import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, pool_from_host

pytestmark = pytest.mark.gpu
SCALE = int(os.environ.get("DYNA_FUZZ_SCALE", "1"))   # longer campaigns: DYNA_FUZZ_SCALE=10


def _case(rng):
    e = int(rng.choice([1, 2, 4]))
    d = int(rng.choice([8, 16, 32, 64, 128])) * (2 // e if e < 2 else 1)
    H = int(rng.integers(1, 9))
    if (H * d * e) % 16:
        d = 16 // e * int(rng.integers(1, 9))
    L = int(rng.integers(1, 5))
    bss, bsd = int(rng.choice([1, 2, 4, 8, 16, 24, 32])), int(rng.choice([1, 2, 4, 8, 16, 32]))
    n_tok = int(rng.integers(1, 600))
    gs = Geom(L, H, d, e, bss, kvgen.blocks_needed(n_tok, bss) + int(rng.integers(0, 20)))
    gd = Geom(L, H, d, e, bsd, kvgen.blocks_needed(n_tok, bsd) + int(rng.integers(0, 20)))
    t0 = int(rng.integers(0, n_tok))
    t1 = int(rng.integers(t0, n_tok + 1))
    l0 = int(rng.integers(0, L))
    l1 = int(rng.integers(l0, L + 1))
    c = int(rng.choice([1, 3, 16, 17, 64, 100, 257, 1000]))
    variant = int(rng.choice([1, 2]))
    engine = int(rng.choice([0, 1, 2, 3]))        # 0 = AUTO: short runs as TMA tiles
    piece = int(rng.choice([0, 256, 1024, 4096, 16384, 32768]))
    stages = int(rng.choice([0, 2, 3, 4, 6, 8]))
    unroll = int(rng.choice([0, 4, 8, 16]))
    signal = bool(rng.integers(0, 2))
    return gs, gd, n_tok, (t0, t1), (l0, l1), c, dict(variant=variant, engine=engine, piece_bytes=piece,
                                                        stages=stages, unroll=unroll,
                                                        flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0)


@pytest.mark.parametrize("block", range(8 * SCALE))
def test_fuzz_migrate(block):
    rng = np.random.default_rng(kvgen.MASTER_SEED + 500 + block)
    for i in range(40):
        gs, gd, n_tok, tr, lr, c, kw = _case(rng)
        ts, td = kvgen.table_pair(int(rng.integers(1 << 30)), n_tok, gs, gd)
        hs = kvgen.fill_bytes(int(rng.integers(1 << 30)), gs.pool_bytes)
        hd = kvgen.fill_bytes(int(rng.integers(1 << 30)), gd.pool_bytes)
        want = hd.copy()
        oracle.migrate(hs, gs, ts, want, gd, td, tr, lr)
        src, dst = pool_from_host(gs, hs, instance=int(rng.integers(0, 8))), pool_from_host(gd, hd)
        st, dt = dev_table(src, ts), dev_table(dst, td)
        x = dk.migrate(st, dt, tr, lr, c, **kw)
        dk.dyna_kv_wait(x)
        got = dst.tensor.cpu().numpy()
        assert np.array_equal(src.tensor.cpu().numpy(), hs), (i, gs, gd, tr, lr, c, kw)
        assert np.array_equal(got, want), (i, gs, gd, tr, lr, c, kw)


@pytest.mark.parametrize("block", range(4 * SCALE))
def test_fuzz_migrate_heads(block):
    rng = np.random.default_rng(kvgen.MASTER_SEED + 900 + block)
    for i in range(40):
        e = int(rng.choice([2, 4]))
        d = 16 // e * int(rng.integers(1, 9))
        Hs, Hd = int(rng.integers(1, 9)), int(rng.integers(1, 9))
        n = int(rng.integers(0, min(Hs, Hd) + 1))
        h0 = int(rng.integers(0, Hs - n + 1))
        hd0 = int(rng.integers(0, Hd - n + 1))
        L = int(rng.integers(1, 4))
        bss, bsd = int(rng.choice([1, 4, 8, 16])), int(rng.choice([2, 8, 16, 32]))
        n_tok = int(rng.integers(1, 500))
        gs = Geom(L, Hs, d, e, bss, kvgen.blocks_needed(n_tok, bss) + 3)
        gd = Geom(L, Hd, d, e, bsd, kvgen.blocks_needed(n_tok, bsd) + 3)
        t0 = int(rng.integers(0, n_tok))
        tr = (t0, int(rng.integers(t0, n_tok + 1)))
        c = int(rng.choice([1, 7, 16, 100, 1000]))
        piece = int(rng.choice([0, 256, 4096]))
        sig = dk.DYNA_MIGRATE_SIGNAL if rng.integers(0, 2) else 0
        engine = int(rng.choice([0, 1]))          # AUTO (TMA tiles) / VEC (row kernel)
        ts, td = kvgen.table_pair(int(rng.integers(1 << 30)), n_tok, gs, gd)
        hs = kvgen.fill_bytes(int(rng.integers(1 << 30)), gs.pool_bytes)
        hdst = kvgen.fill_bytes(int(rng.integers(1 << 30)), gd.pool_bytes)
        want = hdst.copy()
        oracle.migrate_heads(hs, gs, ts, want, gd, td, tr, None, (h0, h0 + n), hd0)
        src, dst = pool_from_host(gs, hs), pool_from_host(gd, hdst)
        st, dt = dev_table(src, ts), dev_table(dst, td)
        dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(st, dt, tr, (0, L), (h0, h0 + n), hd0, c, 0,
                                                 dk.opts(piece_bytes=piece, flags=sig, engine=engine)))
        assert np.array_equal(dst.tensor.cpu().numpy(), want), (i, gs, gd, tr, (h0, n, hd0), c, piece, engine)


@pytest.mark.parametrize("block", range(2 * SCALE))
def test_fuzz_batch(block):
    """Random batches: 1-12 requests with own ranges into one or two destination pools, random
    engine / piece, with or without per-request flags (each request's flags checked)."""
    rng = np.random.default_rng(kvgen.MASTER_SEED + 1300 + block)
    for i in range(12):
        H = int(rng.integers(1, 9))
        gs = Geom(int(rng.integers(1, 4)), H, 64, 2, int(rng.choice([8, 16])), 900)
        gd1 = gs.with_(block_size=int(rng.choice([8, 16, 32])), num_blocks=900)
        gd2 = gs.with_(block_size=16, num_blocks=900)
        nreq = int(rng.integers(1, 13))
        lens = [int(rng.integers(0, 300)) for _ in range(nreq)]
        hs = kvgen.fill_bytes(int(rng.integers(1 << 30)), gs.pool_bytes)
        h1, h2 = kvgen.fill_bytes(int(rng.integers(1 << 30)), gd1.pool_bytes), kvgen.fill_bytes(7, gd2.pool_bytes)
        w1, w2 = h1.copy(), h2.copy()
        free_s, free1, free2 = np.arange(900), np.arange(900), np.arange(900)
        ents = []
        for n in lens:
            t0 = int(rng.integers(0, 20))
            which = int(rng.integers(0, 2))
            gd = gd1 if which == 0 else gd2
            ts, free_s = kvgen.fragmented_table(rng, free_s, kvgen.blocks_needed(t0 + n + 1, gs.block_size))
            if which == 0:
                td, free1 = kvgen.fragmented_table(rng, free1, kvgen.blocks_needed(t0 + n + 1, gd.block_size))
            else:
                td, free2 = kvgen.fragmented_table(rng, free2, kvgen.blocks_needed(t0 + n + 1, gd.block_size))
            oracle.migrate(hs, gs, ts, w1 if which == 0 else w2, gd, td, (t0, t0 + n))
            ents.append((ts, td, (t0, t0 + n), which))
        src = pool_from_host(gs, hs, instance=1)
        d1, d2 = pool_from_host(gd1, h1), pool_from_host(gd2, h2)
        migs = [(dev_table(src, ts), dev_table(d1 if w == 0 else d2, td), tr) for ts, td, tr, w in ents]
        sig = bool(rng.integers(0, 2))
        c = int(rng.choice([16, 33, 128, 1000]))
        kw = dict(engine=int(rng.choice([0, 1, 2, 3])), piece_bytes=int(rng.choice([0, 1024, 16384])))
        if sig:
            kw["flags"] = dk.DYNA_MIGRATE_SIGNAL
        x = dk.migrate_batch(migs, (0, gs.num_layers), c, **kw)
        infos = [dk.dyna_kv_batch_info(x, j) for j in range(len(migs))] if sig else []
        dk.dyna_kv_wait(x)
        assert np.array_equal(d1.tensor.cpu().numpy(), w1), (i, kw)
        assert np.array_equal(d2.tensor.cpu().numpy(), w2), (i, kw)
        for (ts, td, tr, w), (epoch, first, nck, sender) in zip(ents, infos):
            if nck:
                fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
                dk.dyna_kv_copy_flags((d1 if w == 0 else d2).handle, sender, first, nck, fl.data_ptr(), 0)
                torch.cuda.synchronize()
                assert (fl.numpy() == epoch).all(), (i, first, nck)


def test_fuzz_channel():
    """Random receiver-steered transfers: slots, slot sizes (down to one token), chunk sizes,
    ranges, whole rows or head slices; push and place on separate streams."""
    rng = np.random.default_rng(kvgen.MASTER_SEED + 1700)
    for i in range(12):
        H = int(rng.choice([2, 4, 8]))
        L = int(rng.integers(1, 4))
        gs = Geom(L, H, 64, 2, int(rng.choice([8, 16])), 300)
        heads = bool(rng.integers(0, 2))
        n = int(rng.integers(1, H + 1)) if heads else H
        h0 = int(rng.integers(0, H - n + 1)) if heads else 0
        gd = gs.with_(num_kv_heads=n if heads else H, block_size=int(rng.choice([8, 16, 32])), num_blocks=300)
        n_tok = int(rng.integers(1, 1500))
        ts, td = kvgen.table_pair(int(rng.integers(1 << 30)), n_tok, gs, gd)
        t0 = int(rng.integers(0, n_tok))
        tr = (t0, int(rng.integers(t0 + 1, n_tok + 1)))
        c = int(rng.choice([1, 16, 100, 512, 5000]))
        tok = 2 * L * n * 128
        slot_bytes = tok * int(rng.choice([1, 3, 64, 1000]))
        slots = int(rng.integers(2, 5))
        hs = kvgen.fill_bytes(int(rng.integers(1 << 30)), gs.pool_bytes)
        hd = kvgen.fill_bytes(int(rng.integers(1 << 30)), gd.pool_bytes)
        want = hd.copy()
        if heads:
            oracle.migrate_heads(hs, gs, ts, want, gd, td, tr, None, (h0, h0 + n), 0)
        else:
            oracle.migrate(hs, gs, ts, want, gd, td, tr)
        src, dst = pool_from_host(gs, hs), pool_from_host(gd, hd)
        st, dt = dev_table(src, ts), dev_table(dst, td)
        ch = dk.dyna_kv_channel_create(dst.handle, 2, slots, slot_bytes)
        dk.dyna_kv_channel_set_timeout(ch, 120_000_000_000)
        try:
            sp, sq = torch.cuda.Stream(), torch.cuda.Stream()
            if heads:
                xp = dk.dyna_kv_push_heads(st, tr, (0, L), (h0, h0 + n), c, ch, sp.cuda_stream)
                xq = dk.dyna_kv_place_heads(ch, dt, tr, (0, L), 0, n, c, sq.cuda_stream)
            else:
                xp = dk.dyna_kv_push(st, tr, (0, L), c, ch, sp.cuda_stream)
                xq = dk.dyna_kv_place(ch, dt, tr, (0, L), c, sq.cuda_stream)
            dk.dyna_kv_wait(xp)
            dk.dyna_kv_wait(xq)
            assert np.array_equal(dst.tensor.cpu().numpy(), want), (i, heads, tr, c, slots, slot_bytes)
        finally:
            dk.dyna_kv_channel_destroy(ch)


@pytest.mark.parametrize("block", range(4 * SCALE))
def test_fuzz_overlapped_chains(block):
    """Random chains of DYNA_MIGRATE_OVERLAP_PREV calls: one request cut at random points into
    consecutive calls (each its own chunk size, variant, engine and flags), all enqueued back to back
    after a plain first call; the destination equals one oracle migration of the whole range."""
    rng = np.random.default_rng(kvgen.MASTER_SEED + 1300 + block)
    for i in range(20):
        gs, gd, n_tok, (t0, t1), lr, _, _ = _case(rng)
        ts, td = kvgen.table_pair(int(rng.integers(1 << 30)), n_tok, gs, gd)
        hs = kvgen.fill_bytes(int(rng.integers(1 << 30)), gs.pool_bytes)
        hd = kvgen.fill_bytes(int(rng.integers(1 << 30)), gd.pool_bytes)
        want = hd.copy()
        oracle.migrate(hs, gs, ts, want, gd, td, (t0, t1), lr)
        src, dst = pool_from_host(gs, hs, instance=int(rng.integers(0, 8))), pool_from_host(gd, hd)
        st, dt = dev_table(src, ts), dev_table(dst, td)
        cuts = sorted(set([t0, t1] + [int(x) for x in rng.integers(t0, t1 + 1, int(rng.integers(0, 6)))]))
        xs = []
        for j, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
            kw = _case(rng)[6]
            kw["flags"] |= dk.DYNA_MIGRATE_OVERLAP_PREV if j else 0
            xs.append(dk.migrate(st, dt, (a, b), lr, int(rng.choice([1, 7, 16, 64, 300])), **kw))
        for x in xs:
            dk.dyna_kv_wait(x)
        assert np.array_equal(src.tensor.cpu().numpy(), hs), (i, gs, gd, cuts, lr)
        assert np.array_equal(dst.tensor.cpu().numpy(), want), (i, gs, gd, cuts, lr)
