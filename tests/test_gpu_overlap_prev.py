"""DYNA_MIGRATE_OVERLAP_PREV: back-to-back independent migrations start copying while the previous
kernel on the stream drains (§4.3: chunk k+1 pushed while chunk k is in flight).
Bit-exact against the oracle for every engine and call kind; per-chunk flags and their self-resetting
counters stay correct when the slot ring wraps under overlapped launches; and a migration never
completes before its predecessor (events / dyna_kv_wait keep stream order)."""
import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, mapped_mask, pool_filled, pool_from_host, torch_rows_equal, untouched_equal

pytestmark = pytest.mark.gpu
OV = dk.DYNA_MIGRATE_OVERLAP_PREV


@pytest.mark.parametrize("engine", [dk.DYNA_ENGINE_AUTO, dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK, dk.DYNA_ENGINE_TILES])
@pytest.mark.parametrize("signal", [False, True])
def test_per_chunk_calls_overlapped_match_oracle(engine, signal):
    """One request pushed as per-chunk calls (c = 100: chunks straddle blocks), each overlapping the last."""
    g = Geom(3, 8, 128, 2, 16, 200)
    ts, td = kvgen.table_pair(4, 3000, g, g)
    hs, hd = kvgen.fill_bytes(1, g.pool_bytes), kvgen.fill_bytes(2, g.pool_bytes)
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (7, 2911))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    torch.cuda.synchronize()   # the first flagged call must not overlap the uploads' kernels (contract)
    flags = OV | (dk.DYNA_MIGRATE_SIGNAL if signal else 0)
    xs = [dk.migrate(st, dt, (a, min(a + 100, 2911)), (0, 3), 100, engine=engine, flags=flags)
          for a in range(7, 2911, 100)]
    infos = [dk.dyna_kv_xfer_info(x) for x in xs]
    for x in xs:
        dk.dyna_kv_wait(x)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)
    assert np.array_equal(src.tensor.cpu().numpy(), hs)
    if signal:
        for epoch, nck, sender, first in infos:
            fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
            dk.dyna_kv_copy_flags(dst.handle, sender, first, nck, fl.data_ptr(), 0)
            torch.cuda.synchronize()
            assert nck == 1 and (fl.numpy() == epoch).all()


def test_signalled_slot_ring_wraps_under_overlap():
    """Signalled overlapped calls of 1500 chunks each wrap the 4096-slot inbox row every third call:
    a call's counters are touched only after its predecessor finished resetting them, so every flag
    reaches its epoch and nothing is lost (20 calls back to back, one token per chunk)."""
    g = Geom(1, 1, 8, 2, 16, 4000)        # 16-B rows
    src, dst = pool_filled(g, 5), pool_filled(g, 6)
    rng = np.random.default_rng(3)
    ts, td = rng.permutation(4000).astype(np.int32), rng.permutation(4000).astype(np.int32)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    torch.cuda.synchronize()   # the fills are kernels the first flagged call must not overlap
    xs = []
    for i in range(20):
        a = (i % 40) * 1500
        xs.append(dk.migrate(st, dt, (a, a + 1500), (0, 1), 1, flags=OV | dk.DYNA_MIGRATE_SIGNAL))
    infos = [dk.dyna_kv_xfer_info(x) for x in xs]
    for x in xs:
        dk.dyna_kv_wait(x)
    firsts = [f for (_, _, _, f) in infos]
    assert 0 in firsts[1:], firsts                       # the ring wrapped at least once
    last = {}
    for (epoch, nck, sender, first) in infos:          # later calls overwrite earlier slots: check the latest
        for k in range(nck):
            last[first + k] = epoch
    fl = torch.zeros(4096, dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(dst.handle, infos[0][2], 0, 4096, fl.data_ptr(), 0)
    torch.cuda.synchronize()
    for slot, epoch in last.items():
        assert fl[slot].item() == epoch, (slot, fl[slot].item(), epoch)
    for i in range(20):
        a = (i % 40) * 1500
        assert torch_rows_equal(src, ts, dst, td, (a, a + 1500), (0, 1))


def test_overlapped_call_never_completes_before_its_predecessor():
    """A 1-GiB ring migration, then a tiny overlapped VEC migration that can run beside it: when the
    tiny one's wait returns, the big one has completed too (its query no longer says in flight)."""
    g = kvgen.LLAMA3_8B.with_(num_blocks=2048)
    src, dst = pool_filled(g, 7), pool_filled(g, 8)
    ts, td = kvgen.table_pair(9, 8192, g, g)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    g2 = Geom(1, 1, 8, 2, 16, 64)
    s2, d2 = pool_filled(g2, 9), pool_filled(g2, 10)
    t2s, t2d = kvgen.table_pair(1, 64, g2, g2)
    a2, b2 = dev_table(s2, t2s), dev_table(d2, t2d)
    torch.cuda.synchronize()
    for _ in range(3):
        big = dk.migrate(st, dt, (0, 8192), (0, 32), 8192, engine=dk.DYNA_ENGINE_BULK)
        tiny = dk.migrate(a2, b2, (0, 64), (0, 1), 64, engine=dk.DYNA_ENGINE_VEC, flags=OV)
        dk.dyna_kv_wait(tiny)
        assert dk.dyna_kv_query(big), "overlapped migration completed before the kernel before it"
        dk.dyna_kv_wait(big)
    assert torch_rows_equal(src, ts, dst, td, (0, 8192), (0, 32))
    assert torch_rows_equal(s2, t2s, d2, t2d, (0, 64), (0, 1))


@pytest.mark.parametrize("engine", [dk.DYNA_ENGINE_AUTO, dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK])
def test_batches_heads_reshard_pack_overlapped(engine):
    g = Geom(2, 8, 128, 2, 16, 300)
    reqs = [700, 1200, 333]
    tabs = kvgen.batch_tables(3, reqs, g, g)
    src, dst = pool_filled(g, 11), pool_filled(g, 12)
    keep = [(dev_table(src, a), dev_table(dst, b)) for a, b in tabs]
    gd = g.with_(num_kv_heads=4, num_blocks=200)
    r0, r1 = pool_filled(gd, 13), pool_filled(gd, 14)
    ts, td0 = kvgen.table_pair(5, 900, g, gd)
    _, td1 = kvgen.table_pair(6, 900, g, gd)
    sT, t0, t1 = dev_table(src, ts), dev_table(r0, td0), dev_table(r1, td1)
    buf = torch.empty(900 * 2 * 2 * g.row_bytes, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()   # fills done: then a chain of mutually independent flagged calls
    # a batch, a TP-1 -> TP-2 reshard and a pack, each overlapping the calls before it
    xs = [dk.migrate_batch([(a, b, (0, n)) for (a, b), n in zip(keep, reqs)], (0, 2), 256, engine=engine, flags=OV)]
    xs.append(dk.dyna_kv_reshard([(sT, t0, (0, 4), 0), (sT, t1, (4, 8), 0)], (0, 900), (0, 2), 300, 0,
                                 dk.opts(engine=engine, flags=OV)))
    xs.append(dk.dyna_kv_pack(sT, (0, 900), (0, 2), buf.data_ptr(), buf.numel(), 0, dk.opts(flags=OV)))
    for x in xs:
        dk.dyna_kv_wait(x)
    for (a, b), n in zip(tabs, reqs):
        assert torch_rows_equal(src, a, dst, b, (0, n), (0, 2))
    assert untouched_equal(dst, 12, mapped_mask(g, [(b, (0, n)) for (_, b), n in zip(tabs, reqs)]))
    for pool, tdx, seed, h0 in ((r0, td0, 13, 0), (r1, td1, 14, 4)):
        want = kvgen.fill_bytes(seed, gd.pool_bytes)
        oracle.migrate_heads(kvgen.fill_bytes(11, g.pool_bytes), g, ts, want, gd, tdx, (0, 900), (0, 2), (h0, h0 + 4), 0)
        assert np.array_equal(pool.tensor.cpu().numpy(), want)
    assert np.array_equal(buf.cpu().numpy(), oracle.pack(kvgen.fill_bytes(11, g.pool_bytes), g, ts, (0, 900), (0, 2)))


def test_prepared_batches_overlapped():
    """Two prepared batches with the flag after a plain migration, all three on disjoint rows (a chain of
    flagged launches must be mutually independent: launch 3 may still overlap launch 1)."""
    g = Geom(2, 8, 128, 2, 16, 400)
    tabs = kvgen.batch_tables(8, [500, 640, 300], g, g)
    src, dst = pool_filled(g, 21), pool_filled(g, 22)
    keep = [(dev_table(src, a), dev_table(dst, b)) for a, b in tabs]
    preps = [dk.dyna_kv_prepare_batch([(keep[i][0], keep[i][1], (0, n))], (0, 2), 128, dk.opts(flags=OV))
             for i, n in ((1, 640), (2, 300))]
    try:
        st = torch.cuda.current_stream().cuda_stream
        xs = [dk.migrate(keep[0][0], keep[0][1], (0, 500), (0, 2), 128)]
        xs += [dk.dyna_kv_prepared_launch(p, st) for p in preps]
        for x in xs:
            dk.dyna_kv_wait(x)
        for (a, b), n in zip(tabs, (500, 640, 300)):
            assert torch_rows_equal(src, a, dst, b, (0, n), (0, 2))
        assert untouched_equal(dst, 22, mapped_mask(g, [(b, (0, n)) for (_, b), n in zip(tabs, (500, 640, 300))]))
    finally:
        for p in preps:
            dk.dyna_kv_prepared_destroy(p)


def test_overlap_flag_ignored_where_it_cannot_apply():
    """STAGED chains, dynamic scheduling and producer-coupled launches accept the flag and keep the wait."""
    g = Geom(2, 8, 128, 2, 16, 100)
    ts, td = kvgen.table_pair(2, 1000, g, g)
    hs, hd = kvgen.fill_bytes(1, g.pool_bytes), kvgen.fill_bytes(2, g.pool_bytes)
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (0, 1000))
    for kw in (dict(variant=dk.DYNA_VARIANT_STAGED), dict(engine=dk.DYNA_ENGINE_VEC, schedule=dk.DYNA_SCHED_DYNAMIC)):
        src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
        st, dt = dev_table(src, ts), dev_table(dst, td)
        xs = [dk.migrate(st, dt, (a, a + 250), (0, 2), 100, flags=OV, **kw) for a in range(0, 1000, 250)]
        for x in xs:
            dk.dyna_kv_wait(x)
        assert np.array_equal(dst.tensor.cpu().numpy(), want), kw


def test_auto_picks_vec_for_overlapped_calls():
    """AUTO's rule for overlapped calls (measured): the VEC engine — 8 KiB x U4 for
    2-KiB rows, 4 KiB x U8 below — except 8-KiB rows from 4096 tokens, which keep the ring."""
    for g, n, want in ((Geom(2, 8, 128, 2, 16, 300), 1024, (dk.DYNA_ENGINE_VEC, 8192)),
                       (Geom(2, 1, 128, 2, 16, 300), 2048, (dk.DYNA_ENGINE_VEC, 4096)),
                       (Geom(2, 32, 128, 2, 16, 300), 4096, (dk.DYNA_ENGINE_BULK, 32768))):
        src, dst = pool_filled(g, 1), pool_filled(g, 2)
        ts, td = kvgen.table_pair(3, n, g, g)
        st, dt = dev_table(src, ts), dev_table(dst, td)
        torch.cuda.synchronize()
        x = dk.migrate(st, dt, (0, n), (0, 2), n, flags=OV)
        plan = dk.dyna_kv_xfer_plan(x)
        dk.dyna_kv_wait(x)
        assert (plan["engine"], plan["piece_bytes"]) == want, (g, plan)
        assert torch_rows_equal(src, ts, dst, td, (0, n), (0, 2))
