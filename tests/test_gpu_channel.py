"""Receiver-steered placement through a channel (push on the sender, place on the
receiver with its own block table) — bit-exact vs the oracle, in one process
(two streams, loopback) and across two processes (CUDA IPC)."""
import multiprocessing as mp

import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, pool_from_host

pytestmark = pytest.mark.gpu
G = Geom(4, 8, 128, 2, 16, 400)     # 2 KiB rows


@pytest.mark.parametrize("slots,slot_bytes,c", [(2, 4 * 2 * 4 * 2048 * 16, 100), (3, 1 << 20, 256), (4, 1 << 22, 1000)])
@pytest.mark.parametrize("signal", [False, True])
def test_push_place_loopback(slots, slot_bytes, c, signal):
    ts, td = kvgen.table_pair(7, 5000, G, G)
    hs, hd = kvgen.fill_bytes(1, G.pool_bytes), kvgen.fill_bytes(2, G.pool_bytes)
    tr = (13, 4321)
    want = hd.copy()
    oracle.migrate(hs, G, ts, want, G, td, tr)
    src, dst = pool_from_host(G, hs), pool_from_host(G, hd)
    ch = dk.dyna_kv_channel_create(dst.handle, 9, slots, slot_bytes)
    dk.dyna_kv_channel_set_timeout(ch, 120_000_000_000)   # a slow shared box must not turn into ETIMEDOUT
    try:
        s_push, s_place = torch.cuda.Stream(), torch.cuda.Stream()
        # tables must outlive the enqueued work (dyna_block_table contract): keep them in variables
        st, dt = dev_table(src, ts), dev_table(dst, td)
        for rep in range(2):   # the channel's sequence numbers carry over between migrations
            xp = dk.dyna_kv_push(st, tr, (0, 4), c, ch, s_push.cuda_stream)
            xq = dk.dyna_kv_place(ch, dt, tr, (0, 4), c, s_place.cuda_stream,
                                  dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0))
            epoch, nchunks, sender, first = dk.dyna_kv_xfer_info(xq)
            dk.dyna_kv_wait(xp)
            dk.dyna_kv_wait(xq)
            assert np.array_equal(dst.tensor.cpu().numpy(), want)
            if signal:
                flags = torch.zeros(nchunks, dtype=torch.int64).pin_memory()
                dk.dyna_kv_copy_flags(dst.handle, sender, first, nchunks, flags.data_ptr(), 0)
                torch.cuda.synchronize()
                assert sender == 9 and (flags.numpy() == epoch).all()
            dst.tensor.copy_(torch.from_numpy(hd).cuda())
            torch.cuda.synchronize()   # torch side streams are non-blocking: finish the reset first
    finally:
        dk.dyna_kv_channel_destroy(ch)


def test_channel_errors():
    src, dst = pool_from_host(G, kvgen.fill_bytes(1, G.pool_bytes)), pool_from_host(G, kvgen.fill_bytes(2, G.pool_bytes))
    ts, td = kvgen.table_pair(7, 5000, G, G)
    with pytest.raises(dk.DynaKVError):
        dk.dyna_kv_channel_create(dst.handle, 0, 1, 1 << 20)          # slots >= 2
    ch = dk.dyna_kv_channel_create(dst.handle, 0, 2, 4096)          # 4 KiB slots: < one token of 4 layers
    try:
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_push(dev_table(src, ts), (0, 10), (0, 4), 4, ch)
        assert e.value.status == dk.DYNA_EINVAL
        other = pool_from_host(G, kvgen.fill_bytes(3, G.pool_bytes))
        with pytest.raises(dk.DynaKVError):
            dk.dyna_kv_place(ch, dev_table(other, td), (0, 10), (0, 1), 4)   # not the channel's pool
    finally:
        dk.dyna_kv_channel_destroy(ch)


def _sender(handle, q):
    try:
        import torch
        import kvgen
        import paper_2504_09285_b200 as dk
        from gpu_util import dev_table, pool_from_host
        torch.cuda.set_device(0)
        src = pool_from_host(G, kvgen.fill_bytes(1, G.pool_bytes), instance=3)
        ts, _ = kvgen.table_pair(7, 5000, G, G)
        ch = dk.dyna_kv_channel_import(handle, 0)
        dk.dyna_kv_channel_set_timeout(ch, 120_000_000_000)
        q.put("ready")
        st = dev_table(src, ts)
        x = dk.dyna_kv_push(st, (0, 3000), (0, 4), 512, ch, torch.cuda.current_stream().cuda_stream)
        dk.dyna_kv_wait(x)
        dk.dyna_kv_channel_destroy(ch)
        q.put("ok")
    except Exception as e:  # surface to the parent
        q.put(repr(e))


def test_push_place_across_processes():
    ts, td = kvgen.table_pair(7, 5000, G, G)
    hs, hd = kvgen.fill_bytes(1, G.pool_bytes), kvgen.fill_bytes(2, G.pool_bytes)
    want = hd.copy()
    oracle.migrate(hs, G, ts, want, G, td, (0, 3000))
    dst = pool_from_host(G, hd)
    ch = dk.dyna_kv_channel_create(dst.handle, 3, 8, 1 << 23)   # 8 x 8 MiB: the sender never waits for credit
    dk.dyna_kv_channel_set_timeout(ch, 120_000_000_000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_sender, args=(dk.dyna_kv_channel_export(ch), q))
    p.start()
    assert q.get(timeout=300) == "ready"
    # On one GPU the receiver's place kernel is launched only after the sender's push finished:
    # kernels of two processes that spin on each other's words are not guaranteed to be
    # co-scheduled on one device (B200_PROFILING: Xid 109 under context switching).  Every slot
    # is full by then, so place finds each full word already raised; on two GPUs the two
    # processes run concurrently (test_gpu_peer.py).
    assert q.get(timeout=300) == "ok"
    p.join(timeout=60)
    dt = dev_table(dst, td)
    x = dk.dyna_kv_place(ch, dt, (0, 3000), (0, 4), 512)
    dk.dyna_kv_wait(x)
    dk.dyna_kv_channel_destroy(ch)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


@pytest.mark.parametrize("slots,slot_bytes,c", [(2, 4 * 2 * 2 * 1024 * 8, 100), (3, 1 << 20, 256)])
@pytest.mark.parametrize("signal", [False, True])
def test_push_place_heads_tp1_to_tp2(slots, slot_bytes, c, signal):
    """Receiver-steered TP resharding (reading R14): a TP-1 sender (8 heads) feeds two TP-2
    receivers (4 heads each) through their own channels; each receiver places with its own
    table.  Bit-exact against oracle.migrate_heads, flags per receiver."""
    gd = G.with_(num_kv_heads=4, block_size=32, num_blocks=200)
    ts, _ = kvgen.table_pair(17, 5000, G, G)
    hs = kvgen.fill_bytes(1, G.pool_bytes)
    tr = (7, 3333)
    src = pool_from_host(G, hs)
    st = dev_table(src, ts)
    keep = []
    for r in range(2):
        hd = kvgen.fill_bytes(10 + r, gd.pool_bytes)
        td = kvgen.table_pair(20 + r, 5000, gd, gd)[1]
        want = hd.copy()
        oracle.migrate_heads(hs, G, ts, want, gd, td, tr, None, (4 * r, 4 * r + 4), 0)
        dst = pool_from_host(gd, hd)
        ch = dk.dyna_kv_channel_create(dst.handle, 3, slots, slot_bytes)
        dk.dyna_kv_channel_set_timeout(ch, 120_000_000_000)
        try:
            s_push, s_place = torch.cuda.Stream(), torch.cuda.Stream()
            dt = dev_table(dst, td)
            keep.append((dt, dst))
            xp = dk.dyna_kv_push_heads(st, tr, (0, 4), (4 * r, 4 * r + 4), c, ch, s_push.cuda_stream)
            xq = dk.dyna_kv_place_heads(ch, dt, tr, (0, 4), 0, 4, c, s_place.cuda_stream,
                                        dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0))
            epoch, nchunks, sender, first = dk.dyna_kv_xfer_info(xq)
            dk.dyna_kv_wait(xp)
            dk.dyna_kv_wait(xq)
            assert np.array_equal(dst.tensor.cpu().numpy(), want)
            if signal:
                flags = torch.zeros(nchunks, dtype=torch.int64).pin_memory()
                dk.dyna_kv_copy_flags(dst.handle, sender, first, nchunks, flags.data_ptr(), 0)
                torch.cuda.synchronize()
                assert sender == 3 and (flags.numpy() == epoch).all()
        finally:
            dk.dyna_kv_channel_destroy(ch)


def test_push_place_heads_errors():
    gd = G.with_(num_kv_heads=4)
    src, dst = pool_from_host(G, kvgen.fill_bytes(1, G.pool_bytes)), pool_from_host(gd, kvgen.fill_bytes(2, gd.pool_bytes))
    ts, td = kvgen.table_pair(7, 1000, G, gd)
    ch = dk.dyna_kv_channel_create(dst.handle, 0, 2, 1 << 20)
    try:
        for heads in [(0, 9), (6, 9), (3, 3)]:
            with pytest.raises(dk.DynaKVError) as e:
                dk.dyna_kv_push_heads(dev_table(src, ts), (0, 100), (0, 4), heads, 32, ch, 0)
            assert e.value.status == dk.DYNA_ERANGE
        with pytest.raises(dk.DynaKVError) as e:        # receiver heads outside its pool
            dk.dyna_kv_place_heads(ch, dev_table(dst, td), (0, 100), (0, 4), 2, 4, 32, 0)
        assert e.value.status == dk.DYNA_ERANGE
        with pytest.raises(dk.DynaKVError) as e:        # whole-row push into a 4-head channel: geometry differs
            dk.dyna_kv_push(dev_table(src, ts), (0, 100), (0, 4), 32, ch, 0)
        assert e.value.status == dk.DYNA_EGEOM
    finally:
        dk.dyna_kv_channel_destroy(ch)
