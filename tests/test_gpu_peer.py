"""The NVLink form in one process (source on cuda:0, destination pool on cuda:1, P2P): parity
against the oracle for every variant / engine, per-chunk flags raised in the peer's inbox, head
resharding across devices.  Skipped on a one-GPU box (the cross-process form over CUDA IPC is
covered on one GPU by test_ipc.py)."""
import itertools

import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import pool_from_host

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NVLink peer)")]

G = Geom(4, 8, 128, 2, 16, 400)


def _tab(pool, ids, dev):
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    return dk.table(pool, torch.from_numpy(ids).to(f"cuda:{dev}"), ids)


@pytest.mark.parametrize("variant,engine", list(itertools.product([1, 2], [1, 2, 3])))
@pytest.mark.parametrize("signal", [False, True])
def test_peer_parity(variant, engine, signal):
    ts, td = kvgen.table_pair(5, 3000, G, G)
    hs, hd = kvgen.fill_bytes(1, G.pool_bytes), kvgen.fill_bytes(2, G.pool_bytes)
    tr = (11, 2900)
    want = hd.copy()
    oracle.migrate(hs, G, ts, want, G, td, tr)
    dk.dyna_kv_enable_peer(0, 1)
    src, dst = pool_from_host(G, hs, device=0, instance=6), pool_from_host(G, hd, device=1)
    st = _tab(src, ts, 0)
    dt = _tab(dst, td, 0 if variant == 1 else 1)     # the fused kernel reads both tables on cuda:0
    torch.cuda.set_device(0)
    x = dk.dyna_kv_migrate_ex(st, dt, tr, (0, 4), 512, 0,
                              dk.opts(variant=variant, engine=engine, flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0))
    epoch, nck, sender, first = dk.dyna_kv_xfer_info(x)
    dk.dyna_kv_wait(x)
    torch.cuda.synchronize(1)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)
    if signal:
        fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
        with torch.cuda.device(1):
            dk.dyna_kv_copy_flags(dst.handle, sender, first, nck, fl.data_ptr(), 0)
            torch.cuda.synchronize()
        assert (fl.numpy() == epoch).all()


@pytest.mark.parametrize("engine", [0, 1, 2], ids=["auto", "vec", "tiles"])
def test_peer_head_reshard(engine):
    gd = G.with_(num_kv_heads=2, block_size=32, num_blocks=200)
    ts, _ = kvgen.table_pair(8, 3000, G, G)
    td = kvgen.table_pair(9, 3000, gd, gd)[1]
    hs, hd = kvgen.fill_bytes(3, G.pool_bytes), kvgen.fill_bytes(4, gd.pool_bytes)
    want = hd.copy()
    oracle.migrate_heads(hs, G, ts, want, gd, td, (0, 2500), None, (6, 8), 0)
    dk.dyna_kv_enable_peer(0, 1)
    src, dst = pool_from_host(G, hs, device=0), pool_from_host(gd, hd, device=1)
    torch.cuda.set_device(0)
    dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(_tab(src, ts, 0), _tab(dst, td, 0), (0, 2500), (0, 4), (6, 8), 0, 256, 0,
                                             dk.opts(engine=engine)))
    torch.cuda.synchronize(1)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


# ---------------------------------------------------------------- round 2: the NVLink forms the verdict listed
@pytest.mark.parametrize("engine", [dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK])
def test_peer_flag_litmus_consumer_on_destination_gpu(engine):
    """Flag protocol over NVLink (SURVEY §5 "prove it with a litmus stress test"): the consumer
    stream lives on cuda:1 (the destination's GPU), waits for chunk k's flag and at once snapshots
    chunk k's rows there, while the (slow: 2 CTAs) migration from cuda:0 still stores later chunks.
    Every snapshot must hold the source rows: a flag visible before its chunk's remote stores
    would show the zeros."""
    g = Geom(32, 8, 128, 2, 16, 200)
    rng = np.random.default_rng(77)
    hs = kvgen.fill_bytes(31, g.pool_bytes)
    dk.dyna_kv_enable_peer(0, 1)
    src = pool_from_host(g, hs, device=0, instance=6)
    dst = pool_from_host(g, np.zeros(g.pool_bytes, np.uint8), device=1)
    ts, td = kvgen.table_pair(33, 3000, g, g)
    s, row = 3000, g.row_bytes
    S = torch.from_numpy(hs).view(g.num_layers, 2, g.num_blocks, g.block_size, row)
    D = dst.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, row)
    Td = torch.as_tensor(td.astype(np.int64), device="cuda:1")
    st, dt = _tab(src, ts, 0), _tab(dst, td, 0)
    with torch.cuda.device(1):
        consumer = torch.cuda.Stream()
    for rep in range(6):
        c = int(rng.choice([64, 200, 512]))
        with torch.cuda.device(1):
            dst.tensor.zero_()
            torch.cuda.synchronize()
        torch.cuda.set_device(0)
        x = dk.migrate(st, dt, (0, s), (0, g.num_layers), c, engine=engine, max_ctas=2,
                       flags=dk.DYNA_MIGRATE_SIGNAL)
        epoch, nchunks, sender, first = dk.dyna_kv_xfer_info(x)
        snaps = {}
        with torch.cuda.device(1), torch.cuda.stream(consumer):
            for k in rng.permutation(nchunks):
                dk.dyna_kv_stream_wait_chunk(dst.handle, sender, first + int(k), epoch, 10_000_000_000,
                                             consumer.cuda_stream)
                t = torch.arange(int(k) * c, min((int(k) + 1) * c, s), device="cuda:1")
                snaps[int(k)] = D[:, :, Td[t // g.block_size], t % g.block_size].clone()
        consumer.synchronize()
        dk.dyna_kv_wait(x)
        dk.dyna_kv_poll_error()
        for k, snap in snaps.items():
            t = np.arange(k * c, min((k + 1) * c, s))
            want = S[:, :, torch.as_tensor(ts[t // g.block_size].astype(np.int64)),
                     torch.as_tensor(t % g.block_size)]
            assert torch.equal(snap.cpu(), want), (rep, c, k)


def test_peer_channel_push_place_across_devices():
    """Receiver-steered placement with the receiver on cuda:1: the sender on cuda:0 fills the
    receiver's slots over NVLink, the receiver places with its own table, flags on cuda:1."""
    hs, hd = kvgen.fill_bytes(1, G.pool_bytes), kvgen.fill_bytes(2, G.pool_bytes)
    ts, td = kvgen.table_pair(7, 5000, G, G)
    tr = (13, 4321)
    want = hd.copy()
    oracle.migrate(hs, G, ts, want, G, td, tr)
    dk.dyna_kv_enable_peer(0, 1)
    src, dst = pool_from_host(G, hs, device=0), pool_from_host(G, hd, device=1)
    ch = dk.dyna_kv_channel_create(dst.handle, 9, 3, 16 << 20)
    dk.dyna_kv_channel_set_timeout(ch, 120_000_000_000)
    try:
        st = _tab(src, ts, 0)
        dt = _tab(dst, td, 1)
        s_push = torch.cuda.Stream(device=0)
        with torch.cuda.device(1):
            s_place = torch.cuda.Stream()
        xp = dk.dyna_kv_push(st, tr, (0, 4), 700, ch, s_push.cuda_stream)
        with torch.cuda.device(1):
            xq = dk.dyna_kv_place(ch, dt, tr, (0, 4), 700, s_place.cuda_stream, dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL))
            epoch, nchunks, sender, first = dk.dyna_kv_xfer_info(xq)
        dk.dyna_kv_wait(xp)
        dk.dyna_kv_wait(xq)
        assert np.array_equal(dst.tensor.cpu().numpy(), want)
        fl = torch.zeros(nchunks, dtype=torch.int64).pin_memory()
        with torch.cuda.device(1):
            dk.dyna_kv_copy_flags(dst.handle, sender, first, nchunks, fl.data_ptr(), 0)
            torch.cuda.synchronize()
        assert (fl.numpy() == epoch).all()
    finally:
        dk.dyna_kv_channel_destroy(ch)


def test_peer_4prime_full_size():
    """The north-star shape over NVLink: one 4096-token Llama-3-8B chunk (512 MiB), fragmented
    tables, cuda:0 -> cuda:1, every engine; whole check by torch indexing on the destination GPU
    plus sampled rows against the oracle's offsets of the kvgen source stream."""
    from gpu_util import pool_filled, sampled_rows_match
    g = kvgen.LLAMA3_8B.with_(num_blocks=1024)
    dk.dyna_kv_enable_peer(0, 1)
    src = pool_filled(g, 81, device=0)
    dst = pool_filled(g, 82, device=1)
    ts, td = kvgen.table_pair(83, 4096, g, g)
    for engine in (0, dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK):
        torch.cuda.set_device(0)
        x = dk.migrate(_tab(src, ts, 0), _tab(dst, td, 0), (0, 4096), (0, 32), 4096, engine=engine,
                       flags=dk.DYNA_MIGRATE_SIGNAL)
        dk.dyna_kv_wait(x)
        torch.cuda.synchronize(1)
        S = src.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, g.row_bytes)
        D = dst.tensor.view_as(S)
        t = torch.arange(0, 4096)
        Ts, Td = torch.as_tensor(ts.astype(np.int64)), torch.as_tensor(td.astype(np.int64))
        got = D[:, :, Td.to("cuda:1")[t.to("cuda:1") // 16], t.to("cuda:1") % 16].cpu()
        want = S[:, :, Ts.to("cuda:0")[t.to("cuda:0") // 16], t.to("cuda:0") % 16].cpu()
        assert torch.equal(got, want), engine
        assert sampled_rows_match(81, g, ts, dst, g, td, (0, 4096), (0, 32), 64, np.random.default_rng(engine)) == 0


def _ipc_receiver_on_gpu1(q_handle, q_done):
    """Destination instance on cuda:1 (own process): export its pool, wait for the sender."""
    try:
        import torch as th
        import paper_2504_09285_b200 as dkk
        from gpu_util import pool_filled as pf
        th.cuda.set_device(1)
        dst = pf(Geom(4, 8, 128, 2, 16, 400), 72, device=1)
        th.cuda.synchronize()
        q_handle.put(dkk.dyna_kv_pool_export(dst.handle))
        info = q_done.get(timeout=300)
        epoch, nchunks, sender, first = info
        fl = th.zeros(nchunks, dtype=th.int64).pin_memory()
        dkk.dyna_kv_copy_flags(dst.handle, sender, first, nchunks, fl.data_ptr(), 0)
        th.cuda.synchronize()
        q_handle.put(("flags", bool((fl.numpy() == epoch).all()), dst.tensor.cpu().numpy()))
    except Exception as e:
        q_handle.put(("err", repr(e), None))


def test_peer_two_processes_over_ipc():
    """One process per GPU (the deployment shape): the receiver on cuda:1 exports its pool, the
    sender on cuda:0 imports it and pushes with per-chunk flags over NVLink; the receiver sees
    every flag at its epoch and the oracle's bytes."""
    import multiprocessing as mp
    g = Geom(4, 8, 128, 2, 16, 400)
    ctx = mp.get_context("spawn")
    qh, qd = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_ipc_receiver_on_gpu1, args=(qh, qd))
    p.start()
    handle = qh.get(timeout=300)
    hs = kvgen.fill_bytes(71, g.pool_bytes)
    ts, td = kvgen.table_pair(9, 4000, g, g)
    torch.cuda.set_device(0)
    src = pool_from_host(g, hs, device=0, instance=3)
    dst = dk.Pool.imported(handle, 0)
    x = dk.migrate(_tab(src, ts, 0), dk.table(dst, torch.from_numpy(td).to("cuda:0"), td), (0, 3001), (0, 4), 512,
                   engine=dk.DYNA_ENGINE_BULK, flags=dk.DYNA_MIGRATE_SIGNAL)
    info = dk.dyna_kv_xfer_info(x)
    dk.dyna_kv_wait(x)
    dst.close()
    qd.put(info)
    tag, ok, got = qh.get(timeout=300)
    p.join(timeout=60)
    assert tag == "flags", ok
    assert ok
    want = kvgen.fill_bytes(72, g.pool_bytes)
    oracle.migrate(hs, g, ts, want, g, td, (0, 3001))
    assert np.array_equal(got, want)
