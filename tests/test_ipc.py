"""Cross-process path on one GPU: the destination instance exports its pool over
CUDA IPC, the source instance (another process) imports it and pushes its
request's KV into it with per-chunk flags (§3.1, §4.3).

On the 8-GPU box the two processes sit on different GPUs and the same kernel
stores over NVLink; here both map the same B200, which exercises the export /
import / offset / inbox / system-scope-fence logic end to end.
"""
import multiprocessing as mp

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SRC_SEED, DST_SEED, SENDER = 71, 72, 3
S, CHUNK = 3001, 512


def _geom():
    from kvgen import Geom
    return Geom(4, 8, 128, 2, 16, 400)


def _sender(handle: bytes, q, engine: int, reps: int = 1):
    try:
        import torch

        import kvgen
        import paper_2504_09285_b200 as dk
        from gpu_util import dev_table, pool_filled
        torch.cuda.set_device(0)
        g = _geom()
        src = pool_filled(g, SRC_SEED, instance=SENDER)
        dst = dk.Pool.imported(handle, 0)
        ts, td = kvgen.table_pair(9, 4000, g, g)
        src_t = dev_table(src, ts)
        dst_t = dk.table(dst, torch.from_numpy(td).cuda(), td)
        for _ in range(reps):
            x = dk.migrate(src_t, dst_t, (0, S), (0, 4), CHUNK, engine=engine, flags=dk.DYNA_MIGRATE_SIGNAL)
            info = dk.dyna_kv_xfer_info(x)
            dk.dyna_kv_wait(x)
        dst.close()
        q.put(("ok", info))
    except Exception as e:  # surface the failure to the parent
        q.put(("err", repr(e)))


@pytest.mark.parametrize("engine", [1, 2])
def test_ipc_push_with_chunk_flags(engine):
    import torch

    import kvgen
    import paper_2504_09285_b200 as dk
    from gpu_util import pool_filled, torch_rows_equal, untouched_equal, mapped_mask
    torch.cuda.set_device(0)
    g = _geom()
    dst = pool_filled(g, DST_SEED)
    torch.cuda.synchronize()
    handle = dk.dyna_kv_pool_export(dst.handle)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_sender, args=(handle, q, engine))
    p.start()
    status, info = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", info
    epoch, nchunks, sender, first = info
    assert sender == SENDER and nchunks == -(-S // CHUNK) and epoch >= 1
    # the owner waits on every chunk flag (already released) and reads them back
    st = torch.cuda.current_stream()
    for k in range(nchunks):
        dk.dyna_kv_stream_wait_chunk(dst.handle, sender, first + k, epoch, 2_000_000_000, st.cuda_stream)
    flags = torch.zeros(nchunks, dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(dst.handle, sender, first, nchunks, flags.data_ptr(), st.cuda_stream)
    torch.cuda.synchronize()
    dk.dyna_kv_poll_error()
    assert (flags.numpy() == epoch).all()
    # contents: the sender's source pool is the kvgen stream SRC_SEED; rebuild it here to compare
    src = pool_filled(g, SRC_SEED)
    ts, td = kvgen.table_pair(9, 4000, g, g)
    assert torch_rows_equal(src, ts, dst, td, (0, S), (0, 4))
    assert untouched_equal(dst, DST_SEED, mapped_mask(g, [(td, (0, S))]))


def _heads_sender(handle: bytes, q, engine: int = 0):
    """TP-1 sender (8 heads) pushes heads [4, 8) into the importer's TP-2 rank-1 pool (4 heads)."""
    try:
        import torch

        import kvgen
        import paper_2504_09285_b200 as dk
        from gpu_util import dev_table, pool_filled
        torch.cuda.set_device(0)
        g = _geom()
        src = pool_filled(g, SRC_SEED, instance=SENDER)
        dst = dk.Pool.imported(handle, 0)
        ts, _ = kvgen.table_pair(9, 4000, g, g)
        _, td = kvgen.table_pair(10, 4000, g.with_(num_kv_heads=4), g.with_(num_kv_heads=4))
        x = dk.dyna_kv_migrate_heads(dev_table(src, ts), dk.table(dst, torch.from_numpy(td).cuda(), td), (0, S),
                                     (0, 4), (4, 8), 0, CHUNK, 0, dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL, engine=engine))
        info = dk.dyna_kv_xfer_info(x)
        assert engine != dk.DYNA_ENGINE_BULK or dk.dyna_kv_xfer_plan(x)["engine"] == dk.DYNA_ENGINE_TILES
        dk.dyna_kv_wait(x)
        dst.close()
        q.put(("ok", info))
    except Exception as e:
        q.put(("err", repr(e)))


@pytest.mark.parametrize("engine", [0, 2], ids=["auto", "tiles"])
def test_ipc_head_reshard_with_chunk_flags(engine):
    """TP resharding across processes (reading R14): bit-exact against oracle.migrate_heads.  AUTO keeps
    an imported destination on VEC; explicit BULK runs the TMA tile kernel's tensor stores into the
    IPC-mapped pool (on a multi-GPU box: over NVLink)."""
    import torch

    import kvgen
    import oracle
    import paper_2504_09285_b200 as dk
    from gpu_util import pool_filled
    torch.cuda.set_device(0)
    g = _geom()
    gd = g.with_(num_kv_heads=4)
    dst = pool_filled(gd, DST_SEED)
    torch.cuda.synchronize()
    handle = dk.dyna_kv_pool_export(dst.handle)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_heads_sender, args=(handle, q, engine))
    p.start()
    status, info = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", info
    epoch, nchunks, sender, first = info
    flags = torch.zeros(nchunks, dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(dst.handle, sender, first, nchunks, flags.data_ptr(), 0)
    torch.cuda.synchronize()
    assert (flags.numpy() == epoch).all()
    ts, _ = kvgen.table_pair(9, 4000, g, g)
    _, td = kvgen.table_pair(10, 4000, gd, gd)
    want = kvgen.fill_bytes(DST_SEED, gd.pool_bytes)
    oracle.migrate_heads(kvgen.fill_bytes(SRC_SEED, g.pool_bytes), g, ts, want, gd, td, (0, S), None, (4, 8), 0)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_restarted_sender_never_reuses_an_epoch():
    """epochs were counted per importing process from 1, so a restarted
    sender (same instance id, fresh import of the same pool) handed out epochs that stale
    flags of its previous incarnation already satisfied.  Epochs now start above the inbox
    row's largest flag: the second process's epoch exceeds every epoch of the first."""
    import torch

    import paper_2504_09285_b200 as dk
    from gpu_util import pool_filled
    torch.cuda.set_device(0)
    dst = pool_filled(_geom(), DST_SEED)
    torch.cuda.synchronize()
    handle = dk.dyna_kv_pool_export(dst.handle)
    ctx = mp.get_context("spawn")
    infos = []
    for reps in (3, 1):                       # first incarnation: three migrations; then a restart
        q = ctx.Queue()
        p = ctx.Process(target=_sender, args=(handle, q, 2, reps))
        p.start()
        status, info = q.get(timeout=300)
        p.join(timeout=60)
        assert status == "ok", info
        infos.append(info)
    assert infos[1][0] > infos[0][0], infos
