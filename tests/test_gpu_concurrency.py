"""Concurrent use of the library (round-2 fixes):
per-migration deferred errors, disjoint per-chunk flag slots for concurrent signalled
migrations and interleaved chunk streams, the staged variant's staging lease, alias checks
without host ids and across batch entries, and a timed-out producer wait raising no flag."""
import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, pool_filled, pool_from_host, torch_rows_equal

pytestmark = pytest.mark.gpu


def _flags(pool, sender, first, n):
    fl = torch.zeros(max(n, 1), dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(pool.handle, sender, first, n, fl.data_ptr(), 0)
    torch.cuda.synchronize()
    return fl.numpy()[:n]


@pytest.mark.parametrize("bad_first", [False, True])
@pytest.mark.parametrize("engine", [dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK])
def test_deferred_errors_are_per_migration(bad_first, engine):
    """Two migrations in flight at once on two streams, one with an out-of-range device-side
    block id: its wait returns DYNA_ERANGE, the other's DYNA_OK, whichever is waited first."""
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    td2 = kvgen.table_pair(2, 256, g, g)[1]
    bad = td.copy()
    bad[2] = g.num_blocks + 7
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        torch.cuda._sleep(20_000_000)       # both in flight together
    good_t = (dev_table(src, ts, False), dev_table(dst, td2, False))
    bad_t = (dev_table(src, ts, False), dev_table(dst, bad, False))
    o = dict(engine=engine, flags=dk.DYNA_MIGRATE_UNCHECKED)
    xb = dk.migrate(*bad_t, (0, 100), (0, 2), 32, stream=s1, **o)
    xg = dk.migrate(*good_t, (100, 200), (0, 2), 32, stream=s2, **o)
    order = [(xb, dk.DYNA_ERANGE), (xg, dk.DYNA_OK)]
    if not bad_first:
        order.reverse()
    for x, want in order:
        if want == dk.DYNA_OK:
            dk.dyna_kv_wait(x)
        else:
            with pytest.raises(dk.DynaKVError) as e:
                dk.dyna_kv_wait(x)
            assert e.value.status == want
    dk.dyna_kv_poll_error()                  # nothing left on the process-wide word


def test_concurrent_signalled_migrations_get_disjoint_slots():
    """Signalled migrations from one sender into one pool on four streams at once: every one gets
    its own slot range, and after all waits each range holds exactly its own epoch."""
    g = Geom(2, 8, 128, 2, 16, 1200)
    src, dst = pool_filled(g, 3, instance=4), pool_filled(g, 4)
    tabs = kvgen.batch_tables(9, [1000] * 4, g, g)
    streams = [torch.cuda.Stream() for _ in tabs]
    keep, xs = [], []
    for (ts, td), st in zip(tabs, streams):
        t = (dev_table(src, ts), dev_table(dst, td))
        keep.append(t)
        xs.append(dk.migrate(*t, (0, 1000), (0, 2), 96, stream=st, flags=dk.DYNA_MIGRATE_SIGNAL))
    infos = [dk.dyna_kv_xfer_info(x) for x in xs]
    for x in xs:
        dk.dyna_kv_wait(x)
    spans = sorted((f, f + n) for _, n, _, f in infos)
    assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:])), spans
    assert len({e for e, _, _, _ in infos}) == 4
    for epoch, n, sender, first in infos:
        assert (_flags(dst, sender, first, n) == epoch).all()
    for ts, td in tabs:
        assert torch_rows_equal(src, ts, dst, td, (0, 1000), (0, 2))


def test_interleaved_chunk_streams_one_stream():
    """two open chunk streams from one instance into one pool, pushes
    interleaved on ONE CUDA stream.  Each stream's chunk flags live in its own slots: waiting on
    stream A's chunk k is never satisfied by stream B's chunk k."""
    g = Geom(2, 8, 128, 2, 16, 600)
    hs, hd = kvgen.fill_bytes(51, g.pool_bytes), kvgen.fill_bytes(52, g.pool_bytes)
    tabs = kvgen.batch_tables(13, [1024, 1024], g, g)
    want = hd.copy()
    for ts, td in tabs:
        oracle.migrate(hs, g, ts, want, g, td, (0, 1000))
    src, dst = pool_from_host(g, hs, instance=6), pool_from_host(g, hd)
    T = [(dev_table(src, ts), dev_table(dst, td)) for ts, td in tabs]
    o = dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL)
    cs = [dk.dyna_kv_chunkstream_open(st, dt, 0, (0, 2), 128, 0, o) for st, dt in T]
    for step in (256, 128, 300, 316):
        for s in cs:
            dk.dyna_kv_chunkstream_produced(s, step)
    for s in cs:
        dk.dyna_kv_chunkstream_close(s)
    infos = [dk.dyna_kv_chunkstream_info(s) for s in cs]
    for s in cs:
        dk.dyna_kv_chunkstream_finish(s)
    a, b = infos
    assert a["epoch"] != b["epoch"]
    ra = set(range(a["first_slot"], a["first_slot"] + 8))
    rb = set(range(b["first_slot"], b["first_slot"] + 8))
    assert not ra & rb
    for i in infos:
        assert (_flags(dst, i["sender"], i["first_slot"], 8) == i["epoch"]).all()
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_staged_migrations_on_two_streams_share_staging_safely():
    """STAGED migrations of one (source, destination) pair on two streams use
    the pair's staging slots one after the other (the second is ordered after the first)."""
    g = Geom(4, 8, 128, 2, 16, 900)
    hs, hd = kvgen.fill_bytes(61, g.pool_bytes), kvgen.fill_bytes(62, g.pool_bytes)
    tabs = kvgen.batch_tables(17, [3000, 3000], g, g)
    want = hd.copy()
    for ts, td in tabs:
        oracle.migrate(hs, g, ts, want, g, td, (0, 3000))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    T = [(dev_table(src, ts), dev_table(dst, td)) for ts, td in tabs]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    xs = [dk.migrate(*T[0], (0, 3000), (0, 4), 1024, stream=s1, variant=dk.DYNA_VARIANT_STAGED, max_ctas=4),
          dk.migrate(*T[1], (0, 3000), (0, 4), 1024, stream=s2, variant=dk.DYNA_VARIANT_STAGED)]
    for x in xs:
        dk.dyna_kv_wait(x)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_alias_rules_without_host_ids_and_across_batch_entries():
    """Reading R7 enforced in every form: a destination table without host ids needs
    DYNA_MIGRATE_UNCHECKED; two batch entries writing one row, or one entry reading a row
    another entry writes, are refused; distinct pool objects over overlapping memory too."""
    g = kvgen.TOY                                            # 64 blocks of 16 tokens per pool
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, ts2 = np.arange(0, 16, dtype=np.int32), np.arange(16, 32, dtype=np.int32)
    td, td2 = np.arange(20, 36, dtype=np.int32), np.arange(40, 56, dtype=np.int32)

    def expect(status, fn):
        with pytest.raises(dk.DynaKVError) as e:
            fn()
        assert e.value.status == status, e.value

    expect(dk.DYNA_EINVAL, lambda: dk.migrate(dev_table(src, ts), dev_table(dst, td, False), (0, 100), (0, 2), 32))
    dk.dyna_kv_wait(dk.migrate(dev_table(src, ts), dev_table(dst, td, False), (0, 100), (0, 2), 32,
                               flags=dk.DYNA_MIGRATE_UNCHECKED))
    # same pool on both sides: the source table needs host ids too
    expect(dk.DYNA_EINVAL, lambda: dk.migrate(dev_table(src, ts, False), dev_table(src, td), (0, 100), (0, 2), 32))
    # batch: two entries write the same destination block
    overlap = td2.copy()
    overlap[0] = td[3]
    expect(dk.DYNA_EALIAS, lambda: dk.migrate_batch(
        [(dev_table(src, ts), dev_table(dst, td), (0, 100)), (dev_table(src, ts2), dev_table(dst, overlap), (0, 100))],
        (0, 2), 32))
    # batch: entry 1 writes rows of `src` that entry 0 reads
    expect(dk.DYNA_EALIAS, lambda: dk.migrate_batch(
        [(dev_table(src, ts), dev_table(dst, td), (0, 100)), (dev_table(dst, td2), dev_table(src, ts), (0, 40))],
        (0, 2), 32))
    # ... but rows of one block that do not overlap are fine: [0, 10) and [10, 20) of block ts[0]
    dk.dyna_kv_wait(dk.migrate_batch(
        [(dev_table(dst, td2), dev_table(src, ts), (0, 10)), (dev_table(src, ts), dev_table(dst, td), (10, 20))],
        (0, 2), 32))
    # two pool objects over overlapping memory (not the same pool)
    big = torch.zeros(g.pool_bytes + 4096, dtype=torch.uint8, device="cuda")
    p1, p2 = dk.Pool(g, 0, tensor=big), dk.Pool(g, 0, tensor=big[4096:])
    expect(dk.DYNA_EALIAS, lambda: dk.migrate(dev_table(p1, ts), dev_table(p2, td), (0, 100), (0, 2), 32))


def test_ready_wait_timeout_raises_no_flag():
    """a producer-coupled chunk whose mark never comes times out; the chunk is
    skipped and gets no flag (before, its flag was raised over rows never marked)."""
    g = kvgen.TOY
    src, dst = pool_filled(g, 1, instance=2), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    board = dk.dyna_kv_ready_create(0, 8)
    dk.dyna_kv_ready_set_timeout(board, 50_000_000)         # 50 ms
    try:
        epoch = dk.dyna_kv_ready_begin(board)
        prod = torch.cuda.Stream()
        dk.dyna_kv_ready_mark(board, 0, epoch, prod.cuda_stream)   # chunk 0 marked, chunk 1 never
        prod.synchronize()
        x = dk.dyna_kv_migrate_on_ready(st, dt, (0, 64), (0, 2), 32, board, epoch, 0,
                                        dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL, max_ctas=2))
        ep, n, sender, first = dk.dyna_kv_xfer_info(x)
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_wait(x)
        assert e.value.status == dk.DYNA_ETIMEDOUT
        fl = _flags(dst, sender, first, n)
        assert fl[0] == ep and fl[1] < ep, fl
    finally:
        dk.dyna_kv_ready_destroy(board)
