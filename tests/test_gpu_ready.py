"""Producer-coupled push: one migration launch waits on the device for the
producer's per-chunk marks (§4.3).  The producer REWRITES each
chunk's source rows just before marking it, so a migration that did not wait
would copy stale bytes and fail the comparison."""
import numpy as np
import pytest
import torch

import kvgen
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, mapped_mask, pool_filled, torch_rows_equal, untouched_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _no_gc_during_coupled_waits():
    """A garbage-collected Pool left over from an earlier test destroys itself, and its inbox
    cudaFree synchronises the device: inside a coupled migration's wait window that deadlocks
    until the board's timeout (dyna_kv.h HAZARD).  Collect before each test, keep the collector
    off while it runs."""
    import gc
    gc.collect()
    gc.disable()
    try:
        yield
    finally:
        gc.enable()


def _produce_chunk(fresh_t, src_t, g, a, b, stream):
    """Stand-in producer for chunk [a, b): ~1 ms of "prefill compute", then the chunk's KV
    lands in the source pool (copied from `fresh` with the library's own fused kernel).
    Nothing here allocates device memory: a cudaMalloc that synchronises the device while
    the coupled migration waits would deadlock (see dyna_kv.h, producer-coupled push)."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000)
    x = dk.dyna_kv_migrate_ex(fresh_t, src_t, (a, b), (0, g.num_layers), b - a, stream.cuda_stream, None)
    return x


@pytest.mark.parametrize("c", [64, 100, 256])
@pytest.mark.parametrize("signal", [False, True])
def test_migration_waits_for_each_chunk(c, signal):
    g = Geom(4, 8, 128, 2, 16, 300)
    s = 1000
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    fresh = pool_filled(g, 3)                      # the values the producer will write
    ts, td = kvgen.table_pair(5, 1200, g, g)
    src_t, dst_t, fresh_t = dev_table(src, ts), dev_table(dst, td), dev_table(fresh, ts)
    prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
    board = dk.dyna_kv_ready_create(0, 64)
    dk.dyna_kv_ready_set_timeout(board, 20_000_000_000)
    # warm every library path used below so nothing allocates while the migration waits
    flags = dk.DYNA_MIGRATE_SIGNAL if signal else 0
    e0 = dk.dyna_kv_ready_begin(board)
    for k in range(-(-s // c)):
        dk.dyna_kv_ready_mark(board, k, e0, prod.cuda_stream)
    prod.synchronize()
    dk.dyna_kv_wait(dk.dyna_kv_migrate_on_ready(src_t, dst_t, (0, s), (0, 4), c, board, e0, mig.cuda_stream,
                                                dk.opts(max_ctas=8, flags=flags)))
    dk.dyna_kv_wait(_produce_chunk(fresh_t, src_t, g, 0, 1, prod))
    src = pool_filled(g, 1)                        # back to the stale values
    src_t = dev_table(src, ts)
    torch.cuda.synchronize()
    try:
        epoch = dk.dyna_kv_ready_begin(board)
        x = dk.dyna_kv_migrate_on_ready(src_t, dst_t, (0, s), (0, 4), c, board, epoch,
                                        mig.cuda_stream, dk.opts(max_ctas=8, flags=flags))
        nck = -(-s // c)
        px = []
        for k in range(nck):                         # prefill chunk k, then mark it ready
            px.append(_produce_chunk(fresh_t, src_t, g, k * c, min((k + 1) * c, s), prod))
            dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
        dk.dyna_kv_wait(x)
        for y in px:
            dk.dyna_kv_wait(y)
        torch.cuda.synchronize()
        assert torch_rows_equal(src, ts, dst, td, (0, s), (0, 4))        # fresh values arrived
        assert untouched_equal(dst, 2, mapped_mask(g, [(td, (0, s))]))
        # the same board serves the next request with a new epoch
        e2 = dk.dyna_kv_ready_begin(board)
        assert e2 == epoch + 1
    finally:
        dk.dyna_kv_ready_destroy(board)


def test_ready_errors():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    board = dk.dyna_kv_ready_create(0, 2)
    try:
        with pytest.raises(dk.DynaKVError) as e:       # 4 chunks > 2 slots
            dk.dyna_kv_migrate_on_ready(dev_table(src, ts), dev_table(dst, td), (0, 100), (0, 2), 32, board, 1)
        assert e.value.status == dk.DYNA_ERANGE
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_migrate_on_ready(dev_table(src, ts), dev_table(dst, td), (0, 50), (0, 2), 32, board, 1,
                                        opts=dk.opts(engine=dk.DYNA_ENGINE_BULK))
        assert e.value.status == dk.DYNA_ENOTSUP
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_ready_mark(board, 2, 1)
        assert e.value.status == dk.DYNA_ERANGE
    finally:
        dk.dyna_kv_ready_destroy(board)


def test_missing_mark_times_out_instead_of_hanging():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    board = dk.dyna_kv_ready_create(0, 8)
    try:
        dk.dyna_kv_ready_set_timeout(board, 2_000_000)          # 2 ms
        epoch = dk.dyna_kv_ready_begin(board)
        dk.dyna_kv_ready_mark(board, 0, epoch)                  # chunk 1..3 never marked
        x = dk.dyna_kv_migrate_on_ready(dev_table(src, ts), dev_table(dst, td), (0, 100), (0, 2), 32, board, epoch)
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_wait(x)
        assert e.value.status == dk.DYNA_ETIMEDOUT
    finally:
        dk.dyna_kv_ready_destroy(board)


_FRESH = r"""
import sys, torch
sys.path.insert(0, {root!r})
import kvgen, paper_2504_09285_b200 as dk
torch.cuda.set_device(0)
g = kvgen.TOY.with_(num_blocks=256)
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)          # first device use: the library preloads its kernels
ts, td = kvgen.table_pair(1, 1024, g, g)
st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
board = dk.dyna_kv_ready_create(0, 16)
dk.dyna_kv_ready_set_timeout(board, 5_000_000_000)
prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
with torch.cuda.stream(prod):
    torch.cuda._sleep(1000)                        # warm the producer's own kernel only
torch.cuda.synchronize()
epoch = dk.dyna_kv_ready_begin(board)
x = dk.dyna_kv_migrate_on_ready(st, dt, (0, 1000), (0, 2), 100, board, epoch, mig.cuda_stream, dk.opts(max_ctas=4))
for k in range(10):                                # first-ever k_mark_ready launches happen now
    with torch.cuda.stream(prod):
        torch.cuda._sleep(100000)
    dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
dk.dyna_kv_wait(x)
print("ok")
"""


def test_first_mark_during_wait_does_not_deadlock():
    """Regression: CUDA's lazy module loading synchronises the context; a first-ever launch of the
    mark kernel while the coupled migration waits used to deadlock (until the device timeout)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _FRESH.format(root=root)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


# ---------------------------------------------------------------- layer-granular marks

def _oracle_expect(fresh_seed, g, ts, dst_seed, td, tr, lr=None, rows=None):
    """Destination bytes the oracle computes from the fresh source values (host numpy)."""
    import oracle
    hs = kvgen.fill_bytes(fresh_seed, g.pool_bytes)
    want = kvgen.fill_bytes(dst_seed, g.pool_bytes)
    oracle.migrate(hs, g, ts, want, g, td, tr, lr)
    return want


@pytest.mark.parametrize("c", [64, 100])
def test_per_layer_marks_copy_each_layer_after_its_mark(c):
    """The producer rewrites layer l of chunk k, then marks slot k*lm + l; every row must
    arrive with the rewritten (fresh) bytes, bit-exact against the oracle."""
    g = Geom(4, 8, 128, 2, 16, 200)
    s, lm = 700, 4
    src, dst, fresh = pool_filled(g, 1), pool_filled(g, 2), pool_filled(g, 3)
    ts, td = kvgen.table_pair(6, 800, g, g)
    src_t, dst_t, fresh_t = dev_table(src, ts), dev_table(dst, td), dev_table(fresh, ts)
    prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
    nck = -(-s // c)
    board = dk.dyna_kv_ready_create(0, nck * lm)
    dk.dyna_kv_ready_set_timeout(board, 20_000_000_000)
    try:
        o = dk.opts(max_ctas=8, flags=dk.DYNA_MIGRATE_SIGNAL | dk.DYNA_READY_PER_LAYER)
        e0 = dk.dyna_kv_ready_begin(board)           # warm-up pass: every path runs once
        for k in range(nck * lm):
            dk.dyna_kv_ready_mark(board, k, e0, prod.cuda_stream)
        prod.synchronize()
        dk.dyna_kv_wait(dk.dyna_kv_migrate_on_ready(src_t, dst_t, (0, s), (0, lm), c, board, e0, mig.cuda_stream, o))
        # warm every kernel the producer will launch while the coupled migration waits (a first
        # launch loads its module lazily, which synchronises the context: dyna_kv.h HAZARD)
        with torch.cuda.stream(prod):
            torch.cuda._sleep(1000)
        for n in sorted({c, s - (nck - 1) * c}):
            dk.dyna_kv_wait(dk.dyna_kv_migrate_ex(fresh_t, src_t, (0, n), (0, 1), n, prod.cuda_stream, None))
        src = pool_filled(g, 1)
        dst = pool_filled(g, 2)
        src_t, dst_t = dev_table(src, ts), dev_table(dst, td)
        torch.cuda.synchronize()

        epoch = dk.dyna_kv_ready_begin(board)
        x = dk.dyna_kv_migrate_on_ready(src_t, dst_t, (0, s), (0, lm), c, board, epoch, mig.cuda_stream, o)
        info = dk.dyna_kv_xfer_info(x)
        px = []
        for k in range(nck):
            a, b = k * c, min((k + 1) * c, s)
            for l in range(lm):                       # layer l of chunk k: compute, write KV, mark
                with torch.cuda.stream(prod):
                    torch.cuda._sleep(200_000)
                px.append(dk.dyna_kv_migrate_ex(fresh_t, src_t, (a, b), (l, l + 1), b - a, prod.cuda_stream, None))
                dk.dyna_kv_ready_mark(board, dk.ready_slot(k, l, (0, lm)), epoch, prod.cuda_stream)
        dk.dyna_kv_wait(x)
        for y in px:
            dk.dyna_kv_wait(y)
        torch.cuda.synchronize()
        want = _oracle_expect(3, g, ts, 2, td, (0, s))
        assert np.array_equal(dst.tensor.cpu().numpy(), want)
        flags = torch.zeros(nck, dtype=torch.int64).pin_memory()
        dk.dyna_kv_copy_flags(dst.handle, info[2], info[3], nck, flags.data_ptr(), 0)
        torch.cuda.synchronize()
        assert int(flags.min()) == info[0]
    finally:
        dk.dyna_kv_ready_destroy(board)


def test_per_layer_errors():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    board = dk.dyna_kv_ready_create(0, 7)
    try:
        with pytest.raises(dk.DynaKVError) as e:       # 4 chunks x 2 layers > 7 slots
            dk.dyna_kv_migrate_on_ready(dev_table(src, ts), dev_table(dst, td), (0, 100), (0, 2), 32, board, 1,
                                        opts=dk.opts(flags=dk.DYNA_READY_PER_LAYER))
        assert e.value.status == dk.DYNA_ERANGE
        with pytest.raises(dk.DynaKVError) as e:       # per-layer marks need a board
            dk.dyna_kv_migrate_ex(dev_table(src, ts), dev_table(dst, td), (0, 100), (0, 2), 32, 0,
                                  dk.opts(flags=dk.DYNA_READY_PER_LAYER))
        assert e.value.status == dk.DYNA_EINVAL
        with pytest.raises(dk.DynaKVError) as e:       # unknown flag bits
            dk.dyna_kv_migrate_ex(dev_table(src, ts), dev_table(dst, td), (0, 100), (0, 2), 32, 0, dk.opts(flags=16))
        assert e.value.status == dk.DYNA_EINVAL
    finally:
        dk.dyna_kv_ready_destroy(board)


# ---------------------------------------------------------------- cancellation

@pytest.mark.parametrize("per_layer", [False, True])
def test_cancel_delivers_marked_chunks_and_stops(per_layer):
    """alpha ends early: chunks 0..m-1 were marked, the rest never will be.  After the cancel the
    migration returns at once with DYNA_ECANCELED; marked chunks are delivered whole with their
    flags, unmarked chunks have no flag, rows outside the range are untouched, and the channel's
    per-chunk counters are clean for the next signalled migration."""
    import time
    g = Geom(2, 8, 128, 2, 16, 160)
    s, c, m = 900, 128, 3
    lm = g.num_layers
    nck = -(-s // c)
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(7, 1000, g, g)
    src_t, dst_t = dev_table(src, ts), dev_table(dst, td)
    prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
    board = dk.dyna_kv_ready_create(0, nck * lm)
    dk.dyna_kv_ready_set_timeout(board, 30_000_000_000)   # a cancel must not wait for this
    flags = dk.DYNA_MIGRATE_SIGNAL | (dk.DYNA_READY_PER_LAYER if per_layer else 0)
    try:
        epoch = dk.dyna_kv_ready_begin(board)
        x = dk.dyna_kv_migrate_on_ready(src_t, dst_t, (0, s), (0, lm), c, board, epoch, mig.cuda_stream,
                                        dk.opts(max_ctas=8, flags=flags))
        ep, nchunks, sender, first = dk.dyna_kv_xfer_info(x)
        for k in range(m):
            for l in (range(lm) if per_layer else [0]):
                dk.dyna_kv_ready_mark(board, dk.ready_slot(k, l, (0, lm)) if per_layer else k, epoch,
                                      prod.cuda_stream)
        prod.synchronize()
        time.sleep(0.05)
        t = time.perf_counter()
        dk.dyna_kv_ready_cancel(board, epoch)
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_wait(x)
        assert e.value.status == dk.DYNA_ECANCELED
        assert time.perf_counter() - t < 5.0
        torch.cuda.synchronize()
        fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
        dk.dyna_kv_copy_flags(dst.handle, sender, first, nck, fl.data_ptr(), 0)
        torch.cuda.synchronize()
        got = fl.numpy()
        assert (got[:m] == ep).all() and (got[m:] < ep).all(), got
        want = _oracle_expect(1, g, ts, 2, td, (0, m * c))
        D = dst.tensor.cpu().numpy()
        marked = mapped_mask(g, [(td, (0, m * c))]).cpu().numpy()
        rows = D.reshape(marked.shape + (-1,))
        assert np.array_equal(rows[marked], want.reshape(rows.shape)[marked])        # delivered chunks
        assert untouched_equal(dst, 2, mapped_mask(g, [(td, (0, s))]))                 # outside the range
        # the next signalled migration over the same (src, dst) channel gets every flag
        dst2_seed = 2
        y = dk.dyna_kv_migrate_ex(src_t, dst_t, (0, s), (0, lm), c, 0, dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL))
        ep2, _, _, first2 = dk.dyna_kv_xfer_info(y)
        dk.dyna_kv_wait(y)
        dk.dyna_kv_copy_flags(dst.handle, sender, first2, nck, fl.data_ptr(), 0)
        torch.cuda.synchronize()
        assert (fl.numpy() == ep2).all()
        assert np.array_equal(dst.tensor.cpu().numpy(), _oracle_expect(1, g, ts, dst2_seed, td, (0, s)))
    finally:
        dk.dyna_kv_ready_destroy(board)


def test_cancel_before_launch_and_later_epochs_unaffected():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    board = dk.dyna_kv_ready_create(0, 8)
    try:
        dk.dyna_kv_ready_set_timeout(board, 30_000_000_000)
        e1 = dk.dyna_kv_ready_begin(board)
        dk.dyna_kv_ready_cancel(board, e1)
        x = dk.dyna_kv_migrate_on_ready(st, dt, (0, 100), (0, 2), 32, board, e1)   # nothing marked
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_wait(x)
        assert e.value.status == dk.DYNA_ECANCELED
        torch.cuda.synchronize()
        assert np.array_equal(dst.tensor.cpu().numpy(), kvgen.fill_bytes(2, g.pool_bytes))   # untouched
        dk.dyna_kv_ready_cancel(board, 0)                                           # monotone: no-op
        e2 = dk.dyna_kv_ready_begin(board)
        for k in range(4):
            dk.dyna_kv_ready_mark(board, k, e2)
        dk.dyna_kv_wait(dk.dyna_kv_migrate_on_ready(st, dt, (0, 100), (0, 2), 32, board, e2))
        assert np.array_equal(dst.tensor.cpu().numpy(), _oracle_expect(1, g, ts, 2, td, (0, 100)))
    finally:
        dk.dyna_kv_ready_destroy(board)


def test_destroy_during_coupled_wait_does_not_deadlock():
    """Destroying a pool, a ready board and a channel while a coupled migration waits for marks
    must not synchronise the device (their memory is retired, released by a later allocating call)."""
    import time
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    victim, victim_dst = pool_filled(g, 3), pool_filled(g, 4)
    ts, td = kvgen.table_pair(1, 256, g, g)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    vt, vdt = dev_table(victim, ts), dev_table(victim_dst, td)
    dk.dyna_kv_wait(dk.migrate(vt, vdt, (0, 100), (0, 2), 32, flags=dk.DYNA_MIGRATE_SIGNAL))  # channel counters
    ch = dk.dyna_kv_channel_create(victim_dst.handle, 5, 2, 1 << 16)
    other = dk.dyna_kv_ready_create(0, 4)
    board = dk.dyna_kv_ready_create(0, 8)
    dk.dyna_kv_ready_set_timeout(board, 30_000_000_000)
    prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
    try:
        torch.cuda.synchronize()
        epoch = dk.dyna_kv_ready_begin(board)
        x = dk.dyna_kv_migrate_on_ready(st, dt, (0, 100), (0, 2), 32, board, epoch, mig.cuda_stream,
                                        dk.opts(max_ctas=2))
        t = time.perf_counter()
        victim.close()                        # inbox + channel counters retired, not freed
        victim_dst.close()
        dk.dyna_kv_channel_destroy(ch)
        dk.dyna_kv_ready_destroy(other)
        for k in range(4):
            dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
        dk.dyna_kv_wait(x)
        assert time.perf_counter() - t < 10.0
        torch.cuda.synchronize()
        want = kvgen.fill_bytes(2, g.pool_bytes)
        import oracle
        oracle.migrate(kvgen.fill_bytes(1, g.pool_bytes), g, ts, want, g, td, (0, 100))
        assert np.array_equal(dst.tensor.cpu().numpy(), want)
        extra = pool_filled(g, 9)             # an allocating call releases the retired memory
        extra.close()
    finally:
        dk.dyna_kv_ready_destroy(board)


def test_first_use_of_a_channel_during_coupled_wait_does_not_deadlock():
    """While a producer-coupled migration waits on the device for its marks, the FIRST signalled
    (and small-row, tiled) migration of a new pool pair allocates that pair's chunk counters and
    fills the source pool's tile-map cache.  Those fills run on a non-blocking library stream and
    are waited for on the host; a legacy-stream cudaMemset there would wait for the coupled
    kernel, whose marks this thread only issues afterwards (a deadlock until the board timeout)."""
    import time
    g = Geom(4, 8, 128, 2, 16, 300)
    gs = Geom(3, 1, 128, 2, 16, 300)                     # 256-B rows: AUTO tiles
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(5, 1200, g, g)
    a, b = pool_filled(gs, 3), pool_filled(gs, 4)        # a pair never used before
    ta, tb = kvgen.table_pair(6, 3200, gs, gs)
    prod = torch.cuda.Stream()
    side = torch.cuda.Stream()
    board = dk.dyna_kv_ready_create(0, 64)
    dk.dyna_kv_ready_set_timeout(board, 8_000_000_000)
    # every torch allocation / copy before the coupled launch: torch's own H2D copies run on the
    # legacy stream, which the coupled kernel below occupies until its marks arrive
    st, dt, at, bt = dev_table(src, ts), dev_table(dst, td), dev_table(a, ta), dev_table(b, tb)
    torch.cuda.synchronize()
    epoch = dk.dyna_kv_ready_begin(board)
    x = dk.dyna_kv_migrate_on_ready(st, dt, (0, 1000), (0, 4), 250, board, epoch,
                                    torch.cuda.default_stream().cuda_stream, dk.opts(max_ctas=8))
    t0 = time.perf_counter()
    y = dk.dyna_kv_migrate_ex(at, bt, (0, 3000), (0, 3), 750, side.cuda_stream, dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL))
    issue_s = time.perf_counter() - t0
    for k in range(4):
        dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
    dk.dyna_kv_wait(y)
    dk.dyna_kv_wait(x)                                   # DYNA_ETIMEDOUT here would mean the fill blocked
    assert issue_s < 4.0, issue_s
    assert torch_rows_equal(src, ts, dst, td, (0, 1000), (0, 4))
    assert torch_rows_equal(a, ta, b, tb, (0, 3000), (0, 3))
    dk.dyna_kv_ready_destroy(board)
