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
