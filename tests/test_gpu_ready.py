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


def _produce_chunk(src, g, ts, a, b, fresh, stream):
    """Stand-in producer: write tokens [a, b) of the request (all layers, K and V) from `fresh`."""
    with torch.cuda.stream(stream):
        torch.cuda._sleep(2_000_000)  # ~1 ms of "prefill compute" before the KV lands
        S = src.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, g.row_bytes)
        F = fresh.view_as(S)
        t = torch.arange(a, b, device="cuda")
        T = torch.as_tensor(ts, device="cuda").long()
        idx = (slice(None), slice(None), T[t // g.block_size], t % g.block_size)
        S[idx] = F[idx]


@pytest.mark.parametrize("c", [64, 100, 256])
@pytest.mark.parametrize("signal", [False, True])
def test_migration_waits_for_each_chunk(c, signal):
    g = Geom(4, 8, 128, 2, 16, 300)
    s = 1000
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    fresh = pool_filled(g, 3).tensor               # the values the producer will write
    ts, td = kvgen.table_pair(5, 1200, g, g)
    torch.cuda.synchronize()
    board = dk.dyna_kv_ready_create(0, 64)
    try:
        prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
        epoch = dk.dyna_kv_ready_begin(board)
        flags = dk.DYNA_MIGRATE_SIGNAL if signal else 0
        x = dk.dyna_kv_migrate_on_ready(dev_table(src, ts), dev_table(dst, td), (0, s), (0, 4), c, board, epoch,
                                        mig.cuda_stream, dk.opts(max_ctas=8, flags=flags))
        nck = -(-s // c)
        for k in range(nck):                         # prefill chunk k, then mark it ready
            _produce_chunk(src, g, ts, k * c, min((k + 1) * c, s), fresh, prod)
            dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
        dk.dyna_kv_wait(x)
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
