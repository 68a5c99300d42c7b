"""DMA engine (copy engines via cudaMemcpyBatchAsync, no SM copying; "DMA-pushed"):
bit-exact against the oracle, per-chunk flags, and its restrictions."""
import itertools

import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, pool_filled, pool_from_host

pytestmark = pytest.mark.gpu
DMA = dk.DYNA_ENGINE_DMA


def _parity(gs, gd, n_tok, tr, lr, c, seed=1, flags=0, device_ids=True):
    ts, td = kvgen.table_pair(seed + 100, n_tok, gs, gd)
    hs, hd = kvgen.fill_bytes(seed, gs.pool_bytes), kvgen.fill_bytes(seed + 1, gd.pool_bytes)
    want = hd.copy()
    oracle.migrate(hs, gs, ts, want, gd, td, tr, lr)
    src, dst = pool_from_host(gs, hs), pool_from_host(gd, hd)
    if device_ids:
        st, dt = dev_table(src, ts), dev_table(dst, td)
    else:
        st, dt = dk.table(src, None, ts), dk.table(dst, None, td)
    x = dk.dyna_kv_migrate_ex(st, dt, tr, lr, c, 0, dk.opts(engine=DMA, flags=flags))
    info = dk.dyna_kv_xfer_info(x)
    plan = dk.dyna_kv_xfer_plan(x)
    dk.dyna_kv_wait(x)
    assert plan["engine"] == DMA
    got = dst.tensor.cpu().numpy()
    assert np.array_equal(src.tensor.cpu().numpy(), hs)
    assert np.array_equal(got, want)
    return dst, info


@pytest.mark.parametrize("c", [1, 15, 16, 17, 32, 100, 1000])
@pytest.mark.parametrize("tr,lr", [((0, 100), (0, 2)), ((37, 100), (0, 2)), ((0, 100), (1, 2)), ((0, 256), (0, 2))])
def test_dma_toy(c, tr, lr):
    _parity(kvgen.TOY, kvgen.TOY, 256, tr, lr, c)


@pytest.mark.parametrize("bss,bsd", [(16, 32), (32, 16), (16, 24), (8, 16)])
def test_dma_reblocking(bss, bsd):
    gs = kvgen.TOY.with_(block_size=bss, num_blocks=64 * 16 // bss)
    gd = kvgen.TOY.with_(block_size=bsd, num_blocks=64 * 16 // bsd + 8)
    _parity(gs, gd, 256, (3, 201), (0, 2), 40)


@pytest.mark.parametrize("device_ids", [True, False])
def test_dma_llama3_rows_with_flags(device_ids):
    g = Geom(4, 8, 128, 2, 16, 400)
    dst, (epoch, nck, sender) = _parity(g, g, 3000, (0, 2999), (0, 4), 512, flags=dk.DYNA_MIGRATE_SIGNAL,
                                        device_ids=device_ids)
    fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
    dk.dyna_kv_copy_flags(dst.handle, sender, 0, nck, fl.data_ptr(), 0)
    torch.cuda.synchronize()
    assert nck == 6 and (fl.numpy() == epoch).all()


def test_dma_contiguous_tables_merge_runs():
    g = kvgen.TOY
    hs, hd = kvgen.fill_bytes(5, g.pool_bytes), kvgen.fill_bytes(6, g.pool_bytes)
    ts, td = kvgen.table_pair(0, 256, g, g, "contiguous")
    want = hd.copy()
    oracle.migrate(hs, g, ts, want, g, td, (0, 256))
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    dk.dyna_kv_wait(dk.dyna_kv_migrate_ex(dev_table(src, ts), dev_table(dst, td), (0, 256), (0, 2), 256, 0,
                                          dk.opts(engine=DMA)))
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_dma_restrictions():
    g = kvgen.TOY
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(1, 256, g, g)
    st_dev_only = dev_table(src, ts, with_host=False)
    dt = dev_table(dst, td)
    for args, status in [((st_dev_only, dt, dk.opts(engine=DMA)), dk.DYNA_ENOTSUP),
                         ((dev_table(src, ts), dt, dk.opts(engine=DMA, variant=dk.DYNA_VARIANT_STAGED)),
                          dk.DYNA_ENOTSUP)]:
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_migrate_ex(args[0], args[1], (0, 100), (0, 2), 32, 0, args[2])
        assert e.value.status == status
    board = dk.dyna_kv_ready_create(0, 8)
    try:
        with pytest.raises(dk.DynaKVError) as e:
            dk.dyna_kv_migrate_on_ready(dev_table(src, ts), dt, (0, 100), (0, 2), 32, board, 1,
                                        opts=dk.opts(engine=DMA))
        assert e.value.status == dk.DYNA_ENOTSUP
    finally:
        dk.dyna_kv_ready_destroy(board)
