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


def test_peer_head_reshard():
    gd = G.with_(num_kv_heads=2, block_size=32, num_blocks=200)
    ts, _ = kvgen.table_pair(8, 3000, G, G)
    td = kvgen.table_pair(9, 3000, gd, gd)[1]
    hs, hd = kvgen.fill_bytes(3, G.pool_bytes), kvgen.fill_bytes(4, gd.pool_bytes)
    want = hd.copy()
    oracle.migrate_heads(hs, G, ts, want, gd, td, (0, 2500), None, (6, 8), 0)
    dk.dyna_kv_enable_peer(0, 1)
    src, dst = pool_from_host(G, hs, device=0), pool_from_host(gd, hd, device=1)
    torch.cuda.set_device(0)
    dk.dyna_kv_wait(dk.dyna_kv_migrate_heads(_tab(src, ts, 0), _tab(dst, td, 0), (0, 2500), (0, 4), (6, 8), 0, 256, 0))
    torch.cuda.synchronize(1)
    assert np.array_equal(dst.tensor.cpu().numpy(), want)
