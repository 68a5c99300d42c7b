"""Helpers shared by the GPU tests (plumbing only: memory, tables, checks)."""
from __future__ import annotations

import numpy as np
import torch

import kvgen
import paper_2504_09285_b200 as dk


def pool_from_host(geom, host: np.ndarray, device: int = 0, instance: int = 0) -> dk.Pool:
    t = torch.from_numpy(host).to(f"cuda:{device}")
    return dk.Pool(geom, device, instance, tensor=t)


def pool_filled(geom, seed: int, device: int = 0, instance: int = 0) -> dk.Pool:
    """Pool filled on the device with the kvgen stream of `seed` (dyna_kv_debug_fill)."""
    p = dk.Pool(geom, device, instance)
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0,
                          torch.cuda.current_stream(device).cuda_stream)
    return p


def dev_table(pool: dk.Pool, ids, with_host: bool = True):
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    d = torch.from_numpy(ids).to(pool.tensor.device if pool.tensor is not None else "cuda")
    return dk.table(pool, d, ids if with_host else None)


def migrate_and_wait(src: dk.Pool, ts, dst: dk.Pool, td, tr, lr, c, with_host=True, **kw):
    st, dt = dev_table(src, ts, with_host), dev_table(dst, td, with_host)  # alive until the wait
    if not with_host:  # device-only tables: the caller vouches for distinct destination rows
        kw["flags"] = kw.get("flags", 0) | dk.DYNA_MIGRATE_UNCHECKED
    x = dk.migrate(st, dt, tr, lr, c, **kw)
    dk.dyna_kv_wait(x)


def torch_rows_equal(src: dk.Pool, ts, dst: dk.Pool, td, tr, lr) -> bool:
    """Independent full check at any size: dst rows == src rows through both tables (torch advanced indexing)."""
    gs, gd = src.geom, dst.geom
    row = gs.row_bytes
    S = src.tensor.view(gs.num_layers, 2, gs.num_blocks, gs.block_size, row)
    D = dst.tensor.view(gd.num_layers, 2, gd.num_blocks, gd.block_size, row)
    dev = src.tensor.device
    Ts = torch.as_tensor(np.asarray(ts, np.int64), device=dev)
    Td = torch.as_tensor(np.asarray(td, np.int64), device=dev)
    ok = True
    step = 4096  # bound the temporaries
    for a in range(tr[0], tr[1], step):
        t = torch.arange(a, min(a + step, tr[1]), device=dev)
        ok &= bool(torch.equal(D[lr[0]:lr[1], :, Td[t // gd.block_size], t % gd.block_size],
                               S[lr[0]:lr[1], :, Ts[t // gs.block_size], t % gs.block_size]))
    return ok


def mapped_mask(geom, tables_ranges, lr=None) -> torch.Tensor:
    """Bool [L, 2, NB, bs] of destination rows written by the given (table, token range) list."""
    m = torch.zeros(geom.num_layers, 2, geom.num_blocks, geom.block_size, dtype=torch.bool, device="cuda")
    l0, l1 = lr or (0, geom.num_layers)
    for td, (t0, t1) in tables_ranges:
        t = torch.arange(t0, t1, device="cuda")
        Td = torch.as_tensor(np.asarray(td, np.int64), device="cuda")
        m[l0:l1, :, Td[t // geom.block_size], t % geom.block_size] = True
    return m


def untouched_equal(dst: dk.Pool, seed: int, mask: torch.Tensor) -> bool:
    """Rows outside `mask` still hold the kvgen stream of `seed`."""
    g = dst.geom
    ref = torch.empty_like(dst.tensor)
    dk.dyna_kv_debug_fill(ref.data_ptr(), ref.numel(), seed, 0, torch.cuda.current_stream().cuda_stream)
    D = dst.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, g.row_bytes)
    R = ref.view_as(D)
    keep = ~mask
    return bool(torch.equal(D[keep], R[keep]))


def sampled_rows_match(src_seed: int, gs, ts, dst: dk.Pool, gd, td, tr, lr, n: int, rng) -> int:
    """Sample n (l, kv, t): the dst row must equal the kvgen bytes at the oracle's source offset."""
    import oracle
    row = gs.row_bytes
    host = None
    bad = 0
    for _ in range(n):
        l = int(rng.integers(lr[0], lr[1]))
        kv = int(rng.integers(0, 2))
        t = int(rng.integers(tr[0], tr[1]))
        so = oracle.logical_off(gs, ts, l, kv, t)
        do = oracle.logical_off(gd, td, l, kv, t)
        want = kvgen.bytes_at(src_seed, so, row)
        got = dst.tensor[do:do + row].cpu().numpy()
        bad += int(not np.array_equal(want, got))
    return bad
