#!/usr/bin/env python
"""Comparison baseline B1: library gather -> NCCL send/recv of the
packed chunk -> library scatter.  NOT the product path — this is what "fully
offloaded to high-speed libraries like NCCL" (§4.3) looks like
with stock PyTorch ops, on the same workload as bench.py (configs[1], rank r
pushes its request's [0, s) KV to rank (r+1) % N), chunk by chunk.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/nccl_baseline.py [--steps K]

The pack/unpack uses torch advanced indexing on the pool view
[L][2][NB][bs][row]; the bytes moved are identical to dyna_kv_migrate's, and
--check compares the destination rows with the source rows.  The same code runs
on CPU with gloo (tests/test_dist_gloo.py) to cover its host logic.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pool_view(t, g):
    return t.view(g.num_layers, 2, g.num_blocks, g.block_size, g.row_bytes)


def gather(pool, g, table, a, b):
    """Pack tokens [a, b) of one request (all layers, K and V) into [L][2][b-a][row]."""
    import torch
    t = torch.arange(a, b, device=pool.device)
    T = table.to(pool.device).long()
    return pool_view(pool, g)[:, :, T[t // g.block_size], t % g.block_size].contiguous()


def scatter(pool, g, table, a, b, packed):
    import torch
    t = torch.arange(a, b, device=pool.device)
    T = table.to(pool.device).long()
    pool_view(pool, g)[:, :, T[t // g.block_size], t % g.block_size] = packed


def push_chunks(rank, world, src_pool, dst_pool, g, ts, td_of_sender, s, chunk):
    """Every rank sends [0, s) of its request to (rank+1) % world and receives
    from (rank-1) % world, one chunk at a time, grouped send/recv."""
    import torch.distributed as dist
    nxt, prv = (rank + 1) % world, (rank - 1) % world
    for a in range(0, s, chunk):
        b = min(a + chunk, s)
        out = gather(src_pool, g, ts, a, b)
        inc = out.new_empty(out.shape)
        ops = [dist.P2POp(dist.isend, out, nxt), dist.P2POp(dist.irecv, inc, prv)]
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        scatter(dst_pool, g, td_of_sender, a, b, inc)


def main():
    import torch
    import torch.distributed as dist

    import kvgen
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    rank, world, lr = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr}"))
    g, s, chunk = kvgen.LLAMA2_7B, 1024, 256
    src = torch.empty(g.pool_bytes, dtype=torch.uint8, device="cuda")
    dst = torch.empty_like(src)
    src.random_(0, 256)
    # tables: my outgoing request's (src, dst-on-next-rank) and the incoming one's dst table
    ts, _ = kvgen.table_pair(500 + rank, 2048, g, g)
    _, td_in = kvgen.table_pair(500 + (rank - 1) % world, 2048, g, g)
    ts, td_in = torch.from_numpy(ts).cuda(), torch.from_numpy(td_in).cuda()
    for _ in range(args.warmup):
        push_chunks(rank, world, src, dst, g, ts, td_in, s, chunk)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        push_chunks(rank, world, src, dst, g, ts, td_in, s, chunk)
    torch.cuda.synchronize()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    payload = s * 2 * g.num_layers * g.row_bytes
    if rank == 0:
        print(json.dumps({"impl": "nccl_baseline", "n_gpus": world, "steps": args.steps,
                          "GBps": world * args.steps * payload / dt.item() / 1e9,
                          "per_pair_GBps": args.steps * payload / dt.item() / 1e9}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
