#!/usr/bin/env python
"""configs[4]: all ordered instance pairs migrate concurrently (8 x B200).

    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 scripts/allpairs.py [--steps K] [--check]

Every rank owns a Qwen2-72B-shaped KV shard (80 layers, 8 KV heads, d128,
bf16, block 16, 6144 blocks = 30 GiB) as the source pool and a second pool of
the same shape that receives its peers' micro-requests (§3.1).
The plan (kvgen.allpairs_plan: 4 skewed requests per ordered pair, seeds
1000 + 8i + j) is identical on every rank.  Receive pools are exported over
CUDA IPC and imported by every peer; each rank then issues ONE
dyna_kv_migrate_batch covering all its outgoing requests into 7 different
peer pools — in-kernel NVLink stores, no NCCL on the data path.

Reported: aggregate GB/s = all bytes / max-over-ranks device time, and the
load-aware NVLink bound (busiest egress or ingress port at 900 GB/s nominal /
770 GB/s measured peer copy) — SURVEY §8d.  --check samples received rows
against the senders' generator streams.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import kvgen
    import paper_2504_09285_b200 as dk
    from paper_2504_09285_b200 import dist as dd

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--num-blocks", type=int, default=6144)
    a = ap.parse_args()
    rank, world, lr = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
    # DYNA_BENCH_SAME_DEVICE=1 + DYNA_BENCH_BACKEND=gloo: functional check with every rank on cuda:0
    if os.environ.get("DYNA_BENCH_SAME_DEVICE") == "1":
        lr = 0
    torch.cuda.set_device(lr)
    if os.environ.get("DYNA_BENCH_BACKEND", "nccl") == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr}"))
    else:
        dist.init_process_group(os.environ["DYNA_BENCH_BACKEND"])
    red_dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{lr}"
    g = kvgen.QWEN2_72B.with_(num_blocks=a.num_blocks)
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    src = dk.Pool(g, lr, instance=rank)
    recv = dk.Pool(g, lr, instance=rank)
    dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 3000 + rank, 0, cs)
    dk.dyna_kv_debug_fill(recv.tensor.data_ptr(), recv.tensor.numel(), 4000 + rank, 0, cs)
    torch.cuda.synchronize()
    handles = dd.exchange_handles(dk.dyna_kv_pool_export(recv.handle))
    peers = {j: dk.Pool.imported(handles[j], lr) for j in range(world) if j != rank}
    plan = kvgen.allpairs_plan(world, g)
    mine = [m for m in plan if m.src_rank == rank]
    keep = []
    migs = []
    for m in mine:
        ts = torch.from_numpy(m.src_table).to(f"cuda:{lr}")
        td = torch.from_numpy(m.dst_table).to(f"cuda:{lr}")
        keep += [ts, td]
        migs.append((dk.table(src, ts, m.src_table), dk.table(peers[m.dst_rank], td, m.dst_table), (0, m.req.s)))
    tok_bytes = 2 * g.num_layers * g.row_bytes
    my_bytes = sum(m.req.s for m in mine) * tok_bytes

    def step():
        return dk.dyna_kv_migrate_batch(migs, (0, g.num_layers), 1024, cs, None)

    for _ in range(a.warmup):
        dk.dyna_kv_wait(step())
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    xs = [step() for _ in range(a.steps)]
    e1.record(stream)
    for x in xs:
        dk.dyna_kv_wait(x)
    torch.cuda.synchronize()
    dist.barrier()
    ms = dd.max_over_ranks(e0.elapsed_time(e1) / a.steps, device=red_dev)
    total = torch.tensor([my_bytes], dtype=torch.float64, device=red_dev)
    dist.all_reduce(total)
    bad = 0
    if a.check:
        rng = np.random.default_rng(rank)
        S = recv.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, g.row_bytes)
        for m in [m for m in plan if m.dst_rank == rank]:
            for _ in range(16):
                l, kv, t = int(rng.integers(0, g.num_layers)), int(rng.integers(0, 2)), int(rng.integers(0, m.req.s))
                sb, db = int(m.src_table[t // g.block_size]), int(m.dst_table[t // g.block_size])
                off = ((((l * 2 + kv) * g.num_blocks + sb) * g.block_size) + t % g.block_size) * g.row_bytes
                want = kvgen.bytes_at(3000 + m.src_rank, off, g.row_bytes)
                got = S[l, kv, db, t % g.block_size].cpu().numpy()
                bad += int(not np.array_equal(want, got))
        b = torch.tensor([bad], device=red_dev)
        dist.all_reduce(b)
        bad = int(b.item())
    if rank == 0:
        pb = {}
        for m in plan:
            pb[(m.src_rank, m.dst_rank)] = pb.get((m.src_rank, m.dst_rank), 0) + m.req.s * tok_bytes
        bound_nom = dd.load_aware_bound_s(pb, 900e9) * 1e3
        bound_meas = dd.load_aware_bound_s(pb, 770e9) * 1e3
        gbps = total.item() / (ms / 1e3) / 1e9
        print(json.dumps({"config": "configs[4] all ordered pairs, Qwen2-72B shard", "n_gpus": world,
                          "migrations": len(plan), "bytes": total.item(), "ms": ms, "GBps": gbps,
                          "load_aware_bound_ms_900": bound_nom, "load_aware_bound_ms_770": bound_meas,
                          "frac_of_load_aware_bound_900": bound_nom / ms,
                          "check_bad_rows": bad if a.check else None}))
    for p in peers.values():
        p.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
