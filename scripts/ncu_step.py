#!/usr/bin/env python
"""A few launches of one workload's step, for `ncu --set full` captures.

    ncu --set full --clock-control none --import-source on -k regex:k_copy_ -s 2 -c 1 \
        -o gpurun_out/prof_c2 python scripts/ncu_step.py --work c2

  c2     bench.py's N = 1 step: the configs[2] batch (54 requests) as one dyna_kv_migrate_batch
  t4     one 4096-token Llama-3-8B chunk (the 4' shape, 1-GPU form)
  rows   one head-sliced call: head 1 of 8 of Llama-3-8B rows (256-B slices), 4096 tokens
  small  TP-8 Qwen2-72B shard rows (1 KV head, 256-B rows), 8192 tokens, whole rows
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--work", default="c2")
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--engine", type=int, default=0)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    cs = torch.cuda.current_stream().cuda_stream
    o = dk.opts(engine=a.engine)

    def tab(p, ids):
        return dk.table(p, torch.from_numpy(ids).cuda(), ids)

    if a.work == "c2":
        g = kvgen.LLAMA3_8B
        reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
        tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
        src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
        migs = [(tab(src, x), tab(dst, y), (0, r.s)) for r, (x, y) in zip(reqs, tabs)]
        step = lambda: dk.dyna_kv_migrate_batch(migs, (0, 32), 256, cs, o)  # noqa: E731
    elif a.work == "t4":
        g = kvgen.LLAMA3_8B.with_(num_blocks=2048)
        src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
        ts, td = kvgen.table_pair(3, 4096, g, g)
        st, dt = tab(src, ts), tab(dst, td)
        step = lambda: dk.dyna_kv_migrate_ex(st, dt, (0, 4096), (0, 32), 4096, cs, o)  # noqa: E731
    elif a.work == "rows":
        g = kvgen.LLAMA3_8B.with_(num_blocks=2048)
        g1 = g.with_(num_kv_heads=1)
        src, dst = dk.Pool(g, 0), dk.Pool(g1, 0)
        ts, td = kvgen.table_pair(3, 4096, g, g1)
        st, dt = tab(src, ts), tab(dst, td)
        step = lambda: dk.dyna_kv_migrate_heads(st, dt, (0, 4096), (0, 32), (1, 2), 0, 1024, cs, o)  # noqa: E731
    else:
        g = kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=1024)
        src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
        ts, td = kvgen.table_pair(3, 8192, g, g)
        st, dt = tab(src, ts), tab(dst, td)
        step = lambda: dk.dyna_kv_migrate_ex(st, dt, (0, 8192), (0, 80), 1024, cs, o)  # noqa: E731
    for _ in range(a.reps):
        dk.dyna_kv_wait(step())
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
