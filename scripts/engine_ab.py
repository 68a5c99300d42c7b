#!/usr/bin/env python
"""Engine A/B on the workloads that decide the headline.

Workloads (one B200, intra-device form, fragmented tables, working set > L2):
  l2req    configs[1]: one Llama-2-7B request, s = 1024, c = 256 (round-1 bench step)
  c2calls  configs[2]: the 54 migrating requests of skewed_batch(1, 64), one call each, c = 256
  c2batch  configs[2]: the same 54 requests as ONE dyna_kv_migrate_batch
  t4prime  4' shape: 4096-token Llama-3-8B chunks (512 MiB), one call each
  c3c512   configs[3]: 32k-token Llama-3-8B prompt pushed as 64 per-chunk calls of 512 tokens

Each workload is repeated back to back (`--reps`) between two CUDA events on the launch
stream; GB/s = payload / (region time / reps).  Candidates are engine option sets given
as name=engine:piece:stages:unroll:max_ctas[:flags] (0 = AUTO/default), e.g.
    python scripts/engine_ab.py --cand auto=0:0:0:0:0 --cand vec2=1:8192:0:8:296
Environment switches (DYNA_KV_RING, DYNA_KV_LAG, ...) are set by the caller per process.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cand", action="append", default=[])
    ap.add_argument("--work", default="l2req,c2calls,c2batch,t4prime,c3c512")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--tag", default=os.environ.get("AB_TAG", ""))
    args = ap.parse_args()
    cands = []
    for c in args.cand or ["auto=0:0:0:0:0"]:
        name, spec = c.split("=")
        f = [int(x) for x in spec.split(":")]
        e, p, s, u, m = f[:5]
        fl = f[5] if len(f) > 5 else 0          # optional 6th field: opts.flags (1 = per-chunk flags)
        cands.append((name, dk.opts(engine=e, piece_bytes=p, stages=s, unroll=u, max_ctas=m, flags=fl)))
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    works = args.work.split(",")

    def pools(g, a, b):
        x, y = dk.Pool(g, 0), dk.Pool(g, 0)
        dk.dyna_kv_debug_fill(x.tensor.data_ptr(), x.tensor.numel(), a, 0, cs)
        dk.dyna_kv_debug_fill(y.tensor.data_ptr(), y.tensor.numel(), b, 0, cs)
        return x, y

    def tab(p, ids):
        return dk.table(p, torch.from_numpy(ids).cuda(), ids)

    def timeit(step, n_steps, reps):
        for i in range(3):
            for x in step(i):
                dk.dyna_kv_wait(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        xs = []
        for i in range(reps):
            xs += step(i)
        e1.record(stream)
        for x in xs:
            dk.dyna_kv_wait(x)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    res = []

    def report(work, name, payload, ms, plan):
        r = {"tag": args.tag, "work": work, "cand": name, "ms": ms, "GBps": payload / ms / 1e6,
             "frac": 2 * payload / ms / 1e6 / 6456.2, "plan": plan}
        print(json.dumps(r), flush=True)
        res.append(r)

    def plan_of(x):
        p = dk.dyna_kv_xfer_plan(x)
        dk.dyna_kv_wait(x)
        return f"v{p['variant']} e{p['engine']} p{p['piece_bytes']} s{p['stages']} u{p['unroll']}"

    if "l2req" in works:
        g = kvgen.LLAMA2_7B
        src, dst = pools(g, 3, 4)
        tabs = kvgen.batch_tables(5, [2048] * 4, g, g)
        T = [(tab(src, a), tab(dst, b)) for a, b in tabs]
        for name, o in cands:
            def step(i, o=o):
                t = T[i % 4]
                return [dk.dyna_kv_migrate_ex(t[0], t[1], (0, 1024), (0, 32), 256, cs, o)]
            ms = timeit(step, 1, args.reps * 2)
            report("l2req", name, 1024 * 2 * 32 * g.row_bytes, ms, plan_of(step(0)[0]))
        del src, dst, T

    if "c2calls" in works or "c2batch" in works:
        g = kvgen.LLAMA3_8B
        src, dst = pools(g, 5, 6)
        reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
        tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
        T = [(tab(src, a), tab(dst, b), r.s) for r, (a, b) in zip(reqs, tabs)]
        tot = sum(r.s for r in reqs)
        payload = tot * 2 * 32 * g.row_bytes
        for name, o in cands:
            if "c2calls" in works:
                def step(i, o=o):
                    return [dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 32), 256, cs, o) for t in T]
                ms = timeit(step, len(T), args.reps)
                report("c2calls", name, payload, ms, plan_of(step(0)[0]))
            if "c2batch" in works:
                migs = [(t[0], t[1], (0, t[2])) for t in T]
                def stepb(i, o=o):
                    return [dk.dyna_kv_migrate_batch(migs, (0, 32), 256, cs, o)]
                ms = timeit(stepb, 1, args.reps)
                report("c2batch", name, payload, ms, plan_of(stepb(0)[0]))
        del src, dst, T

    if "t4prime" in works or "c3c512" in works:
        g = kvgen.LLAMA3_8B.with_(num_blocks=4096)
        src, dst = pools(g, 7, 8)
        ts, td = kvgen.table_pair(3, 32768, g, g)
        st, dt = tab(src, ts), tab(dst, td)
        for name, o in cands:
            if "t4prime" in works:
                def step(i, o=o):
                    k = i % 8
                    return [dk.dyna_kv_migrate_ex(st, dt, (k * 4096, (k + 1) * 4096), (0, 32), 4096, cs, o)]
                ms = timeit(step, 1, args.reps * 4)
                report("t4prime", name, 4096 * 2 * 32 * g.row_bytes, ms, plan_of(step(0)[0]))
            if "c3c512" in works:
                def step(i, o=o):
                    return [dk.dyna_kv_migrate_ex(st, dt, (k * 512, (k + 1) * 512), (0, 32), 512, cs, o)
                            for k in range(64)]
                ms = timeit(step, 64, args.reps)
                report("c3c512", name, 32768 * 2 * 32 * g.row_bytes, ms, plan_of(step(0)[0]))
        del src, dst
    if "q8" in works:   # TP-8 Qwen2-72B shard: 1 KV head per rank, 256-B rows (4-KiB block runs), 8192 tokens
        g = kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=2048)
        src, dst = pools(g, 9, 10)
        tabs = kvgen.batch_tables(4, [8192] * 4, g, g)
        T = [(tab(src, a), tab(dst, b)) for a, b in tabs]
        for name, o in cands:
            def step(i, o=o):
                t = T[i % 4]
                return [dk.dyna_kv_migrate_ex(t[0], t[1], (0, 8192), (0, 80), 1024, cs, o)]
            ms = timeit(step, 1, args.reps * 2)
            report("q8", name, 8192 * 2 * 80 * g.row_bytes, ms, plan_of(step(0)[0]))
        del src, dst, T
    out = os.path.join(ROOT, "gpurun_out", f"engine_ab{('_' + args.tag) if args.tag else ''}.json")
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
