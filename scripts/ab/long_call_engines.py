#!/usr/bin/env python
"""Steady-state engine comparison: one long call (Llama-3-8B rows, 32768 tokens = 4 GiB payload, chunk
1024) per engine shape, calls back to back (5 reps behind a gate), plus the configs[2] batch per shape.
JSON per line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

torch.cuda.set_device(0)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
s = torch.cuda.Stream()
B, V = dk.DYNA_ENGINE_BULK, dk.DYNA_ENGINE_VEC
shapes = [("ring 32Kx4", dict(engine=B, piece_bytes=32768, stages=4)),
          ("ring 32Kx4 dyn", dict(engine=B, piece_bytes=32768, stages=4, schedule=dk.DYNA_SCHED_DYNAMIC)),
          ("vec 8K U4", dict(engine=V, piece_bytes=8192, unroll=4)),
          ("vec 4K U8", dict(engine=V, piece_bytes=4096, unroll=8)),
          ("vec 32K U8", dict(engine=V, piece_bytes=32768, unroll=8)),
          ("vec 8K U4 dyn", dict(engine=V, piece_bytes=8192, unroll=4, schedule=dk.DYNA_SCHED_DYNAMIC))]


def timed(calls, reps=5):
    res = []
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(30_000_000)
        e0.record(s)
        xs = [c() for _ in range(reps) for c in calls]
        e1.record(s)
        for x in xs:
            dk.dyna_kv_wait(x)
        e1.synchronize()
        res.append(e0.elapsed_time(e1) / reps)
    return min(res)


g = kvgen.LLAMA3_8B.with_(num_blocks=4096)
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
for p, seed in ((src, 1), (dst, 2)):
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
ts, td = kvgen.table_pair(3, 32768, g, g)
st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
pay = 32768 * 2 * 32 * g.row_bytes
for name, kw in shapes:
    o = dk.opts(**kw)
    ms = timed([lambda: dk.dyna_kv_migrate_ex(st, dt, (0, 32768), (0, 32), 1024, s.cuda_stream, o)])
    print(json.dumps({"case": "one 4-GiB call", "shape": name, "ms": round(ms, 4),
                      "frac_of_measured_hbm": round(2 * pay / (ms / 1e3) / 1e9 / peak, 4)}), flush=True)
    for c in (512, 4096):
        calls = [lambda k=k, c=c: dk.dyna_kv_migrate_ex(st, dt, (k * c, (k + 1) * c), (0, 32), c, s.cuda_stream, o)
                 for k in range(32768 // c)]
        ms = timed(calls, reps=2)
        print(json.dumps({"case": f"per-chunk calls c={c}", "shape": name, "ms": round(ms, 4),
                          "frac_of_measured_hbm": round(2 * pay / (ms / 1e3) / 1e9 / peak, 4)}), flush=True)
del src, dst
g = kvgen.LLAMA3_8B
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
for p, seed in ((src, 1), (dst, 2)):
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
keep = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b)) for a, b in tabs]
migs = [(a, b, (0, r.s)) for (a, b), r in zip(keep, reqs)]
pay = sum(r.s for r in reqs) * 2 * 32 * g.row_bytes
for name, kw in shapes:
    o = dk.opts(**kw)
    ms = timed([lambda: dk.dyna_kv_migrate_batch(migs, (0, 32), 256, s.cuda_stream, o)])
    print(json.dumps({"case": "configs[2] batch", "shape": name, "ms": round(ms, 4),
                      "frac_of_measured_hbm": round(2 * pay / (ms / 1e3) / 1e9 / peak, 4)}), flush=True)
