#!/usr/bin/env python
"""Why do small static ring calls slow down after dynamic ones?  Llama-2 rows: sets of 16 calls of s
tokens (host-issued back to back, device-timed), before and after a batch of dynamic s=1024 calls."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

torch.cuda.set_device(0)
cs = torch.cuda.current_stream().cuda_stream
g = kvgen.LLAMA2_7B
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
tabs = kvgen.batch_tables(5, [2048] * 4, g, g)
T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b)) for a, b in tabs]


def run(s, n=16, reps=5, gate=False, o=None):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if gate:
        torch.cuda._sleep(50_000_000)
    e0.record()
    t0 = time.perf_counter()
    xs = [dk.dyna_kv_migrate_ex(T[i % 4][0], T[i % 4][1], (0, s), (0, 32), 256, cs, o) for i in range(n * reps)]
    host = (time.perf_counter() - t0) / (n * reps) * 1e6
    e1.record()
    for x in xs:
        dk.dyna_kv_wait(x)
    e1.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / (n * reps), 2), round(host, 2)


for phase in ("before", "after"):
    if phase == "after":
        run(1024, reps=2)
    for s in (1, 16, 100):
        dev, host = run(s)
        devg, _ = run(s, gate=True)
        devs, _ = run(s, gate=True, o=dk.opts(schedule=dk.DYNA_SCHED_STATIC))
        devd, _ = run(s, gate=True, o=dk.opts(schedule=dk.DYNA_SCHED_DYNAMIC))
        print(json.dumps({"lib_dyn": os.environ.get("DYNA_KV_RING_DYN", "default"), "phase": phase, "s": s,
                          "us_per_call": dev, "us_per_call_gated": devg, "gated_static": devs, "gated_dynamic": devd, "host_us_per_call": host}), flush=True)
