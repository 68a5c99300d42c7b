#!/usr/bin/env python
"""Per-call device time of back-to-back Llama-3-8B migrations of c tokens, issued behind the
library's calibration gate (host issue time out of the picture), for ring shapes: how much of a
launch is bubble (ramp of the next, tail of the last) and what the ring depth / CTAs per SM do to it.
    python scripts/launch_probe.py [--out gpurun_out/launch_probe.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "launch_probe.json"))
a = ap.parse_args()
torch.cuda.set_device(0)
g = kvgen.LLAMA3_8B.with_(num_blocks=4096)
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
for p, seed in ((src, 1), (dst, 2)):
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
rng = np.random.default_rng(1)
ts, td = rng.permutation(g.num_blocks).astype(np.int32), rng.permutation(g.num_blocks).astype(np.int32)
st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
s = torch.cuda.Stream()
out = []
shapes = [("ring 32K x4", dict(engine=dk.DYNA_ENGINE_BULK, piece_bytes=32768, stages=4)),
          ("ring 32K x3", dict(engine=dk.DYNA_ENGINE_BULK, piece_bytes=32768, stages=3)),
          ("ring 32K x2", dict(engine=dk.DYNA_ENGINE_BULK, piece_bytes=32768, stages=2)),
          ("ring 16K x4", dict(engine=dk.DYNA_ENGINE_BULK, piece_bytes=16384, stages=4)),
          ("ring 16K x6", dict(engine=dk.DYNA_ENGINE_BULK, piece_bytes=16384, stages=6))]
base = dk.dyna_kv_calib_get()
for name, kw in shapes:
    for c in (256, 1024, 4096):
        # gated AUTO timing: time AUTO with the one-entry table
        torch.cuda.synchronize()
        dk.dyna_kv_calib_set([(2048, 0, 1 << 30, 1, kw["engine"], kw["piece_bytes"], kw["stages"], 0)])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 24
        T = g.num_blocks * 16
        with torch.cuda.stream(s):
            torch.cuda._sleep(20_000_000)        # hold the stream while the calls are issued
        e0.record(s)
        xs = []
        for i in range(reps):
            t0 = (i * c) % (T - c)
            xs.append(dk.dyna_kv_migrate_ex(st, dt, (t0, t0 + c), (0, 32), c, s.cuda_stream,
                                            dk.opts(flags=dk.DYNA_MIGRATE_UNCHECKED)))
        e1.record(s)
        for x in xs:
            dk.dyna_kv_wait(x)
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        ideal = 2 * c * 2 * 32 * 2048 / 6451.2e9 * 1e6
        row = {"shape": name, "c": c, "us_per_call": round(us, 2), "ideal_us": round(ideal, 2),
               "bubble_us": round(us - ideal, 2), "frac": round(ideal / us, 3)}
        print(json.dumps(row), flush=True)
        out.append(row)
dk.dyna_kv_calib_set([])
json.dump(out, open(a.out, "w"), indent=1)
