#!/usr/bin/env python
"""Static vs guided-dynamic ring per call size: back-to-back disjoint calls of c tokens (8-KiB and 2-KiB
rows), plain and signalled.  JSON per line."""
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
B = dk.DYNA_ENGINE_BULK
for rname, g in (("llama3_2K", kvgen.LLAMA3_8B.with_(num_blocks=4096)), ("llama2_8K", kvgen.LLAMA2_7B.with_(num_blocks=1024))):
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    for p, seed in ((src, 1), (dst, 2)):
        dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
    T = g.num_blocks * g.block_size
    ts, td = kvgen.table_pair(3, T, g, g)
    st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
    dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
    tok = 2 * g.num_layers * g.row_bytes
    for sig in (0, dk.DYNA_MIGRATE_SIGNAL):
        for c in (256, 512, 1024, 2048, 4096, 8192, 16384):
            if c > T:
                continue
            for sched in (1, 2):
                o = dk.opts(engine=B, piece_bytes=32768, stages=4, schedule=sched, flags=sig | dk.DYNA_MIGRATE_UNCHECKED)
                reps = max(2, min(32, T // c))
                res = []
                for _ in range(3):
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    with torch.cuda.stream(s):
                        torch.cuda._sleep(30_000_000)
                    e0.record(s)
                    xs = [dk.dyna_kv_migrate_ex(st, dt, ((k % (T // c)) * c, (k % (T // c) + 1) * c), (0, g.num_layers),
                                                min(c, 4096), s.cuda_stream, o) for k in range(reps)]
                    e1.record(s)
                    for x in xs:
                        dk.dyna_kv_wait(x)
                    e1.synchronize()
                    res.append(e0.elapsed_time(e1) * 1e3 / reps)
                us = min(res)
                print(json.dumps({"rows": rname, "signal": bool(sig), "c": c, "sched": "dynamic" if sched == 2 else "static",
                                  "us_per_call": round(us, 2),
                                  "frac_of_measured_hbm": round(2 * c * tok / (us * 1e-6) / 1e9 / peak, 4)}), flush=True)
    src.close()
    dst.close()
