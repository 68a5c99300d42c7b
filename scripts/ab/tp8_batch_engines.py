#!/usr/bin/env python
"""configs[4]'s pair of 3 requests as TP-8 shards (256-B rows) and as full Qwen2-72B shards (2-KiB rows),
one dyna_kv_migrate_batch per set, per engine shape (sets back to back behind a gate).  JSON per line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

torch.cuda.set_device(0)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
s = torch.cuda.Stream()
reqs = kvgen.migrating(kvgen.skewed_batch(1000 + 1, 4))
V, T, B, D = dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_TILES, dk.DYNA_ENGINE_BULK, dk.DYNA_SCHED_DYNAMIC
for name, g in (("tp8_256B", kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=6144)), ("qwen_2K", kvgen.QWEN2_72B)):
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    tabs = kvgen.batch_tables(3, [r.s for r in reqs], g, g)
    keep = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b)) for a, b in tabs]
    migs = [(a, b, (0, r.s)) for (a, b), r in zip(keep, reqs)]
    pay = sum(r.s for r in reqs) * 2 * g.num_layers * g.row_bytes
    shapes = [("auto", {}), ("tiles", dict(engine=T)), ("ring", dict(engine=B)),
              ("vec 4K U8", dict(engine=V, piece_bytes=4096, unroll=8)),
              ("vec 8K U4", dict(engine=V, piece_bytes=8192, unroll=4)),
              ("vec 8K U4 dyn", dict(engine=V, piece_bytes=8192, unroll=4, schedule=D)),
              ("vec 4K U8 dyn", dict(engine=V, piece_bytes=4096, unroll=8, schedule=D))]
    for sname, kw in shapes:
        res = []
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(30_000_000)
            e0.record(s)
            try:
                xs = [dk.dyna_kv_migrate_batch(migs, (0, g.num_layers), 1024, s.cuda_stream, dk.opts(**kw)) for _ in range(10)]
            except dk.DynaKVError as e:
                xs = []
                print(json.dumps({"rows": name, "shape": sname, "error": str(e)}))
                break
            e1.record(s)
            for x in xs:
                dk.dyna_kv_wait(x)
            e1.synchronize()
            res.append(e0.elapsed_time(e1) / 10)
        if res:
            ms = min(res)
            print(json.dumps({"rows": name, "shape": sname, "us": round(ms * 1e3, 2),
                              "frac_of_measured_hbm": round(2 * pay / (ms / 1e3) / 1e9 / peak, 4)}), flush=True)
    src.close()
    dst.close()
