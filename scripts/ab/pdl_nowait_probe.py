#!/usr/bin/env python
"""A/B of the launch bubble between back-to-back independent migrations: per-call device time of
disjoint Llama-3-8B chunks (and TP-8 256-B-row chunks) issued behind a sleeping kernel (host issue
time out of the picture), for whichever build DYNA_KV_LIB loads (default vs -DDYNA_DIAG_PDL_NOWAIT,
which skips griddepcontrol.wait), or with DYNA_PROBE_OV=1 the product's opt-in flag
DYNA_MIGRATE_OVERLAP_PREV on every call.  Prints one JSON line per case."""
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
lib = os.path.basename(os.environ.get("DYNA_KV_LIB", "default"))
ov = dk.DYNA_MIGRATE_OVERLAP_PREV if os.environ.get("DYNA_PROBE_OV") == "1" else 0
if ov:
    lib += "+OVERLAP_PREV"
sig = dk.DYNA_MIGRATE_SIGNAL if os.environ.get("DYNA_PROBE_SIG") == "1" else 0
if sig:
    lib += "+SIGNAL"
s = torch.cuda.Stream()
for name, g in (("llama3", kvgen.LLAMA3_8B.with_(num_blocks=4096)),
                ("tp8_256B", kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=8192))):
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    for p, seed in ((src, 1), (dst, 2)):
        dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
    rng = np.random.default_rng(1)
    ts, td = rng.permutation(g.num_blocks).astype(np.int32), rng.permutation(g.num_blocks).astype(np.int32)
    st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
    dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
    T = g.num_blocks * g.block_size
    tok = 2 * g.num_layers * g.row_bytes
    for c in (256, 512, 1024, 4096):
        reps = min(48, T // c)
        res = []
        for trial in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(30_000_000)
            e0.record(s)
            xs = [dk.dyna_kv_migrate_ex(st, dt, (i * c, (i + 1) * c), (0, g.num_layers), c, s.cuda_stream,
                                        dk.opts(flags=dk.DYNA_MIGRATE_UNCHECKED | ov | sig)) for i in range(reps)]
            e1.record(s)
            plan = dk.dyna_kv_xfer_plan(xs[0])
            for x in xs:
                dk.dyna_kv_wait(x)
            e1.synchronize()
            res.append(e0.elapsed_time(e1) * 1e3 / reps)
        us = min(res)
        ok = bool(torch.equal(dst.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, -1)[:, :, td[:reps * c // g.block_size]],
                              src.tensor.view(g.num_layers, 2, g.num_blocks, g.block_size, -1)[:, :, ts[:reps * c // g.block_size]]))
        print(json.dumps({"lib": lib, "rows": name, "c": c, "calls": reps, "us_per_call": round(us, 2),
                          "frac_of_measured_hbm": round(2 * c * tok / (us * 1e-6) / 1e9 / peak, 4),
                          "engine": plan["engine"], "rows_equal": ok}), flush=True)
    src.close()
    dst.close()
