#!/usr/bin/env python
"""Would a stream memory op (cuStreamWriteValue64 after an unsignalled launch) raise a one-chunk call's
flag cheaper than the in-kernel count?  Back-to-back disjoint Llama-3-8B chunks behind a gate: plain,
in-kernel signalled, and plain + stream-written flag.  JSON per line (A/B only, not a product path)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

torch.cuda.set_device(0)
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
s = torch.cuda.Stream()
g = kvgen.LLAMA3_8B.with_(num_blocks=4096)
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
rng = np.random.default_rng(1)
ts, td = rng.permutation(g.num_blocks).astype(np.int32), rng.permutation(g.num_blocks).astype(np.int32)
st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
flags = torch.zeros(4096, dtype=torch.int64, device="cuda")
tok = 2 * 32 * g.row_bytes
for c in (256, 512, 1024, 4096):
    reps = 32
    for mode in ("plain", "signalled", "plain+stream_write", "plain+overlap+stream_write"):
        res = []
        for trial in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(30_000_000)
            e0.record(s)
            xs = []
            for i in range(reps):
                fl = dk.DYNA_MIGRATE_UNCHECKED | (dk.DYNA_MIGRATE_SIGNAL if mode == "signalled" else 0) | \
                    (dk.DYNA_MIGRATE_OVERLAP_PREV if "overlap" in mode else 0)
                xs.append(dk.dyna_kv_migrate_ex(st, dt, (i * c, (i + 1) * c), (0, 32), c, s.cuda_stream, dk.opts(flags=fl)))
                if "stream_write" in mode:
                    cu.cuStreamWriteValue64(cu.CUstream(s.cuda_stream), cu.CUdeviceptr(flags.data_ptr() + 8 * i),
                                            trial * 100 + i + 1, 0)
            e1.record(s)
            for x in xs:
                dk.dyna_kv_wait(x)
            e1.synchronize()
            res.append(e0.elapsed_time(e1) * 1e3 / reps)
        us = min(res)
        print(json.dumps({"c": c, "mode": mode, "us_per_call": round(us, 2),
                          "frac_of_measured_hbm": round(2 * c * tok / (us * 1e-6) / 1e9 / peak, 4)}), flush=True)
