#!/usr/bin/env python
"""Signalled per-chunk pushes with DYNA_MIGRATE_OVERLAP_PREV: which launch shape lets the next call's
CTAs share an SM with this call's tail (ring smem cut to half an SM, grid capped at one CTA per SM)?
Per-call device time of 48 back-to-back disjoint Llama-3-8B chunks behind a gate.  JSON per line."""
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
sms = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.Stream()
B, V, T = dk.DYNA_ENGINE_BULK, dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_TILES
ROWS = {"llama2_8K": kvgen.LLAMA2_7B.with_(num_blocks=1024), "llama3_2K": kvgen.LLAMA3_8B.with_(num_blocks=4096),
        "tp8_256B": kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=8192)}
only = os.environ.get("OV_ROWS")
for rname, g in ROWS.items():
    if only and rname not in only.split(","):
        continue
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    for p, seed in ((src, 1), (dst, 2)):
        dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
    rng = np.random.default_rng(1)
    ts, td = rng.permutation(g.num_blocks).astype(np.int32), rng.permutation(g.num_blocks).astype(np.int32)
    st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
    dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
    tok = 2 * g.num_layers * g.row_bytes
    T_all = g.num_blocks * g.block_size
    shapes = [("auto", {}), ("ring 32Kx4", dict(engine=B, piece_bytes=32768, stages=4)),
              ("vec 8K U4", dict(engine=V, piece_bytes=8192, unroll=4)),
              ("vec 4K U8", dict(engine=V, piece_bytes=4096, unroll=8)),
              ("vec 16K U16", dict(engine=V, piece_bytes=16384, unroll=16))]
    if g.row_bytes < 2048:
        shapes.append(("tiles", dict(engine=T)))
    for sig in (dk.DYNA_MIGRATE_SIGNAL, 0):
        for c in (256, 1024, 4096):
            reps = min(48, T_all // c)
            for ovf in (dk.DYNA_MIGRATE_OVERLAP_PREV, 0):
                for name, kw in shapes:
                    res = []
                    for trial in range(3):
                        torch.cuda.synchronize()
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        with torch.cuda.stream(s):
                            torch.cuda._sleep(30_000_000)
                        e0.record(s)
                        o = dk.opts(flags=dk.DYNA_MIGRATE_UNCHECKED | ovf | sig, **kw)
                        xs = [dk.dyna_kv_migrate_ex(st, dt, (i * c, (i + 1) * c), (0, g.num_layers), c, s.cuda_stream, o)
                              for i in range(reps)]
                        e1.record(s)
                        for x in xs:
                            dk.dyna_kv_wait(x)
                        e1.synchronize()
                        res.append(e0.elapsed_time(e1) * 1e3 / reps)
                    us = min(res)
                    print(json.dumps({"rows": rname, "signal": bool(sig), "overlap_prev": bool(ovf), "c": c,
                                      "shape": name, "us_per_call": round(us, 2),
                                      "frac_of_measured_hbm": round(2 * c * tok / (us * 1e-6) / 1e9 / peak, 4)}),
                          flush=True)
    src.close()
    dst.close()
