#!/usr/bin/env python
"""dyna_kv_calibrate on one GPU for the paper's row geometries: GB/s of every candidate
(FUSED x VEC/BULK, STAGED x VEC/BULK) per chunk size, as the library measures them.

    python scripts/calib_native.py [--out gpurun_out/calib_native.json]
"""
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

NAMES = ["FUSED VEC 4K U8", "FUSED VEC 8K U4", "FUSED VEC 16K U16", "FUSED BULK ring 32K x4",
         "STAGED VEC 8K U8", "STAGED BULK 32K x4", "FUSED TILES"]
GEOMS = {"Llama-2-7B rows (8 KiB)": kvgen.LLAMA2_7B,
         "Llama-3-8B rows (2 KiB)": kvgen.LLAMA3_8B.with_(num_blocks=4096),
         "TP-8 shard rows (256 B)": kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=6144),
         "TP-4 shard rows (512 B)": kvgen.LLAMA3_8B.with_(num_kv_heads=2, num_blocks=8192),
         "TP-2 shard rows (1 KiB)": kvgen.LLAMA3_8B.with_(num_kv_heads=4, num_blocks=8192)}

ap = argparse.ArgumentParser()
ap.add_argument("--chunks", default="64,256,1024,4096")
ap.add_argument("--only", default="", help="comma-separated geometry name prefixes")
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "calib_native.json"))
a = ap.parse_args()
chunks = [int(x) for x in a.chunks.split(",")]
torch.cuda.set_device(0)
s = torch.cuda.Stream()
out = []
for name, g in GEOMS.items():
    if a.only and not any(name.startswith(x) for x in a.only.split(",")):
        continue
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    for p, seed in ((src, 1), (dst, 2)):
        dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
    rng = np.random.default_rng(1)
    ts, td = rng.permutation(g.num_blocks).astype(np.int32), rng.permutation(g.num_blocks).astype(np.int32)
    st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
    dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
    entries, rates = dk.dyna_kv_calibrate(st, dt, chunks, reps=a.reps, stream=s.cuda_stream)
    for c, e, r in zip(chunks, entries, rates):
        row = {"geometry": name, "chunk": c, "chosen": e, "GBps": dict(zip(NAMES, [round(x, 1) for x in r]))}
        print(json.dumps(row), flush=True)
        out.append(row)
    del src, dst
    torch.cuda.empty_cache()
dk.dyna_kv_calib_set([])
os.makedirs(os.path.dirname(a.out), exist_ok=True)
json.dump({"k2": "kernel" if os.environ.get("DYNA_KV_K2_KERNEL") == "1" else "copy engine", "results": out},
          open(a.out, "w"), indent=1)
