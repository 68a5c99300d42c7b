#!/usr/bin/env python
"""One TP reshard case (dyna_kv_reshard, one launch) repeated `reps` times on cuda:0, for ncu captures
of the head-slice kernels:  python scripts/tiles_case.py MODEL TP_SRC TP_DST [--s 16384] [--engine tiles|rows]
--whole: instead, a whole-row migration of one TP_SRC-rank shard (H / TP_SRC heads per row) of s tokens,
AUTO (tiles for short runs) vs --engine rows (VEC)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402
from paper_2504_09285_b200 import dist as dd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("model", choices=["llama3", "qwen72"])
ap.add_argument("tp_src", type=int)
ap.add_argument("tp_dst", type=int)
ap.add_argument("--s", type=int, default=16384)
ap.add_argument("--chunk", type=int, default=1024)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--engine", default="tiles")
ap.add_argument("--whole", action="store_true")
a = ap.parse_args()
g0 = kvgen.LLAMA3_8B if a.model == "llama3" else kvgen.QWEN2_72B
H, L, s = g0.num_kv_heads, g0.num_layers, a.s
nb = 2 * kvgen.blocks_needed(s, g0.block_size) + 16
gs = g0.with_(num_kv_heads=H // a.tp_src, num_blocks=nb)
gd = g0.with_(num_kv_heads=H // a.tp_dst, num_blocks=nb)
src = [dk.Pool(gs, 0) for _ in range(a.tp_src)]
dst = [dk.Pool(gd, 0) for _ in range(a.tp_dst)]
for i, p in enumerate(src + dst):
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), 100 + i, 0, 0)
st = [dk.table(p, torch.from_numpy(kvgen.table_pair(10 + i, s, gs, gs)[0]).cuda(), None) for i, p in enumerate(src)]
dt = [dk.table(p, torch.from_numpy(kvgen.table_pair(20 + i, s, gd, gd)[1]).cuda(), None) for i, p in enumerate(dst)]
if a.whole:
    o = dk.opts(engine=0 if a.engine == "tiles" else dk.DYNA_ENGINE_VEC, flags=dk.DYNA_MIGRATE_UNCHECKED)
    for _ in range(a.reps):
        x = dk.dyna_kv_migrate_ex(st[0], dt[0], (0, s), (0, L), a.chunk, 0, o)
        dk.dyna_kv_wait(x)
    print(dk.dyna_kv_xfer_plan(x))
    print(f"payload_bytes_per_launch {s * 2 * L * gs.row_bytes}")
    sys.exit(0)
plan = dd.tp_reshard_plan(H, a.tp_src, a.tp_dst)
o = dk.opts(engine=dk.DYNA_ENGINE_BULK if a.engine == "tiles" else dk.DYNA_ENGINE_VEC, flags=dk.DYNA_MIGRATE_UNCHECKED)
migs = [(st[x], dt[y], heads, hd0) for x, y, heads, hd0 in plan]
for _ in range(a.reps):
    dk.dyna_kv_wait(dk.dyna_kv_reshard(migs, (0, s), (0, L), a.chunk, 0, o))
torch.cuda.synchronize()
print(f"payload_bytes_per_launch {s * 2 * L * g0.row_bytes}")
