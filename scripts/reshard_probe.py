#!/usr/bin/env python
"""One TP reshard case (Llama-3-8B rows, 1 -> 8 by default), per-pair calls vs one dyna_kv_reshard
launch: device time per launch (events around each launch after a synchronize, so host work is
outside) and host time per call."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402
from paper_2504_09285_b200 import dist as dd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", default="1,8")
    ap.add_argument("--s", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    ts_, td_ = (int(x) for x in a.tp.split(","))
    torch.cuda.set_device(0)
    st_ = torch.cuda.Stream()
    cs = st_.cuda_stream
    g0 = kvgen.LLAMA3_8B
    H, L, s, c = 8, 32, a.s, 1024
    nb = 2 * kvgen.blocks_needed(s, 16) + 16
    gs = g0.with_(num_kv_heads=H // ts_, num_blocks=nb)
    gd = g0.with_(num_kv_heads=H // td_, num_blocks=nb)
    src = [dk.Pool(gs, 0) for _ in range(ts_)]
    dst = [dk.Pool(gd, 0) for _ in range(td_)]
    st = [dk.table(p, torch.from_numpy(t).cuda(), t) for p, t in
          ((p, kvgen.table_pair(10 + i, s, gs, gs)[0]) for i, p in enumerate(src))]
    dt = [dk.table(p, torch.from_numpy(t).cuda(), t) for p, t in
          ((p, kvgen.table_pair(20 + i, s, gd, gd)[1]) for i, p in enumerate(dst))]
    plan = dd.tp_reshard_plan(H, ts_, td_)
    migs = [(st[x], dt[y], heads, hd0) for x, y, heads, hd0 in plan]
    out = {}
    for mode in ("calls", "one_launch"):
        dev_ms, host_ms = [], []
        for r in range(a.reps + 3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t = time.perf_counter()
            if mode == "calls":
                xs = [dk.dyna_kv_migrate_heads(st[x], dt[y], (0, s), (0, L), heads, hd0, c, cs) for x, y, heads, hd0
                      in plan]
            else:
                xs = [dk.dyna_kv_reshard(migs, (0, s), (0, L), c, cs)]
            h = time.perf_counter() - t
            if r == a.reps + 2 and mode == "one_launch":   # where the host time goes (one call, profiled)
                import cProfile
                import pstats
                pr = cProfile.Profile()
                pr.enable()
                y = dk.dyna_kv_reshard(migs, (0, s), (0, L), c, cs)
                pr.disable()
                dk.dyna_kv_wait(y)
                pstats.Stats(pr).sort_stats("cumulative").print_stats(6)
            for x in xs:
                dk.dyna_kv_wait(x)
            # device time: re-issue with the host work done first, then events around the launches only
            torch.cuda.synchronize()
            e0.record(st_)
            if mode == "calls":
                xs = [dk.dyna_kv_migrate_heads(st[x], dt[y], (0, s), (0, L), heads, hd0, c, cs) for x, y, heads, hd0
                      in plan]
            else:
                xs = [dk.dyna_kv_reshard(migs, (0, s), (0, L), c, cs)]
            e1.record(st_)
            for x in xs:
                dk.dyna_kv_wait(x)
            e1.synchronize()
            if r >= 3:
                dev_ms.append(e0.elapsed_time(e1))
                host_ms.append(h * 1e3)
        payload = s * 2 * L * g0.row_bytes
        out[mode] = {"ms": statistics.median(dev_ms), "host_ms": statistics.median(host_ms),
                     "GBps": payload / (statistics.median(dev_ms) / 1e3) / 1e9}
        print(json.dumps({"tp": [ts_, td_], "mode": mode, **out[mode]}), flush=True)


if __name__ == "__main__":
    main()
