#!/usr/bin/env python
"""Head-sliced migration (TP resharding) throughput on one B200.

A request's KV is held by the tp_src ranks of the sending instance (each a pool
of H/tp_src heads) and must land in the tp_dst ranks of the receiving instance
(§5 P:595-596 deploys r^alpha / r^beta as TP groups).  Every
overlapping rank pair of dist.tp_reshard_plan gets one dyna_kv_migrate_heads;
here all rank pools live on cuda:0, so the numbers are the HBM (1-GPU) form:
payload = s * 2 * L * H * d * e bytes (every head once), HBM traffic = 2x.
The whole-row migration of the same request (tp 1 -> 1) is the reference line.

    python scripts/reshard_sweep.py [--out gpurun_out/reshard.json]
"""
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


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=4096)
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--quick", action="store_true", help="a few representative cases (A/B runs)")
    ap.add_argument("--engines", default="rows,tiles", help="rows (VEC row kernel) and/or tiles (TMA tensor tiles)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "reshard.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    pk = peak()
    s, c = args.s, args.chunk
    out = []
    cases = [("Llama-3-8B", kvgen.LLAMA3_8B, tp) for tp in
             [(1, 1), (1, 2), (1, 4), (1, 8), (2, 1), (4, 1), (8, 1), (2, 4), (4, 2), (2, 8), (8, 2)]]
    cases += [("Qwen2-72B", kvgen.QWEN2_72B, tp) for tp in [(1, 1), (4, 8), (8, 4), (2, 8)]]
    if args.quick:
        cases = [cases[i] for i in (2, 3, 6, 8, 13)]

    engines = {"rows": dk.DYNA_ENGINE_VEC, "tiles": dk.DYNA_ENGINE_BULK}
    engines = {k: engines[k] for k in args.engines.split(",")}

    def measure(name, g0, gs, gd, ts_, td_, plan, mode, once, eng):
        # reps back to back between two events (the host issues rep k+1 while rep k runs, as a
        # serving loop would); the host time per rep is reported beside it
        for _ in range(3):
            for x in once():
                dk.dyna_kv_wait(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # one untimed rep is enqueued first, so the device is busy when e0 is reached and the timed
        # region does not start with one call's host latency (validation, uploads) of idle device
        xs = once()
        e0.record(stream)
        t = time.perf_counter()
        for _ in range(args.reps):
            xs += once()
        e1.record(stream)
        host_ms = (time.perf_counter() - t) * 1e3 / args.reps
        for x in xs:
            dk.dyna_kv_wait(x)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        payload = s * 2 * g0.num_layers * g0.row_bytes
        gb = payload / (ms / 1e3) / 1e9
        r = {"model": name, "tp_src": ts_, "tp_dst": td_, "mode": mode, "engine": eng, "s": s, "chunk": c, "calls": len(plan),
             "slice_bytes": min(gs.row_bytes, gd.row_bytes), "payload_bytes": payload, "ms": ms, "GBps": gb,
             "hbm_rw_GBps": 2 * gb, "frac_of_measured_hbm": 2 * gb / pk, "host_ms_per_reshard": host_ms}
        print(json.dumps(r), flush=True)
        out.append(r)

    for name, g0, (ts_, td_) in cases:
        H, L = g0.num_kv_heads, g0.num_layers
        nb = 2 * kvgen.blocks_needed(s, g0.block_size) + 16
        gs = g0.with_(num_kv_heads=H // ts_, num_blocks=nb)
        gd = g0.with_(num_kv_heads=H // td_, num_blocks=nb)
        src = [dk.Pool(gs, 0) for _ in range(ts_)]
        dst = [dk.Pool(gd, 0) for _ in range(td_)]
        for i, p in enumerate(src + dst):
            dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), 100 + i, 0, cs)
        st = [dk.table(p, torch.from_numpy(t).cuda(), t) for p, t in
              ((p, kvgen.table_pair(10 + i, s, gs, gs)[0]) for i, p in enumerate(src))]
        dt = [dk.table(p, torch.from_numpy(t).cuda(), t) for p, t in
              ((p, kvgen.table_pair(20 + i, s, gd, gd)[1]) for i, p in enumerate(dst))]
        plan = dd.tp_reshard_plan(H, ts_, td_)

        for eng, e in engines.items():
            o = dk.opts(engine=e)

            def calls():
                return [dk.dyna_kv_migrate_heads(st[a], dt[b], (0, s), (0, L), heads, hd0, c, cs, o)
                        for a, b, heads, hd0 in plan]

            def fused():
                return [dk.dyna_kv_reshard([(st[a], dt[b], heads, hd0) for a, b, heads, hd0 in plan], (0, s), (0, L),
                                           c, cs, o)]
            for mode, once in (("calls", calls), ("one_launch", fused)):
                if ts_ == td_ == 1 and (mode == "one_launch" or eng != "rows"):
                    continue   # whole rows: the plain migration (ring), one line
                measure(name, g0, gs, gd, ts_, td_, plan, mode, once, eng)
        del src, dst, st, dt
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"device": torch.cuda.get_device_name(0), "hbm_peak_gbs": pk, "results": out},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
