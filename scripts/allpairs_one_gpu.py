#!/usr/bin/env python
"""configs[4] all ordered instance pairs, emulated on ONE B200 (measurement + full row check).

    python scripts/allpairs_one_gpu.py [--world 8] [--steps 5] [--warmup 3] [--mode auto|one|per-receiver]

The 8-GPU form (scripts/allpairs.py, bench.py N >= 3) has every rank push its outgoing requests
into its peers' receive pools over NVLink.  With one GPU the ranks are emulated as B200_PROFILING
prescribes — one kernel over all ranks' data, no rank waiting on another: the seeded plan
(kvgen.allpairs_plan, Qwen2-72B shard geometry) with each rank's block ids relabelled onto pools
that fit one device (kvgen.compact_plan), every request of every ordered pair in ONE
dyna_kv_migrate_batch (mode one), or one batch per receiving rank with all its senders (mode
per-receiver, when sixteen pools do not fit).  The bytes cross HBM, not NVLink: the number is the
1-GPU (reblock) form of configs[4] against the HBM copy peak; the NVLink load-aware bound of the
real plan is printed beside it as context.  Every destination row of every request is then checked
on the device against its source row (torch indexing).
"""
from __future__ import annotations

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
from paper_2504_09285_b200 import dist as dd  # noqa: E402


def peak():
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        return float(json.load(f)["hbm_gbs"])


def filled(g, seed, instance, st):
    p = dk.Pool(g, 0, instance)
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, st)
    return p


def rows_equal(src, ts, dst, td, s, g):
    S = src.tensor.view(g.num_layers, 2, -1, g.block_size, g.row_bytes)
    D = dst.tensor.view(g.num_layers, 2, -1, g.block_size, g.row_bytes)
    Ts = torch.as_tensor(np.asarray(ts, np.int64), device="cuda")
    Td = torch.as_tensor(np.asarray(td, np.int64), device="cuda")
    ok = True
    for a in range(0, s, 2048):
        t = torch.arange(a, min(a + 2048, s), device="cuda")
        ok &= bool(torch.equal(D[:, :, Td[t // g.block_size], t % g.block_size],
                               S[:, :, Ts[t // g.block_size], t % g.block_size]))
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--mode", choices=["auto", "one", "per-receiver"], default="auto")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    g = kvgen.QWEN2_72B
    full = kvgen.allpairs_plan(a.world, g)
    plan, ns, nd = kvgen.compact_plan(full, spare=2)
    tok = 2 * g.num_layers * g.row_bytes
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    src = {r: filled(g.with_(num_blocks=ns[r]), 3000 + r, r, cs) for r in range(a.world)}
    free, total = torch.cuda.mem_get_info()
    need = sum(nd.values()) * g.block_size * tok
    mode = a.mode
    if mode == "auto":
        mode = "one" if need < free - (6 << 30) else "per-receiver"
    groups = [list(range(a.world))] if mode == "one" else [[j] for j in range(a.world)]
    out = {"config": f"configs[4] all ordered pairs, Qwen2-72B shard, world {a.world}, emulated on one B200 "
                     f"({'one launch over every rank' if mode == 'one' else 'one launch per receiving rank'})",
           "migrations": len(plan), "chunk_tokens": a.chunk, "mode": mode,
           "src_blocks": ns, "recv_blocks": nd, "groups": []}
    tot_bytes, tot_ms, bad = 0, 0.0, 0
    for grp in groups:
        recv = {j: filled(g.with_(num_blocks=nd[j]), 4000 + j, j, cs) for j in grp}
        ms_ = [m for m in plan if m.dst_rank in recv]
        keep = [(torch.from_numpy(m.src_table).cuda(), torch.from_numpy(m.dst_table).cuda()) for m in ms_]
        migs = [(dk.table(src[m.src_rank], ts, m.src_table), dk.table(recv[m.dst_rank], td, m.dst_table), (0, m.req.s))
                for (ts, td), m in zip(keep, ms_)]
        nbytes = sum(m.req.s for m in ms_) * tok
        torch.cuda.synchronize()

        def step():
            return dk.dyna_kv_migrate_batch(migs, (0, g.num_layers), a.chunk, cs, None)

        for _ in range(a.warmup):
            dk.dyna_kv_wait(step())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        xs = [step() for _ in range(a.steps)]
        e1.record(stream)
        plan_info = dk.dyna_kv_xfer_plan(xs[0])
        for x in xs:
            dk.dyna_kv_wait(x)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        nbad = sum(0 if rows_equal(src[m.src_rank], m.src_table, recv[m.dst_rank], m.dst_table, m.req.s, g) else 1
                   for m in ms_)
        bad += nbad
        tot_bytes += nbytes
        tot_ms += ms
        out["groups"].append({"receivers": grp, "requests": len(ms_), "bytes": nbytes, "ms": ms,
                              "GBps": nbytes / ms / 1e6, "frac_of_measured_hbm": 2 * nbytes / ms / 1e6 / peak(),
                              "plan": plan_info, "bad_requests": nbad})
        for p in recv.values():
            p.close()
        del recv, migs, keep
        torch.cuda.empty_cache()
    pb = {}
    for m in full:
        pb[(m.src_rank, m.dst_rank)] = pb.get((m.src_rank, m.dst_rank), 0) + m.req.s * tok
    out.update({"bytes": tot_bytes, "ms": tot_ms, "GBps": tot_bytes / tot_ms / 1e6,
                "frac_of_measured_hbm": 2 * tot_bytes / tot_ms / 1e6 / peak(), "hbm_peak_gbs": peak(),
                "nvlink_load_aware_bound_ms_900": dd.load_aware_bound_s(pb, 900e9) * 1e3 if a.world > 1 else None,
                "nvlink_load_aware_bound_ms_770": dd.load_aware_bound_s(pb, 770e9) * 1e3 if a.world > 1 else None,
                "bad_requests": bad, "rows_checked": "every row of every request (device, torch indexing)"})
    print(json.dumps(out))
    for p in src.values():
        p.close()
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
