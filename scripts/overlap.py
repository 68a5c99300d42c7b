#!/usr/bin/env python
"""Config 4 overlap experiment: chunked KV migration concurrent with the prefill.

PAPER.md §4.3: r^alpha is processed in equal-sized chunks; once chunk k
completes its KV is pushed while chunk k+1 computes.  §6.6: chunking
"reduces non-overlapped transfer by 94%" (A100, Mini-Reasoning; model and
chunk size not stated) — context, not a target.

Workload (BASELINE.json configs[3]): Llama-3-8B GQA pools (32 L, 8 KV heads,
d128, bf16, block 16), a 32k-token prompt, chunk c in {512, 1024, 2048, 4096}.
Stand-in producer (NOT part of the path; torch.matmul = cuBLAS): per chunk,
N_GEMM bf16 GEMMs of [c, 4096] x [4096, 14336] — 128 of them ~= the dense
prefill FLOPs of Llama-3-8B (2 * ~7e9 * c).  After chunk k's GEMMs an event is
recorded; the migration stream waits on it and pushes chunk k.

Reported per (c, SM budget), all from CUDA events inside the same run:
  exposed_chunked  end of the producer's last chunk -> end of the last per-chunk
                   migration (chunk k pushed as soon as chunk k is computed)
  exposed_whole    end of the producer -> end of one whole-range migration
                   issued after the prefill (no chunking)
  reduction = 1 - exposed_chunked / exposed_whole     (the P:738 analogue)
  producer_slowdown  producer time with concurrent chunked migrations vs alone
  ready_coupled    the same with ONE dyna_kv_migrate_on_ready launch that waits
                   on the device for the producer's per-chunk marks
  --layers adds the layer-granular forms ("can be composed with" layer-
  level transfer): the producer runs a chunk layer by layer (n_gemm/32 GEMMs per
  layer) and
  layered          pushes (chunk k, layer l) as soon as layer l of chunk k is done
                   (one dyna_kv_migrate per chunk x layer, host-enqueued)
  ready_layers     one coupled launch with DYNA_READY_PER_LAYER marks
  ready_tail       a coupled launch (per-chunk marks) for every chunk but the last, and the
                   last chunk pushed by a full-width dyna_kv_migrate once the producer ends
                   (the coupled kernel's CTA budget no longer caps the tail)
On one GPU the migration is an intra-device reblock (HBM); on the 8-GPU box
the same script with a peer destination measures the NVLink form.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

N_GEMM = 128   # 4 per layer: ~= the dense prefill FLOPs of Llama-3-8B per chunk (2 * ~7e9 * c)


OV = dk.DYNA_MIGRATE_OVERLAP_PREV


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--s", type=int, default=32768)
    ap.add_argument("--chunks", default="512,1024,2048,4096")
    ap.add_argument("--budgets", default="0,74,32,16")
    ap.add_argument("--n-gemm", type=int, default=N_GEMM)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ready-ctas", type=int, default=8, help="CTA budget of the coupled launch when budget is 0")
    ap.add_argument("--layers", action="store_true", help="add the layer-granular modes")
    ap.add_argument("--dst-device", type=int, default=0, help="destination pool's GPU (1: the NVLink form)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "overlap.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    g = kvgen.LLAMA3_8B.with_(num_blocks=4096)
    s = args.s
    if args.dst_device:
        dk.dyna_kv_enable_peer(0, args.dst_device)
    src, dst = dk.Pool(g, 0), dk.Pool(g, args.dst_device)
    for p, seed in ((src, 1), (dst, 2)):
        dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
    ts, td = kvgen.table_pair(3, s, g, g)
    st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
    dt = dk.table(dst, torch.from_numpy(td).cuda(), td)   # read by the kernel on the source GPU (cuda:0)
    W = torch.randn(4096, 14336, dtype=torch.bfloat16, device="cuda") * 0.01
    prod, mig, mig2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    payload = s * 2 * g.num_layers * g.row_bytes
    results = []

    def producer_chunk(X):
        for _ in range(args.n_gemm):
            torch.matmul(X, W)

    def producer_layer(X):
        for _ in range(max(1, args.n_gemm // g.num_layers)):
            torch.matmul(X, W)

    def run(c, mode, budget):
        """One run.  Returns (T_prod_ms, exposed_ms): exposed = time from the end of the
        producer's last chunk to the end of the last migration (the non-overlapped transfer)."""
        X = xs_in[c]
        nck = -(-s // c)
        torch.cuda.synchronize()
        e0, e_prod, e_mig = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(prod)
        mig.wait_event(e0)
        handles = []
        if mode in ("ready", "ready_layers", "ready_tail"):   # one launch; waits on the device for marks
            epoch = dk.dyna_kv_ready_begin(board)
            fl = dk.DYNA_READY_PER_LAYER if mode == "ready_layers" else 0
            end = (nck - 1) * c if mode == "ready_tail" else s
            if end > 0:
                handles.append(dk.dyna_kv_migrate_on_ready(st, dt, (0, end), (0, 32), c, board, epoch,
                                                           mig.cuda_stream,
                                                           dk.opts(max_ctas=budget or args.ready_ctas, flags=fl)))
        for k in range(nck):
            if mode in ("layered", "ready_layers", "layered_ov"):
                for l in range(g.num_layers):
                    with torch.cuda.stream(prod):
                        producer_layer(X)
                    if mode == "ready_layers":
                        dk.dyna_kv_ready_mark(board, dk.ready_slot(k, l, (0, 32)), epoch, prod.cuda_stream)
                    else:                             # layer l of chunk k complete -> push it now
                        ev = torch.cuda.Event()
                        ev.record(prod)
                        mig.wait_event(ev)
                        handles.append(dk.migrate(st, dt, (k * c, min((k + 1) * c, s)), (l, l + 1), c, stream=mig,
                                                  max_ctas=budget, flags=OV if mode == "layered_ov" else 0))
                continue
            with torch.cuda.stream(prod):
                producer_chunk(X)
            if mode == "ready" or (mode == "ready_tail" and k < nck - 1):
                dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
            if mode == "ready_tail" and k == nck - 1:   # the last chunk: full width, beside the coupled kernel
                ev = torch.cuda.Event()
                ev.record(prod)
                mig2.wait_event(ev)
                handles.append(dk.migrate(st, dt, (k * c, s), (0, 32), c, stream=mig2, max_ctas=budget))
                e_tail = torch.cuda.Event(enable_timing=True)
                e_tail.record(mig2)
                mig.wait_event(e_tail)
            if mode in ("chunked", "chunked_ov"):    # chunk k complete -> push it now
                ev = torch.cuda.Event()
                ev.record(prod)
                mig.wait_event(ev)
                # chunked_ov: DYNA_MIGRATE_OVERLAP_PREV — push k may start while push k-1 drains (disjoint rows)
                handles.append(dk.migrate(st, dt, (k * c, min((k + 1) * c, s)), (0, 32), c, stream=mig,
                                          max_ctas=budget, flags=OV if mode == "chunked_ov" else 0))
        e_prod.record(prod)
        if mode == "whole":                           # no chunking: push everything after the prefill
            mig.wait_event(e_prod)
            handles.append(dk.migrate(st, dt, (0, s), (0, 32), c, stream=mig, max_ctas=budget))
        e_mig.record(mig)
        torch.cuda.synchronize()
        for x in handles:
            dk.dyna_kv_wait(x)
        return e0.elapsed_time(e_prod), max(0.0, e_prod.elapsed_time(e_mig))

    board = dk.dyna_kv_ready_create(0, 1 << 16)
    xs_in = {}
    for c in [int(x) for x in args.chunks.split(",")]:
        xs_in[c] = torch.randn(c, 4096, dtype=torch.bfloat16, device="cuda")
        # migration alone (whole range), for reference
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(mig)
        x = dk.migrate(st, dt, (0, s), (0, 32), c, stream=mig)
        a1.record(mig)
        dk.dyna_kv_wait(x)
        t_mig = a0.elapsed_time(a1)
        prod_alone = statistics.median(run(c, "none", 0)[0] for _ in range(args.reps))
        for budget in [int(x) for x in args.budgets.split(",")]:
            W_, C_, R_, LY, RL, RT, CO, LO = [], [], [], [], [], [], [], []
            run(c, "whole", budget)
            run(c, "chunked", budget)   # warm
            run(c, "chunked_ov", budget)
            run(c, "ready", budget)
            run(c, "ready_tail", budget)
            if args.layers:
                run(c, "layered", budget)
                run(c, "layered_ov", budget)
                run(c, "ready_layers", budget)
            for _ in range(args.reps):  # interleaved so drift hits all modes alike
                W_.append(run(c, "whole", budget))
                C_.append(run(c, "chunked", budget))
                CO.append(run(c, "chunked_ov", budget))
                R_.append(run(c, "ready", budget))
                RT.append(run(c, "ready_tail", budget))
                if args.layers:
                    LY.append(run(c, "layered", budget))
                    LO.append(run(c, "layered_ov", budget))
                    RL.append(run(c, "ready_layers", budget))
            exp_w = statistics.median(e for _, e in W_)
            exp_c = statistics.median(e for _, e in C_)
            exp_r = statistics.median(e for _, e in R_)
            prod_c = statistics.median(p for p, _ in C_)
            prod_r = statistics.median(p for p, _ in R_)
            r = {"chunk": c, "sm_budget_ctas": budget, "T_migrate_alone_ms": t_mig,
                 "migrate_alone_GBps": payload / (t_mig / 1e3) / 1e9,
                 "T_prod_alone_ms": prod_alone, "T_prod_with_chunked_ms": prod_c,
                 "producer_slowdown": prod_c / prod_alone - 1,
                 "exposed_whole_ms": exp_w, "exposed_chunked_ms": exp_c,
                 "reduction": 1 - exp_c / exp_w if exp_w > 0 else None,
                 "ready_coupled": {"ctas": budget or args.ready_ctas, "exposed_ms": exp_r, "T_prod_ms": prod_r,
                                   "producer_slowdown": prod_r / prod_alone - 1,
                                   "reduction": 1 - exp_r / exp_w if exp_w > 0 else None}}
            exp_t = statistics.median(e for _, e in RT)
            prod_t = statistics.median(p for p, _ in RT)
            r["ready_tail"] = {"ctas": budget or args.ready_ctas, "exposed_ms": exp_t, "T_prod_ms": prod_t,
                               "producer_slowdown": prod_t / prod_alone - 1,
                               "reduction": 1 - exp_t / exp_w if exp_w > 0 else None}
            exp_o = statistics.median(e for _, e in CO)
            prod_o = statistics.median(p for p, _ in CO)
            r["chunked_overlap_prev"] = {"exposed_ms": exp_o, "T_prod_ms": prod_o,
                                         "producer_slowdown": prod_o / prod_alone - 1,
                                         "reduction": 1 - exp_o / exp_w if exp_w > 0 else None}
            if args.layers:
                for name, runs in (("layered", LY), ("layered_overlap_prev", LO), ("ready_layers", RL)):
                    exp_l = statistics.median(e for _, e in runs)
                    prod_l = statistics.median(p for p, _ in runs)
                    r[name] = {"exposed_ms": exp_l, "T_prod_ms": prod_l, "producer_slowdown": prod_l / prod_alone - 1,
                               "reduction": 1 - exp_l / exp_w if exp_w > 0 else None}
                    if name == "ready_layers":
                        r[name]["ctas"] = budget or args.ready_ctas
            print(json.dumps(r), flush=True)
            results.append(r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"workload": "configs[3] Llama-3-8B 32k prompt, 1-GPU reblock", "n_gemm_per_chunk": args.n_gemm,
               "exposed": "end of producer's last chunk -> end of last migration (CUDA events, same run)",
               "gemm": "[c,4096]x[4096,14336] bf16 (torch.matmul, stand-in producer)", "results": results},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
