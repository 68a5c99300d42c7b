#!/usr/bin/env python
"""Throughput vs SM budget (opts.max_ctas) of the fused migration: how many CTAs (SMs) a
migration needs to saturate HBM on one GPU, and by extension the ~900 GB/s of one NVLink
direction — the SM cost of overlapping the push with the prefill (SURVEY §8 "sweep the SM
budget").  One 4096-token Llama-3-8B chunk (512 MiB payload) and the bench request."""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402


def main():
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    cs = st.cuda_stream
    out = []
    for name, g, s, c in (("Llama-3-8B 4096-token chunk", kvgen.LLAMA3_8B.with_(num_blocks=2048), 4096, 4096),
                          ("Llama-2-7B bench request", kvgen.LLAMA2_7B, 1024, 256)):
        src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
        dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 1, 0, cs)
        dk.dyna_kv_debug_fill(dst.tensor.data_ptr(), dst.tensor.numel(), 2, 0, cs)
        tabs = kvgen.batch_tables(3, [s] * 2, g, g)
        T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b)) for a, b in tabs]
        payload = s * 2 * g.num_layers * g.row_bytes
        for engine in (1, 2):
            for ctas in (2, 4, 8, 16, 32, 64, 148, 0):
                o = dk.opts(variant=1, engine=engine, max_ctas=ctas)
                for i in range(3):
                    dk.dyna_kv_wait(dk.dyna_kv_migrate_ex(T[i % 2][0], T[i % 2][1], (0, s), (0, g.num_layers), c, cs, o))
                ms = []
                for i in range(8):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    x = dk.dyna_kv_migrate_ex(T[i % 2][0], T[i % 2][1], (0, s), (0, g.num_layers), c, cs, o)
                    b.record(st)
                    dk.dyna_kv_wait(x)
                    b.synchronize()
                    ms.append(a.elapsed_time(b))
                m = statistics.median(ms)
                r = {"case": name, "engine": "VEC" if engine == 1 else "BULK", "max_ctas": ctas or "all",
                     "us": round(m * 1e3, 1), "GBps": round(payload / m / 1e6)}
                print(json.dumps(r), flush=True)
                out.append(r)
        del src, dst, T
        torch.cuda.empty_cache()
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sm_budget.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
