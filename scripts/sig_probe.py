#!/usr/bin/env python
"""Cost of per-chunk signalling per engine on the bench workload (configs[1]: Llama-2-7B rows,
s = 1024, c = 256, 4 rotating requests): device time per launch, signalled vs not."""
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
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    g = kvgen.LLAMA2_7B
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 1, 0, cs)
    dk.dyna_kv_debug_fill(dst.tensor.data_ptr(), dst.tensor.numel(), 2, 0, cs)
    s, c = int(os.environ.get("S", 1024)), int(os.environ.get("C", 256))
    engines = [int(e) for e in os.environ.get("ENGINES", "1,2,3,4").split(",")]
    tabs = kvgen.batch_tables(500, [max(s, 2048)] * 4, g, g) if s <= 2048 else kvgen.batch_tables(500, [s] * 2, g, g) * 2
    T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b)) for a, b in tabs]
    payload = s * 2 * g.num_layers * g.row_bytes
    out = []
    cands = ((1, 8192, 0, 8), (2, 32768, 6, 0), (3, 32768, 6, 0), (4, 0, 0, 0))
    if os.environ.get("VEC_SWEEP"):  # VEC shapes only
        cands = ((1, 8192, 0, 8), (1, 4096, 0, 8), (1, 16384, 0, 8), (1, 8192, 0, 16), (1, 16384, 0, 16),
                 (1, 32768, 0, 16), (1, 8192, 0, 4), (1, 4096, 0, 4))
    for engine, piece, stages, unroll in [e for e in cands if e[0] in engines]:
        for sig in (0, 1):
            o = dk.opts(variant=1, engine=engine, piece_bytes=piece, stages=stages, unroll=unroll,
                        flags=dk.DYNA_MIGRATE_SIGNAL if sig else 0)
            for i in range(8):
                dk.dyna_kv_wait(dk.dyna_kv_migrate_ex(T[i % 4][0], T[i % 4][1], (0, s), (0, 32), c, cs, o))
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(int(os.environ.get("N", 200)))]
            xs = []
            for i, (a, b) in enumerate(ev):
                a.record(stream)
                xs.append(dk.dyna_kv_migrate_ex(T[i % 4][0], T[i % 4][1], (0, s), (0, 32), c, cs, o))
                b.record(stream)
            for x in xs:
                dk.dyna_kv_wait(x)
            torch.cuda.synchronize()
            ms = statistics.median(a.elapsed_time(b) for a, b in ev)
            r = {"engine": engine, "piece": piece, "unroll": unroll, "signal": sig, "us": ms * 1e3,
                 "GBps": payload / ms / 1e6}
            print(json.dumps(r), flush=True)
            out.append(r)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sig_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
