#!/usr/bin/env python
"""BULK engine with small rings and several issuing CTAs per SM: k_copy_bulk is a 32-thread
CTA whose only issuing thread drives `stages` x `piece` bytes of shared memory, so a small
ring lets 2-7 CTAs (issuers) share an SM.  Device time per launch, signalled or not, on the
bench workload (Llama-2 rows, s = 1024, c = 256) and one Llama-3 4096-token chunk."""
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
    out = []
    cands = [(1, 8192, 0, 8), (2, 32768, 6, 0), (2, 49152, 4, 0), (2, 32768, 3, 0), (2, 16384, 6, 0), (2, 16384, 4, 0),
             (2, 16384, 3, 0), (2, 8192, 6, 0), (2, 8192, 4, 0), (2, 8192, 3, 0), (2, 4096, 6, 0), (2, 4096, 4, 0),
             (2, 24576, 4, 0), (2, 24576, 3, 0)]
    for name, g, s, c in (("llama2 s1024 c256", kvgen.LLAMA2_7B, 1024, 256),
                          ("llama3 s4096 c512", kvgen.LLAMA3_8B.with_(num_blocks=2048), 4096, 512)):
        src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
        dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 1, 0, cs)
        dk.dyna_kv_debug_fill(dst.tensor.data_ptr(), dst.tensor.numel(), 2, 0, cs)
        n = max(s, 2048)
        nset = 4 if kvgen.blocks_needed(n, g.block_size) * 4 <= g.num_blocks else 2
        tabs = kvgen.batch_tables(500, [n] * nset, g, g)
        T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b))
             for a, b in tabs]
        payload = s * 2 * g.num_layers * g.row_bytes
        for engine, piece, stages, unroll in cands:
            for sig in (0, 1):
                o = dk.opts(variant=1, engine=engine, piece_bytes=piece, stages=stages, unroll=unroll,
                            flags=dk.DYNA_MIGRATE_SIGNAL if sig else 0)
                try:
                    for i in range(6):
                        dk.dyna_kv_wait(dk.dyna_kv_migrate_ex(T[i % nset][0], T[i % nset][1], (0, s),
                                                              (0, g.num_layers), c, cs, o))
                except dk.DynaKVError as e:
                    print(json.dumps({"case": name, "engine": engine, "piece": piece, "stages": stages, "err": str(e)}))
                    continue
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(60)]
                xs = []
                for i, (a, b) in enumerate(ev):
                    a.record(stream)
                    xs.append(dk.dyna_kv_migrate_ex(T[i % nset][0], T[i % nset][1], (0, s), (0, g.num_layers), c, cs, o))
                    b.record(stream)
                for x in xs:
                    dk.dyna_kv_wait(x)
                torch.cuda.synchronize()
                ms = statistics.median(a.elapsed_time(b) for a, b in ev)
                r = {"case": name, "engine": engine, "piece": piece, "stages": stages, "signal": sig,
                     "us": round(ms * 1e3, 1), "GBps": round(payload / ms / 1e6)}
                print(json.dumps(r), flush=True)
                out.append(r)
        del src, dst, T
        torch.cuda.empty_cache()
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "bulk_ring_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
