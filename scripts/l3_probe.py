#!/usr/bin/env python
"""Why Llama-3-8B rows (2 KiB rows, 32-KiB blocks) stream at ~0.90 of the HBM
peak while Llama-2-7B rows (8 KiB, 128-KiB blocks) reach ~0.97: one 4096-token
chunk (512 MiB payload, the 4' target shape, 1-GPU form) per call, swept over
engine / piece / stages, pool size (TLB reach) and table kind (fragmented vs
contiguous).  Device time with CUDA events, 4 rotating requests (> L2)."""
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
    s = 4096
    res = []
    for gname, g0 in (("llama3", kvgen.LLAMA3_8B), ("llama2", kvgen.LLAMA2_7B)):
        for nb_mult, kind in ((1, "fragmented"), (1, "contiguous"), (4, "fragmented"), (16, "fragmented")):
            need = 4 * kvgen.blocks_needed(s, g0.block_size)
            g = g0.with_(num_blocks=need * nb_mult)
            if g.pool_bytes > 40 << 30:
                continue
            src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
            if kind == "contiguous":
                nblk = kvgen.blocks_needed(s, g.block_size)
                tabs = [(kvgen.contiguous_table(i * nblk, nblk), kvgen.contiguous_table(i * nblk, nblk)) for i in range(4)]
            else:
                tabs = kvgen.batch_tables(7, [s] * 4, g, g)
            T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b))
                 for a, b in tabs]
            payload = s * 2 * g.num_layers * g.row_bytes
            cands = [("auto", dk.opts())]
            if nb_mult == 1 and kind == "fragmented":
                cands += [(f"bulk p{p//1024}k st{st}", dk.opts(variant=1, engine=2, piece_bytes=p, stages=st))
                          for p, st in ((32768, 6), (32768, 4), (16384, 12), (16384, 8), (32768, 3), (8192, 16))]
                cands += [("bulk_ws p32k st6", dk.opts(variant=1, engine=3, piece_bytes=32768, stages=6)),
                          ("vec p8k u8", dk.opts(variant=1, engine=1, piece_bytes=8192, unroll=8)),
                          ("vec p16k u16", dk.opts(variant=1, engine=1, piece_bytes=16384, unroll=16))]
            for name, o in cands:
                def once(i):
                    return dk.dyna_kv_migrate_ex(T[i % 4][0], T[i % 4][1], (0, s), (0, g.num_layers), s, cs, o)
                for i in range(8):
                    dk.dyna_kv_wait(once(i))
                ms = []
                for i in range(24):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    x = once(i)
                    e1.record(stream)
                    dk.dyna_kv_wait(x)
                    e1.synchronize()
                    ms.append(e0.elapsed_time(e1))
                m = statistics.median(ms)
                r = {"rows": gname, "pool_GiB": round(g.pool_bytes / 2**30, 1), "tables": kind, "cand": name,
                     "ms": m, "payload_GBps": payload / m / 1e6, "rw_GBps": 2 * payload / m / 1e6}
                print(json.dumps(r), flush=True)
                res.append(r)
            del src, dst, T
            torch.cuda.empty_cache()
    json.dump(res, open(os.path.join(ROOT, "gpurun_out", "l3_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
