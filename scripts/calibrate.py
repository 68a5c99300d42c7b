#!/usr/bin/env python
"""Variant / engine calibration sweep ("chosen over the staged
variant per chunk size by measured bandwidth").

For each row geometry and chunk size c, migrate one c-token chunk per call
(the paper's per-chunk push), cycling through the whole 4 GiB pool so
the working set never sits in L2, and time every candidate
(variant x engine x piece/stages/unroll) with CUDA events around each call.
The best candidate per (row bytes, chunk bucket) becomes the built-in table
(paper_2504_09285_b200/csrc/calib_default.inc); all measurements go to JSON.

    python scripts/calibrate.py [--out gpurun_out/calibration.json] [--inc gpurun_out/calib_default.inc]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

F, S = dk.DYNA_VARIANT_FUSED, dk.DYNA_VARIANT_STAGED
V, B, W = dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK, dk.DYNA_ENGINE_BULK_WS
CANDIDATES = [  # (variant, engine, piece, stages, unroll)
    (F, V, 8192, 0, 4), (F, V, 8192, 0, 8), (F, V, 4096, 0, 8), (F, V, 16384, 0, 8),
    (F, V, 16384, 0, 16), (F, V, 32768, 0, 16),
    (F, B, 16384, 8, 0), (F, B, 24576, 6, 0), (F, B, 32768, 3, 0), (F, B, 32768, 4, 0), (F, B, 32768, 6, 0),
    (F, B, 49152, 3, 0), (F, B, 49152, 4, 0), (F, B, 65536, 3, 0),
    (S, V, 8192, 0, 8), (S, B, 32768, 6, 0),
]
GEOMS = {8192: kvgen.LLAMA2_7B, 2048: kvgen.LLAMA3_8B.with_(num_blocks=2048),
         256: kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=6144)}   # TP-8 shard: 1 KV head per rank
CHUNKS = [16, 32, 64, 128, 256, 512, 1024, 2048, 4096]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "calibration.json"))
    ap.add_argument("--inc", default=os.path.join(ROOT, "gpurun_out", "calib_default.inc"))
    ap.add_argument("--min-ms", type=float, default=15.0)
    ap.add_argument("--select", help="re-run only the selection on a saved calibration.json")
    ap.add_argument("--peer", action="store_true",
                    help="also calibrate peer (NVLink) entries: source on cuda:0, destination on cuda:1 (needs 2 GPUs)")
    args = ap.parse_args()
    if args.select:
        d = json.load(open(args.select))
        write_outputs(args, d["measurements"], d["device"])
        return
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    rows, chosen = [], []
    pairs = [(0, 0)]
    if args.peer:
        if torch.cuda.device_count() < 2:
            print("--peer: fewer than 2 GPUs visible, peer entries skipped", file=sys.stderr)
        else:
            dk.dyna_kv_enable_peer(0, 1)
            pairs.append((0, 1))
    for (sdev, ddev), (row, g) in [(pr, rg) for pr in pairs for rg in GEOMS.items()]:
        peer = int(sdev != ddev)
        ntok = g.num_blocks * g.block_size
        src, dst = dk.Pool(g, sdev), dk.Pool(g, ddev)
        for p, seed in ((src, 1), (dst, 2)):
            dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
        torch.cuda.synchronize(ddev)
        rng = np.random.default_rng(row)
        ts, td = rng.permutation(g.num_blocks).astype(np.int32), rng.permutation(g.num_blocks).astype(np.int32)
        st = dk.table(src, torch.from_numpy(ts).to(f"cuda:{sdev}"), ts)
        dt = dk.table(dst, torch.from_numpy(td).to(f"cuda:{ddev}"), td)
        tok_bytes = 2 * g.num_layers * g.row_bytes
        for c in CHUNKS:
            n_calls = min(2000, max(20, int(args.min_ms * 1e-3 * 3.0e12 / (c * tok_bytes))))
            offs = [(i * c) % (ntok - c + 1) for i in range(n_calls)]
            results = []
            for (var, eng, piece, stages, unroll) in CANDIDATES:
                o = dk.opts(variant=var, engine=eng, piece_bytes=piece, stages=stages, unroll=unroll)

                def batch():
                    evs, xs = [], []
                    for off in offs:
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        a.record(stream)
                        xs.append(dk.dyna_kv_migrate_ex(st, dt, (off, off + c), (0, g.num_layers), c, cs, o))
                        b.record(stream)
                        evs.append((a, b))
                    for x in xs:
                        dk.dyna_kv_wait(x)
                    return statistics.median(a.elapsed_time(b) for a, b in evs)

                batch()  # warm-up
                ms = min(batch() for _ in range(2))
                gbps = c * tok_bytes / (ms / 1e3) / 1e9
                r = {"row_bytes": row, "peer": peer, "chunk": c, "variant": var, "engine": eng, "piece": piece,
                     "stages": stages, "unroll": unroll, "ms_per_call": ms, "GBps": gbps}
                results.append(r)
                rows.append(r)
                print(json.dumps(r), flush=True)
            best = max(results, key=lambda r: r["GBps"])
            chosen.append(best)
        src.close()
        dst.close()
    write_outputs(args, rows, torch.cuda.get_device_name(0))


def select(rows):
    """Per (row bytes, chunk bucket) pick the candidate with the best geometric-mean GB/s over the
    bucket and its two neighbours — event timing of one call is quantised (~0.5 us), so a plain
    per-bucket argmax flips between candidates that are within noise of each other."""
    import math
    chosen, entries = [], []
    classes = sorted({(r["row_bytes"], r.get("peer", 0)) for r in rows}, key=lambda x: (x[1], -x[0]))
    for row, peer in classes:
        mine = [r for r in rows if r["row_bytes"] == row and r.get("peer", 0) == peer]
        chunks = sorted({r["chunk"] for r in mine})
        key = lambda r: (r["variant"], r["engine"], r["piece"], r["stages"], r["unroll"])  # noqa: E731
        perf = {}
        for r in mine:
            perf[(r["chunk"], key(r))] = r["GBps"]
        cands = sorted({key(r) for r in mine})
        seq = []
        for i, c in enumerate(chunks):
            win = chunks[max(0, i - 1): i + 2]
            score = {k: sum(math.log(perf[(w, k)]) for w in win) / len(win) for k in cands}
            best = max(cands, key=lambda k: (score[k], perf[(c, k)]))
            # sticky: keep the previous bucket's choice while it is within 1% (fewer, stabler entries)
            if seq and score[seq[-1][1]] >= score[best] + math.log(0.99):
                best = seq[-1][1]
            seq.append((c, best, perf[(c, best)]))
            chosen.append({"row_bytes": row, "peer": peer, "chunk": c, "choice": best, "GBps": perf[(c, best)],
                           "best_single": max(perf[(c, k)] for k in cands)})
        for i, (c, best, _) in enumerate(seq):
            nxt = seq[i + 1] if i + 1 < len(seq) else None
            if nxt and nxt[1] == best:
                continue
            entries.append((row, peer, c if nxt else (1 << 30)) + tuple(best))
    return chosen, entries


def write_outputs(args, rows, device):
    chosen, entries = select(rows)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"device": device, "candidates": CANDIDATES, "measurements": rows,
               "chosen": chosen, "entries": entries}, open(args.out, "w"), indent=1)
    with open(args.inc, "w") as f:
        f.write(f"// Built-in calibration table, generated by scripts/calibrate.py on {device}\n")
        if any(e[1] for e in entries):
            f.write("// (measurements and choices: profiles/*calibration*.json).  Same-GPU and peer (NVLink) entries.\n")
        else:
            f.write("// (measurements and choices: profiles/*calibration*.json).  Same-GPU entries only;\n")
            f.write("// peer (NVLink) migrations fall back to FUSED + VEC until measured on a multi-GPU box.\n")
        f.write("// row_bytes, peer, max_chunk_tokens, variant, engine, piece_bytes, stages, unroll\n")
        for e in entries:
            f.write("    {" + ", ".join(str(x) for x in e) + "},\n")
        # generic fallback for other row sizes: the table of the most common (GQA, 2 KiB) row, per locality
        for peer in sorted({e[1] for e in entries}):
            gen = [e for e in entries if e[0] == 2048 and e[1] == peer] or [e for e in entries if e[1] == peer]
            f.write(f"    // generic fallback (row_bytes 0, peer {peer}) = the 2 KiB-row choices\n")
            for e in gen:
                f.write("    {" + ", ".join(str(x) for x in (0,) + tuple(e[1:])) + "},\n")
    print(json.dumps({"entries": entries}))


if __name__ == "__main__":
    main()
