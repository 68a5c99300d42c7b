#!/usr/bin/env python
"""Throughput of every BASELINE.json config on one B200 (intra-device form).

For each config: the exact workload shape, migrated through the C ABI with
AUTO selection, timed with CUDA events on the launch stream over repeated
runs (after warm-up), with the working set rotated or larger than L2.
Reported: payload GB/s, tokens/s, HBM read+write GB/s and its fraction of
the measured copy peak (MEASURED_PEAKS.json), launches per run.

    python scripts/configs_sweep.py [--out gpurun_out/configs.json]
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

OV = dk.opts(flags=dk.DYNA_MIGRATE_OVERLAP_PREV)  # the requests / chunks of each set are disjoint


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def run_set(stream, calls, reps=10, warm=3):
    """calls: list of zero-arg functions each enqueuing one migrate and returning its handle.
    Device time per set of calls, sets issued back to back (as a serving loop issues them): one
    untimed set is enqueued before the start event, so the timed region does not open with one
    call's host latency on an idle device; the host issues set k+1 while set k runs."""
    def once():
        xs = [c() for c in calls]
        return xs
    for _ in range(warm):
        for x in once():
            dk.dyna_kv_wait(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xs = once()
    a.record(stream)
    for _ in range(reps):
        xs += once()
    b.record(stream)
    for x in xs:
        dk.dyna_kv_wait(x)
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "configs.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream
    pk = peak()
    out = []

    def report(name, payload, ms, ntok, launches, note=""):
        gb = payload / (ms / 1e3) / 1e9
        r = {"config": name, "payload_bytes": payload, "ms": ms, "GBps": gb, "tokens_per_s": ntok / (ms / 1e3),
             "hbm_rw_GBps": 2 * gb, "frac_of_measured_hbm": 2 * gb / pk, "launches": launches, "note": note}
        print(json.dumps(r), flush=True)
        out.append(r)

    def pools(g, s1, s2):
        a, b = dk.Pool(g, 0), dk.Pool(g, 0)
        dk.dyna_kv_debug_fill(a.tensor.data_ptr(), a.tensor.numel(), s1, 0, cs)
        dk.dyna_kv_debug_fill(b.tensor.data_ptr(), b.tensor.numel(), s2, 0, cs)
        return a, b

    def tab(p, ids):
        return dk.table(p, torch.from_numpy(ids).cuda(), ids)

    # configs[0] toy: 100 tokens, chunk 32 (latency-bound; rotate 8 requests over the pool)
    g = kvgen.TOY
    src, dst = pools(g, 1, 2)
    tabs = kvgen.batch_tables(1, [256] * 4, g, g)
    T = [(tab(src, a), tab(dst, b)) for a, b in tabs]
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, 100), (0, 2), 32, cs, None) for t in T]
    ms = run_set(stream, calls * 25, reps=5)
    report("configs[0] toy s=100 c=32", 100 * 2 * 2 * g.row_bytes * 100, ms, 100 * 100, 100, "100 calls")
    del src, dst

    # configs[1] Llama-2-7B, s = 1024 of 2048, chunk 256 (the bench workload), plus the R12 edge sweep
    g = kvgen.LLAMA2_7B
    src, dst = pools(g, 3, 4)
    tabs = kvgen.batch_tables(5, [2048] * 4, g, g)
    T = [(tab(src, a), tab(dst, b)) for a, b in tabs]
    for s in (1024, 1, 16, 17, 100, 1000, 2047, 2048):
        calls = [lambda t=t, s=s: dk.dyna_kv_migrate_ex(t[0], t[1], (0, s), (0, 32), 256, cs, None) for t in T]
        ms = run_set(stream, calls * 4, reps=5)
        report(f"configs[1] Llama-2-7B s={s} c=256", 16 * s * 2 * 32 * g.row_bytes, ms, 16 * s, 16)
    del src, dst, T

    # configs[2] Llama-3-8B skewed batch of 64 (one call per migrating request)
    g = kvgen.LLAMA3_8B
    src, dst = pools(g, 5, 6)
    reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
    tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
    T = [(tab(src, a), tab(dst, b), r.s) for r, (a, b) in zip(reqs, tabs)]
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 32), 256, cs, None) for t in T]
    tot = sum(r.s for r in reqs)
    ms = run_set(stream, calls, reps=5)
    report(f"configs[2] Llama-3-8B skewed batch ({len(reqs)} migrating of 64, sum s={tot}) c=256",
           tot * 2 * 32 * g.row_bytes, ms, tot, len(calls), "one dyna_kv_migrate per request")
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 32), 256, cs, OV) for t in T]
    ms = run_set(stream, calls, reps=5)
    report(f"configs[2] Llama-3-8B skewed batch ({len(reqs)} migrating of 64, sum s={tot}) c=256, OVERLAP_PREV",
           tot * 2 * 32 * g.row_bytes, ms, tot, len(calls), "one dyna_kv_migrate per request, overlapping each other")
    migs = [(t[0], t[1], (0, t[2])) for t in T]
    ms = run_set(stream, [lambda: dk.dyna_kv_migrate_batch(migs, (0, 32), 256, cs, None)], reps=5)
    report(f"configs[2] Llama-3-8B skewed batch ({len(reqs)} migrating of 64, sum s={tot}) c=256, batched",
           tot * 2 * 32 * g.row_bytes, ms, tot, 1, "one dyna_kv_migrate_batch launch")
    del src, dst, T

    # configs[3] Llama-3-8B 32k prompt, chunk sweep: one call per chunk (the per-chunk push) and one call per range
    g = kvgen.LLAMA3_8B.with_(num_blocks=4096)
    src, dst = pools(g, 7, 8)
    ts, td = kvgen.table_pair(3, 32768, g, g)
    st, dt = tab(src, ts), tab(dst, td)
    payload = 32768 * 2 * 32 * g.row_bytes
    for c in (512, 1024, 2048, 4096):
        calls = [lambda k=k, c=c: dk.dyna_kv_migrate_ex(st, dt, (k * c, (k + 1) * c), (0, 32), c, cs, None)
                 for k in range(32768 // c)]
        ms = run_set(stream, calls, reps=5)
        report(f"configs[3] Llama-3-8B s=32768 per-chunk calls c={c}", payload, ms, 32768, len(calls))
        calls = [lambda k=k, c=c: dk.dyna_kv_migrate_ex(st, dt, (k * c, (k + 1) * c), (0, 32), c, cs, OV)
                 for k in range(32768 // c)]
        ms = run_set(stream, calls, reps=5)
        report(f"configs[3] Llama-3-8B s=32768 per-chunk calls c={c}, OVERLAP_PREV", payload, ms, 32768, len(calls),
               "chunks are disjoint: each call starts while the previous drains")
    ms = run_set(stream, [lambda: dk.dyna_kv_migrate_ex(st, dt, (0, 32768), (0, 32), 1024, cs, None)], reps=5)
    report("configs[3] Llama-3-8B s=32768 one call c=1024", payload, ms, 32768, 1)
    # 4' target shape: one 4096-token chunk (here intra-device; the target is 2 GPUs over NVLink)
    calls = [lambda k=k: dk.dyna_kv_migrate_ex(st, dt, (k * 4096, (k + 1) * 4096), (0, 32), 4096, cs, None)
             for k in range(8)]
    ms = run_set(stream, calls, reps=5)
    report("target 4' shape: 4096-token Llama-3-8B chunk (1-GPU form)", payload, ms, 32768, 8,
           "NVLink form needs 2 GPUs")
    calls = [lambda k=k: dk.dyna_kv_migrate_ex(st, dt, (k * 4096, (k + 1) * 4096), (0, 32), 4096, cs, OV)
             for k in range(8)]
    ms = run_set(stream, calls, reps=5)
    report("target 4' shape: 4096-token Llama-3-8B chunk (1-GPU form), OVERLAP_PREV", payload, ms, 32768, 8,
           "NVLink form needs 2 GPUs")
    # the push's halves and the staged variant on the 4' shape (SURVEY 8a a2 / a3 / a4, 1-GPU form):
    # K1 pack (paged -> contiguous buffer), K3 unpack (buffer -> paged), and STAGED K1 -> K2 -> K3
    chunk_bytes = 4096 * 2 * 32 * g.row_bytes
    buf = torch.empty(chunk_bytes, dtype=torch.uint8, device="cuda")
    calls = [lambda k=k: dk.dyna_kv_pack(st, (k * 4096, (k + 1) * 4096), (0, 32), buf.data_ptr(), chunk_bytes, cs)
             for k in range(8)]
    ms = run_set(stream, calls, reps=5)
    report("4' shape: K1 pack (paged -> packed chunk), 8 chunks", payload, ms, 32768, 8, "a2 gather")
    calls = [lambda k=k: dk.dyna_kv_unpack(buf.data_ptr(), chunk_bytes, dt, (k * 4096, (k + 1) * 4096), (0, 32), cs)
             for k in range(8)]
    ms = run_set(stream, calls, reps=5)
    report("4' shape: K3 unpack (packed chunk -> paged), 8 chunks", payload, ms, 32768, 8, "a4 scatter")
    calls = [lambda k=k: dk.dyna_kv_migrate_ex(st, dt, (k * 4096, (k + 1) * 4096), (0, 32), 4096, cs,
                                               dk.opts(variant=dk.DYNA_VARIANT_STAGED))
             for k in range(8)]
    ms = run_set(stream, calls, reps=5)
    report("4' shape: STAGED variant (K1 -> K2 copy engine -> K3), 8 chunks", payload, ms, 32768, 8,
           "3x the fused variant's HBM traffic on one GPU")
    del src, dst, buf

    # configs[4] Qwen2-72B-shaped shard (80 layers): one ordered pair's 4 requests, chunk 1024
    g = kvgen.QWEN2_72B
    src, dst = pools(g, 9, 10)
    reqs = kvgen.migrating(kvgen.skewed_batch(1000 + 1, 4))
    tabs = kvgen.batch_tables(3, [r.s for r in reqs], g, g)
    T = [(tab(src, a), tab(dst, b), r.s) for r, (a, b) in zip(reqs, tabs)]
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 80), 1024, cs, None) for t in T]
    tot = sum(r.s for r in reqs)
    ms = run_set(stream, calls, reps=5)
    report(f"configs[4] Qwen2-72B shard, one pair's {len(reqs)} requests (sum s={tot}) c=1024",
           tot * 2 * 80 * g.row_bytes, ms, tot, len(calls), "all-pairs 8-GPU form needs 8 GPUs")
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 80), 1024, cs, OV) for t in T]
    ms = run_set(stream, calls, reps=5)
    report(f"configs[4] Qwen2-72B shard, one pair's {len(reqs)} requests (sum s={tot}) c=1024, OVERLAP_PREV",
           tot * 2 * 80 * g.row_bytes, ms, tot, len(calls), "per-request calls overlapping each other")
    migs = [(t[0], t[1], (0, t[2])) for t in T]
    ms = run_set(stream, [lambda: dk.dyna_kv_migrate_batch(migs, (0, 80), 1024, cs, None)], reps=5)
    report(f"configs[4] Qwen2-72B shard, one pair's {len(reqs)} requests (sum s={tot}) c=1024, batched",
           tot * 2 * 80 * g.row_bytes, ms, tot, 1, "one dyna_kv_migrate_batch launch")
    del src, dst, T
    # NEXT-3 shape: TP-8 Qwen2-72B shard (1 KV head per rank: 256-B rows, 4-KiB segments)
    g = kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=6144)
    src, dst = pools(g, 11, 12)
    tabs = kvgen.batch_tables(3, [r.s for r in reqs], g, g)
    T = [(tab(src, a), tab(dst, b), r.s) for r, (a, b) in zip(reqs, tabs)]
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 80), 1024, cs, None) for t in T]
    ms = run_set(stream, calls, reps=5)
    report(f"TP-8 Qwen2-72B shard (1 KV head, 256-B rows), {len(reqs)} requests (sum s={tot}) c=1024",
           tot * 2 * 80 * g.row_bytes, ms, tot, len(calls))
    calls = [lambda t=t: dk.dyna_kv_migrate_ex(t[0], t[1], (0, t[2]), (0, 80), 1024, cs, OV) for t in T]
    ms = run_set(stream, calls, reps=5)
    report(f"TP-8 Qwen2-72B shard (1 KV head, 256-B rows), {len(reqs)} requests (sum s={tot}) c=1024, OVERLAP_PREV",
           tot * 2 * 80 * g.row_bytes, ms, tot, len(calls), "per-request calls overlapping each other")
    migs = [(t[0], t[1], (0, t[2])) for t in T]
    ms = run_set(stream, [lambda: dk.dyna_kv_migrate_batch(migs, (0, 80), 1024, cs, None)], reps=5)
    report(f"TP-8 Qwen2-72B shard (1 KV head, 256-B rows), {len(reqs)} requests (sum s={tot}) c=1024, batched",
           tot * 2 * 80 * g.row_bytes, ms, tot, 1, "one dyna_kv_migrate_batch launch")
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"device": torch.cuda.get_device_name(0), "hbm_peak_gbs": pk, "results": out},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
