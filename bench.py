#!/usr/bin/env python
"""bench.py — KV-migrate throughput of the B200-native chunked KV-cache push.

One "step" = one dyna_kv_migrate of one split request's first-segment KV
(§3.1, §4.3) on BASELINE.json configs[1]: Llama-2-7B
shape (32 layers, 32 KV heads, d128, fp16, block 16), a 2048-token prompt
split mid-prefill at s = 1024, chunk 256.  At N = 1 the destination pool is a
second pool on the same B200 (intra-device reblocking, HBM roofline); at N > 1
each rank r pushes into rank (r+1) % N's pool, mapped over CUDA IPC, with
in-kernel NVLink stores (NVLink roofline).  Per-GPU work is fixed: weak
scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dyna|reference]

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (the
test-infrastructure program in oracle/) on a bounded sample of the same
workload — the only other place this file runs oracle/ code besides the
cpu_baseline leg.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV-migrate GB/s & tokens/s per pair and aggregate at 1/2/4/8 B200; % of roofline"
WORKLOAD = "configs[1]: Llama-2-7B shape (32L, 32 KV heads, d128, fp16, block 16), 2048-token prompt split at s=1024, chunk 256"
N_TOKENS, S_SPLIT, CHUNK, N_SETS = 2048, 1024, 256, 4
HBM_FALLBACK = 6650.0         # B200_PROFILING.md fallback (GB/s, read+write copy)
NVLINK_MEASURED = 770.0       # B200_PROFILING.md measured peer copy per direction (GB/s)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, read+write copy)"
    return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p)).get("bytes_per_launch")
        except Exception:
            return None
    return None


class Clocks:
    """nvidia-smi sampler running during warm-up + timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.split(", ") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------------------- oracle (CPU) timing
class OracleSample:
    """oracle.migrate (single-threaded plain C, as it stands) on a bounded sample of the
    workload: the configs[1] request shape (Llama-2-7B rows, s = 1024) on 1 of its 32 layers.
    Pools are generated once; each run() repeats the migration to fill a time budget."""

    def __init__(self):
        import kvgen
        import oracle
        self.oracle = oracle
        g = kvgen.LLAMA2_7B
        self.row = g.row_bytes
        self.gp = g.with_(num_layers=1, num_blocks=N_TOKENS // g.block_size)
        self.ts, self.td = kvgen.table_pair(7, N_TOKENS, self.gp, self.gp)
        self.hs, self.hd = kvgen.fill_bytes(1, self.gp.pool_bytes), kvgen.fill_bytes(2, self.gp.pool_bytes)
        t = time.perf_counter()
        self._once(S_SPLIT)
        self.per_rep = time.perf_counter() - t

    def _once(self, ntok):
        self.oracle.migrate(self.hs, self.gp, self.ts, self.hd, self.gp, self.td, (0, ntok), (0, 1))

    def run(self, budget_s: float):
        reps = max(1, int(budget_s / self.per_rep))
        ntok = S_SPLIT if budget_s >= self.per_rep else max(16, int(S_SPLIT * budget_s / self.per_rep))
        t = time.perf_counter()
        for _ in range(reps):
            self._once(ntok)
        dt = time.perf_counter() - t
        payload = reps * ntok * 2 * self.row
        sample = (f"oracle.migrate (plain C, 1 thread) of the configs[1] request (Llama-2-7B rows, "
                  f"tokens [0,{ntok}) of s=1024) on 1 of 32 layers, x{reps} = {payload / 2**20:.1f} MiB")
        return payload / dt / 1e9, sample, dt


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    total_budget = float(os.environ.get("DYNA_BENCH_REF_BUDGET_S", 90.0))  # seconds of oracle work in all
    per_step_budget = max(0.02, total_budget / max(1, args.steps + args.warmup))
    o = OracleSample()
    for _ in range(args.warmup):
        o.run(per_step_budget)
    vals, total, sample = [], 0.0, ""
    for _ in range(args.steps):
        v, sample, dt = o.run(per_step_budget)
        vals.append(v)
        total += dt
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "kv_dtype": "fp16"},
            "tokens_per_s": v * 1e9 / (2 * 32 * o.row),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "host_cpus": os.cpu_count(), "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
def run_dyna(args, rank, world, local_rank):
    import numpy as np
    import torch

    import kvgen
    import paper_2504_09285_b200 as dk
    from paper_2504_09285_b200 import dist as dd

    # DYNA_BENCH_SAME_DEVICE=1 + DYNA_BENCH_BACKEND=gloo: every rank on cuda:0 (functional
    # check of the N > 1 path — IPC pools, pairing, timing — on a one-GPU box; not a measurement)
    dev = 0 if os.environ.get("DYNA_BENCH_SAME_DEVICE") == "1" else local_rank
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("DYNA_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)

    g = kvgen.LLAMA2_7B
    payload = S_SPLIT * 2 * g.num_layers * g.row_bytes  # bytes per step (one request's [0, s) KV)
    stream = torch.cuda.Stream()
    cs = stream.cuda_stream

    src = dk.Pool(g, dev, instance=rank)
    dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 1000 + rank, 0, cs)
    if world == 1:
        dst = dk.Pool(g, dev, instance=rank)
        dk.dyna_kv_debug_fill(dst.tensor.data_ptr(), dst.tensor.numel(), 2000, 0, cs)
        peer = None
    else:
        mine = dk.Pool(g, dev, instance=rank)
        dk.dyna_kv_debug_fill(mine.tensor.data_ptr(), mine.tensor.numel(), 2000 + rank, 0, cs)
        torch.cuda.synchronize()
        handles = dd.exchange_handles(dk.dyna_kv_pool_export(mine.handle))
        peer = dd.ring_pairs(world)[rank][1]
        dst = dk.Pool.imported(handles[peer], dev)
    # N_SETS disjoint request placements per pool, rotated every step: each step
    # reads 512 MiB and writes 512 MiB that the previous steps did not touch (> 126 MB L2).
    tabs = kvgen.batch_tables(500 + rank, [N_TOKENS] * N_SETS, g, g)
    dts = [(torch.from_numpy(ts).to(f"cuda:{dev}"), torch.from_numpy(td).to(f"cuda:{dev}")) for ts, td in tabs]
    tables = [(dk.table(src, a, ts), dk.table(dst, b, td)) for (a, b), (ts, td) in zip(dts, tabs)]
    mopts = dk.opts(variant=args.variant, engine=args.engine, piece_bytes=args.piece, unroll=args.unroll)
    torch.cuda.synchronize()

    def step(i, o=mopts):
        st, dt_ = tables[i % N_SETS]
        return dk.dyna_kv_migrate_ex(st, dt_, (0, S_SPLIT), (0, g.num_layers), CHUNK, cs, o)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        on_cpu = dist is not None and dist.get_backend() == "gloo"
        return dd.max_over_ranks(x, device="cpu" if on_cpu else f"cuda:{dev}")

    probe = step(0)
    plan = dk.dyna_kv_xfer_plan(probe)
    dk.dyna_kv_wait(probe)
    clocks = Clocks(dev)
    # warm-up (untimed), then ~0.5 s of untimed load so the clock samples see the part under load
    xs = [step(i) for i in range(args.warmup)]
    for x in xs:
        dk.dyna_kv_wait(x)
    t_end = time.perf_counter() + 0.5
    i = 0
    while time.perf_counter() < t_end:
        xs = [step(i + j) for j in range(50)]
        for x in xs:
            dk.dyna_kv_wait(x)
        i += 50

    # ---------------- timed region: exactly K steps, device-timed with CUDA events on the launch stream.
    # The steps run back to back (one migration kernel each, nothing between them, so
    # programmatic dependent launch can overlap one launch's drain with the next one's start);
    # a kernel's average launch duration is then the region's time / the launches in it.
    # (DYNA_BENCH_STEP_EVENTS=1 brackets every step with its own events instead — those event
    # records sit between the kernels and cost the overlap.)
    step_events = os.environ.get("DYNA_BENCH_STEP_EVENTS") == "1"
    ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps if step_events else 0)]
    ev_b = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps if step_events else 0)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    n_launch0 = dk.dyna_kv_launch_count()
    t0.record(stream)
    xs = []
    for k in range(args.steps):
        if step_events:
            ev_a[k].record(stream)
        xs.append(step(k))
        if step_events:
            ev_b[k].record(stream)
    t1.record(stream)
    for x in xs:
        dk.dyna_kv_wait(x)
    barrier()
    launches = dk.dyna_kv_launch_count() - n_launch0
    clk = clocks.stop()
    total_ms = max_over_ranks(t0.elapsed_time(t1))
    if step_events:
        kern_ms = statistics.fmean(a.elapsed_time(b) for a, b in zip(ev_a, ev_b))
    else:
        kern_ms = t0.elapsed_time(t1) / max(launches, 1)
    kern_ms = max_over_ranks(kern_ms)

    # ---------------- e2e through the public API with host buffers: every step passes the
    # request's two block tables as HOST arrays (the library copies the entries it needs to
    # the device on the stream), migrates with per-chunk flags, and reads the chunk flags
    # back into pinned host memory; completion is taken from dyna_kv_wait.  Steps are
    # issued one ahead of the wait (the async API as a serving loop uses it), so host work
    # for step k+1 overlaps the device work of step k.
    nchunks = -(-S_SPLIT // CHUNK)
    e2e_tables = [(dk.table(src, None, ts), dk.table(dst, None, td)) for ts, td in tabs]
    flags_host = [torch.zeros(nchunks, dtype=torch.int64).pin_memory() for _ in range(N_SETS)]
    sig_opts = dk.opts(variant=args.variant, engine=args.engine, flags=dk.DYNA_MIGRATE_SIGNAL,
                       piece_bytes=args.piece, unroll=args.unroll)
    sender = rank
    flag_pool = dst.handle
    blocks = -(-S_SPLIT // g.block_size)
    h2d = 2 * blocks * 4            # the table entries [0, s) reaches, both tables
    d2h = nchunks * 8

    flag_stream = torch.cuda.Stream()       # the read-back runs beside the next step's migration

    def e2e_issue(k):
        i = k % N_SETS
        st, dt_ = e2e_tables[i]
        x = dk.dyna_kv_migrate_ex(st, dt_, (0, S_SPLIT), (0, g.num_layers), CHUNK, cs, sig_opts)
        epoch, _, _, first = dk.dyna_kv_xfer_info(x)
        dk.dyna_kv_stream_wait(x, flag_stream.cuda_stream)
        dk.dyna_kv_copy_flags(flag_pool, sender, first, nchunks, flags_host[i].data_ptr(), flag_stream.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(flag_stream)
        return x, epoch, ev, i

    def e2e_finish(h):
        x, epoch, ev, i = h
        dk.dyna_kv_wait(x)
        ev.synchronize()
        return int(flags_host[i].min()) == epoch

    def e2e_run(n):
        ok, prev = True, None
        for k in range(n):
            cur = e2e_issue(k)
            if prev is not None:
                ok &= e2e_finish(prev)
            prev = cur
        return ok & e2e_finish(prev)

    e2e_run(args.warmup)
    barrier()
    t = time.perf_counter()
    flags_ok = e2e_run(args.steps)
    e2e_s = max_over_ranks(time.perf_counter() - t)
    assert flags_ok, "chunk flags did not reach the migration's epoch"
    barrier()

    # context for the roofline: torch's own copy_ of a contiguous buffer of the same payload size
    a = torch.empty(payload, dtype=torch.uint8, device=f"cuda:{dev}")
    b = torch.empty_like(a)
    a.fill_(1)
    ref_ms = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        e1.synchronize()
        ref_ms.append(e0.elapsed_time(e1))
    same_size_copy = 2 * payload / (statistics.median(ref_ms[5:]) / 1e3) / 1e9
    del a, b

    if rank == 0:
        hbm_peak, hbm_src = load_peaks()
        gbps = world * args.steps * payload / (total_ms / 1e3) / 1e9
        if world == 1:
            achieved = 2 * payload / (kern_ms / 1e3) / 1e9  # HBM read + write bytes per launch / duration
            roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                    "frac_of_nominal_8000": achieved / 8000.0,
                    "traffic": ncu_traffic(), "peak_source": hbm_src,
                    "kernel": ("dynakv::k_copy_bulk" if plan["engine"] == dk.DYNA_ENGINE_BULK
                               else "dynakv::k_copy_vec") + " (K4-local fused reblock)",
                    "algorithmic_bytes_per_launch": 2 * payload, "kernel_ms": kern_ms,
                    "kernel_ms_source": "per-step CUDA events" if step_events else
                                        "timed region / launches (back-to-back, one kernel per step)",
                    "same_size_torch_copy_gbs": same_size_copy}
        else:
            achieved = payload / (kern_ms / 1e3) / 1e9      # bytes crossing NVLink per launch / duration
            roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_MEASURED, "unit": "GB/s",
                    "frac": achieved / NVLINK_MEASURED, "traffic": None,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md); nominal 900",
                    "algorithmic_bytes_per_launch": payload, "kernel_ms": kern_ms}
        line = {
            "metric": METRIC, "value": gbps, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "kv_dtype": "fp16", "payload_bytes_per_step": payload,
                       "pairs": "rank r -> rank (r+1) % N over CUDA IPC" if world > 1 else "intra-device reblock",
                       "variant": args.variant, "engine": args.engine, "resolved_plan": plan,
                       "l2": f"{N_SETS} disjoint block-table sets rotated per step; 1 GiB of HBM traffic per step > 126 MB L2"},
            "tokens_per_s": world * args.steps * S_SPLIT / (total_ms / 1e3),
            "roofline": roof,
            "e2e": {"value": world * args.steps * payload / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu_baseline:
            v, sample, dt = OracleSample().run(12.0)
            line["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                                    "seconds": dt, "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="dyna", choices=["dyna", "reference"])
    ap.add_argument("--engine", type=int, default=0, help="0 auto, 1 VEC, 2 BULK")
    ap.add_argument("--variant", type=int, default=0, help="0 auto, 1 FUSED, 2 STAGED")
    ap.add_argument("--piece", type=int, default=0, help="bytes per work item (0 = calibrated)")
    ap.add_argument("--unroll", type=int, default=0, help="VEC loads in flight per lane (0 = calibrated)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, world, local_rank = env_rank()
    if world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_dyna(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
