#!/usr/bin/env python
"""bench.py — KV-migrate throughput of the B200-native chunked KV-cache push.

The step is DynaServe's push of split requests' first-segment KV (§3.1
P:306-308; §4.3): for every request, tokens [0, s) x all layers x K/V
x all KV heads, out of the source instance's paged pool into freshly allocated
blocks of the destination pool.  The workload is BASELINE.json's configuration for
the number of GPUs:

  N = 1   configs[2]: Llama-3-8B (32 L, 8 KV heads, d128, bf16, block 16) pools of 8192
          blocks; the 54 migrating requests of the seeded 64-request skewed batch
          (kvgen.skewed_batch(1, 64), split at s = ceil(phi L)), chunk 256,
          as ONE dyna_kv_migrate_batch per step; destination = a second pool on the same
          B200 (intra-device reblock, HBM roofline).
  N = 2   target 4': each rank pushes one 4096-token Llama-3-8B chunk (512 MiB) into its
          partner's pool (rank r -> r ^ 1, both directions at once) with in-kernel NVLink
          stores (CUDA-IPC mapped pool), NVLink roofline; beside it the NCCL baseline B1
          on identical bytes (dyna_kv_pack -> NCCL send/recv -> dyna_kv_unpack).
  N >= 3  configs[4]: Qwen2-72B-shaped shards (80 L, 8 KV heads, bf16, 6144 blocks); every
          ordered pair of the N ranks migrates 4 skewed requests concurrently (kvgen.
          allpairs_plan), each rank ONE batch into its peers' imported pools; reported
          against the load-aware bound (busiest NVLink port) and with B1 beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dyna|reference]

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (test
infrastructure, oracle/) on a bounded sample of the same workload — the only other
place this file executes oracle/ code besides the cpu_baseline leg.
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
HBM_FALLBACK = 6650.0         # B200_PROFILING.md fallback (GB/s, read+write copy)
NVLINK_MEASURED = 770.0       # B200_PROFILING.md: measured peer copy per direction (GB/s)
NVLINK_NOMINAL = 900.0
C2_SEED, C2_TABLE_SEED, C2_CHUNK = 1, 2, 256
T4_TOKENS, T4_SETS = 4096, 4
C4_REQS, C4_SEED, C4_CHUNK = 4, 1000, 1024

WORKLOADS = {
    "c2": "configs[2]: Llama-3-8B (32L, 8 KV heads, d128, bf16, block 16), the 54 migrating requests of the "
          "seeded 64-request skewed batch (sum s = 57,781 tokens), chunk 256, one dyna_kv_migrate_batch per step, "
          "1-GPU reblock",
    "t4": "target 4': one 4096-token Llama-3-8B chunk (512 MiB) per rank per step into the partner rank's pool "
          "(r -> r^1) over NVLink, fragmented tables",
    "c4": "configs[4]: Qwen2-72B-shaped shards (80L, 8 KV heads, d128, bf16, block 16), all ordered pairs of the "
          "N ranks x 4 skewed requests concurrently, chunk 1024, one dyna_kv_migrate_batch per rank per step",
}


def workload_for(world: int) -> str:
    return "c2" if world == 1 else "t4" if world == 2 else "c4"


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


def ncu_traffic(workload: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            if d.get("workload") == workload:
                return d.get("bytes_per_launch")
        except Exception:
            return None
    return None


class Clocks:
    """nvidia-smi sampler running during warm-up + timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
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


# ---------------------------------------------------------------------------- the JSON line
def make_line(*, world, steps, warmup, workload, payload_per_rank, tokens_per_rank, total_ms, roofline, e2e,
              launches, clocks, config_extra=None, extra=None, impl=None):
    """The contract line (tests/test_bench_cpu.py pins its keys for every N).  value = the
    bytes all ranks moved / the slowest rank's device time; per-GPU work is fixed as N grows
    at N <= 2 (weak); all-pairs work grows with N (reported as weak: every rank's share of
    the step is its own concurrent outgoing batch)."""
    gbps = world * steps * payload_per_rank / (total_ms / 1e3) / 1e9
    cfg = {"workload": WORKLOADS[workload], "workload_id": workload, "kv_dtype": "bf16",
           "payload_bytes_per_step_per_rank": payload_per_rank,
           "l2": "working set >> 126 MB L2 (see workload); no step re-reads a previous step's bytes from L2"}
    cfg.update(config_extra or {})
    line = {
        "metric": METRIC, "value": gbps, "unit": "GB/s", "n_gpus": world, "steps": steps, "warmup": warmup,
        "ms_per_step": total_ms / steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic (seeded kvgen pools and tables; bitwise copy, dtype-agnostic)",
        "config": cfg,
        "tokens_per_s": world * steps * tokens_per_rank / (total_ms / 1e3),
        "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
    }
    if impl:
        line["impl"] = impl
    else:
        line["paper_context"] = PAPER_CONTEXT
    line.update(extra or {})
    return line


# The paper's own numbers on this path (context, not the target: it reports no
# transfer GB/s, latency or tokens/s).
PAPER_CONTEXT = {
    "non_overlapped_transfer_reduction_by_chunking": "94% (PAPER.md §6.6 P:738; 2 servers x 4 A100-80GB, NVLink "
                                                     "600 GB/s bidirectional, Mini-Reasoning, Qwen-2.5; chunk size "
                                                     "not stated)",
    "kv_tokens_transferred_decode_merged_vs_disaggregation": "3x (P:369)",
    "transfer_mechanism": "fully offloaded to NCCL or Mooncake (P:556); no kernel-level figure",
    "this_build_analogue": "profiles/r02_overlap.json: per-chunk pushes cut exposed transfer by 86.8-98.3%, "
                           "per-(chunk, layer) pushes by 98.8-99.8% (configs[3], one B200)",
}


# ---------------------------------------------------------------------------- oracle (CPU) timing
class OracleSample:
    """oracle.migrate (single-threaded plain C, as it stands) on a bounded sample of the
    workload of N: its geometry on 1 layer (of 32 / 80), its requests in order, repeated
    to fill a time budget."""

    def __init__(self, workload: str):
        import kvgen
        import oracle
        self.oracle = oracle
        if workload == "c2":
            g = kvgen.LLAMA3_8B
            reqs = kvgen.migrating(kvgen.skewed_batch(C2_SEED, 64))
            lens = [r.s for r in reqs]
            tabs = kvgen.batch_tables(C2_TABLE_SEED, lens, g, g)
            self.what = "the configs[2] batch (54 requests)"
        elif workload == "t4":
            g = kvgen.LLAMA3_8B.with_(num_blocks=T4_SETS * T4_TOKENS // 16)
            lens = [T4_TOKENS]
            tabs = kvgen.batch_tables(500, lens, g, g)
            self.what = "one 4096-token Llama-3-8B chunk"
        else:
            g = kvgen.QWEN2_72B
            plan = [m for m in kvgen.allpairs_plan(2, g, C4_REQS, C4_SEED) if m.src_rank == 0]
            lens = [m.req.s for m in plan]
            tabs = [(m.src_table, m.dst_table) for m in plan]
            self.what = "rank 0's configs[4] requests"
        self.layers = g.num_layers
        self.row = g.row_bytes
        self.gp = g.with_(num_layers=1)
        self.jobs = list(zip(lens, tabs))
        self.hs = kvgen.fill_bytes(1, self.gp.pool_bytes)
        import numpy as np
        self.hd = np.zeros(self.gp.pool_bytes, np.uint8)
        t = time.perf_counter()
        self._once(self.jobs[:1])
        self.per_tok = (time.perf_counter() - t) / max(1, self.jobs[0][0])

    def _once(self, jobs):
        for n, (ts, td) in jobs:
            self.oracle.migrate(self.hs, self.gp, ts, self.hd, self.gp, td, (0, n), (0, 1))

    def run(self, budget_s: float):
        jobs, tot = [], 0
        while tot * self.per_tok < budget_s or not jobs:      # requests in order, cycled, within the budget
            n, tt = self.jobs[len(jobs) % len(self.jobs)]
            jobs.append((n, tt))
            tot += n
            if len(jobs) > 10 * len(self.jobs):
                break
        t = time.perf_counter()
        self._once(jobs)
        dt = time.perf_counter() - t
        payload = tot * 2 * self.row
        sample = (f"oracle.migrate (plain C, 1 thread) of {self.what} on 1 of {self.layers} layers, "
                  f"{len(jobs)} request migrations = {payload / 2**20:.1f} MiB")
        return payload / dt / 1e9, sample, dt, tot


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    workload = workload_for(world)
    total_budget = float(os.environ.get("DYNA_BENCH_REF_BUDGET_S", 90.0))
    per_step = max(0.02, total_budget / max(1, args.steps + args.warmup))
    o = OracleSample(workload)
    for _ in range(args.warmup):
        o.run(per_step)
    vals, total, sample, toks = [], 0.0, "", 0
    for _ in range(args.steps):
        v, sample, dt, tk = o.run(per_step)
        vals.append(v)
        total += dt
        toks += tk
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOADS[workload], "workload_id": workload, "kv_dtype": "bf16"},
            "tokens_per_s": toks / total / o.layers,
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                             "host_cpus": os.cpu_count(), "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
class Ctx:
    """Per-rank plumbing: device, stream, process group, timing helpers."""

    def __init__(self, rank, world, local_rank):
        import torch
        self.torch = torch
        self.rank, self.world = rank, world
        self.same_device = os.environ.get("DYNA_BENCH_SAME_DEVICE") == "1"
        self.dev = 0 if self.same_device else local_rank
        torch.cuda.set_device(self.dev)
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            backend = os.environ.get("DYNA_BENCH_BACKEND", "nccl")
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device(f"cuda:{self.dev}"))
            else:
                dist.init_process_group(backend)
            self.dist = dist
        self.stream = torch.cuda.Stream()
        self.cs = self.stream.cuda_stream

    @property
    def nccl(self):
        return self.dist is not None and self.dist.get_backend() == "nccl"

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def max(self, x: float) -> float:
        from paper_2504_09285_b200 import dist as dd
        return dd.max_over_ranks(x, device=f"cuda:{self.dev}" if self.nccl else "cpu")

    def sum(self, x: float) -> float:
        if self.dist is None:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=f"cuda:{self.dev}" if self.nccl else "cpu")
        self.dist.all_reduce(t)
        return float(t.item())

    def timed(self, step, steps, warmup):
        """W untimed steps, then exactly K steps back to back between two CUDA events on the
        launch stream (barrier + synchronize on both sides); returns (max-over-ranks ms of the
        region, this rank's ms, library kernel launches in the region)."""
        import paper_2504_09285_b200 as dk
        torch = self.torch
        xs = [step(i) for i in range(warmup)]
        for x in xs:
            _wait_any(x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.barrier()
        n0 = dk.dyna_kv_launch_count()
        e0.record(self.stream)
        xs = [step(i) for i in range(steps)]
        e1.record(self.stream)
        for x in xs:
            _wait_any(x)
        self.barrier()
        launches = dk.dyna_kv_launch_count() - n0
        mine = e0.elapsed_time(e1)
        return self.max(mine), mine, launches


def flag_runs(entries):
    """Contiguous inbox slot runs [(pool_handle, sender, first, n, [(epoch, offset, n)...])] of
    signalled entries, so one copy reads each run back."""
    runs = []
    for pool, sender, first, n, epoch in sorted(entries, key=lambda e: (e[0], e[1], e[2])):
        if n == 0:
            continue
        if runs and runs[-1][0] == pool and runs[-1][1] == sender and runs[-1][2] + runs[-1][3] == first:
            r = runs[-1]
            r[4].append((epoch, r[3], n))
            r[3] += n
        else:
            runs.append([pool, sender, first, n, [(epoch, 0, n)]])
    return runs


class E2E:
    """The end-to-end leg through the public API: host-resident tables in (the library uploads
    them on the stream), per-chunk flags on, the flags of every migration read back into
    pinned host memory and checked against their epochs.  Steps are issued one ahead of the
    wait (the async API as a serving loop uses it)."""

    def __init__(self, ctx, issue):
        self.ctx, self.issue = ctx, issue      # issue(k) -> (xfer, [(pool_handle, sender, first, n, epoch)])
        self.flag_stream = ctx.torch.cuda.Stream()
        self.d2h = 0

    def _start(self, k):
        import paper_2504_09285_b200 as dk
        torch = self.ctx.torch
        x, entries = self.issue(k)
        dk.dyna_kv_stream_wait(x, self.flag_stream.cuda_stream)
        checks = []
        for pool, sender, first, n, parts in flag_runs(entries):
            buf = torch.zeros(n, dtype=torch.int64).pin_memory()
            dk.dyna_kv_copy_flags(pool, sender, first, n, buf.data_ptr(), self.flag_stream.cuda_stream)
            checks.append((buf, parts))
        self.d2h = sum(8 * b.numel() for b, _ in checks)
        ev = torch.cuda.Event()
        ev.record(self.flag_stream)
        return x, checks, ev

    def _finish(self, h):
        import paper_2504_09285_b200 as dk
        x, checks, ev = h
        dk.dyna_kv_wait(x)
        ev.synchronize()
        ok = True
        for buf, parts in checks:
            v = buf.numpy()
            for epoch, off, n in parts:
                ok &= bool((v[off:off + n] == epoch).all())
        return ok

    def run(self, n):
        ok, prev = True, None
        for k in range(n):
            cur = self._start(k)
            if prev is not None:
                ok &= self._finish(prev)
            prev = cur
        return ok & self._finish(prev)

    def timed(self, steps, warmup):
        assert self.run(warmup)
        self.ctx.barrier()
        t = time.perf_counter()
        ok = self.run(steps)
        s = self.ctx.max(time.perf_counter() - t)
        assert ok, "chunk flags did not reach their migrations' epochs"
        self.ctx.barrier()
        return s


def dev_tab(pool, ids, dev):
    import torch
    import paper_2504_09285_b200 as dk
    return dk.table(pool, torch.from_numpy(ids).to(f"cuda:{dev}"), ids)


def run_dyna(args, rank, world, local_rank):
    import numpy as np
    import torch

    import kvgen
    import paper_2504_09285_b200 as dk
    from paper_2504_09285_b200 import dist as dd

    ctx = Ctx(rank, world, local_rank)
    workload = workload_for(world)
    dev, cs = ctx.dev, ctx.cs
    mopts = dk.opts(engine=args.engine, piece_bytes=args.piece, stages=args.stages)
    sig = dk.DYNA_MIGRATE_SIGNAL
    small = os.environ.get("DYNA_BENCH_SMALL") == "1"   # functional runs of N > 1 on one GPU only
    clocks = Clocks(dev)
    extra, cfg_extra = {}, {}

    def fill(p, seed):
        dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, cs)

    if workload == "c2":
        g = kvgen.LLAMA3_8B
        reqs = kvgen.migrating(kvgen.skewed_batch(C2_SEED, 64))
        tabs = kvgen.batch_tables(C2_TABLE_SEED, [r.s for r in reqs], g, g)
        src, dst = dk.Pool(g, dev), dk.Pool(g, dev)
        fill(src, 5)
        fill(dst, 6)
        dtabs = [(dev_tab(src, a, dev), dev_tab(dst, b, dev)) for a, b in tabs]
        migs = [(a, b, (0, r.s)) for r, (a, b) in zip(reqs, dtabs)]
        tokens = sum(r.s for r in reqs)
        payload = tokens * 2 * g.num_layers * g.row_bytes
        lr = (0, g.num_layers)

        def step(i):
            return dk.dyna_kv_migrate_batch(migs, lr, C2_CHUNK, cs, mopts)

        htabs = [(dk.table(src, None, a), dk.table(dst, None, b)) for a, b in tabs]
        hmigs = [(a, b, (0, r.s)) for r, (a, b) in zip(reqs, htabs)]
        sig_opts = dk.opts(engine=args.engine, piece_bytes=args.piece, stages=args.stages, flags=sig)

        def e2e_issue(k):
            x = dk.dyna_kv_migrate_batch(hmigs, lr, C2_CHUNK, cs, sig_opts)
            ents = []
            for i in range(len(hmigs)):
                epoch, first, n, sender = dk.dyna_kv_batch_info(x, i)
                ents.append((dst.handle, sender, first, n, epoch))
            return x, ents

        h2d = sum(2 * 4 * kvgen.blocks_needed(r.s, g.block_size) for r in reqs)
        cfg_extra = {"requests": len(reqs), "sum_s_tokens": tokens, "chunk_tokens": C2_CHUNK,
                     "pools": "two Llama-3-8B pools of 8192 blocks (16 GiB each) on one B200",
                     "tables": "fragmented (kvgen.batch_tables seed 2: blocks drawn from shared free lists)",
                     "l2": f"{payload / 2**30:.2f} GiB read + written per step >> 126 MB L2"}
        kernel_name = "dynakv::k_copy_ring<false, BatchSource> (K4-local fused reblock, decoder-fed TMA ring)"
    elif workload == "t4":
        g = kvgen.LLAMA3_8B.with_(num_blocks=T4_SETS * T4_TOKENS // 16 // (4 if small else 1))
        n_tok = T4_TOKENS // (4 if small else 1)
        peer = rank ^ 1
        src, mine = dk.Pool(g, dev, instance=rank), dk.Pool(g, dev, instance=rank)
        fill(src, 1000 + rank)
        fill(mine, 2000 + rank)
        torch.cuda.synchronize()
        handles = dd.exchange_handles(dk.dyna_kv_pool_export(mine.handle))
        dst = dk.Pool.imported(handles[peer], dev)
        tabs = kvgen.batch_tables(500 + rank, [n_tok] * T4_SETS, g, g)
        dtabs = [(dev_tab(src, a, dev), dev_tab(dst, b, dev)) for a, b in tabs]
        payload = n_tok * 2 * g.num_layers * g.row_bytes
        tokens = n_tok
        lr = (0, g.num_layers)

        def step(i):
            a, b = dtabs[i % T4_SETS]
            return dk.dyna_kv_migrate_ex(a, b, (0, n_tok), lr, n_tok, cs, mopts)

        htabs = [(dk.table(src, None, a), dk.table(dst, None, b)) for a, b in tabs]
        sig_opts = dk.opts(engine=args.engine, piece_bytes=args.piece, stages=args.stages, flags=sig)

        def e2e_issue(k):
            a, b = htabs[k % T4_SETS]
            x = dk.dyna_kv_migrate_ex(a, b, (0, n_tok), lr, n_tok, cs, sig_opts)
            epoch, n, sender, first = dk.dyna_kv_xfer_info(x)
            return x, [(dst.handle, sender, first, n, epoch)]

        h2d = 2 * 4 * kvgen.blocks_needed(n_tok, g.block_size)
        cfg_extra = {"pairs": "rank r -> rank r^1 over CUDA IPC (both directions concurrently)",
                     "chunk_tokens": n_tok, "tables": f"fragmented, {T4_SETS} table sets rotated per step",
                     "l2": f"{T4_SETS} disjoint 512 MiB placements per pool rotated per step (> 126 MB L2)"}
        kernel_name = "dynakv::k_copy_ring<false, SingleSource> (K4 fused, NVLink peer stores)"
    else:
        g = kvgen.QWEN2_72B.with_(num_layers=8, num_blocks=1536) if small else kvgen.QWEN2_72B
        plan = kvgen.allpairs_plan(world, g, C4_REQS, C4_SEED)
        src, mine = dk.Pool(g, dev, instance=rank), dk.Pool(g, dev, instance=rank)
        fill(src, 3000 + rank)
        fill(mine, 4000 + rank)
        torch.cuda.synchronize()
        handles = dd.exchange_handles(dk.dyna_kv_pool_export(mine.handle))
        peers = {j: dk.Pool.imported(handles[j], dev) for j in range(world) if j != rank}
        out_m = [m for m in plan if m.src_rank == rank]
        migs = [(dev_tab(src, m.src_table, dev), dev_tab(peers[m.dst_rank], m.dst_table, dev), (0, m.req.s))
                for m in out_m]
        tok_bytes = 2 * g.num_layers * g.row_bytes
        tokens = sum(m.req.s for m in out_m)
        payload = tokens * tok_bytes
        lr = (0, g.num_layers)

        def step(i):
            return dk.dyna_kv_migrate_batch(migs, lr, C4_CHUNK, cs, mopts)

        hmigs = [(dk.table(src, None, m.src_table), dk.table(peers[m.dst_rank], None, m.dst_table), (0, m.req.s))
                 for m in out_m]
        sig_opts = dk.opts(engine=args.engine, piece_bytes=args.piece, stages=args.stages, flags=sig)

        def e2e_issue(k):
            x = dk.dyna_kv_migrate_batch(hmigs, lr, C4_CHUNK, cs, sig_opts)
            ents = []
            for i, m in enumerate(out_m):
                epoch, first, n, sender = dk.dyna_kv_batch_info(x, i)
                ents.append((peers[m.dst_rank].handle, sender, first, n, epoch))
            return x, ents

        h2d = sum(2 * 4 * kvgen.blocks_needed(m.req.s, g.block_size) for m in out_m)
        pb = {}
        for m in plan:
            pb[(m.src_rank, m.dst_rank)] = pb.get((m.src_rank, m.dst_rank), 0) + m.req.s * tok_bytes
        eg, ing = dd.link_loads(pb)
        cfg_extra = {"migrations": len(plan), "ordered_pairs": world * (world - 1), "chunk_tokens": C4_CHUNK,
                     "total_bytes_per_step": sum(pb.values()),
                     "busiest_egress_bytes": max(eg.values()), "busiest_ingress_bytes": max(ing.values()),
                     "load_aware_bound_ms_900": dd.load_aware_bound_s(pb, NVLINK_NOMINAL * 1e9) * 1e3,
                     "load_aware_bound_ms_770": dd.load_aware_bound_s(pb, NVLINK_MEASURED * 1e9) * 1e3,
                     "l2": "tens of GiB per step (> 126 MB L2)"}
        kernel_name = "dynakv::k_copy_ring<false, BatchSource> (K4 fused, NVLink peer stores)"
    if small:
        cfg_extra["functional_run"] = "DYNA_BENCH_SMALL=1: reduced pools, not a measurement"
    torch.cuda.synchronize()

    # N > 1 with AUTO: the built-in calibration has no NVLink entries (it was measured on one GPU), so
    # before the timed region each rank measures its own peer pair with the library's native
    # calibration (dyna_kv_calibrate: every candidate variant x engine at the workload's chunk size,
    # device-timed) and AUTO then uses the installed choice
    if world > 1 and args.engine == 0:
        if workload == "t4":
            cal_st, cal_dt, cal_c = dtabs[0][0], dtabs[0][1], n_tok
        else:
            big = max(range(len(out_m)), key=lambda k: out_m[k].req.s)
            cal_st, cal_dt, cal_c = migs[big][0], migs[big][1], min(C4_CHUNK, out_m[big].req.s)
        entries, rates = dk.dyna_kv_calibrate(cal_st, cal_dt, [cal_c], reps=4, stream=cs)
        names = ["FUSED VEC 4K U8", "FUSED VEC 8K U4", "FUSED VEC 16K U16", "FUSED BULK ring 32K x4",
                 "STAGED VEC 8K U8", "STAGED BULK 32K x4", "FUSED TILES"]
        extra["calibration"] = {"chunk_tokens": cal_c, "entry": entries[0],
                                "GBps": dict(zip(names, [round(x, 1) for x in rates[0]])),
                                "how": "dyna_kv_calibrate on this rank's peer pair before the timed region "
                                       "(4 device-timed calls per candidate; 0 = not applicable)"}
        ctx.barrier()

    probe = step(0)
    plan_used = dk.dyna_kv_xfer_plan(probe)
    dk.dyna_kv_wait(probe)
    # ~0.5 s of untimed load so the clock sampler sees the part under load, then the contract's warm-up
    t_end = time.perf_counter() + 0.5
    i = 0
    while time.perf_counter() < t_end:
        xs = [step(i + j) for j in range(4)]
        for x in xs:
            dk.dyna_kv_wait(x)
        i += 4
    total_ms, mine_ms, launches = ctx.timed(step, args.steps, args.warmup)
    clk = clocks.stop()
    kern_ms = ctx.max(mine_ms / max(1, launches))        # average launch duration (one launch per step)
    payload_all = ctx.sum(payload)
    tokens_all = ctx.sum(tokens)

    # ---------------- e2e through the public API with host buffers
    e2e = E2E(ctx, e2e_issue)
    e2e_s = e2e.timed(args.steps, args.warmup)
    e2e_line = {"value": payload_all * args.steps / e2e_s / 1e9, "unit": "GB/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": e2e.d2h,
                "how": "host-resident block tables (uploaded by the library on the stream) + per-chunk flags; "
                       "every migration's flags read back to pinned host memory and checked; h2d counts the "
                       "table entries (plus one descriptor record per request for batches)"}

    # ---------------- NCCL baseline B1 (N > 1): identical bytes, pack -> NCCL send/recv -> unpack
    if world > 1:
        extra["nccl_b1"] = run_b1(ctx, workload, g, locals_for_b1(workload, locals()), args) if ctx.nccl else \
            {"unavailable": f"backend {ctx.dist.get_backend()} (functional run): NCCL needs one GPU per rank"}

    # ---------------- N = 1 context: the same requests as per-request calls, and configs[1]
    if world == 1 and not args.quick:
        extra["secondary"] = secondary_n1(ctx, src, dst, dtabs, reqs, g, mopts, args)
    del probe

    if rank == 0:
        if world == 1:
            hbm_peak, hbm_src = load_peaks()
            achieved = 2 * payload / (kern_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                    "frac": achieved / hbm_peak, "frac_of_nominal_8000": achieved / 8000.0,
                    "traffic": ncu_traffic(workload), "peak_source": hbm_src, "kernel": kernel_name,
                    "algorithmic_bytes_per_launch": 2 * payload,
                    "algorithmic_bytes_per_token": 2 * 2 * g.num_layers * g.row_bytes, "kernel_ms": kern_ms,
                    "kernel_ms_source": "timed region / launches (back-to-back, one kernel per step)"}
        else:
            per_dir = payload / (kern_ms / 1e3) / 1e9    # this rank's egress over NVLink per launch / duration
            roof = {"bound": "nvlink", "achieved": per_dir, "peak": NVLINK_MEASURED, "unit": "GB/s",
                    "frac": per_dir / NVLINK_MEASURED, "frac_of_nominal_900": per_dir / NVLINK_NOMINAL,
                    "traffic": None, "kernel": kernel_name,
                    "peak_source": "measured peer copy per direction (B200_PROFILING.md); nominal 900",
                    "algorithmic_bytes_per_launch": payload, "kernel_ms": kern_ms,
                    "note": "ncu is single-GPU only: no DRAM/NVLink counter capture of the multi-rank run"}
            if workload == "c4":
                roof["load_aware_frac_900"] = cfg_extra["load_aware_bound_ms_900"] / (total_ms / args.steps)
                roof["load_aware_frac_770"] = cfg_extra["load_aware_bound_ms_770"] / (total_ms / args.steps)
            if workload == "t4":
                extra["per_pair_GBps"] = payload / (total_ms / args.steps / 1e3) / 1e9
                extra["target_4prime"] = {"per_pair_GBps_needed": 720.0, "chunk_ms_needed": 0.7457,
                                          "chunk_ms": total_ms / args.steps}
        cfg_extra["resolved_plan"] = plan_used
        eng = {dk.DYNA_ENGINE_VEC: "VEC", dk.DYNA_ENGINE_BULK: "BULK", dk.DYNA_ENGINE_BULK_WS: "BULK",
               dk.DYNA_ENGINE_TILES: "TILES"}
        roof["engine"] = eng.get(plan_used["engine"], str(plan_used["engine"]))
        if roof["engine"] == "VEC":
            roof["kernel"] = roof["kernel"].replace("k_copy_ring<false,", "k_copy_lanes<8, false,")
        line = make_line(world=world, steps=args.steps, warmup=args.warmup, workload=workload,
                         payload_per_rank=payload_all / world, tokens_per_rank=tokens_all / world,
                         total_ms=total_ms, roofline=roof, e2e=e2e_line, launches=launches, clocks=clk,
                         config_extra=cfg_extra, extra=extra)
        if world == 1 and not args.no_cpu_baseline:
            v, sample, dt, _ = OracleSample(workload).run(12.0)
            line["cpu_baseline"] = {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": sample,
                                    "seconds": dt, "host_cpus": os.cpu_count(), "cpu_model": cpu_model()}
        print(json.dumps(line), flush=True)
    if ctx.dist is not None:
        ctx.dist.barrier()
        ctx.dist.destroy_process_group()
    return 0


def locals_for_b1(workload, loc):
    """What the NCCL baseline needs from run_dyna's setup."""
    keys = {"t4": ("src", "mine", "tabs", "n_tok", "peer", "dev"),
            "c4": ("src", "mine", "plan", "dev")}[workload]
    return {k: loc[k] for k in keys}


def b1_exchange(plan, rank, tok_bytes):
    """configs[4] B1 exchange of one rank: per peer, the migrations it packs for that peer (in
    plan order) and the ones it unpacks from it (in plan order, i.e. the sender's order), and
    the buffer bytes of each (tests/test_dist_gloo.py checks both sides agree)."""
    out, inn = {}, {}
    for m in plan:
        if m.src_rank == rank:
            out.setdefault(m.dst_rank, []).append(m)
        if m.dst_rank == rank:
            inn.setdefault(m.src_rank, []).append(m)
    return {"out": out, "in": inn,
            "send_bytes": {p: sum(m.req.s for m in v) * tok_bytes for p, v in out.items()},
            "recv_bytes": {p: sum(m.req.s for m in v) * tok_bytes for p, v in inn.items()}}


def run_b1(ctx, workload, g, d, args):
    """SURVEY §2c B1, the paper's "fully offloaded to NCCL" transfer on identical
    bytes: the sender packs its rows with the library's K1 (dyna_kv_pack) into one contiguous
    buffer per peer, NCCL grouped send/recv moves the buffers, the receiver places them with
    the library's K3 (dyna_kv_unpack) through its own tables.  Device-timed per step with CUDA
    events on the launch stream (NCCL ordered on it), max over ranks."""
    import torch
    import kvgen
    import paper_2504_09285_b200 as dk
    dist = ctx.dist
    dev, cs = d["dev"], ctx.cs
    tok_bytes = 2 * g.num_layers * g.row_bytes
    lr = (0, g.num_layers)
    if workload == "t4":
        peer, n = d["peer"], d["n_tok"]
        # the partner's chunk lands in MY pool through the tables the partner drew for it
        peer_tabs = kvgen.batch_tables(500 + peer, [n] * T4_SETS, g, g)
        src_tab = [dev_tab(d["src"], a, dev) for a, _ in d["tabs"]]
        rcv_tab = [dk.table(d["mine"], torch.from_numpy(b).to(f"cuda:{dev}"), b) for _, b in peer_tabs]

        def pieces_out(i):
            return {peer: [(src_tab[i % T4_SETS], (0, n))]}

        def pieces_in(i):
            return {peer: [(rcv_tab[i % T4_SETS], (0, n))]}
    else:
        ex = b1_exchange(d["plan"], ctx.rank, tok_bytes)
        o_t = {p: [(dev_tab(d["src"], m.src_table, dev), (0, m.req.s)) for m in v] for p, v in ex["out"].items()}
        i_t = {p: [(dk.table(d["mine"], torch.from_numpy(m.dst_table).to(f"cuda:{dev}"), m.dst_table), (0, m.req.s))
                   for m in v] for p, v in ex["in"].items()}

        def pieces_out(i):
            return o_t

        def pieces_in(i):
            return i_t
    # one send and one receive buffer per peer, sized for that peer's bytes
    sizes_out = {p: sum((tr[1] - tr[0]) * tok_bytes for _, tr in v) for p, v in pieces_out(0).items()}
    sizes_in = {p: sum((tr[1] - tr[0]) * tok_bytes for _, tr in v) for p, v in pieces_in(0).items()}
    sbuf = {p: torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}") for p, n in sizes_out.items()}
    rbuf = {p: torch.empty(n, dtype=torch.uint8, device=f"cuda:{dev}") for p, n in sizes_in.items()}
    opts = dk.opts(engine=args.engine, piece_bytes=args.piece, stages=args.stages)

    def b1_step(i):
        xs = []
        for p, lst in pieces_out(i).items():
            off = 0
            for tab, tr in lst:
                nb = (tr[1] - tr[0]) * tok_bytes
                xs.append(dk.dyna_kv_pack(tab, tr, lr, sbuf[p].data_ptr() + off, nb, cs, opts))
                off += nb
        with torch.cuda.stream(ctx.stream):
            ops = [dist.P2POp(dist.isend, sbuf[p], p) for p in sorted(sbuf)] + \
                  [dist.P2POp(dist.irecv, rbuf[p], p) for p in sorted(rbuf)]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for p, lst in pieces_in(i).items():
            off = 0
            for tab, tr in lst:
                nb = (tr[1] - tr[0]) * tok_bytes
                xs.append(dk.dyna_kv_unpack(rbuf[p].data_ptr() + off, nb, tab, tr, lr, cs, opts))
                off += nb
        return xs

    def wait_all(xss):
        for xs in xss:
            for x in xs:
                dk.dyna_kv_wait(x)

    wait_all([b1_step(i) for i in range(args.warmup)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    e0.record(ctx.stream)
    xss = [b1_step(i) for i in range(args.steps)]
    e1.record(ctx.stream)
    wait_all(xss)
    ctx.barrier()
    ms = ctx.max(e0.elapsed_time(e1)) / args.steps
    moved = ctx.sum(sum(sizes_out.values()))
    return {"value": moved / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
            "how": "dyna_kv_pack (K1) -> torch.distributed NCCL batch_isend_irecv -> dyna_kv_unpack (K3), "
                   "same bytes and tables as the fused push, device-timed, max over ranks"}


def secondary_n1(ctx, src, dst, dtabs, reqs, g, mopts, args):
    """Context for N = 1 (not the headline): the configs[2] requests as one dyna_kv_migrate
    per request, configs[1] (one Llama-2-7B request, s = 1024, chunk 256), and the 4' shape
    in its 1-GPU form — each device-timed the same way, fewer steps."""
    import kvgen
    import paper_2504_09285_b200 as dk
    cs = ctx.cs
    out = {}
    k = max(3, min(args.steps, 10))
    tokens = sum(r.s for r in reqs)
    payload = tokens * 2 * g.num_layers * g.row_bytes

    def per_req(i):
        return [dk.dyna_kv_migrate_ex(a, b, (0, r.s), (0, 32), C2_CHUNK, cs, mopts) for r, (a, b) in zip(reqs, dtabs)]

    ms, _, n = ctx.timed(lambda i: _Multi(per_req(i)), k, 2)
    out["configs2_per_request_calls"] = {"GBps": payload / (ms / k / 1e3) / 1e9, "ms_per_step": ms / k,
                                         "launches_per_step": n // k}
    # the same calls with DYNA_MIGRATE_OVERLAP_PREV: the requests' rows are disjoint, so each call may
    # start while the previous one drains
    ov = dk.opts(engine=args.engine, piece_bytes=args.piece, stages=args.stages, flags=dk.DYNA_MIGRATE_OVERLAP_PREV)

    def per_req_ov(i):
        return [dk.dyna_kv_migrate_ex(a, b, (0, r.s), (0, 32), C2_CHUNK, cs, ov) for r, (a, b) in zip(reqs, dtabs)]

    ms, _, n = ctx.timed(lambda i: _Multi(per_req_ov(i)), k, 2)
    out["configs2_per_request_calls_overlap_prev"] = {"GBps": payload / (ms / k / 1e3) / 1e9, "ms_per_step": ms / k,
                                                      "launches_per_step": n // k}
    # 4' shape, 1-GPU form: 4096-token chunks of the same pools (8 disjoint placements)
    ts, td = kvgen.table_pair(3, 8 * 4096, g.with_(num_blocks=4096), g.with_(num_blocks=4096))
    st, dt = dev_tab(src, ts, ctx.dev), dev_tab(dst, td, ctx.dev)

    def t4(i):
        j = i % 8
        return dk.dyna_kv_migrate_ex(st, dt, (j * 4096, (j + 1) * 4096), (0, 32), 4096, cs, mopts)

    ms, _, _ = ctx.timed(t4, 4 * k, 3)
    out["t4prime_1gpu_form"] = {"GBps": 4096 * 2 * 32 * g.row_bytes / (ms / (4 * k) / 1e3) / 1e9,
                                "ms_per_chunk": ms / (4 * k)}

    def t4_ov(i):
        j = i % 8
        return dk.dyna_kv_migrate_ex(st, dt, (j * 4096, (j + 1) * 4096), (0, 32), 4096, cs, ov)

    ms, _, _ = ctx.timed(t4_ov, 4 * k, 3)
    out["t4prime_1gpu_form_overlap_prev"] = {"GBps": 4096 * 2 * 32 * g.row_bytes / (ms / (4 * k) / 1e3) / 1e9,
                                             "ms_per_chunk": ms / (4 * k)}
    # configs[1]: Llama-2-7B rows, s = 1024 of 2048, chunk 256 (round 1's bench step)
    g2 = kvgen.LLAMA2_7B
    s2, d2 = dk.Pool(g2, ctx.dev), dk.Pool(g2, ctx.dev)
    tabs2 = kvgen.batch_tables(500, [2048] * 4, g2, g2)
    T2 = [(dev_tab(s2, a, ctx.dev), dev_tab(d2, b, ctx.dev)) for a, b in tabs2]

    def c1(i):
        a, b = T2[i % 4]
        return dk.dyna_kv_migrate_ex(a, b, (0, 1024), (0, 32), 256, cs, mopts)

    ms, _, _ = ctx.timed(c1, 4 * k, 3)
    out["configs1_llama2_request"] = {"GBps": 1024 * 2 * 32 * g2.row_bytes / (ms / (4 * k) / 1e3) / 1e9,
                                      "ms_per_step": ms / (4 * k)}
    del s2, d2, T2
    return out


class _Multi:
    """Several handles as one step (per-request calls)."""

    def __init__(self, xs):
        self.xs = xs


def _wait_any(x):
    import paper_2504_09285_b200 as dk
    if isinstance(x, _Multi):
        for y in x.xs:
            dk.dyna_kv_wait(y)
    else:
        dk.dyna_kv_wait(x)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dyna", choices=["dyna", "reference"])
    ap.add_argument("--engine", type=int, default=0, help="0 auto, 1 VEC, 2 BULK")
    ap.add_argument("--piece", type=int, default=0, help="bytes per work item (0 = calibrated)")
    ap.add_argument("--stages", type=int, default=0, help="BULK ring depth (0 = calibrated)")
    ap.add_argument("--quick", action="store_true", help="skip the N = 1 secondary measurements")
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
