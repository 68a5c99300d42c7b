#!/usr/bin/env python
"""Summarise ncu captures (run on the CPU box) into profiles/.

    python scripts/ncu_summary.py ROUND gpurun_out/prof_e1.ncu-rep [...] [--launches gpurun_out/launches.csv]

Writes profiles/<ROUND>_ncu_summary.md (key counters per captured launch, the
launch list's per-kernel share of device time) and profiles/ncu_traffic.json
(DRAM bytes per launch of the dominant kernel, read by bench.py's roofline).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read BW"),
    ("dram__bytes_write.sum.per_second", "DRAM write BW"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs)"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle / issue"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall drain / issue"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall membar / issue"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (r[i], units[i]) for i, h in enumerate(hdr)} for r in rows[2:]]


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("round")
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--launches")
    ap.add_argument("--dominant", default="k_copy_ring")
    ap.add_argument("--workload", default="c2", help="bench.py workload id the dominant capture belongs to")
    a = ap.parse_args()
    md = [f"# ncu summary — {a.round}", "",
          "Captured with `ncu --set full --clock-control none --import-source on -k regex:k_copy` on one B200",
          "(per-launch, cold-cache, serialised: compare shares and counters, not absolute bench times).", ""]
    traffic = None
    for rep in a.reps:
        md.append(f"## {os.path.basename(rep)}")
        for r in raw_rows(rep):
            name = r.get("Kernel Name", ("?", ""))[0]
            md.append(f"### `{name}`")
            md.append("| counter | value |")
            md.append("|---|---|")
            for k, label in KEYS:
                if k in r:
                    v, u = r[k]
                    md.append(f"| {label} (`{k}`) | {v} {u} |")
            if a.dominant in name and "dram__bytes_read.sum" in r:
                rd = to_bytes(*r["dram__bytes_read.sum"])
                wr = to_bytes(*r["dram__bytes_write.sum"])
                traffic = traffic or {"kernel": name, "bytes_per_launch": rd + wr, "read": rd, "write": wr,
                                      "source": os.path.basename(rep), "round": a.round, "workload": a.workload}
            md.append("")
    if a.launches:
        agg = collections.defaultdict(list)
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        hdr = rows[0]
        iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        for r in rows[1:]:
            v = float(r[ival].replace(",", ""))
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}.get(r[iunit], 1)
            agg[r[iname]].append(v)
        tot = sum(sum(v) for v in agg.values())
        md += ["## Launch list (`--metrics gpu__time_duration.sum`), share of device time", "",
               "| kernel | launches | mean µs | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            md.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / tot:.1f}% |")
        md.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{a.round}_ncu_summary.md"), "w").write("\n".join(md) + "\n")
    if traffic:
        json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
