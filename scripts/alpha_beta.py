#!/usr/bin/env python
"""Fit SPEC's transfer-time model to the measured chunk sweep.

    python scripts/alpha_beta.py profiles/r01_calibration.json [--out profiles/r01_alpha_beta.json]

For every row size, take the AUTO choice at each chunk size (one c-token chunk
per call) and fit ms_per_call = alpha + bytes_per_call / beta.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_09285_b200.model import fit_alpha_beta  # noqa: E402

LAYERS = {8192: 32, 2048: 32, 256: 80}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("calibration")
    ap.add_argument("--out")
    a = ap.parse_args()
    d = json.load(open(a.calibration))
    meas = {(m["row_bytes"], m["chunk"], m["variant"], m["engine"], m["piece"], m["stages"], m["unroll"]): m
            for m in d["measurements"]}
    out = []
    for row in sorted({c["row_bytes"] for c in d["chosen"]}, reverse=True):
        xs, ys = [], []
        for c in d["chosen"]:
            if c["row_bytes"] != row:
                continue
            m = meas[(row, c["chunk"]) + tuple(c["choice"])]
            xs.append(c["chunk"] * 2 * LAYERS[row] * row)
            ys.append(m["ms_per_call"])
        alpha, beta = fit_alpha_beta(xs, ys)
        r = {"row_bytes": row, "alpha_us": alpha * 1e3, "beta_GBps": beta * 1e3 / 1e9,
             "points": [{"bytes": x, "ms": y} for x, y in zip(xs, ys)]}
        out.append(r)
        print(f"row {row}: latency intercept {alpha * 1e3:.2f} us, bandwidth slope {beta * 1e3 / 1e9:.0f} GB/s")
    if a.out:
        json.dump({"model": "ms = alpha + bytes/beta (SPEC.md S:104)", "source": os.path.basename(a.calibration),
                   "fits": out}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
