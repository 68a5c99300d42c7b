"""Latency-bandwidth (alpha-beta) model of one chunk push — host-side analysis,
not part of the copy path.

SPEC.md's transfer cost (citing PAPER.md §4.3 P:556 "immediately
DMA-pushed"):  transfer_time(tokens) = 0 if tokens == 0, else
link_latency + tokens * kv_bytes_per_token / link_bw.
We fit (link_latency, link_bw) to measured per-call times of the chunk sweep
(scripts/calibrate.py, scripts/configs_sweep.py) — a consistency check on the
measurements, not a parity target.
"""
from __future__ import annotations


def transfer_time_ms(tokens: int, kv_bytes_per_token: float, link_bw_bytes_per_ms: float,
                     link_latency_ms: float) -> float:
    if tokens == 0:
        return 0.0
    return link_latency_ms + tokens * kv_bytes_per_token / link_bw_bytes_per_ms


def fit_alpha_beta(bytes_per_call: list[float], ms_per_call: list[float]) -> tuple[float, float]:
    """Least-squares fit of ms = alpha + bytes / beta.  Returns (alpha_ms, beta_bytes_per_ms)."""
    n = len(bytes_per_call)
    if n < 2:
        raise ValueError("need at least two points")
    mx = sum(bytes_per_call) / n
    my = sum(ms_per_call) / n
    sxx = sum((x - mx) ** 2 for x in bytes_per_call)
    sxy = sum((x - mx) * (y - my) for x, y in zip(bytes_per_call, ms_per_call))
    slope = sxy / sxx
    return my - slope * mx, 1.0 / slope
