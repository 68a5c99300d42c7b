"""Host-side multi-GPU plumbing for concurrent instance-pair migrations.

One process per GPU (torchrun).  The data path has no collective: a source
rank's kernel stores straight into the destination rank's pool over NVLink
(§3.1 P:352 "the instances exchange the required KV cache blocks";
§4.3).  torch.distributed is used only to exchange CUDA-IPC pool
handles at setup and to take the max over ranks of measured times.

Pure functions here (schedules, the load-aware bound) are covered by CPU
tests; the collectives run under gloo in tests/test_dist_gloo.py.
"""
from __future__ import annotations

from collections import defaultdict


def ring_pairs(world: int) -> list[tuple[int, int]]:
    """bench.py's weak-scaling pattern: rank r pushes to rank (r+1) % world.
    world == 1 degenerates to (0, 0), the intra-device reblock."""
    return [(r, (r + 1) % world) for r in range(world)]


def all_pairs(world: int) -> list[tuple[int, int]]:
    """Every ordered pair i != j (configs[4]: 56 pairs at 8 GPUs)."""
    return [(i, j) for i in range(world) for j in range(world) if i != j]


def link_loads(pair_bytes: dict[tuple[int, int], int]) -> tuple[dict[int, int], dict[int, int]]:
    """Per-GPU egress and ingress bytes of a set of concurrent migrations."""
    eg, ing = defaultdict(int), defaultdict(int)
    for (i, j), b in pair_bytes.items():
        if i == j:
            continue
        eg[i] += b
        ing[j] += b
    return dict(eg), dict(ing)


def load_aware_bound_s(pair_bytes: dict[tuple[int, int], int], link_bytes_per_s: float) -> float:
    """Lower bound on the completion time of concurrent migrations through a
    non-blocking switch where every GPU has `link_bytes_per_s` per direction
    (NVSwitch: uniform): the busiest egress or ingress port."""
    eg, ing = link_loads(pair_bytes)
    busiest = max(list(eg.values()) + list(ing.values()) + [0])
    return busiest / link_bytes_per_s


def aggregate_bound_s(pair_bytes: dict[tuple[int, int], int], world: int, link_bytes_per_s: float) -> float:
    """Bound ignoring skew: total bytes over the aggregate egress of all GPUs."""
    total = sum(b for (i, j), b in pair_bytes.items() if i != j)
    return total / (world * link_bytes_per_s)


def tp_heads(num_heads: int, tp: int, rank: int) -> tuple[int, int]:
    """KV heads a rank of a TP-`tp` instance holds: the contiguous partition
    [rank*H/tp, (rank+1)*H/tp) (tp must divide H; §5 P:595-596 runs
    r^alpha and r^beta as TP groups)."""
    if tp <= 0 or num_heads % tp:
        raise ValueError(f"TP degree {tp} must divide the {num_heads} KV heads")
    return rank * num_heads // tp, (rank + 1) * num_heads // tp


def tp_reshard_plan(num_heads: int, tp_src: int, tp_dst: int) -> list[tuple[int, int, tuple[int, int], int]]:
    """Head resharding between a TP-tp_src sender and a TP-tp_dst receiver
    (SURVEY §8f NEXT-3): one entry (src_rank, dst_rank, src_heads, dst_head_begin)
    per rank pair whose head sets overlap, in the local head numbering of each
    rank's pool — the arguments of dyna_kv_migrate_heads.  Equal degrees give
    the rank-i -> rank-i pairs with whole rows."""
    out = []
    for a in range(tp_src):
        sa, sb = tp_heads(num_heads, tp_src, a)
        for b in range(tp_dst):
            da, db = tp_heads(num_heads, tp_dst, b)
            lo, hi = max(sa, da), min(sb, db)
            if lo < hi:
                out.append((a, b, (lo - sa, hi - sa), lo - da))
    return out


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All-gather every rank's exported pool handle (dyna_kv_pool_export bytes)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return out


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Max of a scalar over ranks (timings are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
