"""configs[4] all-pairs plan (input generation for the 8-GPU run) — CPU only."""
import numpy as np

import kvgen
from paper_2504_09285_b200 import dist as dd


def test_plan_is_deterministic_injective_and_balanced_enough():
    g = kvgen.QWEN2_72B
    a = kvgen.allpairs_plan(8, g)
    b = kvgen.allpairs_plan(8, g)
    assert [(m.src_rank, m.dst_rank, m.req) for m in a] == [(m.src_rank, m.dst_rank, m.req) for m in b]
    assert all(np.array_equal(x.src_table, y.src_table) and np.array_equal(x.dst_table, y.dst_table)
               for x, y in zip(a, b))
    pairs = {(m.src_rank, m.dst_rank) for m in a}
    assert len(pairs) <= 56 and all(i != j for i, j in pairs)
    for r in range(8):   # blocks are never shared within one pool, on either side
        s = np.concatenate([m.src_table for m in a if m.src_rank == r])
        d = np.concatenate([m.dst_table for m in a if m.dst_rank == r])
        assert len(np.unique(s)) == len(s) and len(np.unique(d)) == len(d)
        assert s.max() < g.num_blocks and d.max() < g.num_blocks
    for m in a:
        assert len(m.src_table) * g.block_size >= m.req.s and len(m.dst_table) * g.block_size >= m.req.s
    tok_bytes = 2 * g.num_layers * g.row_bytes
    pb = {}
    for m in a:
        pb[(m.src_rank, m.dst_rank)] = pb.get((m.src_rank, m.dst_rank), 0) + m.req.s * tok_bytes
    bound = dd.load_aware_bound_s(pb, 900e9)
    assert bound >= dd.aggregate_bound_s(pb, 8, 900e9) > 0


def test_compact_plan_relabels_order_preserving_and_injective():
    """The one-GPU emulation's relabelling keeps every table's block order, never merges two blocks
    of a pool, and sizes each pool to its used blocks plus the spare ones."""
    g = kvgen.QWEN2_72B
    plan = kvgen.allpairs_plan(4, g)
    cp, ns, nd = kvgen.compact_plan(plan, spare=3)
    assert [(m.src_rank, m.dst_rank, m.req) for m in cp] == [(m.src_rank, m.dst_rank, m.req) for m in plan]
    for r in range(4):
        for side, n in (("src", ns), ("dst", nd)):
            orig = np.concatenate([getattr(m, side + "_table") for m in plan if getattr(m, side + "_rank") == r])
            new = np.concatenate([getattr(m, side + "_table") for m in cp if getattr(m, side + "_rank") == r])
            assert len(np.unique(new)) == len(new) == len(orig)         # injective
            assert sorted(new.tolist()) == list(range(n[r] - 3))        # dense onto [0, used)
            o = np.argsort(orig)
            assert np.all(np.diff(new[o]) > 0)                          # monotone in the old ids
