"""Multi-process host logic of the N > 1 path on CPU (gloo, world size 2):
handle exchange, max-over-ranks timing, pair schedules and the load-aware
bound of concurrent migrations."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2504_09285_b200 import dist as dd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fake_handle = bytes([rank]) * 168          # sizeof(dyna_kv_ipc_handle)
        got = dd.exchange_handles(fake_handle)
        peer = dd.ring_pairs(world)[rank][1]
        t = dd.max_over_ranks(1.5 + rank)
        q.put((rank, [g[0] for g in got], len(got[peer]), t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_handle_exchange_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, firsts, peer_len, t in res:
        assert firsts == [0, 1]          # every rank sees every handle, in rank order
        assert peer_len == 168
        assert t == 2.5                  # max over ranks


def test_pair_schedules():
    assert dd.ring_pairs(1) == [(0, 0)]
    assert dd.ring_pairs(4) == [(0, 1), (1, 2), (2, 3), (3, 0)]
    ap = dd.all_pairs(8)
    assert len(ap) == 56 and len(set(ap)) == 56 and all(i != j for i, j in ap)


def test_load_aware_bound_brute_force():
    # brute force: simulate fluid sharing on a switch with per-port capacity 1 byte/s;
    # completion time >= busiest port, and equals it for a single sender/receiver pair.
    pb = {(0, 1): 100, (0, 2): 50, (2, 1): 70, (3, 1): 10}
    eg, ing = dd.link_loads(pb)
    assert eg == {0: 150, 2: 70, 3: 10} and ing == {1: 180, 2: 50}
    assert dd.load_aware_bound_s(pb, 1.0) == 180
    assert dd.aggregate_bound_s(pb, 4, 1.0) == 230 / 4
    assert dd.load_aware_bound_s({(0, 1): 64}, 2.0) == 32
    assert dd.load_aware_bound_s({(0, 0): 64}, 2.0) == 0      # local reblock uses no link
    for n in (2, 4, 8):
        pb = {p: 1 for p in dd.all_pairs(n)}
        assert dd.load_aware_bound_s(pb, 1.0) == n - 1 == dd.aggregate_bound_s(pb, n, 1.0)


@pytest.mark.parametrize("world", [3, 4, 8])
def test_b1_exchange_plan_matches_between_ranks(world):
    """bench.py's NCCL baseline (B1) for configs[4]: what rank i packs for rank j, in order, is
    exactly what rank j unpacks from rank i, and the buffers are sized for those bytes."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import kvgen
    g = kvgen.QWEN2_72B
    plan = kvgen.allpairs_plan(world, g, bench.C4_REQS, bench.C4_SEED)
    tok = 2 * g.num_layers * g.row_bytes
    ex = [bench.b1_exchange(plan, r, tok) for r in range(world)]
    for i in range(world):
        for j in range(world):
            if i == j:
                continue
            sent = [(m.src_rank, m.dst_rank, m.req.s) for m in ex[i]["out"].get(j, [])]
            got = [(m.src_rank, m.dst_rank, m.req.s) for m in ex[j]["in"].get(i, [])]
            assert sent == got
            assert ex[i]["send_bytes"].get(j, 0) == ex[j]["recv_bytes"].get(i, 0) == sum(s for _, _, s in sent) * tok
    assert sum(sum(e["send_bytes"].values()) for e in ex) == sum(m.req.s for m in plan) * tok


# ---------------------------------------------------------------- TP head resharding plan (host logic)
@pytest.mark.parametrize("H", [8, 32])
@pytest.mark.parametrize("ts", [1, 2, 4, 8])
@pytest.mark.parametrize("td", [1, 2, 4, 8])
def test_tp_reshard_plan_covers_every_head_once(H, ts, td):
    plan = dd.tp_reshard_plan(H, ts, td)
    seen = []
    for a, b, (h0, h1), hd0 in plan:
        sa, sb = dd.tp_heads(H, ts, a)
        da, db = dd.tp_heads(H, td, b)
        assert 0 <= h0 < h1 <= sb - sa and 0 <= hd0 and hd0 + (h1 - h0) <= db - da
        assert sa + h0 == da + hd0                      # the same global heads on both sides
        seen += list(range(sa + h0, sa + h1))
    assert sorted(seen) == list(range(H))               # every global head moved exactly once
    if ts == td:
        assert plan == [(r, r, (0, H // ts), 0) for r in range(ts)]
    assert len(plan) == max(ts, td)                     # nested partitions: one pair per finer rank


def test_tp_heads_rejects_uneven():
    with pytest.raises(ValueError):
        dd.tp_heads(8, 3, 0)
