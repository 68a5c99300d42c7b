"""configs[4] all ordered instance pairs, emulated on ONE GPU as one kernel over every rank's data.

On the 8-GPU box every rank issues one dyna_kv_migrate_batch into its peers' IPC-imported receive
pools (scripts/allpairs.py, bench.py N >= 3).  With one GPU the ranks are emulated the way
B200_PROFILING prescribes — one launch over all ranks' data, no rank waiting on another — at the
full Qwen2-72B shard geometry (80 layers, 8 KV heads, d128, bf16, block 16) and the seeded
all-pairs plan (kvgen.allpairs_plan; §3.1 P:352 "the instances exchange the required KV
cache blocks"), with each rank's block ids relabelled onto pools that fit one device
(kvgen.compact_plan).  Every destination row is checked on the device against its source row
(torch indexing), sampled rows against the oracle's offsets and the kvgen stream, and the spare
blocks of every receive pool stay untouched."""
import numpy as np
import pytest
import torch

import kvgen
import paper_2504_09285_b200 as dk
from gpu_util import dev_table, mapped_mask, pool_filled, sampled_rows_match, torch_rows_equal, untouched_equal

pytestmark = pytest.mark.gpu
SPARE = 4


@pytest.mark.parametrize("world,signal", [(4, False), (4, True), (3, False)])
def test_allpairs_one_launch_all_ranks(world, signal):
    g = kvgen.QWEN2_72B
    plan, ns, nd = kvgen.compact_plan(kvgen.allpairs_plan(world, g), spare=SPARE)
    src = {r: pool_filled(g.with_(num_blocks=ns[r]), 3000 + r, instance=r) for r in range(world)}
    recv = {r: pool_filled(g.with_(num_blocks=nd[r]), 4000 + r, instance=r) for r in range(world)}
    keep = [(dev_table(src[m.src_rank], m.src_table), dev_table(recv[m.dst_rank], m.dst_table)) for m in plan]
    migs = [(a, b, (0, m.req.s)) for (a, b), m in zip(keep, plan)]
    st = torch.cuda.current_stream().cuda_stream
    x = dk.dyna_kv_migrate_batch(migs, (0, g.num_layers), 1024, st,
                                 dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL) if signal else None)
    plan_info = dk.dyna_kv_xfer_plan(x)
    infos = [dk.dyna_kv_batch_info(x, i) for i in range(len(migs))] if signal else []
    dk.dyna_kv_wait(x)
    torch.cuda.synchronize()
    assert plan_info["launches"] == 1
    for m, (epoch, first, nck, sender) in zip(plan, infos):   # every request's chunk flags, in its receiver
        assert sender == m.src_rank and nck == -(-m.req.s // 1024)
        fl = torch.zeros(nck, dtype=torch.int64).pin_memory()
        dk.dyna_kv_copy_flags(recv[m.dst_rank].handle, sender, first, nck, fl.data_ptr(), st)
        torch.cuda.synchronize()
        assert (fl.numpy() == epoch).all(), (m.src_rank, m.dst_rank, fl)
    rng = np.random.default_rng(world)
    for m in plan:
        s, d = src[m.src_rank], recv[m.dst_rank]
        assert torch_rows_equal(s, m.src_table, d, m.dst_table, (0, m.req.s), (0, g.num_layers))
        assert sampled_rows_match(3000 + m.src_rank, s.geom, m.src_table, d, d.geom, m.dst_table,
                                  (0, m.req.s), (0, g.num_layers), 4, rng) == 0
    for r in range(world):   # rows no migration maps (spare blocks, tails of last blocks) are untouched
        tr = [(m.dst_table, (0, m.req.s)) for m in plan if m.dst_rank == r]
        assert untouched_equal(recv[r], 4000 + r, mapped_mask(recv[r].geom, tr))
    for p in list(src.values()) + list(recv.values()):
        p.close()
