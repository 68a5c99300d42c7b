#!/usr/bin/env python
"""One round of configs[2]'s 54 requests as overlapped per-request calls (DYNA_MIGRATE_OVERLAP_PREV,
AUTO -> VEC), for an ncu capture of k_copy_lanes (DRAM bytes per launch vs the request's payload)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

torch.cuda.set_device(0)
g = kvgen.LLAMA3_8B
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
keep = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b)) for a, b in tabs]
o = dk.opts(flags=dk.DYNA_MIGRATE_OVERLAP_PREV)
cs = torch.cuda.current_stream().cuda_stream
for rep in range(2):
    xs = [dk.dyna_kv_migrate_ex(a, b, (0, r.s), (0, 32), 256, cs, o) for (a, b), r in zip(keep, reqs)]
    for x in xs:
        dk.dyna_kv_wait(x)
print("payload of requests 0..3 (bytes):", [r.s * 2 * 32 * g.row_bytes for r in reqs[:4]])
