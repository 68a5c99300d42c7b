import sys, os, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch, kvgen, paper_2504_09285_b200 as dk
torch.cuda.set_device(0)
g = kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=6144)
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
for p, seed in ((src, 11), (dst, 12)):
    dk.dyna_kv_debug_fill(p.tensor.data_ptr(), p.tensor.numel(), seed, 0, 0)
reqs = kvgen.migrating(kvgen.skewed_batch(1000 + 1, 4))
tabs = kvgen.batch_tables(3, [r.s for r in reqs], g, g)
T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b), r.s) for r, (a, b) in zip(reqs, tabs)]
print([t[2] for t in T])
s = torch.cuda.Stream()
tot = sum(t[2] for t in T)
for rep in range(3):
    for name, eng, piece, unroll in (("vec8k", 1, 8192, 4), ("vec4k", 1, 4096, 8), ("tiles", 4, 0, 0), ("auto", 0, 0, 0)):
        o = dk.opts(engine=eng, piece_bytes=piece, unroll=unroll)
        def once():
            return [dk.dyna_kv_migrate_ex(a, b, (0, n), (0, 80), 1024, s.cuda_stream, o) for a, b, n in T]
        for x in once(): dk.dyna_kv_wait(x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(20_000_000)
        e0.record(s)
        xs = []
        for _ in range(10): xs += once()
        e1.record(s)
        for x in xs: dk.dyna_kv_wait(x)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(rep, name, round(ms * 1e3, 1), "us/set", round(2 * tot * 80 * 2 * 256 / (ms * 1e-3) / 6451.2e9, 3))
