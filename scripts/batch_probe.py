#!/usr/bin/env python
"""configs[2] batch probe: one dyna_kv_migrate_batch vs per-request calls, per engine and schedule."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402


def main():
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    cs = st.cuda_stream
    g = kvgen.LLAMA3_8B
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 5, 0, cs)
    dk.dyna_kv_debug_fill(dst.tensor.data_ptr(), dst.tensor.numel(), 6, 0, cs)
    reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
    tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
    T = [(dk.table(src, torch.from_numpy(a).cuda(), a), dk.table(dst, torch.from_numpy(b).cuda(), b), r.s)
         for r, (a, b) in zip(reqs, tabs)]
    migs = [(a, b, (0, s)) for a, b, s in T]
    payload = sum(s for _, _, s in T) * 2 * 32 * g.row_bytes
    only = os.environ.get("ONLY")
    for name, engine, sched in (("vec", 1, 1), ("vec", 1, 2), ("bulk", 2, 1), ("bulk", 2, 2)):
        for mode in ("batch", "calls"):
            if only and only != f"{mode}-{name}-{sched}":
                continue
            o = dk.opts(engine=engine, schedule=sched)

            def run():
                if mode == "batch":
                    return [dk.dyna_kv_migrate_batch(migs, (0, 32), 256, cs, o)]
                return [dk.dyna_kv_migrate_ex(a, b, (0, s), (0, 32), 256, cs, o) for a, b, s in T]
            ts = []
            for rep in range(6):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                xs = run()
                e1.record(st)
                for x in xs:
                    dk.dyna_kv_wait(x)
                e1.synchronize()
                if rep:
                    ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            print(json.dumps({"mode": mode, "engine": name, "schedule": sched, "ms": ms,
                              "GBps": payload / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
