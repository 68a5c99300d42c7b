#!/usr/bin/env python
"""dyna_kv_pack / dyna_kv_unpack throughput (K1 / K3 as calls) for one-head TP-shard rows
(256 B) and 2-KiB rows, VEC vs the tile kernel; calls issued behind a _sleep gate so the events
time device work only.   python scripts/pack_probe.py [--out gpurun_out/pack_probe.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "pack_probe.json"))
a = ap.parse_args()
torch.cuda.set_device(0)
s = torch.cuda.Stream()
out = []
for name, g, n in (("Qwen2-72B TP-8 shard (256-B rows)", kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=2048), 4096),
                   ("Llama-3-8B TP-4 shard (512-B rows)", kvgen.LLAMA3_8B.with_(num_kv_heads=2, num_blocks=2048), 4096)):
    pool = dk.Pool(g, 0)
    dk.dyna_kv_debug_fill(pool.tensor.data_ptr(), pool.tensor.numel(), 1, 0, 0)
    rng = np.random.default_rng(1)
    ids = rng.permutation(g.num_blocks).astype(np.int32)
    t = dk.table(pool, torch.from_numpy(ids).cuda(), None)
    need = n * 2 * g.num_layers * g.row_bytes
    buf = torch.empty(need, dtype=torch.uint8, device="cuda")
    for eng_name, eng in (("VEC", dk.DYNA_ENGINE_VEC), ("TILES", dk.DYNA_ENGINE_TILES)):
        for op in ("pack", "unpack"):
            o = dk.opts(engine=eng, flags=dk.DYNA_MIGRATE_UNCHECKED)
            reps = 10

            def call():
                if op == "pack":
                    return dk.dyna_kv_pack(t, (0, n), (0, g.num_layers), buf.data_ptr(), need, s.cuda_stream, o)
                return dk.dyna_kv_unpack(buf.data_ptr(), need, t, (0, n), (0, g.num_layers), s.cuda_stream, o)
            dk.dyna_kv_wait(call())
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                torch.cuda._sleep(20_000_000)
            e0.record(s)
            xs = [call() for _ in range(reps)]
            e1.record(s)
            for x in xs:
                dk.dyna_kv_wait(x)
            e1.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            frac = 2 * need / (us * 1e-6) / 6451.2e9
            row = {"rows": name, "op": op, "engine": eng_name, "bytes": need, "us_per_call": round(us, 1),
                   "frac_of_measured_hbm": round(frac, 3)}
            print(json.dumps(row), flush=True)
            out.append(row)
    del pool, buf
    torch.cuda.empty_cache()
json.dump(out, open(a.out, "w"), indent=1)
