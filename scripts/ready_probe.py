#!/usr/bin/env python
"""Does a resident, waiting migration starve the producer?  Producer variants: sleep kernels,
cuBLAS GEMMs of the overlap shape, small GEMMs.  Short device timeout: a hang shows as ETIMEDOUT."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import kvgen  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g = kvgen.LLAMA3_8B.with_(num_blocks=1024)
    s, c = 8192, 512
    src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
    ts, td = kvgen.table_pair(3, s, g, g)
    st = dk.table(src, torch.from_numpy(ts).cuda(), ts)
    dt = dk.table(dst, torch.from_numpy(td).cuda(), td)
    board = dk.dyna_kv_ready_create(0, 64)
    dk.dyna_kv_ready_set_timeout(board, 2_000_000_000)
    prod, mig = torch.cuda.Stream(), torch.cuda.Stream()
    W = torch.randn(4096, 14336, dtype=torch.bfloat16, device="cuda")
    X = torch.randn(c, 4096, dtype=torch.bfloat16, device="cuda")
    Ws = torch.randn(1024, 1024, dtype=torch.bfloat16, device="cuda")
    Xs = torch.randn(64, 1024, dtype=torch.bfloat16, device="cuda")
    producers = {
        "sleep": lambda: torch.cuda._sleep(1_000_000),
        "gemm_overlap_shape": lambda: [torch.matmul(X, W) for _ in range(4)],
        "gemm_small": lambda: [torch.matmul(Xs, Ws) for _ in range(4)],
    }
    for name, fn in producers.items():
        with torch.cuda.stream(prod):  # warm the producer (allocations, cuBLAS heuristics)
            fn()
        torch.cuda.synchronize()
        for ctas in (4, 32, 74):
            epoch = dk.dyna_kv_ready_begin(board)
            t = time.perf_counter()
            x = dk.dyna_kv_migrate_on_ready(st, dt, (0, s), (0, 32), c, board, epoch, mig.cuda_stream,
                                            dk.opts(max_ctas=ctas))
            for k in range(s // c):
                with torch.cuda.stream(prod):
                    fn()
                dk.dyna_kv_ready_mark(board, k, epoch, prod.cuda_stream)
            status = "ok"
            try:
                dk.dyna_kv_wait(x)
            except dk.DynaKVError as e:
                status = str(e)
            torch.cuda.synchronize()
            print(json.dumps({"producer": name, "ctas": ctas, "status": status,
                              "wall_s": round(time.perf_counter() - t, 3)}), flush=True)


if __name__ == "__main__":
    main()
