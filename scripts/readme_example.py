"""The README's Python usage example, runnable (kept in sync by hand)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, kvgen, paper_2504_09285_b200 as dk

g = kvgen.LLAMA3_8B                                   # 32 layers, 8 KV heads, d128, bf16, block 16
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)               # paged pools [L][2][NB][bs][H][d] (or dk.Pool.imported(handle, dev))
ts, td = kvgen.table_pair(0, 4096, g, g)              # alpha's blocks, beta's freshly allocated blocks
st = dk.table(src, torch.from_numpy(ts).cuda(), ts)   # device ids (+ host ids: synchronous range/alias checks)
dt = dk.table(dst, None, td)                          # host-only ids: the library uploads them
x = dk.migrate(st, dt, (0, 4096), (0, 32), 512, flags=dk.DYNA_MIGRATE_SIGNAL)
epoch, nchunks, sender, first = dk.dyna_kv_xfer_info(x)  # chunk k landed when inbox[sender][first + k] >= epoch
dk.dyna_kv_wait(x)
print("readme example ok", epoch, nchunks, sender)
