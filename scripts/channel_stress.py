"""Repeat the loopback push/place case that failed intermittently; print every error."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import kvgen  # noqa: E402
import oracle  # noqa: E402
import paper_2504_09285_b200 as dk  # noqa: E402
from gpu_util import dev_table, pool_from_host  # noqa: E402

G = kvgen.Geom(4, 8, 128, 2, 16, 400)
slots, slot_bytes, c, signal = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ts, td = kvgen.table_pair(7, 5000, G, G)
hs, hd = kvgen.fill_bytes(1, G.pool_bytes), kvgen.fill_bytes(2, G.pool_bytes)
tr = (13, 4321)
want = hd.copy()
oracle.migrate(hs, G, ts, want, G, td, tr)
src, dst = pool_from_host(G, hs), pool_from_host(G, hd)
ch = dk.dyna_kv_channel_create(dst.handle, 9, slots, slot_bytes)
s_push, s_place = torch.cuda.Stream(), torch.cuda.Stream()
st, dt = dev_table(src, ts), dev_table(dst, td)
bad = 0
for rep in range(int(sys.argv[5])):
    try:
        xp = dk.dyna_kv_push(st, tr, (0, 4), c, ch, s_push.cuda_stream)
        xq = dk.dyna_kv_place(ch, dt, tr, (0, 4), c, s_place.cuda_stream,
                              dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL if signal else 0))
        errs = []
        for x in (xp, xq):
            try:
                dk.dyna_kv_wait(x)
            except dk.DynaKVError as e:
                errs.append(str(e))
        ok = np.array_equal(dst.tensor.cpu().numpy(), want)
        if errs or not ok:
            bad += 1
            print(f"rep {rep}: data_ok={ok} errors={errs}", flush=True)
    except dk.DynaKVError as e:
        bad += 1
        print(f"rep {rep}: call error {e}", flush=True)
    dst.tensor.copy_(torch.from_numpy(hd).cuda())
    torch.cuda.synchronize()
print(f"slots={slots} slot_bytes={slot_bytes} c={c} signal={signal}: {bad} bad of {sys.argv[5]}")
