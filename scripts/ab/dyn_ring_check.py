#!/usr/bin/env python
"""Spot check of the ring's guided dynamic grabs (explicit DYNA_SCHED_DYNAMIC) against the oracle on a few
shapes, plain and signalled.  Prints one line per case and BAD <count>."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch, kvgen, oracle, paper_2504_09285_b200 as dk
from kvgen import Geom
import sys; sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
from gpu_util import dev_table, pool_from_host
bad = 0
for g, n, tr, c in ((Geom(3, 8, 128, 2, 16, 300), 4000, (7, 3999), 100), (Geom(2, 32, 128, 2, 16, 200), 3000, (0, 3000), 1000),
                    (Geom(2, 8, 128, 2, 16, 100), 1500, (5, 17), 3)):
    ts, td = kvgen.table_pair(4, n, g, g)
    hs, hd = kvgen.fill_bytes(1, g.pool_bytes), kvgen.fill_bytes(2, g.pool_bytes)
    want = hd.copy(); oracle.migrate(hs, g, ts, want, g, td, tr)
    for sig in (0, dk.DYNA_MIGRATE_SIGNAL):
        src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
        x = dk.migrate(dev_table(src, ts), dev_table(dst, td), tr, (0, g.num_layers), c, engine=2, schedule=2, flags=sig)
        dk.dyna_kv_wait(x)
        ok = np.array_equal(dst.tensor.cpu().numpy(), want); bad += not ok
        print(g, tr, c, sig, ok)
print("BAD", bad)
