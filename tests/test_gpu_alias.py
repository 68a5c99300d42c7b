"""Reading R7 on the host, randomized: dyna_kv_migrate_batch and dyna_kv_reshard
refuse a call exactly when a brute-force enumeration of the rows (and heads) it writes finds a
destination row written twice, or a destination row that another entry reads as a source row."""
import numpy as np
import pytest

import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import pool_filled

pytestmark = pytest.mark.gpu


def _brute(entries, bs_of, heads_of=None):
    """entries: (src uid, src ids, dst uid, dst ids, (t0, t1)); True when R7 is violated."""
    written = {}
    for k, (su, sid, du, did, (t0, t1)) in enumerate(entries):
        h = heads_of[k] if heads_of else (0, 1)
        for t in range(t0, t1):
            for hh in range(*h):
                key = (du, int(did[t // bs_of[du]]), t % bs_of[du], hh)
                if key in written:
                    return True
                written[key] = k
    for k, (su, sid, du, did, (t0, t1)) in enumerate(entries):
        h = heads_of[k] if heads_of else (0, 1)
        for t in range(t0, t1):
            for hh in range(*h):
                if (su, int(sid[t // bs_of[su]]), t % bs_of[su], hh) in written:
                    return True
    return False


@pytest.mark.parametrize("seed", range(40))
def test_batch_alias_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    g = Geom(1, 1, 8, 2, 4, 24)                 # tiny: 16-B rows, 4-token blocks, 24 blocks per pool
    pools = [pool_filled(g, 10 + i) for i in range(3)]
    n = int(rng.integers(1, 5))
    entries, migs = [], []
    for _ in range(n):
        a, b = (int(x) for x in rng.integers(0, 3, 2))
        t0 = int(rng.integers(0, 8))
        t1 = t0 + int(rng.integers(1, 9))
        nbk = (t1 - 1) // 4 + 1
        sid = rng.integers(0, 24, nbk).astype(np.int32)
        did = rng.choice(24, nbk, replace=False).astype(np.int32) if rng.random() < 0.7 else \
            rng.integers(0, 24, nbk).astype(np.int32)
        entries.append((a, sid, b, did, (t0, t1)))
        migs.append((dk.table(pools[a], None, sid), dk.table(pools[b], None, did), (t0, t1)))
    want = _brute(entries, {0: 4, 1: 4, 2: 4})
    try:
        dk.dyna_kv_wait(dk.migrate_batch(migs, (0, 1), 4))
        got = False
    except dk.DynaKVError as e:
        assert e.status == dk.DYNA_EALIAS, e
        got = True
    assert got == want, entries


@pytest.mark.parametrize("seed", range(30))
def test_reshard_head_alias_matches_brute_force(seed):
    rng = np.random.default_rng(100 + seed)
    g = Geom(1, 4, 8, 2, 4, 24)                 # 4 heads of 16 B
    srcs = [pool_filled(g, 20 + i, instance=i) for i in range(2)]
    dst = pool_filled(g, 30)
    s = int(rng.integers(1, 12))
    nbk = (s - 1) // 4 + 1
    entries, heads, migs = [], [], []
    for k in range(int(rng.integers(1, 4))):
        a = int(rng.integers(0, 2))
        h0 = int(rng.integers(0, 4))
        hd0 = int(rng.integers(0, 4 - 0))
        n = 1
        sid = rng.integers(0, 24, nbk).astype(np.int32)
        did = rng.integers(0, 24, nbk).astype(np.int32) if rng.random() < 0.5 else np.arange(nbk, dtype=np.int32)
        entries.append((a, sid, 2, did, (0, s)))
        heads.append((hd0, hd0 + n))
        migs.append((dk.table(srcs[a], None, sid), dk.table(dst, None, did), (h0, h0 + n), hd0))
    want = _brute(entries, {0: 4, 1: 4, 2: 4}, heads)
    try:
        dk.dyna_kv_wait(dk.dyna_kv_reshard(migs, (0, s), (0, 1), 4))
        got = False
    except dk.DynaKVError as e:
        assert e.status == dk.DYNA_EALIAS, e
        got = True
    assert got == want, (entries, heads)
