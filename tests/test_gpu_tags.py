"""GPU runs read through coordinate tags (SURVEY §8d debug mode): pools filled with
kvgen.tag_fill, every destination vector decoded and compared with the coordinates the definition
assigns it (tests/tagcheck.py).  Same verdict as byte equality with the oracle, but a failure names
the source row each misplaced vector came from — for every engine, head slices, batches, reshards
and pack / unpack."""
import numpy as np
import pytest
import torch

import kvgen
import paper_2504_09285_b200 as dk
import tagcheck
from kvgen import Geom
from gpu_util import dev_table, pool_from_host

pytestmark = pytest.mark.gpu
E = dk
ENGINES = [(1, E.DYNA_ENGINE_AUTO), (1, E.DYNA_ENGINE_VEC), (1, E.DYNA_ENGINE_BULK), (1, E.DYNA_ENGINE_TILES),
           (2, E.DYNA_ENGINE_VEC), (2, E.DYNA_ENGINE_BULK)]
CASES = [  # (gs, gd, n_tokens, token range, layer range, chunk)
    (kvgen.TOY, kvgen.TOY, 256, (0, 100), (0, 2), 32),                                       # configs[0]
    (Geom(3, 2, 32, 2, 16, 40), Geom(3, 2, 32, 2, 32, 20), 500, (17, 433), (1, 3), 100),      # reblock 16 -> 32
    (Geom(2, 4, 16, 2, 32, 20), Geom(2, 4, 16, 2, 8, 80), 600, (31, 577), (0, 2), 64),        # reblock 32 -> 8
    (Geom(4, 8, 128, 2, 16, 400), Geom(4, 8, 128, 2, 16, 400), 5000, (3, 4999), (0, 4), 1000),  # 2-KiB rows
]


def _img(pool):
    torch.cuda.synchronize()
    return pool.tensor.cpu().numpy()


def _run(fn):
    try:
        return fn()
    except dk.DynaKVError as e:
        if e.status == dk.DYNA_ENOTSUP:
            pytest.skip(f"engine refuses this shape: {e}")
        raise


@pytest.mark.parametrize("variant,engine", ENGINES)
@pytest.mark.parametrize("gs,gd,n,tr,lr,c", CASES)
def test_migrate_tags(variant, engine, gs, gd, n, tr, lr, c):
    ts, td = kvgen.table_pair(11, n, gs, gd)
    src, dst = pool_from_host(gs, kvgen.tag_fill(1, gs)), pool_from_host(gd, kvgen.tag_fill(2, gd))
    st, dt = dev_table(src, ts), dev_table(dst, td)
    x = _run(lambda: dk.migrate(st, dt, tr, lr, c, variant=variant, engine=engine))
    dk.dyna_kv_wait(x)
    tagcheck.check(_img(dst), 2, gd, [(1, gs, ts, td, tr, lr, None)])
    assert np.array_equal(_img(src), kvgen.tag_fill(1, gs))


@pytest.mark.parametrize("engine", [E.DYNA_ENGINE_AUTO, E.DYNA_ENGINE_VEC, E.DYNA_ENGINE_BULK])
def test_heads_and_reshard_tags(engine):
    """TP-1 (4 heads) -> TP-2: heads [0, 2) to rank 0, [2, 4) to rank 1, one dyna_kv_reshard launch;
    then one dyna_kv_migrate_heads back-filling head 3 of rank 1 from a second source."""
    gs = Geom(3, 4, 64, 2, 16, 60)
    gd = gs.with_(num_kv_heads=2, num_blocks=70)
    ts, td0 = kvgen.table_pair(5, 900, gs, gd)
    _, td1 = kvgen.table_pair(6, 900, gs, gd)
    src = pool_from_host(gs, kvgen.tag_fill(1, gs))
    d0, d1 = pool_from_host(gd, kvgen.tag_fill(2, gd)), pool_from_host(gd, kvgen.tag_fill(3, gd))
    st, t0, t1 = dev_table(src, ts), dev_table(d0, td0), dev_table(d1, td1)
    tr, lr = (7, 861), (0, 3)
    x = _run(lambda: dk.dyna_kv_reshard([(st, t0, (0, 2), 0), (st, t1, (2, 4), 0)], tr, lr, 256, 0,
                                        dk.opts(engine=engine)))
    dk.dyna_kv_wait(x)
    tagcheck.check(_img(d0), 2, gd, [(1, gs, ts, td0, tr, lr, (0, 2, 0))])
    src2 = pool_from_host(gs, kvgen.tag_fill(4, gs))
    s2 = dev_table(src2, ts)
    x = _run(lambda: dk.dyna_kv_migrate_heads(s2, t1, (100, 400), (1, 3), (0, 1), 1, 128, 0, dk.opts(engine=engine)))
    dk.dyna_kv_wait(x)
    tagcheck.check(_img(d1), 3, gd, [(1, gs, ts, td1, tr, lr, (2, 4, 0)),
                                     (4, gs, ts, td1, (100, 400), (1, 3), (0, 1, 1))])


@pytest.mark.parametrize("engine", [E.DYNA_ENGINE_AUTO, E.DYNA_ENGINE_VEC, E.DYNA_ENGINE_BULK, E.DYNA_ENGINE_TILES])
def test_batch_tags(engine):
    """Four requests from two source pools into two destination pools, one launch."""
    g = Geom(2, 8, 128, 2, 16, 300)
    tabs = kvgen.batch_tables(3, [700, 1200, 333, 900], g, g)
    srcs = [pool_from_host(g, kvgen.tag_fill(i, g)) for i in (1, 2)]
    dsts = [pool_from_host(g, kvgen.tag_fill(i, g)) for i in (5, 6)]
    where = [(0, 0, (0, 700)), (1, 1, (5, 1200)), (0, 1, (0, 333)), (1, 0, (100, 900))]
    # requests 0/3 and 1/2 share a destination pool: their blocks come from one free list (disjoint)
    keep = [(dev_table(srcs[s], tabs[i][0]), dev_table(dsts[d], tabs[i][1])) for i, (s, d, _) in enumerate(where)]
    x = _run(lambda: dk.migrate_batch([(a, b, tr) for (a, b), (_, _, tr) in zip(keep, where)], (0, 2), 256,
                                      engine=engine))
    dk.dyna_kv_wait(x)
    for d in (0, 1):
        moves = [(s + 1, g, tabs[i][0], tabs[i][1], tr, (0, 2), None) for i, (s, dd, tr) in enumerate(where) if dd == d]
        tagcheck.check(_img(dsts[d]), 5 + d, g, moves)


def test_pack_unpack_tags():
    """K1 then K3 through a caller buffer into a destination with another block size."""
    gs, gd = Geom(3, 8, 128, 2, 16, 100), Geom(3, 8, 128, 2, 32, 60)
    ts, td = kvgen.table_pair(8, 1500, gs, gd)
    src, dst = pool_from_host(gs, kvgen.tag_fill(1, gs)), pool_from_host(gd, kvgen.tag_fill(2, gd))
    tr, lr = (40, 1450), (1, 3)
    buf = torch.empty((tr[1] - tr[0]) * 2 * (lr[1] - lr[0]) * gs.row_bytes, dtype=torch.uint8, device="cuda")
    st, dt = dev_table(src, ts), dev_table(dst, td)
    dk.dyna_kv_wait(dk.dyna_kv_pack(st, tr, lr, buf.data_ptr(), buf.numel()))
    dk.dyna_kv_wait(dk.dyna_kv_unpack(buf.data_ptr(), buf.numel(), dt, tr, lr))
    tagcheck.check(_img(dst), 2, gd, [(1, gs, ts, td, tr, lr, None)])
