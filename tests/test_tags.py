"""Coordinate tags (SURVEY §8d debug mode) — CPU: the tag generator against the pool layout of
reading R3, and the oracle against the definition read through tags, so that a misplaced row names
where its bytes came from.  GPU runs of the same checks live in test_gpu_tags.py."""
import numpy as np
import pytest

import kvgen
import oracle
import tagcheck
from kvgen import Geom


def test_tag_layout_pinned_by_hand():
    """R3: off(l, kv, b, slot) = (((l*2 + kv)*NB + b)*bs + slot)*row.  Toy: row = 2*64*2 = 256 B,
    NB = 64, bs = 16; vector 2 of (l 1, kv 0, block 5, slot 3) sits at ((2*64 + 5)*16 + 3)*256 + 32
    = 545568 and reads back as exactly those coordinates."""
    img = kvgen.tag_fill(7, kvgen.TOY)
    w = img[545568:545584].view(np.uint64)
    assert int(w[0]) == (0xA5 << 56) | (7 << 48) | (1 << 40) | (0 << 32) | 5
    assert int(w[1]) == (3 << 32) | 2
    d = kvgen.tag_decode(img)
    assert d["ok"].all() and (d["pool"] == 7).all()
    assert d["vec"].max() == 15 and d["slot"].max() == 15 and d["block"].max() == 63 and d["l"].max() == 1


CASES = [  # (gs, gd, n_tokens, token range, layer range)
    (kvgen.TOY, kvgen.TOY, 256, (0, 100), None),                                        # configs[0]
    (Geom(3, 2, 32, 2, 16, 40), Geom(3, 2, 32, 2, 32, 20), 500, (17, 433), (1, 3)),     # reblock 16 -> 32
    (Geom(2, 4, 16, 2, 32, 20), Geom(2, 4, 16, 2, 8, 80), 600, (31, 577), None),        # reblock 32 -> 8
    (Geom(2, 1, 8, 2, 1, 300), Geom(2, 1, 8, 2, 4, 80), 257, (0, 257), None),           # bs 1 -> 4
]


@pytest.mark.parametrize("gs,gd,n,tr,lr", CASES)
def test_oracle_migrate_reads_back_as_the_definition(gs, gd, n, tr, lr):
    ts, td = kvgen.table_pair(11, n, gs, gd)
    src = kvgen.tag_fill(1, gs)
    dst = kvgen.tag_fill(2, gd)
    oracle.migrate(src, gs, ts, dst, gd, td, tr, lr)
    tagcheck.check(dst, 2, gd, [(1, gs, ts, td, tr, lr or (0, gs.num_layers), None)])
    assert np.array_equal(src, kvgen.tag_fill(1, gs))


def test_oracle_heads_read_back_as_the_definition():
    gs = Geom(2, 4, 64, 2, 16, 40)       # 4 heads of 128 B = 8 vectors each
    gd = gs.with_(num_kv_heads=2, num_blocks=48)
    ts, td = kvgen.table_pair(5, 600, gs, gd)
    dst = kvgen.tag_fill(9, gd)
    oracle.migrate_heads(kvgen.tag_fill(3, gs), gs, ts, dst, gd, td, (10, 555), (0, 2), (1, 3), 0)
    tagcheck.check(dst, 9, gd, [(3, gs, ts, td, (10, 555), (0, 2), (1, 3, 0))])


def test_misplacement_names_its_origin():
    """The checker reports where misplaced bytes came from (here: two destination rows swapped)."""
    g = kvgen.TOY
    ts, td = kvgen.table_pair(11, 256, g, g)
    src, dst = kvgen.tag_fill(1, g), kvgen.tag_fill(2, g)
    oracle.migrate(src, g, ts, dst, g, td, (0, 100))
    row = g.row_bytes
    a, b = int(td[0]) * g.block_size * row, int(td[1]) * g.block_size * row   # slot 0 of two blocks, layer 0 K
    tmp = dst[a:a + row].copy()
    dst[a:a + row] = dst[b:b + row]
    dst[b:b + row] = tmp
    with pytest.raises(AssertionError, match=r"32 misplaced vectors.*holds \{'pool': 1, 'l': 0, 'kv': 0, 'block': "
                                             + str(int(ts[1]))):
        tagcheck.check(dst, 2, g, [(1, g, ts, td, (0, 100), (0, 2), None)])
