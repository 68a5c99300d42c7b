"""Pins for the CPU oracle (oracle/dyna_kv_oracle.c) — CPU only.

The oracle is the plain definition of the migration (PAPER.md
§3.1, §4.3).  These tests tie it to things other
than itself:

* a hand-worked example written from the definition (tests/golden/);
* an independent brute-force formulation (numpy fancy indexing that
  materialises the logical tensor and writes it back), enumerated over tiny
  pools;
* the north_star invariants: element equality, untouched elsewhere, chunk
  size / order independence, A->B->A identity, additivity;
* special cases that reduce to library routines (contiguous slab memcpy,
  torch index_copy_ over whole blocks).
"""
import itertools
import os

import numpy as np
import pytest
import torch

import kvgen
import oracle
from kvgen import Geom

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- helpers
def np_reference(Ps, gs, Ts, Pd, gd, Td, t0, t1, l0, l1):
    """Independent formulation: index the 5-D pool views with token arrays."""
    row = gs.row_bytes
    S = Ps.reshape(gs.num_layers, 2, gs.num_blocks, gs.block_size, row)
    D = Pd.reshape(gd.num_layers, 2, gd.num_blocks, gd.block_size, row)
    t = np.arange(t0, t1)
    Ts, Td = np.asarray(Ts), np.asarray(Td)
    if len(t) and l1 > l0:
        D[l0:l1, :, Td[t // gd.block_size], t % gd.block_size, :] = \
            S[l0:l1, :, Ts[t // gs.block_size], t % gs.block_size, :]


def mapped_row_mask(gd, Td, t0, t1, l0, l1):
    m = np.zeros((gd.num_layers, 2, gd.num_blocks, gd.block_size), bool)
    t = np.arange(t0, t1)
    m[l0:l1, :, np.asarray(Td)[t // gd.block_size], t % gd.block_size] = True
    return m


def pools(gs, gd, seed=1):
    return kvgen.fill_bytes(seed, gs.pool_bytes), kvgen.fill_bytes(seed + 1, gd.pool_bytes)


# ---------------------------------------------------------------- golden
def _parse_golden(path):
    kv = {}
    for line in open(path):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        k, *vals = line.split()
        kv[k] = vals
    g = dict(v.split("=") for v in kv["geom"])
    geom = Geom(int(g["L"]), int(g["H"]), int(g["d"]), int(g["e"]), int(g["bs"]), int(g["NB"]))
    return (geom, [int(x) for x in kv["Ts"]], [int(x) for x in kv["Td"]],
            tuple(int(x) for x in kv["tokens"]), tuple(int(x) for x in kv["layers"]),
            np.array([int(x) for x in kv["expect_dst"]], np.uint8))


def test_golden_hand_example():
    g, Ts, Td, tr, lr, expect = _parse_golden(os.path.join(GOLDEN, "hand_example.txt"))
    Ps = np.arange(g.pool_bytes, dtype=np.uint8)
    Pd = np.full(g.pool_bytes, 255, np.uint8)
    src0 = Ps.copy()
    oracle.migrate(Ps, g, Ts, Pd, g, Td, tr, lr)
    assert np.array_equal(Pd, expect)
    assert np.array_equal(Ps, src0)
    # the chunked model reaches the same bytes for every chunk size and order
    for c in (1, 2, 3):
        n = -(-3 // c)
        for order in itertools.permutations(range(n)):
            Pd2 = np.full(g.pool_bytes, 255, np.uint8)
            oracle.migrate_chunked(Ps, g, Ts, Pd2, g, Td, tr, lr, c, order)
            assert np.array_equal(Pd2, expect), (c, order)


def test_offset_formula_closed_form():
    # pool layout [L][2][NB][bs][H][d] with e-byte elements: offsets are the
    # row-major strides of that shape (numpy's ravel_multi_index).
    g = Geom(3, 2, 4, 2, 4, 5)
    shape = (g.num_layers, 2, g.num_blocks, g.block_size, g.num_kv_heads, g.head_dim)
    rng = np.random.default_rng(0)
    for _ in range(200):
        idx = tuple(int(rng.integers(0, s)) for s in shape)
        assert oracle.off(g, *idx) == np.ravel_multi_index(idx, shape) * g.elem_bytes
    assert oracle.pool_bytes(g) == int(np.prod(shape)) * g.elem_bytes


# ---------------------------------------------------------------- brute force
def _tiny_geoms():
    for L, H, bss, bsd in itertools.product((1, 2), (1, 2), (1, 2, 4), (1, 2, 4)):
        d = 8 // H  # row = 16 B at e = 2
        yield Geom(L, H, d, 2, bss, 6), Geom(L, H, d, 2, bsd, 6)


def test_brute_force_tiny_pools():
    rng = np.random.default_rng(kvgen.MASTER_SEED)
    n_cases = 0
    for gs, gd in _tiny_geoms():
        Ps, Pd0 = pools(gs, gd, seed=n_cases)
        for s in range(0, 9):
            ns, nd = kvgen.blocks_needed(s, gs.block_size), kvgen.blocks_needed(s, gd.block_size)
            if ns > 6 or nd > 6:
                continue
            # all injective dst tables when few, else a random sample of them
            all_td = list(itertools.permutations(range(6), nd))
            tds = all_td if len(all_td) <= 30 else [all_td[i] for i in rng.choice(len(all_td), 30, replace=False)]
            for td in tds:
                ts = rng.choice(6, ns, replace=True).astype(np.int32)  # src may alias (shared prefix)
                t0 = int(rng.integers(0, s + 1))
                for lr in ((0, gs.num_layers), (gs.num_layers - 1, gs.num_layers)):
                    a, b = Pd0.copy(), Pd0.copy()
                    oracle.migrate(Ps, gs, ts, a, gd, td, (t0, s), lr)
                    np_reference(Ps, gs, ts, b, gd, td, t0, s, *lr)
                    assert np.array_equal(a, b), (gs, gd, s, td, ts, t0, lr)
                    n_cases += 1
    assert n_cases > 2000


def test_brute_force_chunked_all_orders():
    rng = np.random.default_rng(7)
    for gs, gd in _tiny_geoms():
        Ps, Pd0 = pools(gs, gd, seed=3)
        for s in (1, 3, 5, 8):
            ns, nd = kvgen.blocks_needed(s, gs.block_size), kvgen.blocks_needed(s, gd.block_size)
            if ns > 6 or nd > 6:
                continue
            ts = rng.permutation(6)[:ns].astype(np.int32)
            td = rng.permutation(6)[:nd].astype(np.int32)
            want = Pd0.copy()
            np_reference(Ps, gs, ts, want, gd, td, 0, s, 0, gs.num_layers)
            for c in range(1, s + 1):
                n = -(-s // c)
                orders = itertools.permutations(range(n)) if n <= 5 else [rng.permutation(n) for _ in range(20)]
                for order in orders:
                    got = Pd0.copy()
                    oracle.migrate_chunked(Ps, gs, ts, got, gd, td, (0, s), (0, gs.num_layers), c, order)
                    assert np.array_equal(got, want), (gs, gd, s, c, order)


# ---------------------------------------------------------------- invariants (toy config shape)
TOY = kvgen.TOY


def _toy_request(seed=11, s=100, n_tok=256):
    ts, td = kvgen.table_pair(seed, n_tok, TOY, TOY)
    Ps, Pd = pools(TOY, TOY, seed)
    return Ps, Pd, ts, td, s


def test_element_equality_and_untouched():
    Ps, Pd0, ts, td, s = _toy_request()
    Pd, src0 = Pd0.copy(), Ps.copy()
    oracle.migrate(Ps, TOY, ts, Pd, TOY, td, (0, s))
    row = TOY.row_bytes
    for l in range(TOY.num_layers):
        for kv in range(2):
            for t in range(s):  # dst KV at (l, h, t) == src KV at t, for every t < s
                a = oracle.logical_off(TOY, ts, l, kv, t)
                b = oracle.logical_off(TOY, td, l, kv, t)
                assert np.array_equal(Pd[b:b + row], Ps[a:a + row])
    mask = np.repeat(mapped_row_mask(TOY, td, 0, s, 0, TOY.num_layers).ravel(), row)
    assert np.array_equal(Pd[~mask], Pd0[~mask])            # untouched elsewhere
    assert np.array_equal(Ps, src0)                          # source read-only
    assert mask.sum() == s * 2 * TOY.num_layers * row        # exactly the range


@pytest.mark.parametrize("c", [1, 15, 16, 17, 32, 64, 100])
def test_chunk_size_and_order_independence(c):
    Ps, Pd0, ts, td, s = _toy_request()
    want = Pd0.copy()
    oracle.migrate(Ps, TOY, ts, want, TOY, td, (0, s))
    n = -(-s // c)
    rng = np.random.default_rng(c)
    orders = list(itertools.permutations(range(n))) if n <= 5 else [rng.permutation(n) for _ in range(5)]
    for order in orders:
        got = Pd0.copy()
        oracle.migrate_chunked(Ps, TOY, ts, got, TOY, td, (0, s), None, c, order)
        assert np.array_equal(got, want)


def test_round_trip_identity():
    gA, gB = TOY, TOY.with_(block_size=32, num_blocks=40)  # reblock 16 -> 32 and back
    A0 = kvgen.fill_bytes(5, gA.pool_bytes)
    B = kvgen.fill_bytes(6, gB.pool_bytes)
    ta, tb = kvgen.table_pair(9, 256, gA, gB)
    s = 100
    A = A0.copy()
    oracle.migrate(A, gA, ta, B, gB, tb, (0, s))
    # poison A's rows in range, then migrate back
    mask = np.repeat(mapped_row_mask(gA, ta, 0, s, 0, gA.num_layers).ravel(), gA.row_bytes)
    A[mask] = 0xA5
    oracle.migrate(B, gB, tb, A, gA, ta, (0, s))
    assert np.array_equal(A, A0)


def test_additivity_tokens_and_layers():
    Ps, Pd0, ts, td, s = _toy_request(s=100)
    whole = Pd0.copy()
    oracle.migrate(Ps, TOY, ts, whole, TOY, td, (0, s))
    for a in (0, 1, 37, 64, 99, 100):
        split = Pd0.copy()
        oracle.migrate(Ps, TOY, ts, split, TOY, td, (0, a))
        oracle.migrate(Ps, TOY, ts, split, TOY, td, (a, s))
        assert np.array_equal(split, whole), a
    split = Pd0.copy()
    oracle.migrate(Ps, TOY, ts, split, TOY, td, (0, s), (0, 1))
    oracle.migrate(Ps, TOY, ts, split, TOY, td, (0, s), (1, 2))
    assert np.array_equal(split, whole)


def test_empty_ranges_are_noops():
    Ps, Pd0, ts, td, _ = _toy_request()
    for tr, lr in (((0, 0), (0, 2)), ((50, 50), (0, 2)), ((0, 100), (1, 1))):
        Pd = Pd0.copy()
        oracle.migrate(Ps, TOY, ts, Pd, TOY, td, tr, lr)
        assert np.array_equal(Pd, Pd0)


# ---------------------------------------------------------------- library special cases
def test_identity_tables_reduce_to_slab_memcpy():
    g = TOY.with_(num_blocks=16)
    Ps, Pd0 = pools(g, g, seed=21)
    n_blk, s = 8, 8 * g.block_size                     # block-aligned range
    Pd = Pd0.copy()
    oracle.migrate(Ps, g, kvgen.contiguous_table(0, n_blk), Pd, g, kvgen.contiguous_table(0, n_blk), (0, s))
    want = Pd0.copy()
    slab = g.num_blocks * g.block_size * g.row_bytes     # one (l, kv) slab
    run = s * g.row_bytes
    for lk in range(g.num_layers * 2):
        want[lk * slab: lk * slab + run] = Ps[lk * slab: lk * slab + run]   # memcpy
    assert np.array_equal(Pd, want)


def test_equal_block_size_aligned_reduces_to_index_copy():
    g = TOY
    Ps, Pd0 = pools(g, g, seed=31)
    ts, td = kvgen.table_pair(17, 128, g, g)             # 8 whole blocks
    Pd = Pd0.copy()
    oracle.migrate(Ps, g, ts, Pd, g, td, (0, 128))
    S = torch.from_numpy(Ps.copy()).view(g.num_layers * 2, g.num_blocks, -1)
    D = torch.from_numpy(Pd0.copy()).view(g.num_layers * 2, g.num_blocks, -1)
    D.index_copy_(1, torch.from_numpy(td).long(), S.index_select(1, torch.from_numpy(ts).long()))
    assert np.array_equal(Pd, D.reshape(-1).numpy())


def test_bitwise_special_values_pass_through():
    # fp16/bf16 NaN payloads, -0, subnormals, Inf: the copy is bitwise (reading R8)
    g = Geom(1, 1, 8, 2, 2, 4)
    specials = np.array([0x7E01, 0xFE55, 0x8000, 0x0001, 0x7C00, 0xFC00, 0x7FFF, 0x0000], np.uint16)
    Ps = np.tile(specials, g.pool_bytes // 16).view(np.uint8).copy()
    Pd = np.zeros(g.pool_bytes, np.uint8)
    oracle.migrate(Ps, g, [3, 1], Pd, g, [0, 2], (0, 4))
    want = np.zeros(g.pool_bytes, np.uint8)
    np_reference(Ps, g, [3, 1], want, g, [0, 2], 0, 4, 0, 1)
    assert np.array_equal(Pd, want) and Pd.any()


# ---------------------------------------------------------------- the pins catch plausible mistakes
def test_pins_detect_mutants():
    """The brute-force check rejects typical slips (swapped K/V, wrong table,
    off-by-one token, block-size mixup)."""
    gs, gd = Geom(2, 1, 8, 2, 2, 6), Geom(2, 1, 8, 2, 4, 6)
    Ps, Pd0 = pools(gs, gd, seed=41)
    ts, td = np.array([4, 1, 3], np.int32), np.array([2, 5], np.int32)
    good = Pd0.copy()
    oracle.migrate(Ps, gs, ts, good, gd, td, (0, 6))
    row = gs.row_bytes
    S = Ps.reshape(2, 2, 6, 2, row)

    def mut(fn):
        D = Pd0.copy().reshape(2, 2, 6, 4, row)
        for l in range(2):
            for kv in range(2):
                for t in range(6):
                    fn(D, l, kv, t)
        return D.reshape(-1)

    mutants = [
        lambda D, l, kv, t: D.__setitem__((l, kv, td[t // 4], t % 4), S[l, 1 - kv, ts[t // 2], t % 2]),
        lambda D, l, kv, t: D.__setitem__((l, kv, td[t // 4], t % 4), S[l, kv, td[t // 4] % 6, t % 2]),
        lambda D, l, kv, t: D.__setitem__((l, kv, td[t // 4], t % 4), S[l, kv, ts[min(t + 1, 5) // 2], (t + 1) % 2]),
        lambda D, l, kv, t: D.__setitem__((l, kv, td[t // 2] if t // 2 < 2 else td[1], t % 4), S[l, kv, ts[t // 2], t % 2]),
    ]
    for m in mutants:
        assert not np.array_equal(mut(m), good)


# ---------------------------------------------------------------- head-restricted definition (reading R14)
def np_reference_heads(Ps, gs, Ts, Pd, gd, Td, t0, t1, l0, l1, h0, h1, hd0):
    """Independent formulation: 6-D views [L][2][NB][bs][H][d*e], head slices assigned with fancy indexing."""
    he = gs.head_dim * gs.elem_bytes
    S = Ps.reshape(gs.num_layers, 2, gs.num_blocks, gs.block_size, gs.num_kv_heads, he)
    D = Pd.reshape(gd.num_layers, 2, gd.num_blocks, gd.block_size, gd.num_kv_heads, he)
    t = np.arange(t0, t1)
    Ts, Td = np.asarray(Ts), np.asarray(Td)
    if len(t) and l1 > l0 and h1 > h0:
        D[l0:l1, :, Td[t // gd.block_size], t % gd.block_size, hd0:hd0 + (h1 - h0)] = \
            S[l0:l1, :, Ts[t // gs.block_size], t % gs.block_size, h0:h1]


def test_heads_full_range_is_the_plain_definition():
    g = Geom(2, 4, 8, 2, 4, 12)
    Ps, Pd0 = pools(g, g, seed=51)
    ts, td = kvgen.table_pair(3, 37, g, g)
    a, b = Pd0.copy(), Pd0.copy()
    oracle.migrate(Ps, g, ts, a, g, td, (5, 37))
    oracle.migrate_heads(Ps, g, ts, b, g, td, (5, 37), None, (0, 4), 0)
    assert np.array_equal(a, b) and not np.array_equal(a, Pd0)


def test_heads_brute_force_tiny_pools():
    rng = np.random.default_rng(kvgen.MASTER_SEED + 14)
    n = 0
    for Hs, Hd, bss, bsd in itertools.product((1, 2, 3, 4), (1, 2, 4), (1, 2, 4), (2, 4)):
        gs, gd = Geom(2, Hs, 8, 2, bss, 6), Geom(2, Hd, 8, 2, bsd, 6)
        Ps, Pd0 = pools(gs, gd, seed=n)
        for h0 in range(Hs):
            for h1 in range(h0, Hs + 1):
                for hd0 in range(0, Hd - (h1 - h0) + 1):
                    s = int(rng.integers(0, 9))
                    ts = rng.choice(6, kvgen.blocks_needed(s, bss), replace=True).astype(np.int32)
                    td = rng.choice(6, kvgen.blocks_needed(s, bsd), replace=False).astype(np.int32)
                    t0 = int(rng.integers(0, s + 1))
                    lr = ((0, 2), (1, 2))[int(rng.integers(0, 2))]
                    a, b = Pd0.copy(), Pd0.copy()
                    oracle.migrate_heads(Ps, gs, ts, a, gd, td, (t0, s), lr, (h0, h1), hd0)
                    np_reference_heads(Ps, gs, ts, b, gd, td, t0, s, *lr, h0, h1, hd0)
                    assert np.array_equal(a, b), (gs, gd, s, t0, lr, h0, h1, hd0)
                    n += 1
    assert n > 500


def _tp_heads(H, T, r):
    """Contiguous head partition of a TP-T instance: rank r holds heads [r*H/T, (r+1)*H/T)."""
    return r * H // T, (r + 1) * H // T


@pytest.mark.parametrize("T", [2, 4, 8])
def test_heads_tp_scatter_gather_round_trip(T):
    """A TP-1 pool scattered head-wise into T shard pools (each its own H/T-head geometry and
    fresh table), then gathered back into a TP-1 pool, equals one plain migration."""
    H, s = 8, 45
    g1 = Geom(2, H, 8, 2, 4, 20)
    gT = Geom(2, H // T, 8, 2, 8, 10)
    Ps, Pd0 = pools(g1, g1, seed=60 + T)
    ts, td = kvgen.table_pair(61, s, g1, g1)
    shards = [kvgen.fill_bytes(70 + r, gT.pool_bytes) for r in range(T)]
    tsh = [kvgen.table_pair(80 + r, s, gT, gT)[1] for r in range(T)]
    for r in range(T):
        oracle.migrate_heads(Ps, g1, ts, shards[r], gT, tsh[r], (0, s), None, _tp_heads(H, T, r), 0)
    got = Pd0.copy()
    for r in range(T):
        h0, h1 = _tp_heads(H, T, r)
        oracle.migrate_heads(shards[r], gT, tsh[r], got, g1, td, (0, s), None, (0, h1 - h0), h0)
    want = Pd0.copy()
    oracle.migrate(Ps, g1, ts, want, g1, td, (0, s))
    assert np.array_equal(got, want)


def test_heads_untouched_outside_the_slice():
    gs, gd = Geom(1, 2, 8, 2, 4, 4), Geom(1, 4, 8, 2, 4, 4)
    Ps, Pd0 = pools(gs, gd, seed=90)
    ts, td = np.array([2, 0], np.int32), np.array([3, 1], np.int32)
    got = Pd0.copy()
    oracle.migrate_heads(Ps, gs, ts, got, gd, td, (1, 7), None, (0, 2), 1)
    D, D0 = got.reshape(1, 2, 4, 4, 4, 16), Pd0.reshape(1, 2, 4, 4, 4, 16)
    S = Ps.reshape(1, 2, 4, 4, 2, 16)
    changed = np.zeros(D.shape[:-1], bool)
    for t in range(1, 7):
        changed[0, :, td[t // 4], t % 4, 1:3] = True
        assert np.array_equal(D[0, :, td[t // 4], t % 4, 1:3], S[0, :, ts[t // 4], t % 4, 0:2])
    assert np.array_equal(D[~changed], D0[~changed])


def test_heads_pins_detect_mutants():
    """The brute force rejects a dropped head offset on either side and swapped head order."""
    gs, gd = Geom(1, 4, 8, 2, 2, 4), Geom(1, 4, 8, 2, 2, 4)
    Ps, Pd0 = pools(gs, gd, seed=91)
    ts, td = np.array([1, 3], np.int32), np.array([2, 0], np.int32)
    good = Pd0.copy()
    oracle.migrate_heads(Ps, gs, ts, good, gd, td, (0, 4), None, (1, 3), 2)
    S = Ps.reshape(1, 2, 4, 2, 4, 16)
    variants = [((1, 3), (0, 2)), ((0, 2), (2, 4)), ((2, 0), (2, 4))]  # (src heads, dst heads) slips
    for (a, b), (c, d_) in variants:
        D = Pd0.copy().reshape(1, 2, 4, 2, 4, 16)
        for t in range(4):
            src = S[0, :, ts[t // 2], t % 2, a:b] if a < b else S[0, :, ts[t // 2], t % 2, [2, 1]]
            D[0, :, td[t // 2], t % 2, c:d_] = src
        assert not np.array_equal(D.reshape(-1), good)


# ---------------------------------------------------------------- pack / unpack (P:556's two halves)
def test_pack_brute_force_tiny_pools():
    """oracle.pack == the logical tensor materialised by numpy fancy indexing (independent
    formulation), laid out [l - l0][kv][t - t0][row]; unpack(pack) == migrate; and
    oracle_unpack writes exactly what np_reference writes from the same buffer."""
    rng = np.random.default_rng(11)
    n_cases = 0
    for gs, gd in _tiny_geoms():
        Ps, Pd0 = pools(gs, gd, seed=n_cases + 5)
        row = gs.row_bytes
        S = Ps.reshape(gs.num_layers, 2, gs.num_blocks, gs.block_size, row)
        for s in range(0, 9, 2):
            ns, nd = kvgen.blocks_needed(s, gs.block_size), kvgen.blocks_needed(s, gd.block_size)
            if ns > 6 or nd > 6:
                continue
            ts = rng.choice(6, ns, replace=True).astype(np.int32)
            td = rng.permutation(6)[:nd].astype(np.int32)
            t0 = int(rng.integers(0, s + 1))
            for lr in ((0, gs.num_layers), (gs.num_layers - 1, gs.num_layers)):
                buf = oracle.pack(Ps, gs, ts, (t0, s), lr)
                t = np.arange(t0, s)
                want = S[lr[0]:lr[1], :, ts[t // gs.block_size], t % gs.block_size, :] if len(t) else \
                    np.zeros((lr[1] - lr[0], 2, 0, row), np.uint8)
                assert np.array_equal(buf, np.ascontiguousarray(want).reshape(-1)), (gs, s, t0, lr)
                a, b = Pd0.copy(), Pd0.copy()
                oracle.unpack(buf, a, gd, td, (t0, s), lr)
                oracle.migrate(Ps, gs, ts, b, gd, td, (t0, s), lr)
                assert np.array_equal(a, b)
                n_cases += 1
    assert n_cases > 150


def test_pack_identity_table_is_slab_concatenation():
    """Identity table, block-aligned range: the packed buffer is each (l, kv) slab's first
    s rows, concatenated (a plain memcpy per slab)."""
    g = TOY.with_(num_blocks=16)
    Ps, _ = pools(g, g, seed=31)
    s = 5 * g.block_size
    buf = oracle.pack(Ps, g, kvgen.contiguous_table(0, 5), (0, s))
    slab, run = g.num_blocks * g.block_size * g.row_bytes, s * g.row_bytes
    want = np.concatenate([Ps[lk * slab: lk * slab + run] for lk in range(g.num_layers * 2)])
    assert np.array_equal(buf, want)
