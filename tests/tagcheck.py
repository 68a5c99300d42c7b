"""Coordinate-tag checks ("a debug coordinate tag mode encodes (pool, l, kv, block,
slot, h, vec) into each 16-B vector, so a misplacement decodes itself").

Pools are filled with kvgen.tag_fill; after a migration every destination vector is decoded and
compared with the coordinates the definition assigns it (§4.3 P:556 / SURVEY §8c:
dst row (l, kv, Td[t div bs_d], t mod bs_d) holds src row (l, kv, Ts[t div bs_s], t mod bs_s) for
t in [t0, t1), l in [l0, l1); every other vector keeps its own tag, reading R6).  A failure lists
the first misplaced vectors with where their bytes actually came from."""
from __future__ import annotations

import numpy as np

import kvgen

FIELDS = ("pool", "l", "kv", "block", "slot", "vec")


def expected_coords(dst_id: int, gd, moves) -> dict[str, np.ndarray]:
    """Expected decoded fields of every vector of the destination image.

    moves: list of (src_id, gs, ts, td, (t0, t1), (l0, l1), heads) with heads = None (whole rows)
    or (h0, h1, hd0): source heads [h0, h1) land at destination heads [hd0, hd0 + h1 - h0)."""
    exp = kvgen.tag_decode(kvgen.tag_fill(dst_id, gd))
    exp.pop("ok")
    vpr_d = gd.row_bytes // 16
    for src_id, gs, ts, td, (t0, t1), (l0, l1), heads in moves:
        if t1 <= t0 or l1 <= l0:
            continue
        vph = gs.head_dim * gs.elem_bytes // 16          # vectors per head (head bytes % 16 == 0 here)
        if heads is None:
            xs_d = np.arange(vpr_d)
            xs_s = xs_d
        else:
            h0, h1, hd0 = heads
            xs_s = np.arange(h0 * vph, h1 * vph)
            xs_d = np.arange(hd0 * vph, (hd0 + h1 - h0) * vph)
        t = np.arange(t0, t1)
        ts_, td_ = np.asarray(ts, np.int64), np.asarray(td, np.int64)
        sb, ss = ts_[t // gs.block_size], t % gs.block_size
        db, ds = td_[t // gd.block_size], t % gd.block_size
        for layer in range(l0, l1):
            for kv in range(2):
                rows_d = ((layer * 2 + kv) * gd.num_blocks + db) * gd.block_size + ds     # [T]
                idx = (rows_d[:, None] * vpr_d + xs_d[None, :]).reshape(-1)
                n = len(t) * len(xs_d)
                exp["pool"][idx] = src_id
                exp["l"][idx] = layer
                exp["kv"][idx] = kv
                exp["block"][idx] = np.repeat(sb, len(xs_d))
                exp["slot"][idx] = np.repeat(ss, len(xs_d))
                exp["vec"][idx] = np.tile(xs_s, len(t))
                assert n == len(idx)
    return exp


def check(img: np.ndarray, dst_id: int, gd, moves, limit: int = 5) -> None:
    """Raise AssertionError naming the first misplaced vectors of `img` (a destination pool image)."""
    got = kvgen.tag_decode(img)
    exp = expected_coords(dst_id, gd, moves)
    bad = ~got["ok"]
    for f in FIELDS:
        bad |= got[f] != exp[f]
    if not bad.any():
        return
    vpr = gd.row_bytes // 16
    lines = []
    for i in np.flatnonzero(bad)[:limit]:
        r, x = divmod(int(i), vpr)
        slot = r % gd.block_size
        r //= gd.block_size
        b = r % gd.num_blocks
        lk = r // gd.num_blocks
        where = f"dst (l {lk // 2}, kv {lk % 2}, block {b}, slot {slot}, vec {x})"
        g = {f: int(got[f][i]) for f in FIELDS}
        e = {f: int(exp[f][i]) for f in FIELDS}
        lines.append(f"{where}: holds {g if got['ok'][i] else 'untagged bytes'}, expected {e}")
    raise AssertionError(f"{int(bad.sum())} misplaced vectors; first: " + "; ".join(lines))
