"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module is the ONLY code both sides use.  It holds no arithmetic of the
method (no offsets through block tables, no copying): it only draws

* pool contents — a counter-based generator over 8-byte words, so any word
  of any pool can be recomputed independently of where it lives;
* block tables — "freshly allocated" destination blocks and source blocks
  sampled from a pool's free list (SURVEY §8d "Tables");
* request shapes — the trace-like length skew of config 3/5 and the split
  point s = ceil(phi * L) of PAPER.md §3.1.

The CUDA side re-implements the same word generator in its test fill kernel
(`dyna_kv_debug_fill`); `tests/test_gpu_parity.py` checks both agree.

Master seed: 250409285.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

MASTER_SEED = 250409285

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_WORD_MUL = np.uint64(0xD1B54A32D192ED03)
_MASK64 = (1 << 64) - 1


def splitmix64_scalar(x: int) -> int:
    """splitmix64 finaliser on a Python int (mod 2**64)."""
    z = (x + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = z + _GOLDEN
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def pool_key(seed: int) -> int:
    return splitmix64_scalar(seed & _MASK64)


def words(seed: int, first_word: int, n_words: int) -> np.ndarray:
    """Words [first_word, first_word + n_words) of the stream for `seed`.

    word(w) = splitmix64(key ^ (w * 0xD1B54A32D192ED03)), key = splitmix64(seed).
    """
    w = np.arange(first_word, first_word + n_words, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _splitmix64(np.uint64(pool_key(seed)) ^ (w * _WORD_MUL))


def fill_bytes(seed: int, nbytes: int) -> np.ndarray:
    """A fresh uint8 buffer of `nbytes` (multiple of 8) filled from `seed`."""
    if nbytes % 8:
        raise ValueError("nbytes must be a multiple of 8")
    return words(seed, 0, nbytes // 8).view(np.uint8).copy()


def bytes_at(seed: int, byte_offset: int, nbytes: int) -> np.ndarray:
    """The bytes [byte_offset, byte_offset + nbytes) of the stream (8-aligned)."""
    if byte_offset % 8 or nbytes % 8:
        raise ValueError("offset and size must be multiples of 8")
    return words(seed, byte_offset // 8, nbytes // 8).view(np.uint8)


# --------------------------------------------------------------------------
# Coordinate tags (SURVEY §8d "debug coordinate tag mode"): every 16-B vector of a
# pool holds its own coordinates, so a misplaced vector names where it came from.
# --------------------------------------------------------------------------
TAG_MAGIC = 0xA5


def tag_fill(pool_id: int, g: "Geom") -> np.ndarray:
    """A pool image ([L][2][NB][bs][row]) whose 16-B vector v of row (l, kv, b, slot)
    holds word0 = A5 | pool_id | l | kv | b and word1 = slot | v (little-endian u64 pair)."""
    if g.row_bytes % 16:
        raise ValueError("row bytes must be a multiple of 16")
    vpr = g.row_bytes // 16
    n = g.pool_bytes // 16
    i = np.arange(n, dtype=np.uint64)
    v = i % np.uint64(vpr)
    r = i // np.uint64(vpr)
    slot = r % np.uint64(g.block_size)
    r //= np.uint64(g.block_size)
    b = r % np.uint64(g.num_blocks)
    r //= np.uint64(g.num_blocks)
    kv = r % np.uint64(2)
    layer = r // np.uint64(2)
    out = np.empty((n, 2), dtype=np.uint64)
    out[:, 0] = ((np.uint64(TAG_MAGIC) << np.uint64(56)) | (np.uint64(pool_id & 0xFF) << np.uint64(48))
                 | (layer << np.uint64(40)) | (kv << np.uint64(32)) | b)
    out[:, 1] = (slot << np.uint64(32)) | v
    return out.view(np.uint8).reshape(-1)


def tag_decode(img: np.ndarray) -> dict[str, np.ndarray]:
    """Per 16-B vector of a tag-filled image: pool, l, kv, block, slot, vec (int64 arrays) and
    `ok` (the magic byte is intact)."""
    w = np.ascontiguousarray(img).view(np.uint64).reshape(-1, 2)
    w0, w1 = w[:, 0], w[:, 1]
    return {"ok": (w0 >> np.uint64(56)) == TAG_MAGIC,
            "pool": ((w0 >> np.uint64(48)) & np.uint64(0xFF)).astype(np.int64),
            "l": ((w0 >> np.uint64(40)) & np.uint64(0xFF)).astype(np.int64),
            "kv": ((w0 >> np.uint64(32)) & np.uint64(0xFF)).astype(np.int64),
            "block": (w0 & np.uint64(0xFFFFFFFF)).astype(np.int64),
            "slot": (w1 >> np.uint64(32)).astype(np.int64),
            "vec": (w1 & np.uint64(0xFFFFFFFF)).astype(np.int64)}


# --------------------------------------------------------------------------
# Geometry presets (BASELINE.json configs) — shapes only.
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Geom:
    num_layers: int
    num_kv_heads: int
    head_dim: int
    elem_bytes: int
    block_size: int
    num_blocks: int

    @property
    def row_bytes(self) -> int:  # one token's K (or V) in one layer
        return self.num_kv_heads * self.head_dim * self.elem_bytes

    @property
    def pool_bytes(self) -> int:  # [L][2][NB][bs][H][d] elements of e bytes
        return self.num_layers * 2 * self.num_blocks * self.block_size * self.row_bytes

    def with_(self, **kw) -> "Geom":
        return replace(self, **kw)


TOY = Geom(2, 2, 64, 2, 16, 64)              # configs[0]
LLAMA2_7B = Geom(32, 32, 128, 2, 16, 512)    # configs[1]  (4 GiB pool)
LLAMA3_8B = Geom(32, 8, 128, 2, 16, 8192)    # configs[2]/[3]
QWEN2_72B = Geom(80, 8, 128, 2, 16, 6144)    # configs[4] per-GPU shard


# --------------------------------------------------------------------------
# Block tables
# --------------------------------------------------------------------------
def blocks_needed(n_tokens: int, block_size: int) -> int:
    return -(-n_tokens // block_size)


def fragmented_table(rng: np.random.Generator, free: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Draw n distinct blocks from the free list `free` (seeded, fragmented).

    Returns (table, remaining_free)."""
    if n > len(free):
        raise ValueError(f"need {n} blocks, only {len(free)} free")
    pick = rng.choice(len(free), size=n, replace=False)
    table = free[pick].astype(np.int32)
    mask = np.ones(len(free), dtype=bool)
    mask[pick] = False
    return table, free[mask]


def contiguous_table(base: int, n: int) -> np.ndarray:
    return np.arange(base, base + n, dtype=np.int32)


def table_pair(seed: int, n_tokens: int, gs: Geom, gd: Geom, kind: str = "fragmented"):
    """(src_table, dst_table) for one request of n_tokens tokens."""
    ns, nd = blocks_needed(n_tokens, gs.block_size), blocks_needed(n_tokens, gd.block_size)
    if kind == "contiguous":
        return contiguous_table(0, ns), contiguous_table(0, nd)
    rng = np.random.default_rng(seed)
    ts, _ = fragmented_table(rng, np.arange(gs.num_blocks), ns)
    td, _ = fragmented_table(rng, np.arange(gd.num_blocks), nd)
    return ts, td


# --------------------------------------------------------------------------
# Request shapes with trace-like skew (config 3 / 5).  P:306-308, P:336-337,
# P:421 (phi starts at P/(P+D)); lognormal medians per SURVEY §8d.
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Request:
    P: int   # prompt length
    D: int   # predicted decode length
    s: int   # split point, alpha = tokens [0, s) (0-based, reading R1)

    @property
    def L(self) -> int:
        return self.P + self.D


def skewed_batch(seed: int, n: int = 64) -> list[Request]:
    rng = np.random.default_rng(seed)
    P = np.clip(np.rint(rng.lognormal(math.log(1024), 1.0, n)), 16, 16384).astype(np.int64)
    D = np.clip(np.rint(rng.lognormal(math.log(256), 1.0, n)), 1, 4096).astype(np.int64)
    phi = np.clip(P / (P + D) + rng.uniform(-0.2, 0.2, n), 0.0, 1.0)
    s = np.ceil(phi * (P + D)).astype(np.int64)
    return [Request(int(p), int(d), int(x)) for p, d, x in zip(P, D, s)]


def migrating(reqs: list[Request]) -> list[Request]:
    """Requests that actually ship KV: 0 < s < L (s at 0 or L = no split)."""
    return [r for r in reqs if 0 < r.s < r.L]


def batch_tables(seed: int, lengths: list[int], gs: Geom, gd: Geom):
    """Per-request (src_table, dst_table) drawn from shared free lists of both pools."""
    rng = np.random.default_rng(seed)
    free_s, free_d = np.arange(gs.num_blocks), np.arange(gd.num_blocks)
    out = []
    for n in lengths:
        ts, free_s = fragmented_table(rng, free_s, blocks_needed(n, gs.block_size))
        td, free_d = fragmented_table(rng, free_d, blocks_needed(n, gd.block_size))
        out.append((ts, td))
    return out


# --------------------------------------------------------------------------
# configs[4]: all ordered instance pairs migrate concurrently.
# Every rank computes the same plan from seeds alone.
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class PairMigration:
    src_rank: int
    dst_rank: int
    req: Request
    src_table: np.ndarray   # blocks of the source rank's pool
    dst_table: np.ndarray   # freshly allocated blocks of the destination rank's pool


def allpairs_plan(world: int, g: Geom, n_req: int = 4, seed_base: int = 1000) -> list[PairMigration]:
    """Pair (i, j), i != j, ships the migrating requests of skewed_batch(seed_base + 8i + j, n_req).
    Source blocks come from rank i's free list, destination blocks from rank j's free list
    (both drawn in a fixed order, so the plan is identical on every rank)."""
    reqs = {(i, j): migrating(skewed_batch(seed_base + 8 * i + j, n_req))
            for i in range(world) for j in range(world) if i != j}
    free_s = {i: np.arange(g.num_blocks) for i in range(world)}
    free_d = {j: np.arange(g.num_blocks) for j in range(world)}
    rng_s = {i: np.random.default_rng(seed_base * 7 + i) for i in range(world)}
    rng_d = {j: np.random.default_rng(seed_base * 11 + j) for j in range(world)}
    out = []
    for i in range(world):
        for j in range(world):
            if i == j:
                continue
            for r in reqs[(i, j)]:
                ts, free_s[i] = fragmented_table(rng_s[i], free_s[i], blocks_needed(r.s, g.block_size))
                out.append(PairMigration(i, j, r, ts, None))
    # destination blocks, receiver by receiver in sender order
    res = []
    for m in out:
        td, free_d[m.dst_rank] = fragmented_table(rng_d[m.dst_rank], free_d[m.dst_rank],
                                                  blocks_needed(m.req.s, g.block_size))
        res.append(replace(m, dst_table=td))
    return res


def compact_plan(plan: list[PairMigration], spare: int = 0):
    """The same all-pairs plan with every rank's block ids relabelled onto [0, used + spare).

    configs[4]'s pools are 30 GiB per rank and side; sixteen of them do not fit one GPU.  For the
    one-GPU emulation each rank's used source blocks (and, separately, its used destination
    blocks) are renumbered in increasing order, so a table keeps its block order and its
    fragmentation relative to the other requests of that rank; `spare` unused blocks at the end of
    every pool hold rows no migration may touch.  Returns (plan', src_blocks[rank],
    dst_blocks[rank]) — the pool sizes to allocate."""
    ranks = sorted({m.src_rank for m in plan} | {m.dst_rank for m in plan})
    used_s = {r: np.unique(np.concatenate([m.src_table for m in plan if m.src_rank == r] or [np.zeros(0, np.int32)]))
              for r in ranks}
    used_d = {r: np.unique(np.concatenate([m.dst_table for m in plan if m.dst_rank == r] or [np.zeros(0, np.int32)]))
              for r in ranks}
    out = [replace(m, src_table=np.searchsorted(used_s[m.src_rank], m.src_table).astype(np.int32),
                   dst_table=np.searchsorted(used_d[m.dst_rank], m.dst_table).astype(np.int32)) for m in plan]
    return out, {r: len(used_s[r]) + spare for r in ranks}, {r: len(used_d[r]) + spare for r in ranks}
