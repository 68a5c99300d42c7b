"""ctypes binding to the CPU oracle (oracle/dyna_kv_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / `--impl reference` legs may import this.  The
CUDA path (paper_2504_09285_b200) never imports it and shares no code with it.

Every function here is marshalling only; the arithmetic is in the C file,
which cites PAPER.md §3.1 and §4.3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dyna_kv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


class _Geom(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("L", "H", "d", "e", "bs", "NB")]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.run(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC], check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        gp = ctypes.POINTER(_Geom)
        i32p, u8p, i64p = (ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_uint8),
                           ctypes.POINTER(ctypes.c_int64))
        i64 = ctypes.c_int64
        L.oracle_off.argtypes = [gp, i64, i64, i64, i64, i64, i64]
        L.oracle_off.restype = i64
        L.oracle_logical_off.argtypes = [gp, i32p, i64, i64, i64, i64, i64]
        L.oracle_logical_off.restype = i64
        L.oracle_pool_bytes.argtypes = [gp]
        L.oracle_pool_bytes.restype = i64
        L.oracle_migrate.argtypes = [u8p, gp, i32p, u8p, gp, i32p, i64, i64, i64, i64]
        L.oracle_migrate.restype = None
        L.oracle_migrate_chunked.argtypes = [u8p, gp, i32p, u8p, gp, i32p, i64, i64, i64, i64,
                                             i64, i64p, i64, u8p]
        L.oracle_migrate_chunked.restype = None
        L.oracle_migrate_heads.argtypes = [u8p, gp, i32p, u8p, gp, i32p, i64, i64, i64, i64, i64, i64, i64]
        L.oracle_migrate_heads.restype = None
        L.oracle_pack.argtypes = [u8p, gp, i32p, i64, i64, i64, i64, u8p]
        L.oracle_pack.restype = None
        L.oracle_unpack.argtypes = [u8p, u8p, gp, i32p, i64, i64, i64, i64]
        L.oracle_unpack.restype = None
        _lib = L
    return _lib


def geom(g) -> _Geom:
    """Accept a kvgen.Geom (or anything with the same attributes)."""
    return _Geom(g.num_layers, g.num_kv_heads, g.head_dim, g.elem_bytes, g.block_size, g.num_blocks)


def _u8(a: np.ndarray):
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _i32(a: np.ndarray):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def pool_bytes(g) -> int:
    return lib().oracle_pool_bytes(ctypes.byref(geom(g)))


def off(g, l, kv, b, slot, h=0, i=0) -> int:
    return lib().oracle_off(ctypes.byref(geom(g)), l, kv, b, slot, h, i)


def logical_off(g, table, l, kv, t, h=0, i=0) -> int:
    t_arr, tp = _i32(table)
    return lib().oracle_logical_off(ctypes.byref(geom(g)), tp, l, kv, t, h, i)


def _check(Ps, gs, Ts, Pd, gd, Td, tr, lr):
    assert Ps.nbytes == pool_bytes(gs) and Pd.nbytes == pool_bytes(gd)
    for a in ("num_layers", "num_kv_heads", "head_dim", "elem_bytes"):
        assert getattr(gs, a) == getattr(gd, a), a
    if tr[1] > tr[0]:
        assert len(Ts) * gs.block_size >= tr[1] and len(Td) * gd.block_size >= tr[1]


def migrate(Ps: np.ndarray, gs, Ts, Pd: np.ndarray, gd, Td, token_range, layer_range=None) -> None:
    """In-place: Pd <- the plain definition (dyna_kv_oracle.c oracle_migrate)."""
    layer_range = layer_range or (0, gs.num_layers)
    _check(Ps, gs, Ts, Pd, gd, Td, token_range, layer_range)
    ts, tsp = _i32(Ts)
    td, tdp = _i32(Td)
    lib().oracle_migrate(_u8(Ps), ctypes.byref(geom(gs)), tsp, _u8(Pd), ctypes.byref(geom(gd)), tdp,
                         token_range[0], token_range[1], layer_range[0], layer_range[1])


def migrate_chunked(Ps, gs, Ts, Pd, gd, Td, token_range, layer_range, chunk_tokens, order=None) -> None:
    """In-place chunk-by-chunk model of P:556 with an arbitrary chunk order."""
    layer_range = layer_range or (0, gs.num_layers)
    _check(Ps, gs, Ts, Pd, gd, Td, token_range, layer_range)
    n = token_range[1] - token_range[0]
    n_chunks = -(-n // chunk_tokens) if n > 0 else 0
    order = np.arange(n_chunks, dtype=np.int64) if order is None else np.asarray(order, dtype=np.int64)
    staging = np.zeros(max(1, (layer_range[1] - layer_range[0]) * 2 * chunk_tokens * gs.row_bytes), np.uint8)
    ts, tsp = _i32(Ts)
    td, tdp = _i32(Td)
    lib().oracle_migrate_chunked(_u8(Ps), ctypes.byref(geom(gs)), tsp, _u8(Pd), ctypes.byref(geom(gd)), tdp,
                                 token_range[0], token_range[1], layer_range[0], layer_range[1],
                                 chunk_tokens, order.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                 len(order), _u8(staging))


def migrate_heads(Ps: np.ndarray, gs, Ts, Pd: np.ndarray, gd, Td, token_range, layer_range, src_heads,
                  dst_head_begin: int) -> None:
    """In-place: Pd <- the head-restricted definition (dyna_kv_oracle.c oracle_migrate_heads)."""
    layer_range = layer_range or (0, gs.num_layers)
    assert Ps.nbytes == pool_bytes(gs) and Pd.nbytes == pool_bytes(gd)
    for a in ("num_layers", "head_dim", "elem_bytes"):
        assert getattr(gs, a) == getattr(gd, a), a
    h0, h1 = src_heads
    assert 0 <= h0 <= h1 <= gs.num_kv_heads and 0 <= dst_head_begin and dst_head_begin + h1 - h0 <= gd.num_kv_heads
    if token_range[1] > token_range[0]:
        assert len(Ts) * gs.block_size >= token_range[1] and len(Td) * gd.block_size >= token_range[1]
    ts, tsp = _i32(Ts)
    td, tdp = _i32(Td)
    lib().oracle_migrate_heads(_u8(Ps), ctypes.byref(geom(gs)), tsp, _u8(Pd), ctypes.byref(geom(gd)), tdp,
                               token_range[0], token_range[1], layer_range[0], layer_range[1], h0, h1, dst_head_begin)


def pack(Ps: np.ndarray, gs, Ts, token_range, layer_range=None) -> np.ndarray:
    """The sender half of P:556 (dyna_kv_oracle.c oracle_pack): a new buffer
    [l - l0][kv][t - t0][row] of the source rows reached through Ts."""
    layer_range = layer_range or (0, gs.num_layers)
    assert Ps.nbytes == pool_bytes(gs)
    n = token_range[1] - token_range[0]
    out = np.zeros(max(0, (layer_range[1] - layer_range[0]) * 2 * n * gs.row_bytes), np.uint8)
    if n > 0:
        assert len(Ts) * gs.block_size >= token_range[1]
    ts, tsp = _i32(Ts)
    lib().oracle_pack(_u8(Ps), ctypes.byref(geom(gs)), tsp, token_range[0], token_range[1], layer_range[0],
                      layer_range[1], _u8(out) if out.size else None)
    return out


def unpack(buf: np.ndarray, Pd: np.ndarray, gd, Td, token_range, layer_range=None) -> None:
    """In-place: the receiver half of P:556 (dyna_kv_oracle.c oracle_unpack)."""
    layer_range = layer_range or (0, gd.num_layers)
    assert Pd.nbytes == pool_bytes(gd)
    n = token_range[1] - token_range[0]
    assert buf.nbytes == max(0, (layer_range[1] - layer_range[0]) * 2 * n * gd.row_bytes)
    if n > 0:
        assert len(Td) * gd.block_size >= token_range[1]
    td, tdp = _i32(Td)
    lib().oracle_unpack(_u8(buf) if buf.size else None, _u8(Pd), ctypes.byref(geom(gd)), tdp, token_range[0],
                        token_range[1], layer_range[0], layer_range[1])
