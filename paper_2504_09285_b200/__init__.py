"""Python binding of libdyna_kv.so — the B200 chunked KV-cache migration path.

Argument marshalling only (ctypes).  Every step of the migration runs in the
CUDA kernels behind the C ABI declared in include/dyna_kv.h; PyTorch is used
by callers for device memory, streams and process groups.  There is no CPU
fallback: importing this package without the built library raises.

The C functions are exposed under their own names (dyna_kv_pool_create,
dyna_kv_migrate, dyna_kv_wait, ...).  `Pool` and `table` are small
conveniences that keep the torch tensors backing a pool / block table alive.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# DYNA_KV_LIB: load another build of the same library (A/B experiments on one box)
LIB_PATH = os.environ.get("DYNA_KV_LIB") or os.path.join(_PKG, "libdyna_kv.so")

# ---------------------------------------------------------------- constants (include/dyna_kv.h)
DYNA_OK, DYNA_EINVAL, DYNA_EGEOM, DYNA_ERANGE, DYNA_EALIAS = 0, -1, -2, -3, -4
DYNA_EPEER, DYNA_ENOMEM, DYNA_ECUDA, DYNA_ETIMEDOUT, DYNA_EAGAIN, DYNA_ENOTSUP = -5, -6, -7, -8, -9, -10
DYNA_ECANCELED = -11
STATUS_NAMES = {0: "DYNA_OK", -1: "DYNA_EINVAL", -2: "DYNA_EGEOM", -3: "DYNA_ERANGE", -4: "DYNA_EALIAS",
                -5: "DYNA_EPEER", -6: "DYNA_ENOMEM", -7: "DYNA_ECUDA", -8: "DYNA_ETIMEDOUT", -9: "DYNA_EAGAIN",
                -10: "DYNA_ENOTSUP", -11: "DYNA_ECANCELED"}
DYNA_MAX_INSTANCES, DYNA_MAX_CHUNKS = 64, 4096
DYNA_VARIANT_AUTO, DYNA_VARIANT_FUSED, DYNA_VARIANT_STAGED = 0, 1, 2
DYNA_ENGINE_AUTO, DYNA_ENGINE_VEC, DYNA_ENGINE_BULK, DYNA_ENGINE_BULK_WS, DYNA_ENGINE_TILES = 0, 1, 2, 3, 4
DYNA_MIGRATE_SIGNAL = 1
DYNA_READY_PER_LAYER = 2
DYNA_MIGRATE_UNCHECKED = 4
DYNA_MIGRATE_OVERLAP_PREV = 8
DYNA_SCHED_STATIC, DYNA_SCHED_DYNAMIC = 1, 2

# every symbol include/dyna_kv.h declares
EXPORTS = (
    "dyna_kv_pool_bytes", "dyna_kv_pool_create", "dyna_kv_pool_destroy", "dyna_kv_migrate",
    "dyna_kv_migrate_ex", "dyna_kv_wait", "dyna_kv_query", "dyna_kv_stream_wait", "dyna_kv_xfer_info",
    "dyna_kv_stream_wait_chunk", "dyna_kv_last_error", "dyna_kv_poll_error", "dyna_kv_launch_count",
    "dyna_kv_enable_peer", "dyna_kv_pool_export", "dyna_kv_pool_import", "dyna_kv_debug_fill",
    "dyna_kv_copy_flags", "dyna_kv_calib_set", "dyna_kv_calib_get", "dyna_kv_calibrate", "dyna_kv_migrate_batch",
    "dyna_kv_prepare_batch", "dyna_kv_prepare_reshard", "dyna_kv_prepared_launch", "dyna_kv_prepared_destroy",
    "dyna_kv_xfer_plan", "dyna_kv_ready_create", "dyna_kv_ready_destroy", "dyna_kv_ready_begin",
    "dyna_kv_ready_mark", "dyna_kv_migrate_on_ready", "dyna_kv_ready_set_timeout",
    "dyna_kv_channel_create", "dyna_kv_channel_export", "dyna_kv_channel_import", "dyna_kv_channel_destroy",
    "dyna_kv_push", "dyna_kv_place", "dyna_kv_channel_set_timeout", "dyna_kv_ready_cancel",
    "dyna_kv_migrate_heads", "dyna_kv_batch_info", "dyna_kv_push_heads", "dyna_kv_place_heads",
    "dyna_kv_chunkstream_open", "dyna_kv_chunkstream_produced", "dyna_kv_chunkstream_close",
    "dyna_kv_chunkstream_info", "dyna_kv_chunkstream_finish", "dyna_kv_pack", "dyna_kv_unpack", "dyna_kv_reshard",
)
DYNA_MAX_BATCH = 16384


class dyna_kv_pool_desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("num_layers", "num_kv_heads", "head_dim", "elem_bytes",
                                               "block_size", "num_blocks", "device", "instance")]


class dyna_block_table(ctypes.Structure):
    _fields_ = [("pool", ctypes.c_void_p), ("block_ids", ctypes.c_void_p),
                ("host_block_ids", ctypes.c_void_p), ("len", ctypes.c_int64)]


class dyna_range(ctypes.Structure):
    _fields_ = [("begin", ctypes.c_int64), ("end", ctypes.c_int64)]


class dyna_kv_migration(ctypes.Structure):
    _fields_ = [("src", dyna_block_table), ("dst", dyna_block_table), ("token_range", dyna_range)]


class dyna_kv_head_migration(ctypes.Structure):
    _fields_ = [("src", dyna_block_table), ("dst", dyna_block_table), ("src_heads", dyna_range),
                ("dst_head_begin", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class dyna_kv_opts(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("variant", "engine", "max_ctas", "flags", "piece_bytes", "stages",
                                               "unroll", "schedule")]


class dyna_kv_calib_entry(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("row_bytes", "peer", "max_chunk_tokens", "variant", "engine",
                                               "piece_bytes", "stages", "unroll")]


class dyna_kv_ipc_handle(ctypes.Structure):
    _fields_ = [("pool_mem", ctypes.c_uint8 * 64), ("inbox_mem", ctypes.c_uint8 * 64),
                ("pool_offset", ctypes.c_uint64), ("desc", dyna_kv_pool_desc), ("uid", ctypes.c_uint64)]


class dyna_kv_channel_handle(ctypes.Structure):
    _fields_ = [("mem", ctypes.c_uint8 * 64), ("slot_bytes", ctypes.c_uint64), ("slots", ctypes.c_int32),
                ("sender", ctypes.c_int32), ("desc", dyna_kv_pool_desc)]


class DynaKVError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `python paper_2504_09285_b200/build.py` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    st, vp, p = ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER
    sig = {
        "dyna_kv_pool_bytes": (ctypes.c_size_t, [p(dyna_kv_pool_desc)]),
        "dyna_kv_pool_create": (st, [p(dyna_kv_pool_desc), vp, p(vp)]),
        "dyna_kv_pool_destroy": (st, [vp]),
        "dyna_kv_migrate": (st, [dyna_block_table, dyna_block_table, dyna_range, dyna_range, ctypes.c_int32, vp,
                                 p(vp)]),
        "dyna_kv_migrate_ex": (st, [dyna_block_table, dyna_block_table, dyna_range, dyna_range, ctypes.c_int32,
                                    vp, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_chunkstream_open": (st, [dyna_block_table, dyna_block_table, ctypes.c_int64, dyna_range,
                                          ctypes.c_int32, vp, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_chunkstream_produced": (st, [vp, ctypes.c_int64, p(ctypes.c_int32)]),
        "dyna_kv_chunkstream_close": (st, [vp, p(ctypes.c_int32)]),
        "dyna_kv_chunkstream_info": (st, [vp, p(ctypes.c_uint64), p(ctypes.c_int32), p(ctypes.c_int32),
                                          p(ctypes.c_int64), p(ctypes.c_int64), p(ctypes.c_int32)]),
        "dyna_kv_chunkstream_finish": (st, [vp]),
        "dyna_kv_push_heads": (st, [dyna_block_table, dyna_range, dyna_range, dyna_range, ctypes.c_int32, vp, vp,
                                    p(vp)]),
        "dyna_kv_place_heads": (st, [vp, dyna_block_table, dyna_range, dyna_range, ctypes.c_int32, ctypes.c_int32,
                                     ctypes.c_int32, vp, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_batch_info": (st, [vp, ctypes.c_int32, p(ctypes.c_uint64), p(ctypes.c_int32), p(ctypes.c_int32),
                                    p(ctypes.c_int32)]),
        "dyna_kv_migrate_heads": (st, [dyna_block_table, dyna_block_table, dyna_range, dyna_range, dyna_range,
                                       ctypes.c_int32, ctypes.c_int32, vp, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_migrate_batch": (st, [p(dyna_kv_migration), ctypes.c_int32, dyna_range, ctypes.c_int32, vp,
                                       p(dyna_kv_opts), p(vp)]),
        "dyna_kv_ready_create": (st, [ctypes.c_int32, ctypes.c_int32, p(vp)]),
        "dyna_kv_ready_destroy": (st, [vp]),
        "dyna_kv_ready_begin": (st, [vp, p(ctypes.c_uint64)]),
        "dyna_kv_ready_set_timeout": (st, [vp, ctypes.c_uint64]),
        "dyna_kv_ready_mark": (st, [vp, ctypes.c_int32, ctypes.c_uint64, vp]),
        "dyna_kv_ready_cancel": (st, [vp, ctypes.c_uint64]),
        "dyna_kv_migrate_on_ready": (st, [dyna_block_table, dyna_block_table, dyna_range, dyna_range, ctypes.c_int32,
                                          vp, ctypes.c_uint64, vp, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_channel_create": (st, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, p(vp)]),
        "dyna_kv_channel_export": (st, [vp, p(dyna_kv_channel_handle)]),
        "dyna_kv_channel_import": (st, [p(dyna_kv_channel_handle), ctypes.c_int32, p(vp)]),
        "dyna_kv_channel_destroy": (st, [vp]),
        "dyna_kv_channel_set_timeout": (st, [vp, ctypes.c_uint64]),
        "dyna_kv_push": (st, [dyna_block_table, dyna_range, dyna_range, ctypes.c_int32, vp, vp, p(vp)]),
        "dyna_kv_place": (st, [vp, dyna_block_table, dyna_range, dyna_range, ctypes.c_int32, vp, p(dyna_kv_opts),
                               p(vp)]),
        "dyna_kv_pack": (st, [dyna_block_table, dyna_range, dyna_range, vp, ctypes.c_uint64, vp, p(dyna_kv_opts),
                              p(vp)]),
        "dyna_kv_unpack": (st, [vp, ctypes.c_uint64, dyna_block_table, dyna_range, dyna_range, vp, p(dyna_kv_opts),
                                p(vp)]),
        "dyna_kv_reshard": (st, [p(dyna_kv_head_migration), ctypes.c_int32, dyna_range, dyna_range, ctypes.c_int32,
                                 vp, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_wait": (st, [vp]),
        "dyna_kv_query": (st, [vp]),
        "dyna_kv_stream_wait": (st, [vp, vp]),
        "dyna_kv_xfer_info": (st, [vp, p(ctypes.c_uint64), p(ctypes.c_int32), p(ctypes.c_int32), p(ctypes.c_int32)]),
        "dyna_kv_xfer_plan": (st, [vp] + [p(ctypes.c_int32)] * 6),
        "dyna_kv_stream_wait_chunk": (st, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                           vp]),
        "dyna_kv_copy_flags": (st, [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp]),
        "dyna_kv_calib_set": (st, [p(dyna_kv_calib_entry), ctypes.c_int32]),
        "dyna_kv_calib_get": (ctypes.c_int32, [p(dyna_kv_calib_entry), ctypes.c_int32]),
        "dyna_kv_prepare_batch": (st, [p(dyna_kv_migration), ctypes.c_int32, dyna_range, ctypes.c_int32,
                                       p(dyna_kv_opts), p(vp)]),
        "dyna_kv_prepare_reshard": (st, [p(dyna_kv_head_migration), ctypes.c_int32, dyna_range, dyna_range,
                                         ctypes.c_int32, p(dyna_kv_opts), p(vp)]),
        "dyna_kv_prepared_launch": (st, [vp, vp, p(vp)]),
        "dyna_kv_prepared_destroy": (st, [vp]),
        "dyna_kv_calibrate": (st, [dyna_block_table, dyna_block_table, p(ctypes.c_int32), ctypes.c_int32,
                                   ctypes.c_int32, vp, p(dyna_kv_calib_entry), p(ctypes.c_float)]),
        "dyna_kv_last_error": (ctypes.c_char_p, []),
        "dyna_kv_poll_error": (st, []),
        "dyna_kv_launch_count": (ctypes.c_uint64, []),
        "dyna_kv_enable_peer": (st, [ctypes.c_int32, ctypes.c_int32]),
        "dyna_kv_pool_export": (st, [vp, p(dyna_kv_ipc_handle)]),
        "dyna_kv_pool_import": (st, [p(dyna_kv_ipc_handle), ctypes.c_int32, p(vp)]),
        "dyna_kv_debug_fill": (st, [vp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("DYNA_KV_LIB") and not hasattr(L, name):
            continue  # an older build under A/B test may lack newer entry points
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


lib = _load()


def _check(status: int) -> int:
    if status < 0:
        raise DynaKVError(status, lib.dyna_kv_last_error().decode(errors="replace"))
    return status


# ---------------------------------------------------------------- C functions, same names
def dyna_kv_pool_bytes(desc: dyna_kv_pool_desc) -> int:
    return lib.dyna_kv_pool_bytes(ctypes.byref(desc))


def dyna_kv_pool_create(desc: dyna_kv_pool_desc, device_base: int) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_pool_create(ctypes.byref(desc), ctypes.c_void_p(device_base), ctypes.byref(out)))
    return out.value


def dyna_kv_pool_destroy(pool: int) -> None:
    _check(lib.dyna_kv_pool_destroy(ctypes.c_void_p(pool)))


def dyna_kv_migrate(src: dyna_block_table, dst: dyna_block_table, token_range, layer_range, chunk_tokens: int,
                    stream: int = 0) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_migrate(src, dst, dyna_range(*token_range), dyna_range(*layer_range), chunk_tokens,
                               ctypes.c_void_p(stream), ctypes.byref(out)))
    return out.value


def dyna_kv_migrate_ex(src: dyna_block_table, dst: dyna_block_table, token_range, layer_range, chunk_tokens: int,
                       stream: int = 0, opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_migrate_ex(src, dst, dyna_range(*token_range), dyna_range(*layer_range), chunk_tokens,
                                  ctypes.c_void_p(stream), ctypes.byref(opts) if opts is not None else None,
                                  ctypes.byref(out)))
    return out.value


def dyna_kv_batch_info(xfer: int, index: int) -> tuple[int, int, int, int]:
    """(epoch, first_slot, num_chunks, sender) of entry `index` of a signalled batch."""
    e, f, n, snd = ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib.dyna_kv_batch_info(ctypes.c_void_p(xfer), index, ctypes.byref(e), ctypes.byref(f), ctypes.byref(n),
                                  ctypes.byref(snd)))
    return e.value, f.value, n.value, snd.value


def dyna_kv_migrate_heads(src: dyna_block_table, dst: dyna_block_table, token_range, layer_range, src_heads,
                          dst_head_begin: int, chunk_tokens: int, stream: int = 0,
                          opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_migrate_heads(src, dst, dyna_range(*token_range), dyna_range(*layer_range),
                                     dyna_range(*src_heads), dst_head_begin, chunk_tokens, ctypes.c_void_p(stream),
                                     ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def dyna_kv_migrate_batch(migs, layer_range, chunk_tokens: int, stream: int = 0,
                          opts: dyna_kv_opts | None = None) -> int:
    """migs: list of (src dyna_block_table, dst dyna_block_table, (t0, t1))."""
    arr = (dyna_kv_migration * max(1, len(migs)))(*[dyna_kv_migration(a, b, dyna_range(*tr)) for a, b, tr in migs])
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_migrate_batch(arr, len(migs), dyna_range(*layer_range), chunk_tokens, ctypes.c_void_p(stream),
                                     ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def dyna_kv_prepare_batch(migs, layer_range, chunk_tokens: int, opts: dyna_kv_opts | None = None) -> int:
    """Plan + upload a batch once (dyna_kv_prepared_launch runs it); migs as dyna_kv_migrate_batch."""
    arr = (dyna_kv_migration * max(1, len(migs)))(*[dyna_kv_migration(a, b, dyna_range(*tr)) for a, b, tr in migs])
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_prepare_batch(arr, len(migs), dyna_range(*layer_range), chunk_tokens,
                                     ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def dyna_kv_prepare_reshard(migs, token_range, layer_range, chunk_tokens: int, opts: dyna_kv_opts | None = None) -> int:
    """Plan + upload a TP reshard once; migs as dyna_kv_reshard."""
    arr = (dyna_kv_head_migration * max(1, len(migs)))(
        *[dyna_kv_head_migration(a, b, dyna_range(*hr), hd, 0) for a, b, hr, hd in migs])
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_prepare_reshard(arr, len(migs), dyna_range(*token_range), dyna_range(*layer_range),
                                       chunk_tokens, ctypes.byref(opts) if opts is not None else None,
                                       ctypes.byref(out)))
    return out.value


def dyna_kv_prepared_launch(prepared: int, stream: int = 0) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_prepared_launch(ctypes.c_void_p(prepared), ctypes.c_void_p(stream), ctypes.byref(out)))
    return out.value


def dyna_kv_prepared_destroy(prepared: int) -> None:
    _check(lib.dyna_kv_prepared_destroy(ctypes.c_void_p(prepared)))


def dyna_kv_ready_create(device: int, max_chunks: int) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_ready_create(device, max_chunks, ctypes.byref(out)))
    return out.value


def dyna_kv_ready_destroy(board: int) -> None:
    _check(lib.dyna_kv_ready_destroy(ctypes.c_void_p(board)))


def dyna_kv_ready_set_timeout(board: int, timeout_ns: int) -> None:
    _check(lib.dyna_kv_ready_set_timeout(ctypes.c_void_p(board), timeout_ns))


def dyna_kv_ready_begin(board: int) -> int:
    e = ctypes.c_uint64()
    _check(lib.dyna_kv_ready_begin(ctypes.c_void_p(board), ctypes.byref(e)))
    return e.value


def dyna_kv_ready_mark(board: int, chunk: int, epoch: int, stream: int = 0) -> None:
    _check(lib.dyna_kv_ready_mark(ctypes.c_void_p(board), chunk, epoch, ctypes.c_void_p(stream)))


def dyna_kv_ready_cancel(board: int, epoch: int) -> None:
    _check(lib.dyna_kv_ready_cancel(ctypes.c_void_p(board), epoch))


def ready_slot(chunk: int, layer: int, layer_range) -> int:
    """Board slot of (chunk, layer) for DYNA_READY_PER_LAYER migrations (include/dyna_kv.h)."""
    l0, l1 = layer_range
    return chunk * (l1 - l0) + (layer - l0)


def dyna_kv_migrate_on_ready(src: dyna_block_table, dst: dyna_block_table, token_range, layer_range,
                             chunk_tokens: int, board: int, epoch: int, stream: int = 0,
                             opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_migrate_on_ready(src, dst, dyna_range(*token_range), dyna_range(*layer_range), chunk_tokens,
                                        ctypes.c_void_p(board), epoch, ctypes.c_void_p(stream),
                                        ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def dyna_kv_channel_create(dst_pool: int, sender: int, slots: int, slot_bytes: int) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_channel_create(ctypes.c_void_p(dst_pool), sender, slots, slot_bytes, ctypes.byref(out)))
    return out.value


def dyna_kv_channel_export(ch: int) -> bytes:
    h = dyna_kv_channel_handle()
    _check(lib.dyna_kv_channel_export(ctypes.c_void_p(ch), ctypes.byref(h)))
    return bytes(h)


def dyna_kv_channel_import(handle: bytes, local_device: int) -> int:
    h = dyna_kv_channel_handle.from_buffer_copy(handle)
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_channel_import(ctypes.byref(h), local_device, ctypes.byref(out)))
    return out.value


def dyna_kv_channel_destroy(ch: int) -> None:
    _check(lib.dyna_kv_channel_destroy(ctypes.c_void_p(ch)))


def dyna_kv_channel_set_timeout(ch: int, timeout_ns: int) -> None:
    _check(lib.dyna_kv_channel_set_timeout(ctypes.c_void_p(ch), timeout_ns))


def dyna_kv_push(src: dyna_block_table, token_range, layer_range, chunk_tokens: int, ch: int, stream: int = 0) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_push(src, dyna_range(*token_range), dyna_range(*layer_range), chunk_tokens,
                            ctypes.c_void_p(ch), ctypes.c_void_p(stream), ctypes.byref(out)))
    return out.value


def dyna_kv_place(ch: int, dst: dyna_block_table, token_range, layer_range, chunk_tokens: int, stream: int = 0,
                  opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_place(ctypes.c_void_p(ch), dst, dyna_range(*token_range), dyna_range(*layer_range),
                             chunk_tokens, ctypes.c_void_p(stream), ctypes.byref(opts) if opts is not None else None,
                             ctypes.byref(out)))
    return out.value


def dyna_kv_chunkstream_open(src: dyna_block_table, dst: dyna_block_table, begin: int, layer_range,
                             chunk_tokens: int, stream: int = 0, opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_chunkstream_open(src, dst, begin, dyna_range(*layer_range), chunk_tokens,
                                        ctypes.c_void_p(stream), ctypes.byref(opts) if opts is not None else None,
                                        ctypes.byref(out)))
    return out.value


def dyna_kv_chunkstream_produced(s: int, n_tokens: int) -> int:
    n = ctypes.c_int32()
    _check(lib.dyna_kv_chunkstream_produced(ctypes.c_void_p(s), n_tokens, ctypes.byref(n)))
    return n.value


def dyna_kv_chunkstream_close(s: int) -> int:
    n = ctypes.c_int32()
    _check(lib.dyna_kv_chunkstream_close(ctypes.c_void_p(s), ctypes.byref(n)))
    return n.value


def dyna_kv_chunkstream_info(s: int) -> dict:
    e, snd, fs = ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_int32()
    pe, pu, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    _check(lib.dyna_kv_chunkstream_info(ctypes.c_void_p(s), ctypes.byref(e), ctypes.byref(snd), ctypes.byref(fs),
                                        ctypes.byref(pe), ctypes.byref(pu), ctypes.byref(n)))
    return {"epoch": e.value, "sender": snd.value, "first_slot": fs.value, "produced_end": pe.value,
            "pushed_end": pu.value, "num_pushed": n.value}


def dyna_kv_chunkstream_finish(s: int) -> None:
    _check(lib.dyna_kv_chunkstream_finish(ctypes.c_void_p(s)))


def dyna_kv_push_heads(src: dyna_block_table, token_range, layer_range, src_heads, chunk_tokens: int, ch: int,
                       stream: int = 0) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_push_heads(src, dyna_range(*token_range), dyna_range(*layer_range), dyna_range(*src_heads),
                                  chunk_tokens, ctypes.c_void_p(ch), ctypes.c_void_p(stream), ctypes.byref(out)))
    return out.value


def dyna_kv_place_heads(ch: int, dst: dyna_block_table, token_range, layer_range, dst_head_begin: int,
                        num_heads: int, chunk_tokens: int, stream: int = 0, opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_place_heads(ctypes.c_void_p(ch), dst, dyna_range(*token_range), dyna_range(*layer_range),
                                   dst_head_begin, num_heads, chunk_tokens, ctypes.c_void_p(stream),
                                   ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def dyna_kv_pack(src: dyna_block_table, token_range, layer_range, buf_ptr: int, buf_bytes: int, stream: int = 0,
                 opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_pack(src, dyna_range(*token_range), dyna_range(*layer_range), ctypes.c_void_p(buf_ptr),
                            buf_bytes, ctypes.c_void_p(stream), ctypes.byref(opts) if opts is not None else None,
                            ctypes.byref(out)))
    return out.value


def dyna_kv_unpack(buf_ptr: int, buf_bytes: int, dst: dyna_block_table, token_range, layer_range, stream: int = 0,
                   opts: dyna_kv_opts | None = None) -> int:
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_unpack(ctypes.c_void_p(buf_ptr), buf_bytes, dst, dyna_range(*token_range),
                              dyna_range(*layer_range), ctypes.c_void_p(stream),
                              ctypes.byref(opts) if opts is not None else None, ctypes.byref(out)))
    return out.value


def dyna_kv_reshard(migs, token_range, layer_range, chunk_tokens: int, stream: int = 0,
                    opts: dyna_kv_opts | None = None) -> int:
    """migs: list of (src dyna_block_table, dst dyna_block_table, (h0, h1), dst_head_begin)."""
    arr = (dyna_kv_head_migration * max(1, len(migs)))(
        *[dyna_kv_head_migration(a, b, dyna_range(*hr), hd, 0) for a, b, hr, hd in migs])
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_reshard(arr, len(migs), dyna_range(*token_range), dyna_range(*layer_range), chunk_tokens,
                               ctypes.c_void_p(stream), ctypes.byref(opts) if opts is not None else None,
                               ctypes.byref(out)))
    return out.value


def dyna_kv_wait(xfer: int) -> None:
    _check(lib.dyna_kv_wait(ctypes.c_void_p(xfer)))


def dyna_kv_query(xfer: int) -> bool:
    s = lib.dyna_kv_query(ctypes.c_void_p(xfer))
    if s == DYNA_EAGAIN:
        return False
    _check(s)
    return True


def dyna_kv_stream_wait(xfer: int, stream: int) -> None:
    _check(lib.dyna_kv_stream_wait(ctypes.c_void_p(xfer), ctypes.c_void_p(stream)))


def dyna_kv_xfer_info(xfer: int) -> tuple[int, int, int, int]:
    """(epoch, num_chunks, sender, first_slot): chunk k's flag is inbox slot [sender][first_slot + k]."""
    e, n, s, f = ctypes.c_uint64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib.dyna_kv_xfer_info(ctypes.c_void_p(xfer), ctypes.byref(e), ctypes.byref(n), ctypes.byref(s),
                                 ctypes.byref(f)))
    return e.value, n.value, s.value, f.value


def dyna_kv_xfer_plan(xfer: int) -> dict:
    v = [ctypes.c_int32() for _ in range(6)]
    _check(lib.dyna_kv_xfer_plan(ctypes.c_void_p(xfer), *[ctypes.byref(a) for a in v]))
    return dict(zip(("variant", "engine", "piece_bytes", "stages", "unroll", "launches"), (a.value for a in v)))


def dyna_kv_stream_wait_chunk(dst_pool: int, sender: int, chunk: int, epoch: int, timeout_ns: int = 0,
                              stream: int = 0) -> None:
    _check(lib.dyna_kv_stream_wait_chunk(ctypes.c_void_p(dst_pool), sender, chunk, epoch, timeout_ns,
                                         ctypes.c_void_p(stream)))


def dyna_kv_copy_flags(dst_pool: int, sender: int, first: int, n: int, host_out_ptr: int, stream: int = 0) -> None:
    """host_out_ptr: address of n uint64 (e.g. a pinned torch.int64 tensor's data_ptr())."""
    _check(lib.dyna_kv_copy_flags(ctypes.c_void_p(dst_pool), sender, first, n, ctypes.c_void_p(host_out_ptr),
                                  ctypes.c_void_p(stream)))


def dyna_kv_calib_set(entries) -> None:
    """entries: list of dyna_kv_calib_entry (or tuples in field order); [] restores the built-in table."""
    arr = (dyna_kv_calib_entry * max(1, len(entries)))(*[e if isinstance(e, dyna_kv_calib_entry)
                                                          else dyna_kv_calib_entry(*e) for e in entries])
    _check(lib.dyna_kv_calib_set(arr, len(entries)))


def dyna_kv_calib_get() -> list:
    n = lib.dyna_kv_calib_get(None, 0)
    arr = (dyna_kv_calib_entry * max(1, n))()
    lib.dyna_kv_calib_get(arr, n)
    return [tuple(getattr(arr[i], f) for f, _ in dyna_kv_calib_entry._fields_) for i in range(n)]


DYNA_CALIB_CANDIDATES = 7


def dyna_kv_calibrate(src: dyna_block_table, dst: dyna_block_table, chunk_tokens, reps: int = 8,
                      stream: int = 0) -> tuple[list, list]:
    """Measure and install AUTO's per-chunk-size choice for this pool pair.  Returns (entries, GB/s per
    candidate per chunk size)."""
    n = len(chunk_tokens)
    ct = (ctypes.c_int32 * n)(*chunk_tokens)
    out = (dyna_kv_calib_entry * n)()
    gb = (ctypes.c_float * (n * DYNA_CALIB_CANDIDATES))()
    _check(lib.dyna_kv_calibrate(src, dst, ct, n, reps, ctypes.c_void_p(stream), out, gb))
    entries = [tuple(getattr(out[i], f) for f, _ in dyna_kv_calib_entry._fields_) for i in range(n)]
    rates = [[gb[i * DYNA_CALIB_CANDIDATES + k] for k in range(DYNA_CALIB_CANDIDATES)] for i in range(n)]
    return entries, rates


def dyna_kv_last_error() -> str:
    return lib.dyna_kv_last_error().decode(errors="replace")


def dyna_kv_poll_error() -> None:
    _check(lib.dyna_kv_poll_error())


def dyna_kv_launch_count() -> int:
    return lib.dyna_kv_launch_count()


def dyna_kv_enable_peer(device: int, peer: int) -> None:
    _check(lib.dyna_kv_enable_peer(device, peer))


def dyna_kv_pool_export(pool: int) -> bytes:
    h = dyna_kv_ipc_handle()
    _check(lib.dyna_kv_pool_export(ctypes.c_void_p(pool), ctypes.byref(h)))
    return bytes(h)


def dyna_kv_pool_import(handle: bytes, local_device: int) -> int:
    h = dyna_kv_ipc_handle.from_buffer_copy(handle)
    out = ctypes.c_void_p()
    _check(lib.dyna_kv_pool_import(ctypes.byref(h), local_device, ctypes.byref(out)))
    return out.value


def dyna_kv_debug_fill(dst: int, nbytes: int, seed: int, byte_offset: int = 0, stream: int = 0) -> None:
    _check(lib.dyna_kv_debug_fill(ctypes.c_void_p(dst), nbytes, seed & ((1 << 64) - 1), byte_offset,
                                  ctypes.c_void_p(stream)))


# ---------------------------------------------------------------- conveniences (keep torch memory alive)
class Pool:
    """A paged KV pool in a torch uint8 tensor on `device`, wrapped by the library."""

    def __init__(self, geom, device: int = 0, instance: int = 0, tensor=None):
        import torch
        self.geom = geom
        self.desc = dyna_kv_pool_desc(geom.num_layers, geom.num_kv_heads, geom.head_dim, geom.elem_bytes,
                                      geom.block_size, geom.num_blocks, device, instance)
        nbytes = dyna_kv_pool_bytes(self.desc)
        if nbytes == 0:
            raise DynaKVError(DYNA_EINVAL, "invalid geometry")
        self.tensor = tensor if tensor is not None else torch.empty(nbytes, dtype=torch.uint8,
                                                                    device=f"cuda:{device}")
        assert self.tensor.numel() >= nbytes and self.tensor.dtype == torch.uint8
        self.device = device
        self.handle = dyna_kv_pool_create(self.desc, self.tensor.data_ptr())

    @classmethod
    def imported(cls, handle: bytes, local_device: int):
        self = cls.__new__(cls)
        h = dyna_kv_ipc_handle.from_buffer_copy(handle)
        self.desc, self.geom, self.tensor, self.device = h.desc, None, None, local_device
        self.handle = dyna_kv_pool_import(handle, local_device)
        return self

    def close(self):
        if getattr(self, "handle", None):
            dyna_kv_pool_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def table(pool: Pool, ids, host_ids=None) -> dyna_block_table:
    """Block table over `pool`.  ids: int32 CUDA tensor, or None for a host-resident table
    (host_ids required; the library uploads it); host_ids: numpy int32 (also enables validation)."""
    import numpy as np
    if ids is None and host_ids is None:
        raise DynaKVError(DYNA_EINVAL, "a table needs device ids or host ids")
    n = ids.numel() if ids is not None else len(host_ids)
    t = dyna_block_table(pool.handle, ids.data_ptr() if ids is not None else None, None, n)
    t._keep = [ids]
    if host_ids is not None:
        h = np.ascontiguousarray(host_ids, dtype=np.int32)
        t.host_block_ids = h.ctypes.data
        t._keep.append(h)
    return t


def opts(variant=0, engine=0, max_ctas=0, flags=0, piece_bytes=0, stages=0, unroll=0, schedule=0) -> dyna_kv_opts:
    return dyna_kv_opts(variant, engine, max_ctas, flags, piece_bytes, stages, unroll, schedule)


def migrate(src: dyna_block_table, dst: dyna_block_table, token_range, layer_range, chunk_tokens, stream=None,
            **kw) -> int:
    """dyna_kv_migrate_ex on a torch stream (default: current stream of the source device)."""
    import torch
    if stream is None:
        s = torch.cuda.current_stream().cuda_stream
    else:
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return dyna_kv_migrate_ex(src, dst, token_range, layer_range, chunk_tokens, s, opts(**kw) if kw else None)


def migrate_batch(migs, layer_range, chunk_tokens, stream=None, **kw) -> int:
    """dyna_kv_migrate_batch on a torch stream; migs: list of (src_table, dst_table, (t0, t1))."""
    import torch
    if stream is None:
        s = torch.cuda.current_stream().cuda_stream
    else:
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return dyna_kv_migrate_batch(migs, layer_range, chunk_tokens, s, opts(**kw) if kw else None)
