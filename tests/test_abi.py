"""The C-ABI library loads and exports every symbol include/dyna_kv.h declares
(CPU only; no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dyna_kv.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^DYNA_API [^(]*?\b(dyna_kv_\w+)\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    syms = declared_symbols()
    for s in ("dyna_kv_pool_create", "dyna_kv_migrate", "dyna_kv_wait"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    import paper_2504_09285_b200 as dk
    out = subprocess.run(["nm", "-D", "--defined-only", dk.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r" T (dyna_kv_\w+)$", out.stdout, re.M))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    # and the Python binding binds the same names
    assert set(dk.EXPORTS) == set(declared_symbols())
    for s in dk.EXPORTS:
        assert hasattr(dk, s) and hasattr(dk.lib, s)


def test_library_is_sm100a_only():
    import paper_2504_09285_b200 as dk
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dk.LIB_PATH], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(?!100a)\d+", out.stdout)


def test_sass_has_bulk_copies_and_vector_moves():
    import paper_2504_09285_b200 as dk
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", dk.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UBLKCP" in sass          # TMA bulk copies (cp.async.bulk)
    assert re.search(r"LDG\.E[.A-Z0-9]*\.128", sass)   # 16-B vector loads
    assert re.search(r"STG\.E[.A-Z0-9]*\.128", sass)   # 16-B vector stores
    assert "HMMA" not in sass and "UTCHMMA" not in sass  # no contraction on this path


def test_struct_layouts_match_header(tmp_path):
    """Every struct the binding mirrors has the size and field offsets a C compiler gives the
    header's declaration."""
    import paper_2504_09285_b200 as dk
    structs = {"dyna_kv_pool_desc": dk.dyna_kv_pool_desc, "dyna_block_table": dk.dyna_block_table,
               "dyna_range": dk.dyna_range, "dyna_kv_opts": dk.dyna_kv_opts,
               "dyna_kv_calib_entry": dk.dyna_kv_calib_entry, "dyna_kv_migration": dk.dyna_kv_migration,
               "dyna_kv_channel_handle": dk.dyna_kv_channel_handle, "dyna_kv_ipc_handle": dk.dyna_kv_ipc_handle,
               "dyna_kv_head_migration": dk.dyna_kv_head_migration}
    lines = []
    for name, cls in structs.items():
        lines.append(f'printf("{name} %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name}.{f} %zu\\n", offsetof({name}, {f}));')
    src = tmp_path / "sz.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "dyna_kv.h"\nint main(void) {\n' +
                   "\n".join(lines) + "\nreturn 0;\n}\n")
    exe = tmp_path / "sz"
    r = subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split("\n")
               if line)
    for name, cls in structs.items():
        assert int(got[name]) == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert int(got[f"{name}.{f}"]) == getattr(cls, f).offset, f"{name}.{f}"


def test_status_constants_match_header():
    import paper_2504_09285_b200 as dk
    src = open(HEADER).read()
    for name, val in re.findall(r"#define (DYNA_E\w+|DYNA_OK)\s+\(?(-?\d+)\)?", src):
        assert getattr(dk, name) == int(val), name


def test_flag_engine_variant_schedule_constants_match_header():
    """Every DYNA_MIGRATE_* / DYNA_READY_* flag, engine, variant and schedule the header defines has the
    same value in the binding (a flag added to one side only would silently change meaning)."""
    import paper_2504_09285_b200 as dk
    src = open(HEADER).read()
    found = re.findall(r"#define (DYNA_(?:MIGRATE|READY|ENGINE|VARIANT|SCHED)_\w+)\s+(\d+)", src)
    assert len(found) >= 14 and ("DYNA_MIGRATE_OVERLAP_PREV", "8") in found
    for name, val in found:
        assert getattr(dk, name) == int(val), name
    flags = [int(v) for n, v in found if n.startswith(("DYNA_MIGRATE_", "DYNA_READY_"))]
    assert all(f & (f - 1) == 0 for f in flags) and len(set(flags)) == len(flags)   # distinct single bits


def test_host_validation_without_gpu():
    import paper_2504_09285_b200 as dk
    bad = dk.dyna_kv_pool_desc(2, 2, 64, 2, 16, 64, 0, 0)
    assert dk.dyna_kv_pool_bytes(bad) == 2 * 2 * 64 * 16 * 2 * 64 * 2
    assert dk.dyna_kv_pool_bytes(dk.dyna_kv_pool_desc(0, 2, 64, 2, 16, 64, 0, 0)) == 0
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_pool_create(bad, 0)
    assert e.value.status == dk.DYNA_EINVAL
    # row bytes not a multiple of 16 -> EGEOM before touching the device
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_pool_create(dk.dyna_kv_pool_desc(1, 1, 3, 2, 16, 4, 0, 0), 256)
    assert e.value.status == dk.DYNA_EGEOM
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_migrate(dk.dyna_block_table(), dk.dyna_block_table(), (0, 1), (0, 1), 1)
    assert e.value.status == dk.DYNA_EINVAL
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_wait(0)
    assert e.value.status == dk.DYNA_EINVAL
    # option validation comes first: an unknown flag bit is refused as such, the overlap flag is a valid
    # option (the call then fails on its NULL tables)
    empty = dk.dyna_block_table()
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_migrate_ex(empty, empty, (0, 1), (0, 1), 1, 0, dk.opts(flags=16))
    assert e.value.status == dk.DYNA_EINVAL and "dyna_kv_opts" in str(e.value)
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_migrate_ex(empty, empty, (0, 1), (0, 1), 1, 0,
                              dk.opts(flags=dk.DYNA_MIGRATE_OVERLAP_PREV | dk.DYNA_MIGRATE_SIGNAL))
    assert e.value.status == dk.DYNA_EINVAL and "dyna_kv_opts" not in str(e.value)


def test_calibration_table_roundtrip_without_gpu():
    import paper_2504_09285_b200 as dk
    base = dk.dyna_kv_calib_get()
    entries = [(8192, 0, 64, 2, 2, 16384, 4, 0), (8192, 0, 4096, 1, 1, 0, 0, 8), (0, 1, 1 << 30, 1, 2, 0, 0, 0)]
    dk.dyna_kv_calib_set(entries)
    assert dk.dyna_kv_calib_get() == entries
    with pytest.raises(dk.DynaKVError):
        dk.dyna_kv_calib_set([(8192, 0, 64, 2, 2, 17, 4, 0)])   # piece not a multiple of 16
    with pytest.raises(dk.DynaKVError):
        dk.dyna_kv_calib_set([(8192, 2, 64, 2, 2, 0, 4, 0)])    # peer must be 0/1
    dk.dyna_kv_calib_set([])
    assert dk.dyna_kv_calib_get() == base


def test_batch_host_validation_without_gpu():
    import paper_2504_09285_b200 as dk
    assert dk.lib.dyna_kv_migrate_batch(None, -1, dk.dyna_range(0, 1), 1, None, None,
                                        ctypes.byref(ctypes.c_void_p())) == dk.DYNA_EINVAL
    x = dk.dyna_kv_migrate_batch([], (0, 1), 16)          # nothing to move: nothing enqueued
    assert dk.dyna_kv_query(x)
    dk.dyna_kv_wait(x)
    with pytest.raises(dk.DynaKVError) as e:
        dk.dyna_kv_migrate_batch([], (0, 1), 16, opts=dk.opts(variant=dk.DYNA_VARIANT_STAGED))
    assert e.value.status == dk.DYNA_ENOTSUP


def test_header_is_plain_c_and_links(tmp_path):
    """include/dyna_kv.h compiles as C99 with warnings as errors, and a C program links against
    libdyna_kv.so and calls a host-only entry point (no GPU needed)."""
    import paper_2504_09285_b200 as dk
    src = tmp_path / "t.c"
    src.write_text(r'''
#include <stdio.h>
#include "dyna_kv.h"
int main(void) {
  dyna_kv_pool_desc d = {2, 2, 64, 2, 16, 64, 0, 0};
  size_t b = dyna_kv_pool_bytes(&d);
  dyna_kv_pool_desc bad = {0, 2, 64, 2, 16, 64, 0, 0};
  if (dyna_kv_pool_bytes(&bad) != 0) return 2;
  dyna_kv_xfer_t x = 0;
  if (dyna_kv_wait(x) != DYNA_EINVAL) return 3;          /* NULL handle: an error code, no crash */
  printf("%zu %s\n", b, dyna_kv_last_error());
  return b == (size_t)2 * 2 * 64 * 16 * 2 * 64 * 2 ? 0 : 1;
}
''')
    libdir = os.path.dirname(dk.LIB_PATH)
    exe = tmp_path / "t"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        str(src), "-o", str(exe), "-L", libdir, "-ldyna_kv", f"-Wl,-rpath,{libdir}"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, (out.returncode, out.stdout, out.stderr)
    assert out.stdout.startswith("1048576 ")
