"""Build libdyna_kv.so in-tree with nvcc for sm_100a (no JIT, no torch build helpers).

    python paper_2504_09285_b200/build.py     (standalone: does not import the package)
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdyna_kv.so")
SOURCES = [os.path.join(CSRC, f) for f in ("runtime.cu", "launch.cu", "migrate.cu", "coupling.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("runtime.cuh", "plan.cuh", "dyna_kv_kernels.cuh", "calib_default.inc")] \
    + [os.path.join(ROOT, "include", "dyna_kv.h")]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Build libdyna_kv.so (or, for A/B experiments, a variant with extra -D defines at `out`,
    loaded by the binding through DYNA_KV_LIB)."""
    if not force and os.path.exists(out) and not defines:
        newest = max(os.path.getmtime(p) for p in DEPS)
        if os.path.getmtime(out) >= newest:
            return out
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-shared",
           "-o", out + ".tmp", *SOURCES, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libdyna_kv.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", action="store_true")
    ap.add_argument("--out", default=LIB, help="output path (A/B variants: e.g. ab_libs/libdyna_kv_x.so)")
    ap.add_argument("-D", action="append", default=[], dest="defines", help="extra preprocessor define")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.v, out=os.path.abspath(a.out), defines=a.defines))
