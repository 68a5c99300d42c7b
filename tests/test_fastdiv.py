"""The kernels' invariant-divisor division (dynakv::FastDiv) equals plain
integer division: exhaustive small divisors x edge dividends, 2M random pairs.
Host-compiled with nvcc (no GPU needed)."""
import os
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))


def test_fastdiv_matches_division():
    src = os.path.join(HERE, "native", "fastdiv_check.cu")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "fastdiv_check")
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-o", exe, src], check=True,
                       capture_output=True)
        out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok")
