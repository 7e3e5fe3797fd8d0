"""The shading path's D3 division (common.cuh operator/(D3, double): one
shared reciprocal for three quotients, the compiler's own division sequence)
must give exactly the quotients of `/` — the images' bit-exactness rests on
it. tests/support/divtest.cu draws random operands over, around and beyond
the range where the shared sequence is used (zeros, exact and near-1
quotients included) and compares bit patterns on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_d3_division_matches_ieee_quotients(tmp_path):
    exe = str(tmp_path / "divtest")
    src = os.path.join(HERE, "support", "divtest.cu")
    b = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", "-std=c++17",
                        "-I", os.path.join(HERE, "..", "include"), "-o", exe, src],
                       capture_output=True, text=True, timeout=600)
    assert b.returncode == 0, b.stderr[-3000:]
    r = subprocess.run([exe, str(1 << 28)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
