"""GPU unit test of the warp-segment primitives (csrc/decide.cuh Seg<LPS, MM>):
segment sums / min / max / u64 sums / broadcasts / ballots against plain loops."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_seg_primitives():
    src = os.path.join(HERE, "native", "seg_primitives.cu")
    exe = os.path.join(HERE, "native", "seg_primitives")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-std=c++17", "-I", os.path.join(os.path.dirname(HERE), "include"), "-o", exe, src])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
