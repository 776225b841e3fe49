"""The Morton bit-arithmetic forms of csrc/geometry.cuh (neighbour_k,
near_mask_k: dilated-integer increment / decrement on the interleaved bits)
against the plain decode / offset / encode forms, exhaustively for d = 1, 2, 3 on
small levels.  Host-compiled (nvcc, no GPU).  The kernels use the bit forms for
the standard structure's interaction partners and near-field neighbours
(Def 2.4 and the box geometry)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="nvcc not available")
def test_geometry_bit_forms(tmp_path):
    exe = tmp_path / "geometry_check"
    subprocess.run([NVCC, "-std=c++17", "-O1", "-I", os.path.join(ROOT, "paper_2008_12441_b200", "csrc"),
                    os.path.join(ROOT, "tests", "native", "geometry_check.cu"), "-o", str(exe)],
                   check=True, capture_output=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "bad 0" in out.stdout
