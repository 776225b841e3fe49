"""The C-ABI library loads, exports every symbol include/hmat.h declares, and
rejects invalid arguments before touching a device (runs without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_2008_12441_b200 import hmat as hm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hmat.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hmat_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    decl = declared_symbols()
    assert len(decl) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", hm.LIB_PATH], capture_output=True, text=True, check=True)
    exported = set(re.findall(r" T (hmat_\w+)", out.stdout))
    missing = [s for s in decl if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    assert set(hm.EXPORTS) == set(decl)


def test_binding_names_match_c_names():
    for s in declared_symbols():
        assert hasattr(hm, s), s


def expect(status, fn, *args):
    with pytest.raises(hm.HMatError) as ei:
        fn(*args)
    assert ei.value.status == status
    assert hm.hmat_last_error() != ""
    return str(ei.value)


@pytest.mark.parametrize("args,needle", [
    ((3, 4, 64, 8), "dim"),
    ((3, 0, 64, 8), "dim"),
    ((-1, 2, 64, 8), "depth"),
    ((48, 1, 1, 1), "depth"),
    ((3, 2, 0, 8), "leaf"),
    ((3, 2, 64, 0), "rank"),
    ((40, 2, 64, 1), "overflow"),
])
def test_plan_query_rejects_invalid(args, needle):
    msg = expect(hm.HMAT_ERR_INVALID, hm.hmat_plan_query, *args)
    assert needle in msg


def test_invalid_partitions():
    expect(hm.HMAT_ERR_INVALID, hm.hmat_plan_query, 3, 2, 64, 8, 3, 0)     # not a power of two
    expect(hm.HMAT_ERR_INVALID, hm.hmat_plan_query, 1, 2, 64, 8, 8, 0)     # more ranks than leaves
    expect(hm.HMAT_ERR_INVALID, hm.hmat_plan_query, 3, 2, 64, 8, 2, 2)     # rank id out of range
    expect(hm.HMAT_ERR_UNSUPPORTED, hm.hmat_plan_query, 3, 3, 64, 147, 1, 0)  # W = 1029 > 1024


def test_create_rejects_invalid_before_device_work():
    # invalid shapes are caught by validation even with real pointers
    expect(hm.HMAT_ERR_INVALID, hm.hmat_create_uninit, 3, 5, 64, 8, None)
    # NULL panels
    h = ctypes.c_void_p()
    assert hm._lib.hmat_create(2, 2, 4, 2, None, None, None, None, ctypes.byref(h)) == hm.HMAT_ERR_INVALID
    assert hm._lib.hmat_create(2, 2, 4, 2, None, None, None, None, None) == hm.HMAT_ERR_INVALID
    # P > 1 needs an NCCL id (allreduce and tree exchanges); exchange modes are 0..3
    d = hm._dist(nranks=2, rank=0, device=0)
    expect(hm.HMAT_ERR_INVALID, hm.hmat_create_uninit, 3, 2, 64, 8, d)
    d = hm._dist(nranks=2, rank=0, device=0, exchange=hm.HMAT_EXCHANGE_TREE)
    expect(hm.HMAT_ERR_INVALID, hm.hmat_create_uninit, 3, 2, 64, 8, d)
    d = hm._dist(nranks=2, rank=0, device=0, exchange=4)
    expect(hm.HMAT_ERR_INVALID, hm.hmat_create_uninit, 3, 2, 64, 8, d)


def test_null_handles():
    assert hm._lib.hmat_destroy(None) == hm.HMAT_OK
    assert hm._lib.hmat_num_points(None) == -1
    assert hm._lib.hmat_matvec(None, None, None, 1) == hm.HMAT_ERR_INVALID
    assert "NULL" in hm.hmat_last_error()
    assert hm._lib.hmat_launches_per_matvec(None, 1) == -1


def test_no_gpu_means_error_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    # a valid request on a machine without a GPU must fail loudly (no CPU path)
    status = hm._lib.hmat_create_uninit(1, 1, 2, 1, None, ctypes.byref(ctypes.c_void_p()))
    assert status == hm.HMAT_ERR_CUDA


def test_plan_query_valid():
    info = hm.hmat_plan_query(9, 2, 64, 16)
    assert info.N == 2 ** 24 and info.row_begin == 0 and info.row_end == 2 ** 24
    assert info.W == 48 and info.cross_levels == 0 and info.exchange_rows == 0
    assert 64 % info.Rp == 0 and 64 % info.Re == 0
    assert info.smem_p <= 227 * 1024 and info.smem_e <= 227 * 1024


def test_nccl_unique_id_resolves_the_runtime():
    """hmat_nccl_unique_id dlopens NCCL (csrc/comm.cpp) and returns the 128-byte id
    rank 0 broadcasts for P > 1 (include/hmat.h); two calls give different ids."""
    import torch  # noqa: F401  (loads torch's libnccl first, as bench.py does)
    a, b = hm.hmat_nccl_unique_id(), hm.hmat_nccl_unique_id()
    assert len(a) == 128 and len(b) == 128 and a != b and any(a)


def _build_c_example(tmp_path):
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "matvec_c")
    lib = os.path.join(root, "paper_2008_12441_b200")
    subprocess.run(["gcc", "-std=c99", "-pedantic", "-Wall", "-Wextra", "-Werror", "-O2", "-I" + os.path.join(root, "include"),
                    os.path.join(root, "examples", "matvec.c"), "-L" + lib, "-lhmat", "-Wl,-rpath," + lib, "-lm",
                    "-o", exe], check=True)
    return exe


def test_c_example_compiles_as_plain_c(tmp_path):
    """include/hmat.h is a C header (extern "C", plain pointers): a C99 program
    compiles against it with -pedantic -Werror and links libhmat.so."""
    _build_c_example(tmp_path)


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    """examples/matvec.c on the GPU: linearity and the dense part alone."""
    import subprocess
    out = subprocess.run([_build_c_example(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.strip().endswith("ok")


@pytest.mark.parametrize("L,d,b,r,dmma,narrow", [
    (5, 3, 64, 32, 1, (1, 1, 1, 1)),    # c5: W = 224, every pass width (16, 32, 64, 8)
    (9, 2, 64, 16, 1, (1, 1, 1, 1)),    # c4 shape: W = 48 (8-warp project grid)
    (3, 3, 64, 8, 0, (0, 0, 0, 0)),     # W = 56: not a multiple of 16 -> SIMT only
    (3, 2, 32, 16, 0, (0, 0, 0, 0)),    # leaf 32: not a multiple of the 64-row item
])
def test_plan_query_reports_tensor_core_layouts(L, d, b, r, dmma, narrow):
    """hmat_plan_query (host only) states which products the tensor-core path
    takes and its pass layouts; every layout fits 227 KB of shared memory."""
    info = hm.hmat_plan_query(L, d, b, r)
    assert info.dmma == dmma and tuple(info.dmma_ok) == narrow
    assert info.max_nr == 4
    for i in range(4):
        if info.dmma_ok[i]:
            assert 2 <= info.dmma_stages_p[i] and 2 <= info.dmma_stages_e[i]
            assert info.dmma_smem_p[i] <= 227 * 1024 and info.dmma_smem_e[i] <= 227 * 1024
            # expand: 2 CTAs per SM, 3 for the 16-wide pass (layout 0) of the weak structure
            ctas_e = 3 if i == 0 else 2
            assert info.dmma_grid_p[i] % 148 == 0 and info.dmma_grid_e[i] == 148 * ctas_e
            assert ctas_e * (info.dmma_smem_e[i] + 1024) <= 228 * 1024


def test_every_declaration_cites_the_paper():
    """Each exported declaration of include/hmat.h is preceded by a comment that
    cites the paper passage it implements or serves (PAPER.md:<line>)."""
    src = open(os.path.join(ROOT, "include", "hmat.h")).read()
    missing = []
    for name in declared_symbols():
        m = re.search(r"^[\w\s\*]*\b" + name + r"\s*\(", src, flags=re.M)
        assert m, name
        before = src[:m.start()]
        # the comment block that precedes the declaration (possibly shared by a
        # run of consecutive declarations)
        end = before.rfind("*/")
        start = before.rfind("/*", 0, end)
        between = before[end + 2:]
        decls_between = re.findall(r"\bhmat_[a-z_0-9]+\s*\(", re.sub(r"/\*.*?\*/", "", between, flags=re.S))
        comment = before[start:end]
        if "PAPER.md:" not in comment or len(decls_between) > 3:
            missing.append(name)
    assert not missing, f"declarations without a PAPER.md: citation: {missing}"
