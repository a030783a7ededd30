"""CPU tests of the product's host logic and C-ABI surface (no GPU needed):
the library loads and exports every symbol include/frpca_b200.h declares; the
host-side CSR construction and validation match the reference semantics
(checked against the oracle); seed mixing matches types.hpp:52-57."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "frpca_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(frpca_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(fb):
    from paper_1810_06825_b200 import _lib
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with the header"
    assert L.frpca_version() >= 10000


def test_library_is_sm100a(fb):
    """The shipped cubin targets sm_100a (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess
    from paper_1810_06825_b200 import _lib
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_is_a_loud_error(fb):
    """Without a GPU the context creation fails with a CUDA error (no fallback)."""
    import ctypes
    from paper_1810_06825_b200 import _lib
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    h = ctypes.c_void_p()
    st = _lib.load().frpca_ctx_create(0, ctypes.byref(h))
    assert st == _lib.ERR_CUDA
    assert _lib.load().frpca_last_error()


def test_mix_seed_matches_oracle(fb, orc):
    for seed in [0, 1, 7, 2024, (1 << 64) - 1]:
        for tag in [0, 0xA11CE, 0x5A]:
            assert fb.mix_seed(seed, tag) == orc.mix_seed(seed, tag)


@pytest.mark.parametrize("seed", range(6))
def test_from_triplets_matches_oracle(fb, orc, seed):
    rng = np.random.default_rng(seed)
    n = 400
    r = rng.integers(0, 20, n)
    c = rng.integers(0, 15, n)
    v = rng.integers(-3, 4, n).astype(float) * 0.5  # exact cancellations happen
    trip = list(zip(r.tolist(), c.tolist(), v.tolist()))
    A = fb.SparseMatrixCsr.from_triplets(20, 15, trip)
    O = orc.Csr.from_triplets(20, 15, trip)
    rp, ci, va = O.arrays()
    assert np.array_equal(A.rowPtr(), rp)
    assert np.array_equal(A.colIdx(), ci)
    assert np.array_equal(A.values(), va)


def test_from_triplets_reference_case(fb):  # test_sparse.cpp:28-36
    A = fb.SparseMatrixCsr.from_triplets(3, 3, [(1, 2, 3.0), (0, 1, 1.0), (1, 2, -1.0), (0, 0, 2.0),
                                                (2, 0, 5.0), (2, 0, -5.0)])
    assert A.nonZeros() == 3
    assert A.rowPtr().tolist() == [0, 2, 3, 3]
    assert A.colIdx().tolist() == [0, 1, 2]
    assert A.values().tolist() == [2.0, 1.0, 2.0]


@pytest.mark.parametrize("args,msg", [
    ((2, 2, [0, 1], [0], [1.0]), "row_ptr length must be rows \\+ 1"),
    ((2, 2, [0, 2, 1], [0, 1], [1.0, 1.0]), "row_ptr\\[rows\\] must equal nnz"),
    ((2, 2, [0, 2, 1, ], [0, 1], [1.0, 1.0]), "row_ptr"),
    ((2, 2, [0, 1, 2], [0, 5], [1.0, 1.0]), "column index out of range"),
    ((1, 3, [0, 2], [1, 1], [1.0, 1.0]), "strictly increasing"),
    ((3, 3, [0, 2, 1, 2], [0, 1], [1.0, 1.0]), "non-decreasing"),
])
def test_csr_validation_messages(fb, args, msg):  # test_sparse.cpp:38-44
    rows, cols, rp, ci, va = args
    with pytest.raises(ValueError, match=msg):
        fb.SparseMatrixCsr(rows, cols, rp, ci, va)
    with pytest.raises(ValueError, match="out of bounds"):
        fb.SparseMatrixCsr.from_triplets(2, 2, [(0, 2, 1.0)])


def test_validation_first_failure_order(fb, orc):
    """When several rows are malformed, the first in scan order is reported."""
    # row 0 has a decreasing pair, row 1 an out-of-range column
    args = (2, 3, [0, 2, 3], [2, 1, 7], [1.0, 1.0, 1.0])
    with pytest.raises(ValueError) as e1:
        fb.SparseMatrixCsr(*args)
    with pytest.raises(ValueError) as e2:
        orc.Csr.create(*args)
    assert str(e1.value) == str(e2.value)


def test_jump_polynomials(tmp_path):
    """The device Omega generator's 16-ary jump tree (rng_poly.cpp) reproduces
    std::mt19937_64::discard at levels 0 and 1 (host-only check)."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "jump_check"
    subprocess.run(["g++", "-O2", "-std=c++20", os.path.join(root, "tests/cpp/jump_check.cpp"),
                    os.path.join(root, "paper_1810_06825_b200/csrc/rng_poly.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "bad 0" in out.stdout, out.stdout + out.stderr


def test_glibc_log_restatement(tmp_path):
    """The sketch's log (glibc_log.cuh) is glibc's log restated: bitwise equal
    to this host's std::log on polar-method inputs r2 = x^2 + y^2, densely near
    1 (the second polynomial), at every table subinterval edge in every binade
    down to 2^-106, and on uniform bit patterns over [2^-106, 1]."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "glibc_log_check"
    r = subprocess.run(["g++", "-O2", "-std=c++20", "-ffp-contract=off",
                        os.path.join(root, "tests/cpp/glibc_log_check.cpp"), "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe), "6000000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and " bad 0" in out.stdout, out.stdout + out.stderr
