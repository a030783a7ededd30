"""Uploads of millions of column ids: the device validation that narrows the
int64 ids to int32 (csr.cu k_check_cols) must keep the reference's
first-failure semantics (sparse_matrix.hpp:132-138) at size, including ids
whose low 32 bits would look valid, and leave the context usable. (A host-side
narrowing before the copy was measured and dropped: DESIGN §4, rejected.)"""
import numpy as np
import pytest

from metrics import SPMM_TOL, rel_fro

pytestmark = pytest.mark.gpu

M, N, D = 100_000, 60_000, 45  # 4.5M nonzeros


def big_arrays(seed=0):
    rng = np.random.default_rng(seed)
    x = np.sort(rng.integers(0, N - D, size=(M, D)), axis=1) + np.arange(D)  # strictly increasing rows
    ci = x.reshape(-1).astype(np.int64)
    rp = np.arange(0, M * D + 1, D, dtype=np.int64)
    va = rng.standard_normal(M * D)
    return rp, ci, va


@pytest.fixture(scope="module")
def arrays():
    return big_arrays()


def test_narrowed_upload_spmm_vs_oracle(fb, orc, arrays):
    rp, ci, va = arrays
    A = fb.SparseMatrixCsr(M, N, rp, ci, va)
    oA = orc.Csr.create(M, N, rp, ci, va)
    X = orc.gaussian_matrix(N, 8, 1)
    Y = orc.gaussian_matrix(M, 8, 2)
    assert rel_fro(fb.spmm(A, X), orc.spmm(oA, X)) <= SPMM_TOL
    assert rel_fro(fb.spmm_transpose(A, Y), orc.spmm_transpose(oA, Y)) <= SPMM_TOL


def corrupt(arrays, edits):
    rp, ci, va = arrays
    ci = ci.copy()
    for (row, off), v in edits.items():
        ci[rp[row] + off] = v
    return rp, ci, va


@pytest.mark.parametrize("edits,msg", [
    ({(70_000, 5): N}, "out of range"),
    ({(50_000, 0): -1}, "out of range"),
    ({(90_000, 44): 1 << 40}, "out of range"),
    ({(30_000, 7): (1 << 32) + 5}, "out of range"),          # low 32 bits = 5: must not pass as 5
    ({(30_000, 7): -(1 << 32) + 3}, "out of range"),         # low 32 bits = 3
    ({(10, 3): 0, (90_000, 1): N + 7}, "strictly increasing"),   # first failure is the order in row 10
    ({(10, 2): 0, (10, 3): N}, "strictly increasing"),       # same row: order at entry 2 before range at 3
    ({(10, 2): N, (10, 3): 0}, "out of range"),              # range at entry 2 first
    ({(20, 1): (1 << 33), (20, 2): 1}, "out of range"),
])
def test_narrowed_upload_validation(fb, arrays, edits, msg):
    rp, ci, va = corrupt(arrays, edits)
    A = fb.SparseMatrixCsr(M, N, rp, ci, va, validate=False)
    with pytest.raises(ValueError, match=msg):
        fb.spmm(A, np.ones((N, 2)))


def test_narrowed_upload_context_usable_after_error(fb, orc, arrays):
    rp, ci, va = corrupt(arrays, {(5, 5): 1 << 40})
    bad = fb.SparseMatrixCsr(M, N, rp, ci, va, validate=False)
    with pytest.raises(ValueError, match="out of range"):
        fb.spmm(bad, np.ones((N, 2)))
    rp, ci, va = arrays
    A = fb.SparseMatrixCsr(M, N, rp, ci, va)
    X = orc.gaussian_matrix(N, 4, 5)
    assert rel_fro(fb.spmm(A, X), orc.spmm(orc.Csr.create(M, N, rp, ci, va), X)) <= SPMM_TOL
