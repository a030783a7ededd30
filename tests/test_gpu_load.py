"""SURVEY §8 row f2 on the B200: from_triplets on the device (radix sort,
per-coordinate sums, exact-zero drop) against the host restatement, and the
full load step load_matrix_market -> CSR -> frpcat against the oracle."""
import numpy as np
import pytest

from metrics import SIGMA_TOL, SUBSPACE_TOL, sigma_rel, subspace_dist

pytestmark = pytest.mark.gpu


def _csr_equal(A, B):
    return (A.rows() == B.rows() and A.cols() == B.cols() and np.array_equal(A.rowPtr(), B.rowPtr())
            and np.array_equal(A.colIdx(), B.colIdx()) and np.array_equal(A.values(), B.values()))


@pytest.mark.parametrize("rows,cols,n,seed", [(50, 40, 300, 0), (1000, 3, 5000, 1), (3, 1000, 5000, 2),
                                              (200000, 50000, 2000000, 3)])
def test_device_from_triplets_matches_host(fb, ctx, rows, cols, n, seed):
    """At most two entries per coordinate (sums are then order-independent):
    bitwise equal to the host from_triplets, including exact-zero drops."""
    rng = np.random.default_rng(seed)
    r = rng.integers(0, rows, n)
    c = rng.integers(0, cols, n)
    v = rng.standard_normal(n)
    key = r * cols + c
    _, first = np.unique(key, return_index=True)
    r, c, v = r[first], c[first], v[first]           # unique coordinates
    k = r.size // 3
    r = np.concatenate([r, r[:k]])                     # one duplicate for a third of them
    c = np.concatenate([c, c[:k]])
    v = np.concatenate([v, np.where(np.arange(k) % 2 == 0, -v[:k], rng.standard_normal(k))])  # half cancel
    perm = rng.permutation(r.size)
    r, c, v = r[perm], c[perm], v[perm]
    H = fb.SparseMatrixCsr.from_triplets(rows, cols, (r, c, v))
    D = fb.SparseMatrixCsr.from_triplets(rows, cols, (r, c, v), device=True)
    assert _csr_equal(H, D)
    assert H.nonZeros() < r.size - k // 3  # cancelled pairs dropped


def test_device_from_triplets_many_duplicates(fb, ctx):
    """Three or more entries per coordinate: same structure, sums equal up to
    the summation order (the reference's std::sort is not stable)."""
    rng = np.random.default_rng(5)
    r = rng.integers(0, 30, 20000)
    c = rng.integers(0, 20, 20000)
    v = rng.standard_normal(20000)
    H = fb.SparseMatrixCsr.from_triplets(30, 20, (r, c, v))
    D = fb.SparseMatrixCsr.from_triplets(30, 20, (r, c, v), device=True)
    assert np.array_equal(H.rowPtr(), D.rowPtr()) and np.array_equal(H.colIdx(), D.colIdx())
    assert np.allclose(H.values(), D.values(), rtol=1e-12, atol=1e-12)


def test_device_from_triplets_edges(fb, ctx):
    E = fb.SparseMatrixCsr.from_triplets(4, 5, ([], [], []), device=True)
    assert E.nonZeros() == 0 and np.array_equal(E.rowPtr(), np.zeros(5))
    Z = fb.SparseMatrixCsr.from_triplets(0, 0, ([], [], []), device=True)
    assert Z.rows() == 0 and Z.nonZeros() == 0
    one = fb.SparseMatrixCsr.from_triplets(3, 3, ([2, 2], [1, 1], [1.5, -1.5]), device=True)
    assert one.nonZeros() == 0 and np.array_equal(one.rowPtr(), [0, 0, 0, 0])
    with pytest.raises(ValueError, match="from_triplets: entry out of bounds"):
        fb.SparseMatrixCsr.from_triplets(3, 3, ([0, 3], [0, 0], [1.0, 1.0]), device=True)
    with pytest.raises(ValueError, match="from_triplets: entry out of bounds"):
        fb.SparseMatrixCsr.from_triplets(3, 3, ([0], [-1], [1.0]), device=True)


@pytest.mark.parametrize("symmetric", [False, True])
def test_load_matrix_market_then_frpcat(fb, orc, tmp_path, symmetric):
    """The whole load step: parse (host) + from_triplets (device) gives the
    CSR the reference's load_matrix_market gives (oracle parse + from_triplets),
    and frpcat on it matches the oracle."""
    rng = np.random.default_rng(9 + symmetric)
    n = 3000
    m = n if symmetric else 5000
    nnz = 60000
    i = rng.integers(1, m + 1, nnz)
    j = rng.integers(1, n + 1, nnz)
    if symmetric:
        i, j = np.maximum(i, j), np.minimum(i, j)
    v = rng.standard_normal(nnz)
    p = tmp_path / "m.mtx"
    head = "%%MatrixMarket matrix coordinate real " + ("symmetric" if symmetric else "general")
    p.write_text(head + f"\n{m} {n} {nnz}\n" + "\n".join(f"{a} {b} {float(x)!r}" for a, b, x in zip(i, j, v)) + "\n")
    A = fb.load_matrix_market(str(p))
    rows, cols, r, c, vv = orc.read_matrix_market(str(p))
    oA = orc.Csr.from_triplets(rows, cols, list(zip(r.tolist(), c.tolist(), vv.tolist())))
    rp, ci, va = oA.arrays()
    assert np.array_equal(A.rowPtr(), rp) and np.array_equal(A.colIdx(), ci)
    assert np.allclose(A.values(), va, rtol=1e-13, atol=0)  # >= 3 duplicates: order of the sum
    res = fb.frpcat(A, fb.PcaConfig(k=10, oversample=10, passes=4, seed=0))
    o = orc.pca(orc.Csr.create(rows, cols, A.rowPtr(), A.colIdx(), A.values()), orc.FRPCAT, 10, 10, 4, seed=0)
    assert sigma_rel(res.S, o["S"]) <= SIGMA_TOL
    assert subspace_dist(o["U"], res.U) <= SUBSPACE_TOL and subspace_dist(o["V"], res.V) <= SUBSPACE_TOL


def test_write_load_round_trip(fb, orc, tmp_path):
    oA = orc.Csr.random_sparse(700, 500, 0.02, 4)
    A = fb.SparseMatrixCsr(700, 500, *oA.arrays())
    p = tmp_path / "rt.mtx"
    fb.write_matrix_market(str(p), A)
    assert _csr_equal(fb.load_matrix_market(str(p)), A)
