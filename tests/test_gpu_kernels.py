"""GPU parity of the hot-path kernels against the CPU oracle, through the C ABI
(paper_1810_06825_b200 -> libfrpca_b200.so). Mirrors the hot-path assertions of
proj/tests/test_sparse.cpp and test_dense_kernels.cpp, plus SURVEY §8c's
SpMM bar: Frobenius-relative error <= 1e-12 against the oracle on identical
inputs (FMA vs separate mul/add is the only difference in a row's sum)."""
import numpy as np
import pytest

from metrics import SPMM_TOL, orth, orthonormality, projector_gap_dense, rel_fro, sigma_rel, subspace_dist

pytestmark = pytest.mark.gpu


def to_fb(fb, oA):
    rp, ci, va = oA.arrays()
    return fb.SparseMatrixCsr(oA.rows, oA.cols, rp, ci, va)


def powerlaw_csr(orc, m, n, nnz_target, seed, a_row=1.6, a_col=1.1):
    """Small power-law matrix (long rows and hot columns) for load-balance paths."""
    rng = np.random.default_rng(seed)
    deg = np.minimum(rng.zipf(a_row, m), n)
    deg = np.maximum(1, (deg * nnz_target / deg.sum()).astype(np.int64))
    deg = np.minimum(deg, n)
    rows, cols = [], []
    perm = rng.permutation(n)
    for i, d in enumerate(deg):
        c = np.unique(np.minimum(rng.zipf(a_col, 2 * d + 8), n) - 1)
        c = perm[c[:d]]
        rows.append(np.full(c.size, i))
        cols.append(np.sort(c))
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = rng.standard_normal(r.size)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    return orc.Csr.create(m, n, rp, c, v)

# ------------------------------------------------------------------ SpMM


def test_spmm_identity_and_hand(fb, ctx):  # test_sparse.cpp:46-59
    I = fb.SparseMatrixCsr.from_triplets(3, 3, [(i, i, 1.0) for i in range(3)])
    X = np.random.default_rng(0).standard_normal((3, 2))
    assert np.array_equal(fb.spmm(I, X), X)
    D = fb.SparseMatrixCsr.from_triplets(2, 2, [(0, 0, 2.0), (1, 1, 3.0)])
    Y = fb.spmm(D, np.ones((2, 1)))
    assert Y[0, 0] == 2.0 and Y[1, 0] == 3.0


def test_spmm_transpose_hand(fb, ctx):  # test_sparse.cpp:68-81
    I = fb.SparseMatrixCsr.from_triplets(4, 4, [(i, i, 1.0) for i in range(4)])
    Y = np.random.default_rng(1).standard_normal((4, 3))
    assert np.array_equal(fb.spmm_transpose(I, Y), Y)
    A = fb.SparseMatrixCsr.from_triplets(2, 3, [(0, 0, 1.0), (0, 2, 2.0), (1, 1, 3.0)])
    z = fb.spmm_transpose(A, np.ones((2, 1)))
    assert z.ravel().tolist() == [1.0, 3.0, 2.0]


@pytest.mark.parametrize("ncols", [1, 3, 7, 40, 64, 150, 200, 257, 300])
def test_spmm_vs_oracle_widths(fb, orc, ncols):
    oA = orc.Csr.random_sparse(120, 90, 0.08, 7 + ncols)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(90, ncols, 3)
    Y = orc.gaussian_matrix(120, ncols, 4)
    assert rel_fro(fb.spmm(A, X), orc.spmm(oA, X)) <= SPMM_TOL
    assert rel_fro(fb.spmm_transpose(A, Y), orc.spmm_transpose(oA, Y)) <= SPMM_TOL


@pytest.mark.parametrize("seed", range(4))
def test_spmm_powerlaw_long_rows(fb, orc, seed):
    """Power-law rows/columns: exercises the chunked long-row path and the
    fixed-order partial combine on both A and the transposed CSR."""
    oA = powerlaw_csr(orc, 3000, 2000, 120000, seed)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(2000, 200, seed)
    Y = orc.gaussian_matrix(3000, 200, seed + 1)
    assert rel_fro(fb.spmm(A, X), orc.spmm(oA, X)) <= SPMM_TOL
    assert rel_fro(fb.spmm_transpose(A, Y), orc.spmm_transpose(oA, Y)) <= SPMM_TOL


def test_spmm_empty_rows_and_matrix(fb, orc):
    A = fb.SparseMatrixCsr.from_triplets(5, 4, [(1, 2, 3.0)])
    X = np.ones((4, 6))
    Y = fb.spmm(A, X)
    assert Y.shape == (5, 6) and np.array_equal(Y[1], np.full(6, 3.0)) and not Y[[0, 2, 3, 4]].any()
    Z = fb.SparseMatrixCsr.from_triplets(6, 6, [])
    assert not fb.spmm(Z, np.ones((6, 2))).any()
    assert not fb.spmm_transpose(Z, np.ones((6, 2))).any()


@pytest.mark.parametrize("seed", range(8))
def test_transpose_matches_oracle(fb, orc, seed):  # test_sparse.cpp:90-100
    oA = orc.Csr.random_sparse(30 + 3 * seed, 25 + 2 * seed, 0.15, seed + 100)
    T = fb.transpose(to_fb(fb, oA))
    rp, ci, va = oA.transpose().arrays()
    assert np.array_equal(T.rowPtr(), rp) and np.array_equal(T.colIdx(), ci) and np.array_equal(T.values(), va)


def test_spmm_transpose_equals_spmm_on_transpose(fb, orc):
    """A^T*Y from the load-time transposed CSR == spmm on transpose(A): the
    same gather kernel over the same work list, so bitwise equal."""
    oA = powerlaw_csr(orc, 2000, 1500, 60000, 5)
    A = to_fb(fb, oA)
    At = fb.transpose(A)
    Y = orc.gaussian_matrix(2000, 40, 9)
    assert np.array_equal(fb.spmm_transpose(A, Y), fb.spmm(At, Y))


@pytest.mark.parametrize("ncols", [2, 3])
def test_spmm_tall_output_layout(fb, ncols):
    """A 5M-row output goes back to the host's column-major layout through
    the tiled device transpose: more than 65535 row tiles, which the kernel
    loops over (grid.y limit)."""
    m, n = 5_000_000, 10
    rp = np.arange(m + 1, dtype=np.int64)
    ci = np.arange(m, dtype=np.int64) % n
    va = np.ones(m)
    A = fb.SparseMatrixCsr(m, n, rp, ci, va)
    X = np.arange(n * ncols, dtype=np.float64).reshape(n, ncols) + 0.5
    Y = fb.spmm(A, X)
    assert np.array_equal(Y, X[ci])


@pytest.fixture
def panels(monkeypatch):
    """Forces the panelled A^T*Y (csr.cu ensure_panels) at test sizes: panels
    of a few rows of Y instead of tens of MB."""
    def force(panel_kb=100.0, part_gb=None):
        monkeypatch.setenv("FRPCA_PANEL_MIN_MB", "0")
        monkeypatch.setenv("FRPCA_PANEL_MB", str(panel_kb / 1024.0))
        if part_gb is not None:
            monkeypatch.setenv("FRPCA_PANEL_PART_GB", str(part_gb))
    return force


@pytest.mark.parametrize("ncols", [2, 40, 150, 200, 300])
@pytest.mark.parametrize("seed", range(2))
def test_spmm_transpose_panelled(fb, orc, panels, ncols, seed):
    """Panel-major chunks of the hot rows + fixed-order combine, cold rows
    through their own list: parity with the oracle, deterministic."""
    panels()
    oA = powerlaw_csr(orc, 3000, 2000, 120000, seed)
    A = to_fb(fb, oA)
    Y = orc.gaussian_matrix(3000, ncols, seed + 1)
    Z = fb.spmm_transpose(A, Y)
    assert rel_fro(Z, orc.spmm_transpose(oA, Y)) <= SPMM_TOL
    assert np.array_equal(Z, fb.spmm_transpose(A, Y))


@pytest.mark.parametrize("dynamic", ["0", "1", "2"])
@pytest.mark.parametrize("ncols", [40, 200, 300])
def test_spmm_transpose_cold_concurrent(fb, orc, panels, monkeypatch, ncols, dynamic):
    """Cold rows on a second stream beside the panel chunks
    (FRPCA_COLD_CONCURRENT, own partial slots) and items taken from a global
    counter (FRPCA_SPMM_DYNAMIC): bitwise equal to the serial, statically
    strided order, and to themselves across calls."""
    panels()
    oA = powerlaw_csr(orc, 3000, 2000, 120000, 4)
    A = to_fb(fb, oA)
    Y = orc.gaussian_matrix(3000, ncols, 8)
    Z0 = fb.spmm_transpose(A, Y)
    monkeypatch.setenv("FRPCA_SPMM_DYNAMIC", dynamic)
    assert np.array_equal(Z0, fb.spmm_transpose(A, Y))
    monkeypatch.setenv("FRPCA_COLD_CONCURRENT", "1")
    Z1 = fb.spmm_transpose(A, Y)
    assert np.array_equal(Z0, Z1)
    assert np.array_equal(Z1, fb.spmm_transpose(A, Y))
    assert rel_fro(Z1, orc.spmm_transpose(oA, Y)) <= SPMM_TOL


@pytest.mark.parametrize("ncols", [1, 40, 200, 256, 300])
def test_spmm_dynamic_items(fb, orc, monkeypatch, ncols):
    """A*X with work items from a global counter: bitwise equal to the
    static stride (the item -> warp assignment does not enter the sums)."""
    oA = powerlaw_csr(orc, 4000, 2500, 150000, 12)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(2500, ncols, 3)
    Y0 = fb.spmm(A, X)
    monkeypatch.setenv("FRPCA_SPMM_DYNAMIC", "1")
    Y1 = fb.spmm(A, X)
    assert np.array_equal(Y0, Y1)
    assert rel_fro(Y1, orc.spmm(oA, X)) <= SPMM_TOL


@pytest.mark.parametrize("panel_kb,part_gb", [(3.0, None), (40.0, 1e-4), (1000.0, None)])
def test_spmm_transpose_panel_sizes(fb, orc, panels, panel_kb, part_gb):
    """Tiny panels (many segments per row), a partial budget that forces the
    hot threshold up, and panels larger than Y (one panel)."""
    panels(panel_kb, part_gb)
    oA = powerlaw_csr(orc, 2500, 800, 90000, 3)
    A = to_fb(fb, oA)
    Y = orc.gaussian_matrix(2500, 64, 5)
    assert rel_fro(fb.spmm_transpose(A, Y), orc.spmm_transpose(oA, Y)) <= SPMM_TOL


@pytest.mark.parametrize("ncols", [1, 40, 200, 150, 64])
def test_spmm_l2_hints(fb, orc, monkeypatch, ncols):
    """A*X with sign-bit L2 hints on the popular columns (csr.cu
    ensure_hint, spmm.cu MODE_HINT) forced at test size: only the cache
    policy of the gathers changes, so results are bitwise equal to the plain
    kernel; re-encoding across widths and the masked id download."""
    oA = powerlaw_csr(orc, 3000, 2000, 120000, 11)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(2000, ncols, 4)
    monkeypatch.setenv("FRPCA_HINT_MB", "0")
    Y0 = fb.spmm(A, X)
    monkeypatch.setenv("FRPCA_HINT_MB", "0.02")
    Y1 = fb.spmm(A, X)
    assert np.array_equal(Y0, Y1)
    assert rel_fro(Y1, orc.spmm(oA, X)) <= SPMM_TOL
    X2 = orc.gaussian_matrix(2000, 7, 5)
    assert rel_fro(fb.spmm(A, X2), orc.spmm(oA, X2)) <= SPMM_TOL


@pytest.mark.parametrize("ncols", [2, 8, 40, 150, 200, 256, 300])
@pytest.mark.parametrize("hint", ["0", "0.02"])
def test_spmm_ring_equals_register_gathers(fb, orc, monkeypatch, ncols, hint):
    """A*X and A^T*Y with the X rows moved into per-warp shared-memory rings by
    bulk copies (spmm.cu k_spmm_ring) are bitwise equal to the register-gather
    kernel: per output entry the same FMA chain in CSR order. Power-law rows
    (chunked long rows + combine), empty rows, L2-hinted ids, widths past 256
    (two column slices)."""
    oA = powerlaw_csr(orc, 5000, 3000, 200000, 17)
    trip_extra = None
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(3000, ncols, 9)
    Y = orc.gaussian_matrix(5000, ncols, 10)
    monkeypatch.setenv("FRPCA_HINT_MB", hint)
    monkeypatch.setenv("FRPCA_SPMM_RING", "0")
    Y0, Z0 = fb.spmm(A, X), fb.spmm_transpose(A, Y)
    monkeypatch.setenv("FRPCA_SPMM_RING", "1")
    Y1, Z1 = fb.spmm(A, X), fb.spmm_transpose(A, Y)
    assert np.array_equal(Y0, Y1) and np.array_equal(Z0, Z1)
    assert rel_fro(Y1, orc.spmm(oA, X)) <= SPMM_TOL
    _ = trip_extra


def test_spmm_ring_empty_rows_and_single_nonzeros(fb, orc, monkeypatch):
    trip = [(i, (7 * i) % 50, 1.0 + i) for i in range(0, 400, 3)] + [(5, j, -0.5) for j in range(50)]
    A = fb.SparseMatrixCsr.from_triplets(400, 50, trip)
    X = orc.gaussian_matrix(50, 64, 3)
    monkeypatch.setenv("FRPCA_SPMM_RING", "0")
    Y0 = fb.spmm(A, X)
    monkeypatch.setenv("FRPCA_SPMM_RING", "1")
    Y1 = fb.spmm(A, X)
    assert np.array_equal(Y0, Y1)
    assert np.array_equal(Y1, A.toDense() @ X) or rel_fro(Y1, A.toDense() @ X) <= 1e-15


@pytest.mark.parametrize("ncols", [1, 8, 32, 37, 150, 200, 300])
@pytest.mark.parametrize("sx_kb", ["0", "2", "160"])
def test_spmm_sliced_shared_hot_rows(fb, orc, monkeypatch, ncols, sx_kb):
    """The sliced A*X (spmm.cu k_spmm_sx: 32-column slices, the most popular
    columns' X rows from shared memory, ids re-encoded kColHot | rank) is
    bitwise equal to the full-width kernel: per entry the same FMA chain in
    CSR order. No hot rows, a few (2 KB: 8 rows) and the default budget;
    power-law rows long enough to be chunked (partials + combine); switching
    encodings back and forth; the decoded transpose download."""
    oA = powerlaw_csr(orc, 5000, 3000, 200000, 13)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(3000, ncols, 6)
    monkeypatch.setenv("FRPCA_HINT_MB", "0")
    monkeypatch.setenv("FRPCA_SPMM_SX", "0")
    Y0 = fb.spmm(A, X)
    monkeypatch.setenv("FRPCA_SPMM_SX", "1")
    monkeypatch.setenv("FRPCA_SX_KB", sx_kb)
    Y1 = fb.spmm(A, X)
    assert np.array_equal(Y0, Y1)
    assert rel_fro(Y1, orc.spmm(oA, X)) <= SPMM_TOL
    monkeypatch.setenv("FRPCA_SPMM_SX", "0")
    monkeypatch.setenv("FRPCA_HINT_MB", "0.02")  # hint encoding after the shared-memory one
    assert np.array_equal(fb.spmm(A, X), Y0)
    # A^T*Y reads the transposed CSR, which no encoding touches
    Yt = orc.gaussian_matrix(5000, ncols, 7)
    assert rel_fro(fb.spmm_transpose(A, Yt), orc.spmm_transpose(oA, Yt)) <= SPMM_TOL


def test_spmm_transpose_panelled_empty_rows(fb, orc, panels):
    """Columns of A with no entries (empty rows of A^T) next to hot ones."""
    panels(1.0)
    trip = [(i, 0, 1.0 + i) for i in range(400)] + [(i, 5, -0.5) for i in range(0, 400, 3)]
    A = fb.SparseMatrixCsr.from_triplets(400, 9, trip)
    Y = orc.gaussian_matrix(400, 10, 2)
    Z = fb.spmm_transpose(A, Y)
    ref = np.zeros((9, 10))
    for i, c, v in trip:
        ref[c] += v * Y[i]
    assert rel_fro(Z, ref) <= SPMM_TOL and not Z[[1, 2, 3, 4, 6, 7, 8]].any()


def test_pass_counter(fb, orc):  # test_sparse.cpp:111-118
    A = to_fb(fb, orc.Csr.random_sparse(20, 20, 0.2, 1))
    X = np.ones((20, 3))
    fb.spmm(A, X)
    A.resetPassCount()
    fb.spmm(A, X)
    fb.spmm_transpose(A, X)
    assert A.passCount() == 2


@pytest.mark.parametrize("bad,msg", [
    (dict(row_ptr=[0, 2, 1], col_idx=[0, 1], values=[1.0, 1.0]), "row_ptr"),
    (dict(row_ptr=[0, 1, 2], col_idx=[0, 5], values=[1.0, 1.0]), "out of range"),
])
def test_device_validation_messages(fb, bad, msg):
    """The device upload re-validates (sparse_matrix.hpp:125-142) even when the
    host object was built without checks."""
    A = fb.SparseMatrixCsr(2, 2, validate=False, **bad)
    with pytest.raises(ValueError, match=msg):
        fb.spmm(A, np.ones((2, 1)))


def test_spmm_deterministic(fb, orc):
    oA = powerlaw_csr(orc, 4000, 3000, 200000, 11)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(3000, 200, 2)
    a = fb.spmm(A, X)
    b = fb.spmm(A, X)
    c = fb.spmm_transpose(A, orc.gaussian_matrix(4000, 200, 3))
    d = fb.spmm_transpose(A, orc.gaussian_matrix(4000, 200, 3))
    assert np.array_equal(a, b) and np.array_equal(c, d)

# ------------------------------------------------------------------ LU


def test_lu_identity(fb, ctx):  # test_dense_kernels.cpp:71-75
    M = np.eye(5, 3)
    assert np.abs(fb.lu_basis(M) - M).max() == 0.0


def test_lu_pivoting_range(fb, ctx):  # test_dense_kernels.cpp:77-82
    M = np.array([[0.0, 1.0], [1.0, 0.0], [0.0, 0.0]])
    assert projector_gap_dense(orth(fb.lu_basis(M)), orth(M)) < 1e-14


def test_lu_unit_lower_factor(fb, orc):  # test_dense_kernels.cpp:90-102
    X = fb.lu_basis(orc.gaussian_matrix(20, 6, 9))
    assert abs(np.abs(X).max() - 1.0) < 1e-15
    for j in range(X.shape[1]):
        assert (X[:, j] == 1.0).sum() >= 1


def test_lu_rank_deficiency(fb):  # test_dense_kernels.cpp:104-109
    c0 = np.linspace(1, 4, 4)
    with pytest.raises(fb.NumericalError):
        fb.lu_basis(np.stack([c0, -3.0 * c0], axis=1))


@pytest.mark.parametrize("m,l", [(40, 8), (300, 70), (5000, 150), (20000, 200), (1000, 33)])
def test_lu_vs_oracle(fb, orc, m, l):
    """Same pivots (first max, ties to lowest position) -> the same P^T L up to
    rounding of the updates."""
    M = orc.gaussian_matrix(m, l, m + l)
    X = fb.lu_basis(M)
    Xo = orc.lu_basis(M)
    assert np.array_equal(X == 1.0, Xo == 1.0)          # same pivot rows
    assert np.array_equal(X == 0.0, Xo == 0.0)
    assert np.abs(X - Xo).max() < 1e-9


# ------------------------------------------------------------------ eig_svd


def test_eig_svd_hand(fb):  # test_dense_kernels.cpp:147-157
    _, S, _ = fb.eig_svd(np.eye(3))
    assert np.abs(S - 1).max() < 1e-14
    A = np.zeros((4, 2))
    A[0, 0], A[1, 1] = 2.0, 3.0
    _, S, _ = fb.eig_svd(A)
    assert abs(S[0] - 2) < 1e-12 and abs(S[1] - 3) < 1e-12


def test_eig_svd_vs_oracle(fb, orc):  # test_dense_kernels.cpp:159-165
    A = orc.gaussian_matrix(200, 30, 17)
    U, S, V = fb.eig_svd(A)
    _, So, _ = orc.oracle_svd(A)
    assert np.max(np.abs(S[::-1] - So) / So) < 1e-10
    assert np.linalg.norm(A - (U * S) @ V.T) / np.linalg.norm(A) < 1e-10


def test_eig_svd_rank_deficient(fb, orc):  # test_dense_kernels.cpp:167-172
    A = orc.gaussian_matrix(5, 3, 1)
    A[:, 2] = A[:, 0] + A[:, 1]
    with pytest.raises(fb.NumericalError):
        fb.eig_svd(A)


@pytest.mark.parametrize("m,n", [(50, 7), (3000, 64), (100000, 200), (20000, 150)])
def test_eig_svd_tall(fb, orc, m, n):
    A = orc.gaussian_matrix(m, n, m + n)
    U, S, V = fb.eig_svd(A)
    Uo, So, Vo = orc.eig_svd(A)
    assert np.max(np.abs(S - So) / So) < 1e-12
    assert orthonormality(U) < 1e-10 and orthonormality(V) < 1e-12
    assert subspace_dist(Uo, U) < 1e-10


@pytest.mark.parametrize("seed", range(0, 100, 9))
def test_eig_svd_property(fb, orc, seed):  # test_dense_kernels.cpp:174-186
    n = 2 + seed % 12
    m = n + (seed * 7) % 40
    A = orc.gaussian_matrix(m, n, 1000 + seed)
    U, S, V = fb.eig_svd(A)
    assert orthonormality(U) < 1e-10 and orthonormality(V) < 1e-12
    assert np.all(np.diff(S) >= 0) and S[0] >= 0
    assert np.linalg.norm(A - (U * S) @ V.T) / np.linalg.norm(A) < 1e-10


def _with_spectrum(orc, m, s, seed):
    """m x n matrix with singular values s (any order) and random singular vectors."""
    n = s.size
    Q1, _ = np.linalg.qr(orc.gaussian_matrix(m, n, seed))
    Q2, _ = np.linalg.qr(orc.gaussian_matrix(n, n, seed + 1))
    return (Q1 * s) @ Q2.T


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 9, 16, 17, 31, 33, 64, 100, 150, 200, 231, 232, 233, 300])
def test_eig_solver_sizes(fb, orc, monkeypatch, n):
    """The library's l <= 232 eigensolver (syev.cu: tridiagonalisation, divide
    and conquer, back-transformation) at every leaf/merge shape; larger n goes
    to cuSOLVER. FRPCA_EIG=strict turns a silent fallback into a failure."""
    monkeypatch.setenv("FRPCA_EIG", "strict")
    A = orc.gaussian_matrix(3 * n + 5, n, 40 + n)
    U, S, V = fb.eig_svd(A)
    Sn = np.linalg.svd(A, compute_uv=False)[::-1]
    assert np.max(np.abs(S - Sn) / Sn) < 1e-12
    assert orthonormality(V) < 1e-12 and orthonormality(U) < 1e-10
    assert np.linalg.norm(A - (U * S) @ V.T) / np.linalg.norm(A) < 1e-12


@pytest.mark.parametrize("kind", ["repeated", "clusters", "graded", "two_values", "near_rank"])
@pytest.mark.parametrize("n", [40, 200])
def test_eig_solver_hard_spectra(fb, orc, monkeypatch, kind, n):
    """Repeated and clustered eigenvalues exercise the deflation of the merges
    (both rotation and small-z deflation); a graded spectrum over 6 decades
    (12 in the Gram) the secular solver near its poles."""
    monkeypatch.setenv("FRPCA_EIG", "strict")
    rng = np.random.default_rng(n)
    if kind == "repeated":
        s = np.ones(n)
    elif kind == "clusters":
        s = np.repeat([1.0, 2.0, 3.0, 5.0], n // 4) * (1 + 1e-13 * rng.standard_normal(n))
    elif kind == "graded":
        s = 10.0 ** np.linspace(0, -6, n)
    elif kind == "two_values":
        s = np.where(np.arange(n) % 2 == 0, 1.0, 1e-3)
    else:
        s = np.concatenate([np.linspace(1, 2, n - 3), [1e-6, 2e-6, 3e-6]])
    A = _with_spectrum(orc, 4 * n, s, 7 + n)
    U, S, V = fb.eig_svd(A)
    Sn = np.sort(s)
    # eigenvalues of the Gram to ~eps*||B||: singular values to eps*smax^2/s
    tol = 1e-13 * (Sn[-1] ** 2) / Sn
    assert np.all(np.abs(S - Sn) <= np.maximum(tol, 1e-12 * Sn))
    assert orthonormality(V) < 1e-12
    top = Sn >= 0.1 * Sn[-1]
    assert np.linalg.norm(A - (U * S) @ V.T) / np.linalg.norm(A) < 1e-10
    assert orthonormality(U[:, top]) < 1e-10


@pytest.mark.parametrize("m,l", [(40, 8), (1000, 33), (4000, 40), (4000, 200), (20000, 200), (100000, 200),
                                 (130000, 150)])
def test_lu_smem_equals_global_kernel(fb, orc, monkeypatch, m, l):
    """The shared-memory-resident LU (rows fit one CTA per SM) performs the
    same operations in the same order as the global-panel kernel: bitwise
    equal results; sizes on both sides of the residency limit."""
    M = orc.gaussian_matrix(m, l, 3 * m + l)
    # rows scaled over 16 decades and 20% zero rows (pipeline-like Z)
    rng = np.random.default_rng(m + l)
    M2 = M * (10.0 ** rng.uniform(-8, 8, size=(m, 1)))
    M2[rng.choice(m, m // 5, replace=False)] = 0.0
    for X in (M, M2):
        monkeypatch.delenv("FRPCA_LU_GLOBAL", raising=False)
        X1 = fb.lu_basis(X)
        monkeypatch.setenv("FRPCA_LU_GLOBAL", "1")
        X2 = fb.lu_basis(X)
        assert np.array_equal(X1, X2)


@pytest.mark.parametrize("m,n", [(5000, 200), (100000, 200), (20000, 150), (9000, 96), (30000, 88)])
def test_gram3_equals_gram2(fb, orc, monkeypatch, m, n):
    """The register-blocked Gram (k_gram3) issues the same DMMAs per output
    tile in the same row order as k_gram2: eig_svd results are bitwise equal."""
    A = orc.gaussian_matrix(m, n, m + 3 * n)
    monkeypatch.delenv("FRPCA_GRAM2", raising=False)
    r1 = fb.eig_svd(A)
    monkeypatch.setenv("FRPCA_GRAM2", "1")
    r2 = fb.eig_svd(A)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)



@pytest.mark.parametrize("m,n", [(4096, 80), (5000, 120), (70001, 150), (123457, 200), (4100, 200)])
def test_gram4_bulk_copies_equal_gram3(fb, orc, monkeypatch, m, n):
    """The Gram fed by 1-D bulk copies and mbarriers (k_gram4) issues the same
    DMMAs per tile over the same 4-row groups as k_gram3 (zero-filled tail
    rows included): bitwise equal eig_svd results; CTA row ranges that are
    not whole stages, odd row counts and widths with zero padding columns."""
    A = orc.gaussian_matrix(m, n, m + 7 * n)
    monkeypatch.setenv("FRPCA_GRAM3", "1")
    r1 = fb.eig_svd(A)
    monkeypatch.delenv("FRPCA_GRAM3")
    r2 = fb.eig_svd(A)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("kernel", ["tma", "cpasync"])
def test_rescale_gemm_every_width(fb, orc, monkeypatch, kernel):
    """eig_svd of a 4100-row panel at every width 1..232: the persistent
    rescale GEMM (r >= 4096) splits the output columns into chunks of <= 104
    and each chunk's 8-column tiles over one or two warp groups of <= 7 tiles.
    Found by the randomised sweep: a chunk of exactly 8 tiles (57-64 columns,
    i.e. l or k in 57..64 and 161..168) went to one group and lost its last
    tile."""
    if kernel == "cpasync":
        monkeypatch.setenv("FRPCA_GEMM_CPASYNC", "1")
    G = orc.gaussian_matrix(4100, 232, 77)
    for n in range(1, 233):
        A = np.ascontiguousarray(G[:, :n])
        U, S, V = fb.eig_svd(A)
        assert np.abs((U * S) @ V.T - A).max() <= 1e-10, n
        assert orthonormality(U) <= 1e-10, n


@pytest.mark.parametrize("k,s", [(57, 0), (60, 10), (64, 0), (50, 10), (63, 100), (100, 62)])
def test_run_outputs_at_eight_tile_widths(fb, orc, k, s):
    # the column-major k-of-l outputs of a run (U: 6000 rows) at those widths
    oA = powerlaw_csr(orc, 6000, 400, 150000, 3)
    A = to_fb(fb, oA)
    r = fb.frpcat(A, fb.PcaConfig(k=k, oversample=s, passes=3, seed=2))
    o = orc.pca(oA, orc.FRPCAT, k, s, seed=2, passes=3)
    assert sigma_rel(r.S, o["S"]) <= 1e-10
    assert subspace_dist(o["U"], r.U) <= 1e-8 and subspace_dist(o["V"], r.V) <= 1e-8
    assert np.abs(np.abs(np.sum(r.U * o["U"], axis=0)) - 1).max() <= 1e-8


@pytest.mark.parametrize("m,n", [(4096, 16), (5000, 40), (70001, 150), (123457, 200), (4100, 208)])
def test_gemm_tma_equals_cp_async(fb, orc, monkeypatch, m, n):
    """The rescale GEMM fed by 2-D TMA tiles (k_gemm_tma: 128-byte swizzle,
    zero fill past the last row and column) issues the same DMMAs per output
    tile in the same k order as the cp.async kernel: bitwise equal eig_svd
    U (row-major output) and frpcat U/V (column-major outputs, k of l
    columns)."""
    A = orc.gaussian_matrix(m, n, m + 5 * n)
    monkeypatch.setenv("FRPCA_GEMM_CPASYNC", "1")
    r1 = fb.eig_svd(A)
    monkeypatch.delenv("FRPCA_GEMM_CPASYNC")
    r2 = fb.eig_svd(A)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


def test_gemm_tma_outputs_of_a_run(fb, orc, monkeypatch):
    oA = powerlaw_csr(orc, 9000, 1500, 150000, 21)
    A = to_fb(fb, oA)
    c = fb.PcaConfig(k=60, oversample=44, passes=3, seed=1)
    monkeypatch.setenv("FRPCA_GEMM_CPASYNC", "1")
    r1 = fb.frpcat(A, c)
    monkeypatch.delenv("FRPCA_GEMM_CPASYNC")
    r2 = fb.frpcat(A, c)
    assert np.array_equal(r1.U, r2.U) and np.array_equal(r1.V, r2.V) and np.array_equal(r1.S, r2.S)


@pytest.mark.parametrize("n", [3, 4, 5, 33, 64, 150, 200, 213, 214, 232])
def test_sytrd_fused_vs_unfused(fb, orc, monkeypatch, n):
    """The fused tridiagonalisation (rank-2 update of step j and symmetric
    product of step j + 1 in one pass) against the two-pass kernel: same
    spectrum to ~eps ||B||, both within the solver's accuracy bar."""
    monkeypatch.setenv("FRPCA_EIG", "strict")
    A = orc.gaussian_matrix(3 * n + 7, n, 11 * n)
    monkeypatch.delenv("FRPCA_SYTRD_UNFUSED", raising=False)
    U1, S1, V1 = fb.eig_svd(A)
    monkeypatch.setenv("FRPCA_SYTRD_UNFUSED", "1")
    U2, S2, V2 = fb.eig_svd(A)
    Sn = np.linalg.svd(A, compute_uv=False)[::-1]
    for U, S, V in ((U1, S1, V1), (U2, S2, V2)):
        assert np.max(np.abs(S - Sn) / Sn) < 1e-12
        assert orthonormality(V) < 1e-12 and orthonormality(U) < 1e-10
        assert np.linalg.norm(A - (U * S) @ V.T) / np.linalg.norm(A) < 1e-12
    assert np.max(np.abs(S1 - S2) / S2) < 1e-13


@pytest.mark.parametrize("ncols", [2, 40, 64, 150, 200, 256])
def test_combine2_bitwise(fb, orc, panels, monkeypatch, ncols):
    """The double2 partial combine (k_combine2) keeps k_combine's partition
    and summation order: bitwise equal A*X (chunked long rows) and panelled
    A^T*Y."""
    panels()
    oA = powerlaw_csr(orc, 3000, 2000, 120000, 21)
    A = to_fb(fb, oA)
    X = orc.gaussian_matrix(2000, ncols, 1)
    Y = orc.gaussian_matrix(3000, ncols, 2)
    monkeypatch.setenv("FRPCA_COMBINE1", "2")  # k_combine2 regardless of the partial count
    r1 = (fb.spmm(A, X), fb.spmm_transpose(A, Y))
    monkeypatch.setenv("FRPCA_COMBINE1", "1")
    r2 = (fb.spmm(A, X), fb.spmm_transpose(A, Y))
    for a, b in zip(r1, r2):
        assert np.array_equal(a, b)
    assert rel_fro(r1[1], orc.spmm_transpose(oA, Y)) <= SPMM_TOL


@pytest.mark.parametrize("m,l", [(1000, 33), (40000, 200), (100000, 200), (130000, 150), (200000, 200),
                                 (500000, 150)])
def test_lu_panel_width_bitwise(fb, orc, monkeypatch, m, l):
    """The global-panel LU at panel width 16 (used above ~262k rows to keep
    the panel copy L2-resident) and 32, and the shared-memory kernel (32):
    every element receives the same FMAs in the same order, so all agree
    bitwise, including scaled and zero rows."""
    M = orc.gaussian_matrix(m, l, 7 * m + l)
    rng = np.random.default_rng(m)
    M *= 10.0 ** rng.uniform(-6, 6, size=(m, 1))
    M[rng.choice(m, m // 7, replace=False)] = 0.0
    out = []
    for glob, nb, snb in ((False, None, None), (False, None, "32"), (True, "32", None), (True, "16", None),
                          (True, "8", None)):
        if glob:
            monkeypatch.setenv("FRPCA_LU_GLOBAL", "1")
        else:
            monkeypatch.delenv("FRPCA_LU_GLOBAL", raising=False)
        if nb:
            monkeypatch.setenv("FRPCA_LU_NB", nb)
        if snb:
            monkeypatch.setenv("FRPCA_LU_SMEM_NB", snb)
        else:
            monkeypatch.delenv("FRPCA_LU_SMEM_NB", raising=False)
        out.append(fb.lu_basis(M))
    for o in out[1:]:
        assert np.array_equal(out[0], o)


@pytest.mark.parametrize("m,n", [(5000, 200), (100000, 200), (20000, 150), (4130, 96)])
def test_gram_staging_depth_bitwise(fb, orc, monkeypatch, m, n):
    """k_gram3 with 32- or 64-row stages: the CTA row split is fixed at 32-row
    granularity, so the partials and the result are bitwise equal."""
    A = orc.gaussian_matrix(m, n, 3 * m + n)
    monkeypatch.setenv("FRPCA_GRAM_ROWS", "32")
    r1 = fb.eig_svd(A)
    monkeypatch.setenv("FRPCA_GRAM_ROWS", "64")
    r2 = fb.eig_svd(A)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)
