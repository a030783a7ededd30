"""SURVEY §8 row f4 on the B200: orth (dense_kernels.hpp:30-48) and the
baseline algorithms basic_rpca / basic_rpcat (randsvd.hpp:95-175), against the
oracle and against the reference's own tests (test_dense_kernels.cpp:38-69,
test_randsvd.cpp:55-69, :87-108, :140-180, :200-209, :253-262), including the
paper's Theorems 1/2: the fast algorithms equal the baselines for a shared
sketch."""
import numpy as np
import pytest

from metrics import SIGMA_TOL, SUBSPACE_TOL, orth as np_orth, orthonormality, projector_gap_dense, sigma_rel, \
    subspace_dist
from test_gpu_kernels import powerlaw_csr, to_fb

pytestmark = pytest.mark.gpu


def cfg(fb, k, s, q=2, p=0, seed=0):
    return fb.PcaConfig(k=k, oversample=s, passes=q, power=p, seed=seed)


def recon(r):
    return (r.U * r.S) @ r.V.T

# ------------------------------------------------------------------- orth


def test_orth_identity_single_column(fb, ctx):  # test_dense_kernels.cpp:38-43, :54-60
    Q = fb.orth(np.eye(5, 3))
    assert np.abs(Q.T @ Q - np.eye(3)).max() < 1e-14
    assert projector_gap_dense(Q, np.eye(5, 3)) < 1e-14
    q = fb.orth(np.array([[3.0], [4.0]]))
    assert abs(abs(q[0, 0]) - 0.6) < 1e-15 and abs(abs(q[1, 0]) - 0.8) < 1e-15


def test_orth_near_dependent(fb, ctx):  # test_dense_kernels.cpp:45-52
    M = np.array([[1.0, 1.0], [1.0, 1.0 + 1e-3], [0.0, 0.0]])
    Q = fb.orth(M)
    assert np.abs(Q.T @ Q - np.eye(2)).max() < 1e-13
    assert projector_gap_dense(Q, np_orth(M)) < 1e-10


def test_orth_rejects(fb, orc):  # test_dense_kernels.cpp:62-69
    M = np.zeros((4, 2))
    M[:, 0] = np.linspace(1.0, 4.0, 4)
    M[:, 1] = 2.0 * M[:, 0]
    with pytest.raises(fb.NumericalError, match="rank-deficient"):
        fb.orth(M)
    with pytest.raises(ValueError, match="must be tall"):
        fb.orth(orc.gaussian_matrix(2, 4, 1))
    with pytest.raises(fb.NumericalError):
        fb.orth(np.zeros((4, 2)))


@pytest.mark.parametrize("m,l", [(60, 7), (5000, 64), (100000, 200)])
def test_orth_vs_oracle(fb, orc, m, l):
    M = orc.gaussian_matrix(m, l, m + l)
    Q = fb.orth(M)
    assert orthonormality(Q) < 1e-12
    Qo = orc.orth(M)
    assert subspace_dist(Qo, Q) < 1e-12
    # same Householder sign convention as the reference: Q itself agrees
    assert np.abs(Q - Qo).max() < 1e-10


# the hand-written Householder kernel (csrc/orth.cu): panels of 16 columns,
# thread-per-column chunks of 256, one CTA per 64+ rows; shapes around every
# one of those boundaries, against the oracle entry by entry
@pytest.mark.parametrize("m,l", [(1, 1), (2, 1), (17, 16), (17, 17), (33, 32), (40, 31), (63, 1), (64, 48), (65, 33),
                                 (129, 100), (600, 257), (700, 300), (1000, 513), (9473, 40), (20000, 272),
                                 (400000, 64)])
def test_orth_shapes(fb, orc, m, l):
    M = orc.gaussian_matrix(m, l, 3 * m + l)
    Q = fb.orth(M)
    assert orthonormality(Q) < 1e-12
    assert np.abs(Q - orc.orth(M)).max() < 1e-10


def test_orth_deterministic_and_scaled(fb, orc):
    M = orc.gaussian_matrix(30000, 96, 5)
    Q1, Q2 = fb.orth(M), fb.orth(M)
    assert np.array_equal(Q1, Q2)  # fixed-order reductions
    # column scales over 8 decades (inside the reference's scale-dependent rank check)
    sc = np.logspace(-4, 4, 96)
    Qs = fb.orth(M * sc)
    assert orthonormality(Qs) < 1e-12
    assert np.abs(Qs - orc.orth(M * sc)).max() < 1e-10


def test_orth_zero_tail_column(fb, orc):
    # a column whose entries below the diagonal are exactly zero takes Eigen's
    # tau = 0 branch (beta = c0, no reflection), :makeHouseholderInPlace
    M = orc.gaussian_matrix(50, 4, 9)
    M[1:, 0] = 0.0
    Q = fb.orth(M)
    assert np.abs(Q - orc.orth(M)).max() < 1e-12
    M2 = np.zeros((6, 2))
    M2[0, 0] = -2.0
    M2[1, 1] = 3.0
    assert np.abs(fb.orth(M2) - orc.orth(M2)).max() == 0.0


def test_orth_rank_deficient_late_column(fb, orc):
    # dependence only shows in the last panel; the context stays usable
    M = orc.gaussian_matrix(3000, 40, 2)
    M[:, 37] = M[:, 3] - 2.0 * M[:, 20]
    with pytest.raises(fb.NumericalError, match="orth: numerically rank-deficient input"):
        fb.orth(M)
    G = orc.gaussian_matrix(3000, 40, 2)
    assert np.abs(fb.orth(G) - orc.orth(G)).max() < 1e-10

# --------------------------------------------------------------- baselines


@pytest.mark.parametrize("name", ["basic_rpca", "basic_rpcat"])
def test_basic_diag(fb, name):  # test_randsvd.cpp:55-69
    A = fb.SparseMatrixCsr.from_triplets(5, 5, [(i, i, float(v)) for i, v in enumerate([5, 4, 3, 2, 1])])
    r = getattr(fb, name)(A, cfg(fb, 2, 3, p=2))
    assert abs(r.S[0] - 5) < 1e-8 and abs(r.S[1] - 4) < 1e-8
    assert orthonormality(r.U) < 1e-10 and orthonormality(r.V) < 1e-10
    assert np.all(np.diff(r.S) <= 0)


def test_basic_exact_rank3(fb, orc):  # test_randsvd.cpp:87-96
    u = orc.gaussian_matrix(100, 3, 11)
    v = orc.gaussian_matrix(3, 80, 12)
    D = u @ v
    ii, jj = np.nonzero(D)
    A = fb.SparseMatrixCsr.from_triplets(100, 80, (ii, jj, D[ii, jj]))
    na = np.linalg.norm(D)
    for f in (fb.basic_rpca, fb.basic_rpcat):
        assert np.linalg.norm(D - recon(f(A, cfg(fb, 3, 0)))) < 1e-9 * na


def test_basic_zero_matrix(fb):  # test_randsvd.cpp:106-108
    with pytest.raises(fb.NumericalError):
        fb.basic_rpca(fb.SparseMatrixCsr.from_triplets(6, 6, []), cfg(fb, 2, 1, p=1))


@pytest.mark.parametrize("p", [0, 1, 2, 4])
def test_basic_pass_accounting(fb, orc, p):  # test_randsvd.cpp:200-209
    A = to_fb(fb, orc.Csr.random_sparse(50, 70, 0.3, 55))
    for f in (fb.basic_rpca, fb.basic_rpcat):
        st = fb.RunStats()
        f(A, cfg(fb, 4, 4, p=p), st)
        assert st.passes_over_matrix == 2 * p + 2


def test_basic_preconditions(fb, orc):  # test_randsvd.cpp:253-262
    A = to_fb(fb, orc.Csr.random_sparse(20, 30, 0.3, 1))
    with pytest.raises(ValueError, match="basic_rpca: power p must be >= 0"):
        fb.basic_rpca(A, cfg(fb, 2, 5, p=-1))
    with pytest.raises(ValueError, match="basic_rpcat: k \\+ oversample must be <= min"):
        fb.basic_rpcat(A, cfg(fb, 15, 10))


@pytest.mark.parametrize("name,algo", [("basic_rpca", 3), ("basic_rpcat", 4)])
@pytest.mark.parametrize("p", [0, 1, 3])
def test_basic_parity_random(fb, orc, name, algo, p):
    oA = orc.Csr.random_sparse(300, 200, 0.05, 7 + p)
    r = getattr(fb, name)(to_fb(fb, oA), cfg(fb, 10, 6, p=p, seed=3))
    o = orc.pca(oA, algo, 10, 6, 2, seed=3, power=p)
    assert sigma_rel(r.S, o["S"]) <= SIGMA_TOL
    assert subspace_dist(o["U"], r.U) <= SUBSPACE_TOL and subspace_dist(o["V"], r.V) <= SUBSPACE_TOL


@pytest.mark.parametrize("name,algo,shape", [("basic_rpca", 3, (3000, 30000)), ("basic_rpcat", 4, (20000, 4000))])
def test_basic_parity_powerlaw_l200(fb, orc, name, algo, shape):
    m, n = shape
    oA = powerlaw_csr(orc, m, n, 400000, 31, a_row=1.5, a_col=1.1)
    r = getattr(fb, name)(to_fb(fb, oA), cfg(fb, 100, 100, p=1))
    o = orc.pca(oA, algo, 100, 100, 2, power=1)
    assert sigma_rel(r.S, o["S"]) <= SIGMA_TOL
    assert subspace_dist(o["U"], r.U) <= SUBSPACE_TOL and subspace_dist(o["V"], r.V) <= SUBSPACE_TOL


@pytest.mark.parametrize("q", [4, 6, 10])
@pytest.mark.parametrize("fast,basic,shape,oseed", [("frpca", "basic_rpca", (80, 120), 42),
                                                   ("frpcat", "basic_rpcat", (120, 80), 43)])
def test_theorem_equivalence(fb, orc, q, fast, basic, shape, oseed):  # test_randsvd.cpp:140-172
    m, n = shape
    A = to_fb(fb, orc.Csr.random_sparse(m, n, 0.15, 77 if fast == "frpca" else 78))
    l = 8 + 5
    Om = orc.gaussian_matrix(n, l, oseed) if fast == "frpca" else orc.gaussian_matrix(l, m, oseed)
    c = cfg(fb, 8, 5, q=q, p=(q - 2) // 2, seed=5)
    sf, sb = fb.RunStats(capture_basis=True), fb.RunStats(capture_basis=True)
    f = getattr(fb, fast)(A, c, sf, omega=Om)
    b = getattr(fb, basic)(A, c, sb, omega=Om)
    assert np.linalg.norm(recon(f) - recon(b)) / np.linalg.norm(recon(f)) < 1e-8
    assert projector_gap_dense(sf.basis, sb.basis) < 1e-8


def test_shared_seed_pairs_sketches(fb, orc):  # test_randsvd.cpp:174-180
    A = to_fb(fb, orc.Csr.random_sparse(60, 90, 0.2, 79))
    c = cfg(fb, 5, 5, q=6, p=2, seed=1234)
    f, b = fb.frpca(A, c), fb.basic_rpca(A, c)
    assert np.linalg.norm(recon(f) - recon(b)) / np.linalg.norm(recon(f)) < 1e-8
