"""SURVEY §8 row f3 on the B200: the validation metrics (validation.hpp:125-332)
through the C ABI — the reference's own tests (test_validation.cpp:78-190)
and agreement with the oracle's restatement — and a full-scale spectral
residual of a frpcat run (what the reference's dense oracle cannot reach)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def oracle_factors(orc, oA, k):
    rp, ci, va = oA.arrays()
    D = np.zeros((oA.rows, oA.cols))
    for i in range(oA.rows):
        D[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    U, S, V = orc.oracle_svd(D)
    return U, S, V, D


def svd(fb, U, S, V):
    return fb.SvdResult(np.asfortranarray(U), np.ascontiguousarray(S), np.asfortranarray(V))


def to_fb(fb, oA):
    return fb.SparseMatrixCsr(oA.rows, oA.cols, *oA.arrays())


def test_exact_svd_zero(fb, orc):  # test_validation.cpp:78-84
    oA = orc.Csr.random_sparse(30, 20, 0.3, 7)
    U, S, V, D = oracle_factors(orc, oA, 20)
    A, r = to_fb(fb, oA), svd(fb, U[:, :20], S[:20], V[:, :20])
    na = np.linalg.norm(D)
    assert fb.low_rank_error(A, r, fb.ErrorNorm.Frobenius) < 1e-10 * na
    assert fb.low_rank_error(A, r, fb.ErrorNorm.Spectral) < 1e-10 * na


def test_truncation_tail(fb, orc):  # test_validation.cpp:86-94
    oA = orc.Csr.random_sparse(40, 25, 0.4, 13)
    U, S, V, _ = oracle_factors(orc, oA, 5)
    A, r = to_fb(fb, oA), svd(fb, U[:, :5], S[:5], V[:, :5])
    assert abs(fb.low_rank_error(A, r, fb.ErrorNorm.Spectral) - S[5]) <= 1e-8 * S[5]
    tail = np.sqrt(np.sum(S[5:] ** 2))
    assert abs(fb.low_rank_error(A, r, fb.ErrorNorm.Frobenius) - tail) <= 1e-10 * tail


def test_zero_factors(fb):  # test_validation.cpp:96-104
    A = fb.SparseMatrixCsr.from_triplets(2, 2, [(0, 0, 3.0), (1, 1, 4.0)])
    r = fb.SvdResult(np.eye(2, 1), np.zeros(1), np.eye(2, 1))
    assert abs(fb.low_rank_error(A, r, fb.ErrorNorm.Frobenius) - 5.0) < 1e-12
    assert abs(fb.low_rank_error(A, r, fb.ErrorNorm.Spectral) - 4.0) < 4e-9


def test_cross_term_path(fb, orc):  # test_validation.cpp:106-114
    oA = orc.Csr.random_sparse(50, 30, 0.3, 23)
    U, S, V, _ = oracle_factors(orc, oA, 6)
    A, r = to_fb(fb, oA), svd(fb, U[:, :6], S[:6], V[:, :6])
    e = fb.low_rank_error(A, r, fb.ErrorNorm.Frobenius)
    i = fb.low_rank_error(A, r, fb.ErrorNorm.Frobenius, entry_limit=0)
    assert abs(i - e) <= 1e-9 * e


def test_shape_checks(fb):
    A = fb.SparseMatrixCsr.from_triplets(3, 2, [(0, 0, 1.0)])
    with pytest.raises(ValueError, match="low_rank_error: shape mismatch"):
        fb.low_rank_error(A, fb.SvdResult(np.zeros((2, 1)), np.zeros(1), np.zeros((2, 1))), fb.ErrorNorm.Spectral)
    with pytest.raises(ValueError, match="inconsistent factor widths"):
        fb.low_rank_error(A, fb.SvdResult(np.zeros((3, 2)), np.zeros(1), np.zeros((2, 1))), fb.ErrorNorm.Frobenius)


def test_best_rank_k(fb):  # test_validation.cpp:116-128 (host part)
    assert fb.best_rank_k_error([5.0, 4.0, 3.0], 2, fb.ErrorNorm.Spectral) == 3.0
    assert fb.best_rank_k_error([5.0, 4.0, 3.0], 2, fb.ErrorNorm.Frobenius) == 3.0
    assert fb.best_rank_k_error([5.0], 3, fb.ErrorNorm.Spectral) == 0.0


def test_pc_correlation(fb, orc):  # test_validation.cpp:130-143
    U = orc.gaussian_matrix(50, 4, 3)
    assert np.abs(fb.pc_correlation(U, U) - 1).max() < 1e-14
    assert np.abs(fb.pc_correlation(U, -U) - 1).max() < 1e-14
    with pytest.raises(ValueError, match="pc_correlation: zero-variance column 0"):
        fb.pc_correlation(np.ones((10, 1)), orc.gaussian_matrix(10, 1, 5))
    X, Y = orc.gaussian_matrix(3000, 7, 1), orc.gaussian_matrix(3000, 7, 2)
    assert np.allclose(fb.pc_correlation(X, Y), orc.pc_correlation(X, Y), rtol=1e-11, atol=1e-14)


def test_projector_distance(fb, orc):  # test_validation.cpp:145-168
    Q1 = orc.orth(orc.gaussian_matrix(40, 5, 7))
    R = orc.orth(orc.gaussian_matrix(5, 5, 8))
    assert fb.projector_distance(Q1, Q1 @ R) < 1e-10
    A, B = np.eye(6, 2), np.zeros((6, 2))
    B[2, 0] = B[3, 1] = 1.0
    assert abs(fb.projector_distance(A, B) - 1.0) < 1e-10
    M = orc.gaussian_matrix(60, 8, 21)
    assert fb.projector_distance(fb.orth(M), fb.orth(fb.lu_basis(M))) < 1e-10
    with pytest.raises(ValueError, match="first basis is not orthonormal within 1e-8"):
        fb.projector_distance(2.0 * np.eye(5, 2), 2.0 * np.eye(5, 2))
    Q3 = orc.orth(orc.gaussian_matrix(2000, 9, 3))
    Q4 = orc.orth(orc.gaussian_matrix(2000, 6, 4))
    assert abs(fb.projector_distance(Q3, Q4) - orc.projector_distance(Q3, Q4)) < 1e-10


def test_accuracy_report(fb, orc):  # test_validation.cpp:170-190
    oA = orc.Csr.random_sparse(30, 20, 0.4, 41)
    U, S, V, _ = oracle_factors(orc, oA, 4)
    rep = fb.make_accuracy_report(to_fb(fb, oA), svd(fb, U[:, :4], S[:4], V[:, :4]), S, U)
    assert len(rep.singular_value_rel_err) == 4 and len(rep.pc_correlations) == 4
    assert rep.eps_equivalent >= -1e-10
    assert all(e < 1e-12 for e in rep.singular_value_rel_err)
    assert all(abs(c - 1.0) < 1e-9 for c in rep.pc_correlations)
    assert list(rep.to_json()) == ["singular_value_rel_err", "recon_err_frobenius", "recon_err_spectral",
                                   "best_rank_k_err", "eps_equivalent", "pc_correlations"]


@pytest.mark.parametrize("norm", [0, 1])
def test_metrics_match_oracle_random(fb, orc, norm):
    oA = orc.Csr.random_sparse(400, 300, 0.05, 8)
    r = fb.frpcat(to_fb(fb, oA), fb.PcaConfig(k=10, oversample=10, passes=4))
    got = fb.low_rank_error(to_fb(fb, oA), r, fb.ErrorNorm(norm))
    want = orc.low_rank_error(oA, r.U, r.S, r.V, norm)
    assert abs(got - want) <= 1e-9 * want


def test_full_scale_spectral_residual(fb, ctx):
    """C1 at scale 0.1 (100k x 10k, 1M nnz): the spectral residual of a frpcat
    run, matrix-free on the GPU, lies between sigma_{k+1} estimates: it is at
    least the (k+1)-th computed singular value bound and the eps_equivalent
    against the run's own (k+1)-th value is small."""
    from paper_1810_06825_b200 import synth
    m, n, rp, ci, va = synth.generate("C1", scale=0.1)
    A = fb.SparseMatrixCsr(m, n, rp, ci, va, validate=False)
    r21 = fb.frpcat(A, fb.PcaConfig(k=21, oversample=20, passes=6))
    r = fb.SvdResult(r21.U[:, :20], r21.S[:20], r21.V[:, :20])
    e = fb.low_rank_error(A, r, fb.ErrorNorm.Spectral)
    assert e >= r21.S[20] * (1 - 1e-6)
    assert e / r21.S[20] - 1.0 < 0.1
