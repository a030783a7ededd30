"""SURVEY §8 row f3, pinned on the CPU: the oracle's restatement of the
reference's validation metrics (validation.hpp:125-282) passes the
reference's own tests (test_validation.cpp:78-168). The GPU versions are
checked against these in test_gpu_validation.py."""
import numpy as np
import pytest


def truncate_oracle(orc, A, k):
    U, S, V = orc.oracle_svd(A.to_dense())
    return U[:, :k], S[:k], V[:, :k], S


def dense(A):
    rp, ci, va = A.arrays()
    D = np.zeros((A.rows, A.cols))
    for i in range(A.rows):
        D[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    return D


@pytest.fixture
def todense(orc):
    orc.Csr.to_dense = dense
    return dense


def test_exact_svd_gives_zero(orc, todense):  # test_validation.cpp:78-84
    A = orc.Csr.random_sparse(30, 20, 0.3, 7)
    U, S, V, _ = truncate_oracle(orc, A, 20)
    na = np.linalg.norm(dense(A))
    assert orc.low_rank_error(A, U, S, V, orc.FROBENIUS) < 1e-10 * na
    assert orc.low_rank_error(A, U, S, V, orc.SPECTRAL) < 1e-10 * na


def test_truncation_equals_tail(orc, todense):  # test_validation.cpp:86-94
    A = orc.Csr.random_sparse(40, 25, 0.4, 13)
    U, S, V, Sall = truncate_oracle(orc, A, 5)
    assert abs(orc.low_rank_error(A, U, S, V, orc.SPECTRAL) - Sall[5]) <= 1e-8 * Sall[5]
    tail = np.sqrt(np.sum(Sall[5:] ** 2))
    assert abs(orc.low_rank_error(A, U, S, V, orc.FROBENIUS) - tail) <= 1e-10 * tail


def test_zero_factors(orc):  # test_validation.cpp:96-104
    A = orc.Csr.from_triplets(2, 2, [(0, 0, 3.0), (1, 1, 4.0)])
    U, V, S = np.eye(2, 1), np.eye(2, 1), np.zeros(1)
    assert abs(orc.low_rank_error(A, U, S, V, orc.FROBENIUS) - 5.0) < 1e-12
    assert abs(orc.low_rank_error(A, U, S, V, orc.SPECTRAL) - 4.0) < 4e-9


def test_cross_term_path(orc, todense):  # test_validation.cpp:106-114
    A = orc.Csr.random_sparse(50, 30, 0.3, 23)
    U, S, V, _ = truncate_oracle(orc, A, 6)
    e = orc.low_rank_error(A, U, S, V, orc.FROBENIUS)
    i = orc.low_rank_error(A, U, S, V, orc.FROBENIUS, entry_limit=0)
    assert abs(i - e) <= 1e-9 * e


def test_pc_correlation(orc):  # test_validation.cpp:130-143
    U = orc.gaussian_matrix(50, 4, 3)
    assert np.abs(orc.pc_correlation(U, U) - 1).max() < 1e-14
    assert np.abs(orc.pc_correlation(U, -U) - 1).max() < 1e-14
    with pytest.raises(ValueError, match="zero-variance column 0"):
        orc.pc_correlation(np.ones((10, 1)), orc.gaussian_matrix(10, 1, 5))


def test_projector_distance(orc):  # test_validation.cpp:145-168
    Q1 = orc.orth(orc.gaussian_matrix(40, 5, 7))
    R = orc.orth(orc.gaussian_matrix(5, 5, 8))
    assert orc.projector_distance(Q1, Q1 @ R) < 1e-10
    A, B = np.eye(6, 2), np.zeros((6, 2))
    B[2, 0] = B[3, 1] = 1.0
    assert abs(orc.projector_distance(A, B) - 1.0) < 1e-10
    M = orc.gaussian_matrix(60, 8, 21)
    assert orc.projector_distance(orc.orth(M), orc.orth(orc.lu_basis(M))) < 1e-10
    with pytest.raises(ValueError, match="first basis is not orthonormal"):
        orc.projector_distance(2.0 * np.eye(5, 2), 2.0 * np.eye(5, 2))
