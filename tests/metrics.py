"""Parity metrics (SURVEY §8c / north_star tolerances)."""
import numpy as np

SIGMA_TOL = 1e-10      # max_i |s'_i - s_i| / s_i
SUBSPACE_TOL = 1e-8    # ||U U^T - U' U'^T||_2
SPMM_TOL = 1e-12       # ||Y - Y_ref||_F / ||Y_ref||_F


def rel_fro(A, B) -> float:
    nb = np.linalg.norm(B)
    d = np.linalg.norm(np.asarray(A) - np.asarray(B))
    return float(d / nb) if nb > 0 else float(d)


def sigma_rel(S, S_ref) -> float:
    S, S_ref = np.asarray(S), np.asarray(S_ref)
    return float(np.max(np.abs(S - S_ref) / np.abs(S_ref)))


def subspace_dist(U, U2) -> float:
    """||U U^T - U2 U2^T||_2 for orthonormal U, U2 of equal width, without
    forming m x m matrices: the norm equals ||U2 - U (U^T U2)||_2 (largest
    principal-angle sine), from the k x k Gram of the residual."""
    U, U2 = np.asarray(U), np.asarray(U2)
    R = U2 - U @ (U.T @ U2)
    G = R.T @ R
    return float(np.sqrt(max(np.linalg.eigvalsh(G).max(), 0.0)))


def orthonormality(U) -> float:
    k = U.shape[1]
    return float(np.abs(U.T @ U - np.eye(k)).max())


def projector_gap_dense(Q1, Q2) -> float:
    """test_support.hpp:40-44 (dense projector difference, small sizes only)."""
    D = Q1 @ Q1.T - Q2 @ Q2.T
    return float(np.linalg.svd(D, compute_uv=False)[0])


def orth(M):
    Q, _ = np.linalg.qr(M)
    return Q
