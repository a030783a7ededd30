"""Accuracy of the l x l eigensolvers of eig_svd (syev.cu vs cuSOLVER syevd)
on Gram matrices of graded conditioning: eigenvector orthogonality
||V^T V - I||_max, residual ||B V - V diag(D)||_F / ||B||_F, and the
orthonormality of eig_svd's U = W V S^-1 (what the power iteration feeds on).
    python tools/syev_accuracy.py [--n 150] [--rows 20000]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=150)
    ap.add_argument("--rows", type=int, default=20000)
    a = ap.parse_args()
    out = {}
    rng = np.random.default_rng(0)
    for logc in (2, 4, 6, 7):
        Q, _ = np.linalg.qr(rng.standard_normal((a.rows, a.n)))
        R, _ = np.linalg.qr(rng.standard_normal((a.n, a.n)))
        s = np.logspace(0, -logc, a.n)
        W = np.asfortranarray((Q * s) @ R.T)
        B = W.T @ W
        res = {}
        for mode in ("small", "cusolver"):
            os.environ["FRPCA_EIG"] = mode
            U, S, V = fb.eig_svd(W)
            D = S ** 2
            res[mode] = {
                "V_orth": float(np.abs(V.T @ V - np.eye(a.n)).max()),
                "residual": float(np.linalg.norm(B @ V - V * D) / np.linalg.norm(B)),
                "U_orth": float(np.abs(U.T @ U - np.eye(a.n)).max()),
                "smallest_sigma_rel": float(abs(S[0] - s[-1]) / s[-1]),
            }
        out[f"cond(W)=1e{logc}"] = res
        print(json.dumps({f"cond(W)=1e{logc}": res}), flush=True)
    os.environ.pop("FRPCA_EIG", None)


if __name__ == "__main__":
    main()
