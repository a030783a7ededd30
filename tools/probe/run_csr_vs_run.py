"""frpca_run_csr (one-shot, pipelined upload) against upload + frpca_run on one
saved case, over variants of q, (k, s) and the pipeline knobs. Probe."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1810_06825_b200 as fb  # noqa: E402
from metrics import sigma_rel, subspace_dist  # noqa: E402

z = np.load(sys.argv[1])
m, n, k0, s0, q0, seed, algo = (int(z[x]) for x in ("m", "n", "k", "s", "q", "seed", "algo"))
A = fb.SparseMatrixCsr(m, n, z["rp"], z["ci"], z["va"])
f = fb.frpca if algo == 0 else fb.frpcat
alg = fb.PcaAlgorithm.Frpca if algo == 0 else fb.PcaAlgorithm.Frpcat


def one(k, s, q, env=None, tag=""):
    for kk, vv in (env or {}).items():
        os.environ[kk] = vv
    try:
        cfg = fb.PcaConfig(k=k, oversample=s, passes=q, seed=seed)
        r = f(A, cfg)
        r1, _ = fb.run_csr(A, cfg, alg)
        r2, _ = fb.run_csr(A, cfg, alg)
        print("k=%d s=%d q=%d %s: run_csr vs run sigma %.3g U %.3g | run_csr twice sigma %.3g" % (
            k, s, q, tag or env or "", sigma_rel(r1.S, r.S), subspace_dist(r.U, r1.U), sigma_rel(r2.S, r1.S)), flush=True)
    finally:
        for kk in (env or {}):
            del os.environ[kk]


print(m, n, k0, s0, q0, algo)
one(k0, s0, q0)
one(k0, s0, q0, {"FRPCA_UPLOAD_PIPELINE": "0"})
one(k0, s0, q0, {"FRPCA_EIG_REFINE": "0"})
one(k0, s0, q0, {"FRPCA_EIG": "cusolver"})
for q in (2, 3, 5, 6):
    one(k0, s0, q)
for k, s in ((100, 14), (135, 0), (64, 14), (140, 9), (20, 10), (128, 22), (120, 30)):
    if k + s <= min(m, n):
        one(k, s, q0)
