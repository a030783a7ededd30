import os, sys, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1810_06825_b200 as fb
from paper_1810_06825_b200 import synth
os.environ["FRPCA_SPMM_SLICE"] = sys.argv[1]
sc = float(sys.argv[2])
m, n, rp, ci, va = synth.generate("C2", scale=sc)
A = fb.SparseMatrixCsr(m, n, rp, ci, va, validate=False)
rng = np.random.default_rng(0)
for nc in [150, 128, 22]:
    Y = rng.standard_normal((m, nc))
    try:
        Z = fb.spmm_transpose(A, Y)
        X = rng.standard_normal((n, nc))
        W = fb.spmm(A, X)
        print(sc, nc, "ok", float(np.abs(Z).sum()), float(np.abs(W).sum()), flush=True)
    except Exception as e:
        print(sc, nc, "ERR", e, flush=True)
        sys.exit(1)
