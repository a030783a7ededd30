import os, sys, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1810_06825_b200 as fb
from paper_1810_06825_b200 import synth
os.environ["FRPCA_SPMM_SLICE"] = sys.argv[1]
m, n, rp, ci, va = synth.generate("C2", scale=float(sys.argv[2]))
A = fb.SparseMatrixCsr(m, n, rp, ci, va, validate=False)
for q in [int(x) for x in sys.argv[3].split(",")]:
    try:
        r = fb.frpcat(A, fb.PcaConfig(k=100, oversample=50, passes=q, seed=0))
        print("q", q, "ok", r.S[:3], flush=True)
    except Exception as e:
        print("q", q, "ERR", e, flush=True)
        sys.exit(1)
