import os, sys, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1810_06825_b200 as fb
import oracle as orc
from test_gpu_kernels import powerlaw_csr, to_fb
from metrics import rel_fro
os.environ["FRPCA_SPMM_SLICE"] = "128"
os.environ["FRPCA_PANEL_MIN_MB"] = "0"
for mb in ["0.5", "4"]:
    os.environ["FRPCA_PANEL_MB"] = mb
    for (m, n, nnz) in [(20000, 5000, 400000), (50000, 5000, 1000000)]:
        for nc in [150, 22, 200, 140]:
            oA = powerlaw_csr(orc, m, n, nnz, 3)
            A = to_fb(fb, oA)
            Y = orc.gaussian_matrix(m, nc, 1)
            try:
                Z = fb.spmm_transpose(A, Y)
                print(mb, m, n, nc, "rel", rel_fro(Z, orc.spmm_transpose(oA, Y)), flush=True)
            except Exception as e:
                print(mb, m, n, nc, "ERR", e, flush=True)
                sys.exit(1)
