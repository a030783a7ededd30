import os, sys, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_1810_06825_b200 as fb
import oracle as orc
from test_gpu_kernels import powerlaw_csr

def both(M):
    os.environ.pop("FRPCA_LU_GLOBAL", None)
    a = fb.lu_basis(M)
    os.environ["FRPCA_LU_GLOBAL"] = "1"
    b = fb.lu_basis(M)
    os.environ.pop("FRPCA_LU_GLOBAL", None)
    return a, b

rng = np.random.default_rng(0)
for (m, l) in [(4000, 200), (3000, 200), (5000, 64), (4500, 32), (4000, 40)]:
    M = orc.gaussian_matrix(m, l, m + l)
    a, b = both(M)
    print("gauss", m, l, np.array_equal(a, b), np.abs(a - b).max())
    M2 = M * (10.0 ** rng.uniform(-8, 8, size=(m, 1)))
    M2[rng.choice(m, m // 5, replace=False)] = 0.0
    a, b = both(M2)
    print("scaled+zero rows", m, l, np.array_equal(a, b), np.abs(a - b).max())
oA = powerlaw_csr(orc, 20000, 4000, 400000, 23, a_row=1.8, a_col=1.05)
Om = orc.gaussian_matrix(200, 20000, 5)
Z = orc.spmm_transpose(oA, Om.T.copy())
a, b = both(Z)
print("pipeline Z", np.array_equal(a, b), np.abs(a - b).max(), "pivots equal", np.array_equal(a == 1.0, b == 1.0))
