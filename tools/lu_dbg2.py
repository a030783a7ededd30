import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_06825_b200 as fb
import oracle as orc
for (m, l) in [(300, 70), (40, 8), (5000, 150)]:
    M = orc.gaussian_matrix(m, l, m + l)
    Xo = orc.lu_basis(M)
    po = [int(np.where(Xo[:, j] == 1.0)[0][0]) if np.any(Xo[:, j] == 1.0) else -1 for j in range(l)]
    for rep in range(3):
        X = fb.lu_basis(M)
        p = [int(np.where(X[:, j] == 1.0)[0][0]) if np.any(X[:, j] == 1.0) else -1 for j in range(l)]
        bad = [j for j in range(l) if p[j] != po[j]]
        print(m, l, rep, "first bad col", bad[:5], "gpu", [p[j] for j in bad[:5]], "orc", [po[j] for j in bad[:5]],
              "maxdiff", float(np.max(np.abs(X - Xo))))
