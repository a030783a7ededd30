"""Times orth (Householder QR basis, csrc/orth.cu) on random tall panels (device time via the profiler)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_06825_b200 as fb
ctx = fb.default_context()
for (m, l) in [(100000, 200), (324000, 200), (1000000, 200), (4000000, 100)]:
    M = np.random.default_rng(1).standard_normal((m, l))
    Q = fb.orth(M)
    ctx.profile(True); ctx.profile_reset()
    fb.orth(M)
    rep = ctx.profile_report()
    ctx.profile(False)
    e = np.abs(Q[:, :8].T @ Q[:, :8] - np.eye(8)).max()
    print(m, l, {k: round(v["ms"], 3) for k, v in rep.items()}, "orthonormality(8 cols) %.1e" % e, flush=True)
