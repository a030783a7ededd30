"""Times lu_basis on random tall panels of several shapes (device time via the profiler)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1810_06825_b200 as fb
ctx = fb.default_context()
for (m, l) in [(100000, 200), (200000, 200), (200000, 150), (400000, 200), (500000, 150)]:
    M = np.random.default_rng(1).standard_normal((m, l))
    fb.lu_basis(M)
    ctx.profile(True); ctx.profile_reset()
    fb.lu_basis(M)
    rep = ctx.profile_report()
    ctx.profile(False)
    print(m, l, {k: round(v["ms"], 3) for k, v in rep.items()}, flush=True)
