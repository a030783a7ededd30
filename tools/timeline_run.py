"""Event timeline of one device-resident run (diagnostic): `FRPCA_DEBUG_TIMELINE=1
python tools/timeline_run.py C3` prints each stage bracket's start/end (ms)
relative to the run's first bracket, after a warm-up run."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("FRPCA_DEBUG_TIMELINE", "1")
import torch  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import _lib, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
m, n, rp, ci, va = synth.generate(cfg.name)
ctx = fb.Context(0)
L = _lib.load()
h = C.c_void_p()
_lib.check(L.frpca_dmat_upload(ctx._h, m, n, int(rp[-1]), rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                               C.byref(h)))
k = cfg.k
dU = torch.empty(m * k, dtype=torch.float64, device="cuda")
dS = torch.empty(k, dtype=torch.float64, device="cuda")
dV = torch.empty(n * k, dtype=torch.float64, device="cuda")
c = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=True)
algo = _lib.ALGO_FRPCA if cfg.algorithm == "frpca" else _lib.ALGO_FRPCAT
for r in range(2):
    if r == 1:
        ctx.profile(True)
        print("---- timed run", file=sys.stderr, flush=True)
    _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(c), None, 0, 0, C.c_void_p(dU.data_ptr()),
                           C.c_void_p(dS.data_ptr()), C.c_void_p(dV.data_ptr()), None, None, None))
    torch.cuda.synchronize()
