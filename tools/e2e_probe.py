"""Per-step e2e timing of the host-CSR paths (diagnostic): frpca_run_csr vs
upload + frpca_run + destroy, C1, pinned host outputs."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import _lib, synth  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = synth.CONFIGS[cfgname]
m, n, rp, ci, va = synth.generate(cfg.name)
ctx = fb.Context(0)
L = _lib.load()
k = cfg.k
algo = _lib.ALGO_FRPCA if cfg.algorithm == "frpca" else _lib.ALGO_FRPCAT


def pinned(nbytes):
    p = C.c_void_p()
    _lib.check(L.frpca_host_alloc(nbytes, C.byref(p)))
    return p


pU, pS, pV = pinned(8 * m * k), pinned(8 * k), pinned(8 * n * k)
prp, pci, pva = pinned(rp.nbytes), pinned(ci.nbytes), pinned(va.nbytes)
C.memmove(prp, rp.ctypes.data, rp.nbytes)
C.memmove(pci, ci.ctypes.data, ci.nbytes)
C.memmove(pva, va.ctypes.data, va.nbytes)
ch = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=False)
nnz = int(rp[-1])


def run_csr():
    _lib.check(L.frpca_run_csr(ctx._h, m, n, nnz, prp, pci, pva, algo, C.byref(ch), None, 0, 0, pU, pS, pV,
                               None, None, None))


def run_split():
    h = C.c_void_p()
    _lib.check(L.frpca_dmat_upload(ctx._h, m, n, nnz, prp, pci, pva, C.byref(h)))
    _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(ch), None, 0, 0, pU, pS, pV, None, None, None))
    L.frpca_dmat_destroy(h)


for name, f in (("run_csr", run_csr), ("split", run_split), ("run_csr", run_csr)):
    f()
    ts = []
    for _ in range(8):
        ms = C.c_double()
        t0 = time.perf_counter()
        _lib.check(L.frpca_timer_begin(ctx._h))
        f()
        _lib.check(L.frpca_timer_end(ctx._h, C.byref(ms)))
        ts.append((round(ms.value, 2), round(1e3 * (time.perf_counter() - t0), 2)))
    print(name, ts, flush=True)
