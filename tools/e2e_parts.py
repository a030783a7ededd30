"""e2e breakdown (diagnostic): upload alone, run with device outputs, run with
pinned host outputs, frpca_run_csr; medians of 6 steps, CUDA-event ms."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import _lib, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C1"]
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
nnz = int(rp[-1])
ch_h = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=False)
ch_d = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=True)
dU = torch.empty(m * k, dtype=torch.float64, device="cuda")
dS = torch.empty(k, dtype=torch.float64, device="cuda")
dV = torch.empty(n * k, dtype=torch.float64, device="cuda")
h = C.c_void_p()
_lib.check(L.frpca_dmat_upload(ctx._h, m, n, nnz, prp, pci, pva, C.byref(h)))


def timed(f, reps=6):
    f()
    ts = []
    for _ in range(reps):
        ms = C.c_double()
        _lib.check(L.frpca_timer_begin(ctx._h))
        f()
        _lib.check(L.frpca_timer_end(ctx._h, C.byref(ms)))
        ts.append(ms.value)
    return round(float(np.median(ts)), 2), [round(t, 2) for t in ts]


def upload():
    h2 = C.c_void_p()
    _lib.check(L.frpca_dmat_upload(ctx._h, m, n, nnz, prp, pci, pva, C.byref(h2)))
    L.frpca_dmat_destroy(h2)


def run_dev():
    _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(ch_d), None, 0, 0, C.c_void_p(dU.data_ptr()),
                           C.c_void_p(dS.data_ptr()), C.c_void_p(dV.data_ptr()), None, None, None))


def run_host():
    _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(ch_h), None, 0, 0, pU, pS, pV, None, None, None))


def run_csr():
    _lib.check(L.frpca_run_csr(ctx._h, m, n, nnz, prp, pci, pva, algo, C.byref(ch_h), None, 0, 0, pU, pS, pV,
                               None, None, None))


def d2h_only():
    torch.cuda.synchronize()
    C.c_void_p()
    src = dU
    dst = torch.from_numpy(np.ctypeslib.as_array(C.cast(pU, C.POINTER(C.c_double)), shape=(m * k,)))
    dst.copy_(src, non_blocking=True)


for name, f in (("upload", upload), ("run_dev", run_dev), ("run_host", run_host), ("run_csr", run_csr)):
    print(name, *timed(f), flush=True)

# per-stage profile of one run_csr (main stream only; Omega runs on the side stream)
_lib.check(L.frpca_profile_reset(ctx._h))
_lib.check(L.frpca_profile_enable(ctx._h, 1))
run_csr()
_lib.check(L.frpca_profile_enable(ctx._h, 0))
cnt = C.c_int()
_lib.check(L.frpca_profile_count(ctx._h, C.byref(cnt)))
rows = []
for i in range(cnt.value):
    nm = C.c_char_p(); la = C.c_int64(); ms = C.c_double(); by = C.c_double(); fl = C.c_double()
    _lib.check(L.frpca_profile_get(ctx._h, i, C.byref(nm), C.byref(la), C.byref(ms), C.byref(by), C.byref(fl)))
    rows.append((ms.value, nm.value.decode(), la.value))
for ms, nm, la in sorted(rows, reverse=True):
    print(f"  {nm:24s} {la:3d} {ms:8.3f} ms")
