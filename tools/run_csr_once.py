"""One warm frpca_run_csr call (pinned host CSR in, pinned U/S/V out) with the
CUDA profiler range around the second call only, for an ncu launch list of
the whole e2e path: `ncu --profile-from-start off ... python
tools/run_csr_once.py C3`."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
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
ch = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=False)


def run_csr():
    _lib.check(L.frpca_run_csr(ctx._h, m, n, nnz, prp, pci, pva, algo, C.byref(ch), None, 0, 0, pU, pS, pV,
                               None, None, None))


run_csr()
torch.cuda.synchronize()
torch.cuda.profiler.start()
run_csr()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done", file=sys.stderr)
