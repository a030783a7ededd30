"""e2e A/B (diagnostic): frpca_run_csr (pinned host CSR in, pinned U/S/V out)
timed per call on the host, variants interleaved call by call:
`python tools/e2e_ab.py C3 6 FRPCA_UPLOAD_PIPELINE=0 FRPCA_UPLOAD_PIPELINE=1`.
Also prints the per-stage event profile of one call of each variant."""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import _lib, synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2])
variants = sys.argv[3:]
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


def setenv(v):
    for kv in v.split(","):
        kk, vv = kv.split("=", 1)
        os.environ[kk] = vv


def unsetenv(v):
    for kv in v.split(","):
        os.environ.pop(kv.split("=", 1)[0], None)


times = {v: [] for v in variants}
S0 = None
per_call = os.environ.get("E2E_PER_CALL_PROFILE") == "1"


def profile_rows():
    cnt = C.c_int()
    _lib.check(L.frpca_profile_count(ctx._h, C.byref(cnt)))
    rows = {}
    for i in range(cnt.value):
        nm = C.c_char_p(); la = C.c_int64(); ms = C.c_double(); by = C.c_double(); fl = C.c_double()
        _lib.check(L.frpca_profile_get(ctx._h, i, C.byref(nm), C.byref(la), C.byref(ms), C.byref(by), C.byref(fl)))
        rows[nm.value.decode()] = round(ms.value, 1)
    return rows


for r in range(reps + 1):
    for v in variants:
        setenv(v)
        if per_call:
            _lib.check(L.frpca_profile_reset(ctx._h))
            _lib.check(L.frpca_profile_enable(ctx._h, 1))
        t0 = time.perf_counter()
        run_csr()
        t = (time.perf_counter() - t0) * 1e3
        if per_call:
            _lib.check(L.frpca_profile_enable(ctx._h, 0))
            rows = profile_rows()
            top = dict(sorted(rows.items(), key=lambda x: -x[1])[:8])
            print(f"  profile {v} call {r}: {top}", file=sys.stderr, flush=True)
        S = np.ctypeslib.as_array(C.cast(pS, C.POINTER(C.c_double)), shape=(k,)).copy()
        if S0 is None:
            S0 = S
        if r:
            times[v].append(round(t, 1))
        free, total = torch.cuda.mem_get_info()
        print(f"{v} call {r}: {t:.1f} ms bitwise={np.array_equal(S, S0)} device used {(total - free) / 2**30:.1f} GiB",
              file=sys.stderr, flush=True)
        unsetenv(v)
prof = {}
for v in variants:
    setenv(v)
    _lib.check(L.frpca_profile_reset(ctx._h))
    _lib.check(L.frpca_profile_enable(ctx._h, 1))
    run_csr()
    _lib.check(L.frpca_profile_enable(ctx._h, 0))
    cnt = C.c_int()
    _lib.check(L.frpca_profile_count(ctx._h, C.byref(cnt)))
    rows = {}
    for i in range(cnt.value):
        nm = C.c_char_p(); la = C.c_int64(); ms = C.c_double(); by = C.c_double(); fl = C.c_double()
        _lib.check(L.frpca_profile_get(ctx._h, i, C.byref(nm), C.byref(la), C.byref(ms), C.byref(by), C.byref(fl)))
        rows[nm.value.decode()] = round(ms.value, 2)
    prof[v] = dict(sorted(rows.items(), key=lambda x: -x[1]))
    unsetenv(v)
print(json.dumps({"config": cfg.name, "ms_per_call": times,
                  "median": {v: float(np.median(t)) for v, t in times.items()}, "profile": prof}, indent=1))
