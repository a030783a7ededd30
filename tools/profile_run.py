"""One device-resident frpca/frpcat run of a BASELINE config (for ncu / launch
lists): `python tools/profile_run.py --config C1 [--runs 2]`. Prints the
per-kernel CUDA-event breakdown of the last run as JSON."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--runs", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    import time
    t0 = time.time()
    m, n, rp, ci, va = synth.generate(cfg.name, scale=a.scale)
    print(f"generated {cfg.name}: {m}x{n} nnz={int(rp[-1])} in {time.time() - t0:.1f}s", file=sys.stderr)
    t0 = time.time()
    ctx = fb.Context(0)
    L = _lib.load()
    h = C.c_void_p()
    _lib.check(L.frpca_dmat_upload(ctx._h, m, n, int(rp[-1]), rp.ctypes.data, ci.ctypes.data,
                                   va.ctypes.data, C.byref(h)))
    print(f"upload {time.time() - t0:.2f}s", file=sys.stderr)
    import torch
    k = cfg.k
    dU = torch.empty(m * k, dtype=torch.float64, device="cuda")
    dS = torch.empty(k, dtype=torch.float64, device="cuda")
    dV = torch.empty(n * k, dtype=torch.float64, device="cuda")
    c = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=True)
    algo = _lib.ALGO_FRPCA if cfg.algorithm == "frpca" else _lib.ALGO_FRPCAT
    for r in range(a.runs):
        t0 = time.time()
        if r == a.runs - 1:
            ctx.profile(True)
            ctx.profile_reset()
        _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(c), None, 0, 0, C.c_void_p(dU.data_ptr()),
                               C.c_void_p(dS.data_ptr()), C.c_void_p(dV.data_ptr()), None, None, None))
        print(f"run {r}: {time.time() - t0:.3f}s", file=sys.stderr)
    rep = ctx.profile_report()
    print(json.dumps({"config": cfg.name, "scale": a.scale, "kernels": rep}, indent=1))
    L.frpca_dmat_destroy(h)


if __name__ == "__main__":
    main()
