"""A/B of environment knobs on one uploaded matrix (one process, one
generation): `python tools/ab_env.py --config C1 --runs 5 FRPCA_X=0 FRPCA_X=1`.
Variants are interleaved run by run; each run is a device-resident frpca_run
(synchronous) timed on the host with an L2 flush before it. Prints the median
and min per variant as JSON."""
import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--runs", type=int, default=5)
    ap.add_argument("--reupload", action="store_true", help="one upload per variant (load-time knobs)")
    ap.add_argument("variants", nargs="+", help="NAME=VALUE[,NAME=VALUE...] per variant")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    m, n, rp, ci, va = synth.generate(cfg.name)
    ctx = fb.Context(0)
    L = _lib.load()

    def upload():
        h = C.c_void_p()
        _lib.check(L.frpca_dmat_upload(ctx._h, m, n, int(rp[-1]), rp.ctypes.data, ci.ctypes.data,
                                       va.ctypes.data, C.byref(h)))
        return h

    envs = [dict(kv.split("=", 1) for kv in v.split(",")) for v in a.variants]
    handles = []
    for e in envs:
        if handles and not a.reupload:
            handles.append(handles[0])
            continue
        os.environ.update(e)
        handles.append(upload())
        for kk in e:
            del os.environ[kk]
    import torch
    k = cfg.k
    dU = torch.empty(m * k, dtype=torch.float64, device="cuda")
    dS = torch.empty(k, dtype=torch.float64, device="cuda")
    dV = torch.empty(n * k, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    c = fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0).to_c(device_io=True)
    algo = _lib.ALGO_FRPCA if cfg.algorithm == "frpca" else _lib.ALGO_FRPCAT
    times = {v: [] for v in a.variants}
    S0 = None
    for r in range(a.runs + 1):
        for v, e, h in zip(a.variants, envs, handles):
            for kk, vv in e.items():
                os.environ[kk] = vv
            flush.fill_(r & 0xff)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(L.frpca_run(ctx._h, h, algo, C.byref(c), None, 0, 0, C.c_void_p(dU.data_ptr()),
                                   C.c_void_p(dS.data_ptr()), C.c_void_p(dV.data_ptr()), None, None, None))
            t = time.perf_counter() - t0
            S = dS.cpu().numpy()
            if S0 is None:
                S0 = S
            same = bool(np.array_equal(S, S0))
            if r:  # the first round warms every variant up
                times[v].append(t)
            print(f"{v} run {r}: {t * 1e3:.2f} ms S_bitwise_equal={same}", file=sys.stderr)
            for kk in e:
                del os.environ[kk]
    out = {v: {"median_ms": float(np.median(t) * 1e3), "min_ms": float(np.min(t) * 1e3)} for v, t in times.items()}
    print(json.dumps({"config": cfg.name, "runs": a.runs, "variants": out}))
    for h in set(x.value for x in handles):
        L.frpca_dmat_destroy(C.c_void_p(h))


if __name__ == "__main__":
    main()
