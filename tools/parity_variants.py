"""Which stage sets the GPU path's distance from the oracle? One pinned oracle
run of a config, then the GPU path under several equally valid settings
(eigensolver, Gram kernel, host Omega), each compared with the oracle, next to
the oracle's own floor (FMA-contracted build vs pinned build).

    python tools/parity_variants.py --config C1 [--out file.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import paper_1810_06825_b200 as fb  # noqa: E402
from paper_1810_06825_b200 import synth  # noqa: E402
from metrics import sigma_rel, subspace_dist  # noqa: E402

VARIANTS = [
    ("default", {}, False),
    ("eig=cusolver", {"FRPCA_EIG": "cusolver"}, False),
    ("gram2", {"FRPCA_GRAM2": "1"}, False),
    ("host_omega", {}, True),
    ("host_omega+eig=cusolver", {"FRPCA_EIG": "cusolver"}, True),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--out", default="")
    ap.add_argument("--no-floor", action="store_true")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    m, n, rp, ci, va = synth.generate(a.config)
    oracle.build()
    oracle.set_threads(os.cpu_count() or 1)
    algo_o = oracle.FRPCA if cfg.algorithm == "frpca" else oracle.FRPCAT
    o = oracle.pca(oracle.Csr.create(m, n, rp, ci, va), algo_o, cfg.k, cfg.s, cfg.q, seed=0)
    out = {"config": a.config, "sigma1_over_sigmak": float(o["S"][0] / o["S"][-1]), "variants": {}}
    if not a.no_floor:
        with oracle.variant("fma"):
            oracle.set_threads(os.cpu_count() or 1)
            o2 = oracle.pca(oracle.Csr.create(m, n, rp, ci, va), algo_o, cfg.k, cfg.s, cfg.q, seed=0)
        out["oracle_fma_floor"] = {"sigma_rel": sigma_rel(o2["S"], o["S"]),
                                   "subspace_U": subspace_dist(o["U"], o2["U"]),
                                   "subspace_V": subspace_dist(o["V"], o2["V"])}
        del o2
    A = fb.SparseMatrixCsr(m, n, rp, ci, va)
    run = fb.frpca if cfg.algorithm == "frpca" else fb.frpcat
    for name, env, host in VARIANTS:
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            r = run(A, fb.PcaConfig(k=cfg.k, oversample=cfg.s, passes=cfg.q, seed=0, host_omega=host))
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        out["variants"][name] = {"sigma_rel": sigma_rel(r.S, o["S"]), "subspace_U": subspace_dist(o["U"], r.U),
                                 "subspace_V": subspace_dist(o["V"], r.V)}
        print(name, out["variants"][name], file=sys.stderr, flush=True)
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        with open(a.out, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
