"""Randomised parity sweep of the product (CUDA, through the C ABI) against the
CPU oracle: `python tools/fuzz_parity.py [--cases N] [--seed S]`.

Each case draws a shape, a sparsity law (uniform, power-law rows and columns,
empty rows/columns, a few very long rows), a panel width and an algorithm and
checks the north_star bars: SpMM Frobenius-relative <= 1e-12, sigma <= 1e-10
relative, subspaces <= 1e-8; lu_basis / orth / eig_svd entry by entry. A fast
run above the direct bars (ill-conditioned q-pass products, where two fp64
evaluations of the reference algorithm differ by more than the bar) is judged
against the long-double arbiter: GPU-to-arbiter <= 4 x oracle-to-arbiter, the
oracle evaluated with both of its eigensolvers (Jacobi and the reference's own
class, tridiagonal QL), whichever is farther. A case
the oracle rejects must be rejected by the product with the same message
class. Prints one JSON line with the worst value of every metric and the
failing cases (none expected). Test infrastructure: the oracle is the checker."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
import paper_1810_06825_b200 as fb  # noqa: E402
from metrics import rel_fro, sigma_rel, subspace_dist  # noqa: E402


def random_csr(rng, m, n):
    law = rng.integers(0, 4)
    if law == 0:  # uniform density
        dens = float(rng.choice([0.002, 0.01, 0.05, 0.3]))
        nnz = max(1, int(m * n * dens))
        r = rng.integers(0, m, nnz)
        c = rng.integers(0, n, nnz)
    else:  # power-law rows and columns; law 2 leaves empty rows, law 3 adds very long rows
        a_row = float(rng.choice([1.3, 1.8, 2.5]))
        deg = np.minimum(rng.zipf(a_row, m), n)
        if law == 2:
            deg[rng.random(m) < 0.3] = 0
        if law == 3:
            deg[rng.integers(0, m, 3)] = n
        perm = rng.permutation(n)
        rs, cs = [], []
        for i, d in enumerate(deg):
            if d == 0:
                continue
            cc = np.unique(np.minimum(rng.zipf(1.15, 2 * int(d) + 8), n) - 1)[: int(d)]
            if d == n:
                cc = np.arange(n)
            rs.append(np.full(cc.size, i))
            cs.append(perm[cc])
        if not rs:
            rs, cs = [np.array([0])], [np.array([0])]
        r = np.concatenate(rs)
        c = np.concatenate(cs)
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = key // n, key % n
    kind = rng.integers(0, 3)
    v = rng.standard_normal(r.size) if kind == 0 else (rng.poisson(1.0, r.size) + 1.0 if kind == 1
                                                       else np.exp(rng.standard_normal(r.size) * 3))
    rp = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    return orc.Csr.create(m, n, rp, c.astype(np.int64), v)


def big_csr(rng, m, n, nnz):
    """Large case, vectorised: uniform rows, Zipf columns over a permutation, a few long rows."""
    r = rng.integers(0, m, nnz)
    r[: nnz // 20] = rng.integers(0, 3)  # three long rows (chunked + combined)
    c = rng.permutation(n)[np.minimum(rng.zipf(1.2, nnz), n) - 1]
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = key // n, key % n
    v = rng.standard_normal(r.size)
    rp = np.zeros(m + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    return orc.Csr.create(m, n, np.cumsum(rp), c.astype(np.int64), v)


def to_fb(oA):
    rp, ci, va = oA.arrays()
    return fb.SparseMatrixCsr(oA.rows, oA.cols, rp, ci, va)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=150)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--kinds", default="spmm,pca,pca,dense,basic,load,valid", help="case kinds, dealt round-robin")
    ap.add_argument("--kmax", type=int, default=60)
    ap.add_argument("--smax", type=int, default=40)
    ap.add_argument("--qmax", type=int, default=7, help="largest pass count q of the fast algorithms")
    ap.add_argument("--only", type=int, nargs="*", help="evaluate only these case numbers (same draws)")
    ap.add_argument("--dump", default="", help="directory: save the CSR and parameters of the evaluated pca cases")
    a = ap.parse_args()
    orc.build()
    rng = np.random.default_rng(a.seed)
    worst = {}
    fails = []
    counts = {}
    noisy = []

    def note(name, val, bar, case):
        worst[name] = max(worst.get(name, 0.0), float(val))
        if not val <= bar:
            fails.append({"case": case, "metric": name, "value": float(val), "bar": bar})

    t0 = time.time()
    for it in range(a.cases):
        kinds = a.kinds.split(",")
        kind = kinds[it % len(kinds)]
        case = {"i": it, "kind": kind}
        skip = a.only is not None and it not in a.only
        if not skip:
            counts[kind] = counts.get(kind, 0) + 1
        try:
            if kind == "spmm":
                m, n = int(rng.integers(1, 4000)), int(rng.integers(1, 3000))
                w = int(rng.choice([1, 2, 3, 7, 31, 32, 33, 64, 100, 129, 200, 256, 257, 300]))
                if rng.random() < 0.2:
                    # large enough for the L2 hints of A*X and the panel plan of A^T*Y
                    m, n = int(rng.integers(60000, 400000)), int(rng.integers(20000, 120000))
                    w = int(rng.choice([64, 150, 200, 256]))
                    oA = big_csr(rng, m, n, int(rng.integers(1, 5) * 1000000))
                else:
                    oA = random_csr(rng, m, n)
                A = to_fb(oA)
                case.update(m=m, n=n, w=w)
                X = rng.standard_normal((n, w))
                Y = rng.standard_normal((m, w))
                if skip:
                    continue
                note("spmm", rel_fro(fb.spmm(A, X), orc.spmm(oA, X)), 1e-12, case)
                note("spmm_transpose", rel_fro(fb.spmm_transpose(A, Y), orc.spmm_transpose(oA, Y)), 1e-12, case)
            elif kind in ("pca", "basic"):
                m, n = int(rng.integers(8, 3000)), int(rng.integers(8, 3000))
                # a third of the cases are long in one dimension: the dense
                # kernels switch to their persistent variants at 4096 rows
                stretch = int(rng.integers(0, 3))
                if stretch == 0:
                    if rng.random() < 0.5:
                        m = int(rng.integers(4096, 14000))
                    else:
                        n = int(rng.integers(4096, 14000))
                lmax = min(m, n)
                k = int(rng.integers(1, max(2, min(lmax, a.kmax))))
                s = int(rng.integers(0, max(1, min(lmax - k, a.smax)) + 1))
                s = min(s, lmax - k)
                q = int(rng.integers(2, a.qmax + 1)) if kind == "pca" else int(rng.integers(0, 3))
                oA = random_csr(rng, m, n)
                A = to_fb(oA)
                seed = int(rng.integers(0, 1 << 30))
                if kind == "pca":
                    algo = orc.FRPCA if m <= n else orc.FRPCAT
                    if m == n and rng.random() < 0.5:
                        algo = orc.FRPCAT
                    f = fb.frpca if algo == orc.FRPCA else fb.frpcat
                    cfg = fb.PcaConfig(k=k, oversample=s, passes=q, seed=seed)
                    kw = dict(passes=q)
                else:
                    algo = orc.BASIC_RPCA if rng.random() < 0.5 else orc.BASIC_RPCAT
                    f = fb.basic_rpca if algo == orc.BASIC_RPCA else fb.basic_rpcat
                    cfg = fb.PcaConfig(k=k, oversample=s, power=q, seed=seed)
                    kw = dict(power=q)
                if skip:
                    continue
                case.update(m=m, n=n, k=k, s=s, q=q, algo=int(algo), seed=seed)
                if a.dump and kind == "pca":
                    rp_, ci_, va_ = oA.arrays()
                    np.savez(os.path.join(a.dump, "case_%d_%d.npz" % (a.seed, it)), rp=rp_, ci=ci_, va=va_, m=m, n=n,
                             k=k, s=s, q=q, seed=seed, algo=int(algo))
                try:
                    o = orc.pca(oA, algo, k, s, seed=seed, **kw)
                except (orc.NumericalError, ValueError) as e:
                    try:
                        f(A, cfg)
                        fails.append({"case": case, "metric": "oracle rejected, product accepted", "value": str(e)})
                    except (fb.NumericalError, ValueError):
                        counts["rejected_by_both"] = counts.get("rejected_by_both", 0) + 1
                    continue
                r = f(A, cfg)
                if kind == "pca":
                    # the one-shot call from host buffers (frpca_run_csr: upload
                    # pipelined with the sketch and the first product) must be
                    # the same computation as upload + run
                    r1, _ = fb.run_csr(A, cfg, fb.PcaAlgorithm.Frpca if algo == orc.FRPCA else fb.PcaAlgorithm.Frpcat)
                    same = np.array_equal(r1.S, r.S) and np.array_equal(r1.U, r.U) and np.array_equal(r1.V, r.V)
                    if not same:
                        case["run_csr_vs_upload_run"] = {"sigma": sigma_rel(r1.S, r.S), "U": subspace_dist(r.U, r1.U),
                                                         "V": subspace_dist(r.V, r1.V)}
                    note("run_csr_differs_from_upload_run", 0.0 if same else 1.0, 0.0, case)
                    if it % 4 == 0:
                        # the sharded drivers through the loopback group (2 or 3
                        # ranks on this device) against the unsharded run
                        world = 2 + (it // 4) % 2
                        g = fb.Group([0] * world)
                        try:
                            rg, _ = g.run(A, cfg, fb.PcaAlgorithm.Frpca if algo == orc.FRPCA else fb.PcaAlgorithm.Frpcat)
                        finally:
                            g.close()
                        counts["sharded"] = counts.get("sharded", 0) + 1
                        sharded = {"S": rg.S, "U": rg.U, "V": rg.V}
                else:
                    sharded = None
                if kind != "pca" or it % 4 != 0:
                    sharded = None
                # the bars hold where the k-th singular value is separated from
                # round-off: a numerically rank-deficient case is compared on
                # its well-conditioned leading part only
                good = o["S"] > 1e-6 * o["S"][0]
                kk = int(good.sum())
                if kk < k:
                    counts["partly_degenerate"] = counts.get("partly_degenerate", 0) + 1
                def dist(x, y, kk=kk, k=k):
                    dd = {"sigma": sigma_rel(x["S"][:kk], y["S"][:kk]) if kk else 0.0}
                    if kk == k:
                        dd["U"] = subspace_dist(y["U"], x["U"])
                        dd["V"] = subspace_dist(y["V"], x["V"])
                    return dd
                bars = {"sigma": 1e-10, "U": 1e-8, "V": 1e-8}
                rr = {"S": r.S, "U": r.U, "V": r.V}
                d = dist(rr, o)
                if kind == "pca" and any(d[key] > bars[key] for key in d):
                    # above the direct bar: is it the algorithm's own fp64
                    # noise (eigSVD squares the condition of a q-pass
                    # product)? Judge both evaluations against the same
                    # pipeline in 80-bit long double (oracle/arbiter.cpp): the
                    # GPU must be no farther from it than a few times the
                    # oracle is.
                    rp, ci, va = oA.arrays()
                    arb = orc.arbiter_pca(m, n, rp, ci, va, algo, k, s, q, seed=seed)
                    g, c = dist(rr, arb), dist(o, arb)
                    # the oracle's Jacobi eigensolver resolves graded Gram
                    # matrices to relative accuracy, which the reference's own
                    # Eigen solver (tridiagonal QR, absolute accuracy) does
                    # not: the noise class is the larger of the oracle's two
                    # solvers (oracle.cpp eig_sym_lower_ql)
                    os.environ["FRPCA_ORACLE_EIG"] = "ql"
                    try:
                        cq = dist(orc.pca(oA, algo, k, s, seed=seed, **kw), arb)
                    except orc.NumericalError:
                        cq = {key: 0.0 for key in c}
                    finally:
                        del os.environ["FRPCA_ORACLE_EIG"]
                    noisy.append({"case": case, "gpu_vs_oracle": d, "gpu_vs_arbiter": g, "oracle_vs_arbiter": c,
                                  "oracle_ql_vs_arbiter": cq})
                    if sharded is not None:
                        gs, ds = dist(sharded, arb), dist(sharded, o)
                        for key in gs:
                            if ds[key] <= bars[key]:
                                note("sharded_" + key, ds[key], bars[key], case)
                            else:
                                note("sharded_arbiter_ratio_" + key,
                                     gs[key] / max(c[key], cq[key], bars[key] * 1e-3), 4.0, case)
                    for key in g:
                        if d[key] <= bars[key]:  # this metric meets its direct bar
                            note(kind + "_" + key, d[key], bars[key], case)
                        else:
                            note("arbiter_ratio_" + key, g[key] / max(c[key], cq[key], bars[key] * 1e-3), 4.0, case)
                else:
                    for key in d:
                        note(kind + "_" + key, d[key], bars[key], case)
                    if sharded is not None:
                        ds = dist(sharded, o)
                        if any(ds[key] > bars[key] for key in ds):
                            # a different split of the same sums: judged like the unsharded run
                            rp, ci, va = oA.arrays()
                            arb = orc.arbiter_pca(m, n, rp, ci, va, algo, k, s, q, seed=seed)
                            gs, c = dist(sharded, arb), dist(o, arb)
                            noisy.append({"case": case, "sharded_vs_oracle": ds, "sharded_vs_arbiter": gs,
                                          "oracle_vs_arbiter": c})
                        for key in ds:
                            if ds[key] <= bars[key]:
                                note("sharded_" + key, ds[key], bars[key], case)
                            else:
                                note("sharded_arbiter_ratio_" + key, gs[key] / max(c[key], bars[key] * 1e-3), 4.0, case)
            elif kind == "load":
                # from_triplets on the device (<= 2 entries per coordinate, exact
                # zeros dropped) and the Matrix Market writer/reader round trip
                m, n = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
                nt = int(rng.integers(0, 60000))
                r = rng.integers(0, m, nt)
                c = rng.integers(0, n, nt)
                key = np.unique(r.astype(np.int64) * n + c)
                r, c = key // n, key % n
                v = rng.standard_normal(r.size)
                dup = rng.random(r.size) < 0.2          # a second entry at the same coordinate
                cancel = rng.random(r.size) < 0.3       # ... a third of which cancel exactly
                r2, c2 = r[dup], c[dup]
                v2 = np.where(cancel[dup], -v[dup], rng.standard_normal(int(dup.sum())))
                order = rng.permutation(r.size + r2.size)
                tr = np.concatenate([r, r2])[order]
                tc = np.concatenate([c, c2])[order]
                tv = np.concatenate([v, v2])[order]
                case.update(m=m, n=n, triplets=int(tr.size))
                if skip:
                    continue
                oA = orc.Csr.from_triplets(m, n, list(zip(tr.tolist(), tc.tolist(), tv.tolist())))
                orp, oci, ova = oA.arrays()
                for dev in (False, True):
                    A = fb.SparseMatrixCsr.from_triplets(m, n, (tr, tc, tv), device=dev)
                    same = (np.array_equal(A.rowPtr(), orp) and np.array_equal(A.colIdx(), oci)
                            and np.array_equal(A.values(), ova))
                    note("from_triplets_device" if dev else "from_triplets_host", 0.0 if same else 1.0, 0.0, case)
                import tempfile
                with tempfile.TemporaryDirectory() as td:
                    path = os.path.join(td, "a.mtx")
                    fb.write_matrix_market(path, A)
                    B = fb.load_matrix_market(path)
                    same = (B.rows() == m and B.cols() == n and np.array_equal(B.rowPtr(), orp)
                            and np.array_equal(B.colIdx(), oci) and np.array_equal(B.values(), ova))
                    note("matrix_market_round_trip", 0.0 if same else 1.0, 0.0, case)
            elif kind == "valid":
                # validation metrics on the GPU against the oracle's (validation.hpp:125-332)
                m, n = int(rng.integers(20, 1500)), int(rng.integers(20, 1500))
                oA = random_csr(rng, m, n)
                A = to_fb(oA)
                k = int(rng.integers(1, min(m, n, 40)))
                seed = int(rng.integers(0, 1 << 30))
                case.update(m=m, n=n, k=k, seed=seed)
                if skip:
                    continue
                algo = orc.FRPCA if m <= n else orc.FRPCAT
                try:
                    o = orc.pca(oA, algo, k, min(5, min(m, n) - k), seed=seed, passes=3)
                except (orc.NumericalError, ValueError):
                    continue
                res = fb.SvdResult(o["U"], o["S"], o["V"])
                for norm, name in ((fb.ErrorNorm.Frobenius, "fro"), (fb.ErrorNorm.Spectral, "spec")):
                    e_o = orc.low_rank_error(oA, o["U"], o["S"], o["V"], int(norm))
                    e_g = fb.low_rank_error(A, res, norm)
                    note("low_rank_error_" + name, abs(e_g - e_o) / max(e_o, 1e-300), 1e-6 if name == "spec" else 1e-9, case)
                    e_g2 = fb.low_rank_error(A, res, norm, entry_limit=1)   # the matrix-free / cross-term path
                    note("low_rank_error_" + name + "_matrix_free", abs(e_g2 - e_o) / max(e_o, 1e-300),
                         1e-6 if name == "spec" else 1e-7, case)
                P = np.linalg.qr(rng.standard_normal((m, k)))[0]
                note("pc_correlation", np.abs(fb.pc_correlation(o["U"], P) - orc.pc_correlation(o["U"], P)).max(), 1e-12, case)
                def guarded(f):  # the reference rejects a basis that is not orthonormal within 1e-8
                    try:
                        return f(o["U"], P)
                    except ValueError as e:
                        return str(e)
                pg, po = guarded(fb.projector_distance), guarded(orc.projector_distance)
                if isinstance(pg, str) or isinstance(po, str):
                    note("projector_distance_rejection_differs", 0.0 if pg == po else 1.0, 0.0, case)
                else:
                    note("projector_distance", abs(pg - po), 1e-9, case)
            else:
                m = int(rng.integers(1, 6000))
                if rng.random() < 0.2:
                    m = int(rng.integers(6000, 300000))  # the global-panel LU, split Grams
                l = int(rng.integers(1, min(max(m // 2, 1), 300) + 1))  # well-conditioned Gaussian panels
                case.update(m=m, l=l)
                M = rng.standard_normal((m, l))
                if skip:
                    continue
                note("lu_basis", np.abs(fb.lu_basis(M) - orc.lu_basis(M)).max(), 1e-9, case)
                note("orth", np.abs(fb.orth(M) - orc.orth(M)).max(), 1e-10, case)
                if l <= m:
                    U, S, V = fb.eig_svd(M)
                    Uo, So, Vo = orc.eig_svd(M)
                    note("eig_svd_S", sigma_rel(S, So), 1e-10, case)
                    note("eig_svd_UV", np.abs((U * S) @ V.T - M).max(), 1e-10, case)
        except Exception as e:  # an unexpected failure of either side is a finding
            fails.append({"case": case, "metric": "exception", "value": repr(e)[:300]})
    print(json.dumps({"cases": a.cases, "seed": a.seed, "counts": counts, "worst": worst, "failures": fails,
                      "above_direct_bar_judged_by_arbiter": noisy,
                      "seconds": round(time.time() - t0, 1)}))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
