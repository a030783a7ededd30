"""Where does a graded power-iteration panel lose accuracy? Steps frpcat (q even)
by hand through the product's kernel entry points and through the oracle on one
saved fuzz case and prints, per eig_svd, the loss of orthonormality of Q =
Z V S^-1 and the spectrum's grading; then the effect of a symmetric
re-orthonormalisation Q (Q^T Q)^-1/2 on the final sigma. Probe, not product."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as orc  # noqa: E402
import paper_1810_06825_b200 as fb  # noqa: E402
from metrics import sigma_rel, subspace_dist  # noqa: E402


def steps(lib, A, Om, q, fix=False, tag=""):
    Y = lib.spmm_transpose(A, np.ascontiguousarray(Om.T))
    loops = (q - 1) // 2
    Q = lib.eig_svd(Y)[0] if q == 2 else lib.lu_basis(Y)
    for i in range(1, loops + 1):
        Y = lib.spmm_transpose(A, lib.spmm(A, Q))
        if i == loops:
            U, S, V = lib.eig_svd(Y)
            E = U.T @ U - np.eye(U.shape[1])
            print(tag, "loop eig_svd: S max/min %.3g  |Q^TQ-I|max %.3g" % (S.max() / S.min(), np.abs(E).max()))
            if fix:
                U = U @ (np.eye(U.shape[1]) - E / 2 + 3.0 / 8.0 * (E @ E))
                print(tag, "  after fix |Q^TQ-I|max %.3g" % np.abs(U.T @ U - np.eye(U.shape[1])).max())
            Q = U
        else:
            Q = lib.lu_basis(Y)
    U, S, V = lib.eig_svd(lib.spmm(A, Q))
    print(tag, "final eig_svd: S max/min %.3g |U^TU-I| %.3g" % (S.max() / S.min(), np.abs(U.T @ U - np.eye(U.shape[1])).max()))
    return U, S, Q @ V


def main():
    orc.build()
    z = np.load(sys.argv[1])
    m, n, k, s, q, seed = (int(z[x]) for x in ("m", "n", "k", "s", "q", "seed"))
    rp, ci, va = z["rp"], z["ci"], z["va"]
    oA = orc.Csr.create(m, n, rp, ci, va)
    A = fb.SparseMatrixCsr(m, n, rp, ci, va)
    l = k + s
    Om = orc.gaussian_matrix(l, m, orc.mix_seed(seed, 0xA11CE))
    arb = orc.arbiter_pca(m, n, rp, ci, va, orc.FRPCAT, k, s, q, seed=seed)
    full = orc.pca(oA, orc.FRPCAT, k, s, seed=seed, passes=q)

    def top(U, S, V):
        return {"U": U[:, s:s + k][:, ::-1], "S": S[s:s + k][::-1], "V": V[:, s:s + k][:, ::-1]}

    def report(tag, r):
        print(tag, "vs arbiter: sigma %.3g U %.3g V %.3g" % (sigma_rel(r["S"], arb["S"]), subspace_dist(arb["U"], r["U"]),
                                                         subspace_dist(arb["V"], r["V"])))
    report("oracle.pca      ", full)

    class O:  # oracle through the same stepping code
        spmm = staticmethod(lambda A_, X: orc.spmm(oA, X))
        spmm_transpose = staticmethod(lambda A_, Y: orc.spmm_transpose(oA, Y))
        lu_basis = staticmethod(orc.lu_basis)
        eig_svd = staticmethod(orc.eig_svd)
    report("oracle stepped  ", top(*steps(O, None, Om, q, tag="  [oracle]")))
    report("gpu stepped     ", top(*steps(fb, A, Om, q, tag="  [gpu]")))
    report("gpu stepped+fix ", top(*steps(fb, A, Om, q, fix=True, tag="  [gpu+fix]")))
    for mode in ("small", "cusolver"):
        os.environ["FRPCA_EIG"] = mode
        report("gpu stepped FRPCA_EIG=" + mode, top(*steps(fb, A, Om, q, tag="  [gpu %s]" % mode)))
    del os.environ["FRPCA_EIG"]
    st = fb.RunStats()
    st.capture_basis = True
    r = fb.frpcat(A, fb.PcaConfig(k=k, oversample=s, passes=q, seed=seed), st)
    report("gpu frpcat      ", {"U": r.U, "S": r.S, "V": r.V})
    ob = orc.pca(oA, orc.FRPCAT, k, s, seed=seed, passes=q, want_basis=True)["basis"]
    I = np.eye(l)
    print("captured basis |Q^TQ-I|max: gpu %.3g oracle %.3g" % (np.abs(st.basis.T @ st.basis - I).max(), np.abs(ob.T @ ob - I).max()))
    r2 = fb.frpcat(A, fb.PcaConfig(k=k, oversample=s, passes=q, seed=seed), omega=Om)
    report("gpu frpcat, Omega injected", {"U": r2.U, "S": r2.S, "V": r2.V})


if __name__ == "__main__":
    main()
