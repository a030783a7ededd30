"""GPU parity of frpca / frpcat / auto_pca against the CPU oracle, through the
C ABI. Mirrors proj/tests/test_randsvd.cpp for the fast algorithms and the
north_star bar: with Omega from the same seed, top-k singular values within
1e-10 relative and ||UU^T - U'U'^T||_2 <= 1e-8 (V likewise)."""
import numpy as np
import pytest

from metrics import SIGMA_TOL, SUBSPACE_TOL, orthonormality, sigma_rel, subspace_dist
from test_gpu_kernels import powerlaw_csr, to_fb

pytestmark = pytest.mark.gpu


def cfg(fb, k, s, q, seed=0, host=False):
    return fb.PcaConfig(k=k, oversample=s, passes=q, seed=seed, host_omega=host)


def check_invariants(r):  # test_randsvd.cpp:37-43
    k = r.S.size
    assert orthonormality(r.U) < 1e-10 and orthonormality(r.V) < 1e-10
    assert np.all(np.diff(r.S) <= 0) and r.S[k - 1] >= 0


def assert_parity(r, o):
    assert sigma_rel(r.S, o["S"]) <= SIGMA_TOL
    assert subspace_dist(o["U"], r.U) <= SUBSPACE_TOL
    assert subspace_dist(o["V"], r.V) <= SUBSPACE_TOL


def test_frpca_diag_wide(fb):  # test_randsvd.cpp:71-77
    A = fb.SparseMatrixCsr.from_triplets(5, 8, [(i, i, float(v)) for i, v in enumerate([5, 4, 3, 2, 1])])
    r = fb.frpca(A, cfg(fb, 2, 3, 6))
    assert abs(r.S[0] - 5) < 1e-8 and abs(r.S[1] - 4) < 1e-8
    check_invariants(r)


def test_frpcat_diag_tall(fb):  # test_randsvd.cpp:79-85
    A = fb.SparseMatrixCsr.from_triplets(8, 5, [(i, i, float(v)) for i, v in enumerate([5, 4, 3, 2, 1])])
    r = fb.frpcat(A, cfg(fb, 2, 3, 11))
    assert abs(r.S[0] - 5) < 1e-8 and abs(r.S[1] - 4) < 1e-8
    check_invariants(r)


@pytest.mark.parametrize("q", [2, 3, 4, 5])
def test_exact_rank3_recovery(fb, orc, q):  # test_randsvd.cpp:87-104
    u = orc.gaussian_matrix(100, 3, 11)
    v = orc.gaussian_matrix(3, 80, 12)
    D = u @ v
    ii, jj = np.nonzero(D)
    A = fb.SparseMatrixCsr.from_triplets(100, 80, (ii, jj, D[ii, jj]))
    At = fb.transpose(A)
    na = np.linalg.norm(D)
    f = fb.frpca(At, cfg(fb, 3, 0, q))
    assert np.linalg.norm(D.T - (f.U * f.S) @ f.V.T) < 1e-8 * na
    t = fb.frpcat(A, cfg(fb, 3, 0, q))
    assert np.linalg.norm(D - (t.U * t.S) @ t.V.T) < 1e-8 * na


def test_zero_matrix_rejected(fb):  # test_randsvd.cpp:106-111
    Z = fb.SparseMatrixCsr.from_triplets(6, 6, [])
    with pytest.raises(fb.NumericalError):
        fb.frpcat(Z, cfg(fb, 2, 1, 4))
    with pytest.raises(fb.NumericalError):
        fb.frpca(Z, cfg(fb, 2, 1, 3))


def test_auto_dispatch(fb, orc):  # test_randsvd.cpp:182-190
    c = cfg(fb, 4, 5, 4)
    assert fb.auto_pca(to_fb(fb, orc.Csr.random_sparse(80, 120, 0.2, 91)), c).dispatched == fb.PcaAlgorithm.Frpca
    assert fb.auto_pca(to_fb(fb, orc.Csr.random_sparse(120, 80, 0.2, 92)), c).dispatched == fb.PcaAlgorithm.Frpcat
    assert fb.auto_pca(to_fb(fb, orc.Csr.random_sparse(100, 100, 0.2, 93)), c).dispatched == fb.PcaAlgorithm.Frpcat


@pytest.mark.parametrize("q", [2, 3, 4, 5, 6, 9, 11])
def test_pass_accounting(fb, orc, q):  # test_randsvd.cpp:192-209
    oA = orc.Csr.random_sparse(50, 70, 0.3, 55)
    A = to_fb(fb, oA)
    At = to_fb(fb, oA.transpose())
    st = fb.RunStats()
    fb.frpca(A, cfg(fb, 4, 4, q), st)
    assert st.passes_over_matrix == q
    fb.frpcat(At, cfg(fb, 4, 4, q), st)
    assert st.passes_over_matrix == q


@pytest.mark.parametrize("q", [2, 3, 4, 7])
def test_invariants(fb, orc, q):  # test_randsvd.cpp:211-223
    o = orc.Csr.random_sparse(60, 100, 0.2, 61)
    check_invariants(fb.frpca(to_fb(fb, o), cfg(fb, 6, 5, q, seed=q)))
    check_invariants(fb.frpcat(to_fb(fb, o.transpose()), cfg(fb, 6, 5, q, seed=q)))


@pytest.mark.parametrize("k,s,q,algo,shape,msg", [
    (28, 5, 4, "frpca", (30, 40), "k \\+ oversample"),
    (2, 5, 1, "frpca", (30, 40), "pass count"),
    (0, 5, 4, "frpca", (30, 40), "rank k"),
    (2, 5, 4, "frpcat", (30, 40), "requires rows >= cols"),
    (2, 5, 4, "frpca", (40, 30), "requires rows <= cols"),
])
def test_preconditions(fb, orc, k, s, q, algo, shape, msg):  # test_randsvd.cpp:253-262
    A = to_fb(fb, orc.Csr.random_sparse(shape[0], shape[1], 0.3, 99))
    with pytest.raises(ValueError, match=msg):
        getattr(fb, algo)(A, cfg(fb, k, s, q))


def test_bitwise_determinism(fb, orc):  # test_randsvd.cpp:264-271
    A = to_fb(fb, orc.Csr.random_sparse(50, 80, 0.2, 101))
    a = fb.frpca(A, cfg(fb, 5, 5, 5, seed=2024))
    b = fb.frpca(A, cfg(fb, 5, 5, 5, seed=2024))
    assert np.array_equal(a.S, b.S) and np.array_equal(a.U, b.U) and np.array_equal(a.V, b.V)


def test_injected_sketch_wrong_shape(fb, orc):  # randsvd.hpp:68-74
    A = to_fb(fb, orc.Csr.random_sparse(40, 30, 0.3, 5))
    with pytest.raises(ValueError, match="wrong shape"):
        fb.frpcat(A, cfg(fb, 4, 2, 3), omega=np.zeros((5, 5)))


# ---- parity vs the oracle on identical inputs (seeded Omega) ---------------

@pytest.mark.parametrize("q", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("host", [False, True])
def test_frpcat_parity_random(fb, orc, q, host):
    oA = orc.Csr.random_sparse(600, 300, 0.05, 1234)
    r = fb.frpcat(to_fb(fb, oA), cfg(fb, 10, 10, q, seed=3, host=host))
    o = orc.pca(oA, orc.FRPCAT, 10, 10, q, seed=3)
    assert_parity(r, o)


@pytest.mark.parametrize("q", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("host", [False, True])
def test_frpca_parity_random(fb, orc, q, host):
    oA = orc.Csr.random_sparse(300, 600, 0.05, 4321)
    r = fb.frpca(to_fb(fb, oA), cfg(fb, 10, 10, q, seed=5, host=host))
    o = orc.pca(oA, orc.FRPCA, 10, 10, q, seed=5)
    assert_parity(r, o)


@pytest.mark.parametrize("q", [3, 4, 5])
def test_frpcat_parity_powerlaw_l200(fb, orc, q):
    """l = 200 (the BASELINE width) on a power-law matrix with long rows."""
    oA = powerlaw_csr(orc, 20000, 4000, 400000, 17, a_row=1.8, a_col=1.05)
    r = fb.frpcat(to_fb(fb, oA), cfg(fb, 100, 100, q, seed=0))
    o = orc.pca(oA, orc.FRPCAT, 100, 100, q, seed=0)
    assert_parity(r, o)


@pytest.mark.parametrize("q", [3, 4])
def test_frpca_parity_powerlaw_l200(fb, orc, q):
    oA = powerlaw_csr(orc, 3000, 30000, 400000, 19, a_row=1.2, a_col=1.2)
    r = fb.frpca(to_fb(fb, oA), cfg(fb, 100, 100, q, seed=0))
    o = orc.pca(oA, orc.FRPCA, 100, 100, q, seed=0)
    assert_parity(r, o)


@pytest.mark.parametrize("algo", ["frpcat", "frpca"])
def test_parity_panelled_aty(fb, orc, monkeypatch, algo):
    """The panelled A^T*Y path (engaged by size on C1-C4) forced at test size."""
    monkeypatch.setenv("FRPCA_PANEL_MIN_MB", "0")
    monkeypatch.setenv("FRPCA_PANEL_MB", "0.5")
    if algo == "frpcat":
        oA = powerlaw_csr(orc, 20000, 4000, 400000, 23, a_row=1.8, a_col=1.05)
    else:
        oA = powerlaw_csr(orc, 3000, 30000, 400000, 29, a_row=1.2, a_col=1.2)
    f = fb.frpcat if algo == "frpcat" else fb.frpca
    r = f(to_fb(fb, oA), cfg(fb, 100, 100, 4, seed=0))
    o = orc.pca(oA, orc.FRPCAT if algo == "frpcat" else orc.FRPCA, 100, 100, 4, seed=0)
    assert_parity(r, o)


def test_injected_omega_parity(fb, orc):
    oA = orc.Csr.random_sparse(500, 200, 0.05, 77)
    om = orc.gaussian_matrix(12, 500, 42)  # even q frpcat: Omega is l x m
    r = fb.frpcat(to_fb(fb, oA), cfg(fb, 8, 4, 4), omega=om)
    o = orc.pca(oA, orc.FRPCAT, 8, 4, 4, omega=om)
    assert_parity(r, o)


def test_capture_basis(fb, orc):
    oA = orc.Csr.random_sparse(400, 150, 0.05, 8)
    st = fb.RunStats(capture_basis=True)
    fb.frpcat(to_fb(fb, oA), cfg(fb, 8, 4, 3, host=True), st)
    o = orc.pca(oA, orc.FRPCAT, 8, 4, 3, want_basis=True)
    assert st.basis.shape == o["basis"].shape
    assert subspace_dist(o["basis"], st.basis) < 1e-9


@pytest.mark.parametrize("algo,shape,q", [(1, (20000, 4000), 4), (1, (20000, 4000), 3), (0, (3000, 30000), 4),
                                          (0, (3000, 30000), 5), (3, (3000, 2000), 2), (4, (3000, 2000), 2)])
def test_run_csr_equals_upload_and_run(fb, orc, algo, shape, q):
    """frpca_run_csr (sketch generated on a second stream during the upload)
    gives bitwise the result of upload + frpca_run."""
    m, n = shape
    oA = powerlaw_csr(orc, m, n, 300000, 41, a_row=1.5, a_col=1.1)
    A = to_fb(fb, oA)
    c = fb.PcaConfig(k=20, oversample=12, passes=q, power=1, seed=9)
    r1, d1 = fb.run_csr(A, c, fb.PcaAlgorithm(algo))
    f = {0: fb.frpca, 1: fb.frpcat, 3: fb.basic_rpca, 4: fb.basic_rpcat}[algo]
    r2 = f(to_fb(fb, oA), c)
    assert d1 == algo
    assert np.array_equal(r1.S, r2.S) and np.array_equal(r1.U, r2.U) and np.array_equal(r1.V, r2.V)


@pytest.mark.parametrize("k,s", [(135, 14), (129, 0), (140, 9), (100, 31), (200, 33), (64, 63), (150, 0)])
@pytest.mark.parametrize("algo,shape,q", [(1, (1067, 551), 4), (1, (1067, 551), 2), (1, (1067, 551), 3),
                                          (0, (600, 2400), 4), (0, (600, 2400), 3)])
def test_run_csr_odd_widths(fb, orc, algo, shape, q, k, s):
    """The pipelined one-shot call at odd sketch widths past 128 columns: the
    scalar SpMM path runs in slices of <= 128 columns that re-use the partial
    buffer, so its item chunks must not alternate between two streams (found
    by the randomised sweep: sigma off by 7e-3 at l = 149, even q). Long rows
    (chunked, combined) and several item chunks; bitwise equal to upload + run."""
    m, n = shape
    oA = powerlaw_csr(orc, m, n, 60000, 19, a_row=1.3, a_col=1.1)
    A = to_fb(fb, oA)
    c = fb.PcaConfig(k=k, oversample=s, passes=q, seed=5)
    f = {0: fb.frpca, 1: fb.frpcat}[algo]
    r2 = f(to_fb(fb, oA), c)
    for _ in range(3):
        r1, _ = fb.run_csr(A, c, fb.PcaAlgorithm(algo))
        assert np.array_equal(r1.S, r2.S) and np.array_equal(r1.U, r2.U) and np.array_equal(r1.V, r2.V)


def test_run_csr_sweep_case(fb):
    """The sweep's own reproducer of that defect (tests/golden/run_csr/: case 77 of
    `tools/fuzz_parity.py --seed 52 --kinds pca --kmax 170 --smax 80 --dump`,
    1067 x 551, l = 149, q = 4)."""
    import os
    z = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "run_csr", "case_52_77.npz"))
    m, n, k, s, q, seed = (int(z[x]) for x in ("m", "n", "k", "s", "q", "seed"))
    A = fb.SparseMatrixCsr(m, n, z["rp"], z["ci"], z["va"])
    c = fb.PcaConfig(k=k, oversample=s, passes=q, seed=seed)
    r2 = fb.frpcat(A, c)
    r1, _ = fb.run_csr(A, c, fb.PcaAlgorithm.Frpcat)
    assert np.array_equal(r1.S, r2.S) and np.array_equal(r1.U, r2.U) and np.array_equal(r1.V, r2.V)


def _raw_run_csr(fb, m, n, rp, ci, va, algo, k=8, s=4, q=3):
    """frpca_run_csr straight through the C ABI (no host-side validation on
    the way): the pipelined upload's own checks are what is tested."""
    import ctypes as C
    from paper_1810_06825_b200 import _lib
    ctx = fb.default_context()
    U, S, V = np.empty(m * k), np.empty(k), np.empty(n * k)
    c = fb.PcaConfig(k=k, oversample=s, passes=q, seed=5).to_c()
    _lib.check(_lib.load().frpca_run_csr(ctx._h, m, n, int(rp[-1]), rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                         algo, C.byref(c), None, 0, 0, U.ctypes.data, S.ctypes.data,
                                         V.ctypes.data, None, None, None))
    return S


@pytest.mark.parametrize("algo", [1, 0])
@pytest.mark.parametrize("bad,msg", [("col_range", "csr: column index out of range"),
                                     ("col_order", "csr: column indices must be strictly increasing within a row"),
                                     ("rowptr", "csr: row_ptr must be non-decreasing")])
def test_run_csr_invalid_input_pipelined(fb, orc, algo, bad, msg):
    """The pipelined upload of frpca_run_csr (values in chunks, A^T built by
    a builder thread beside the first A*X) reports an invalid CSR with the
    reference's message (sparse_matrix.hpp:125-142) before any product, and
    the context stays usable: the next call equals upload + run bitwise."""
    shape = (20000, 4000) if algo == 1 else (4000, 20000)
    oA = powerlaw_csr(orc, shape[0], shape[1], 300000, 43, a_row=1.5, a_col=1.1)
    rp, ci, va = (np.ascontiguousarray(x) for x in oA.arrays())
    ci = ci.astype(np.int64).copy()
    rp = rp.astype(np.int64).copy()
    m, n = shape
    lens = np.diff(rp)
    r = int(np.nonzero(lens >= 3)[0][len(np.nonzero(lens >= 3)[0]) // 2])
    if bad == "col_range":
        ci[rp[r] + 1] = n
    elif bad == "col_order":
        ci[rp[r]], ci[rp[r] + 1] = ci[rp[r] + 1], ci[rp[r]]
    else:
        rp[r + 1] = rp[r] - 1 if rp[r] > 0 else rp[r + 2] + 1
    with pytest.raises(ValueError, match=msg):
        _raw_run_csr(fb, m, n, rp, ci, va.astype(np.float64), algo)
    rp0, ci0, va0 = (np.ascontiguousarray(x) for x in oA.arrays())
    S1 = _raw_run_csr(fb, m, n, rp0.astype(np.int64), ci0.astype(np.int64), va0.astype(np.float64), algo)
    f = fb.frpcat if algo == 1 else fb.frpca
    r2 = f(to_fb(fb, oA), fb.PcaConfig(k=8, oversample=4, passes=3, seed=5))
    assert np.array_equal(S1, r2.S)


def test_run_csr_repeated_shapes_reuse_buffers(fb, orc):
    """Large device buffers are recycled between calls (common.cuh BufCache):
    alternating shapes and algorithms through frpca_run_csr still give
    bitwise the results of a fresh upload + run."""
    cases = [(1, (30000, 5000), 600000, 3), (0, (5000, 30000), 600000, 4), (1, (30000, 5000), 600000, 3),
             (1, (40000, 6000), 900000, 4), (0, (5000, 30000), 600000, 4)]
    for algo, shape, nnz, q in cases:
        oA = powerlaw_csr(orc, shape[0], shape[1], nnz, 47 + q, a_row=1.5, a_col=1.1)
        A = to_fb(fb, oA)
        c = fb.PcaConfig(k=16, oversample=8, passes=q, seed=3)
        r1, _ = fb.run_csr(A, c, fb.PcaAlgorithm(algo))
        r2 = (fb.frpcat if algo == 1 else fb.frpca)(to_fb(fb, oA), c)
        assert np.array_equal(r1.S, r2.S) and np.array_equal(r1.U, r2.U) and np.array_equal(r1.V, r2.V)


def test_run_csr_errors(fb, orc):
    A = to_fb(fb, orc.Csr.random_sparse(50, 40, 0.2, 3))
    with pytest.raises(ValueError, match="frpca: requires rows <= cols"):
        fb.run_csr(A, fb.PcaConfig(k=3, oversample=2, passes=4), fb.PcaAlgorithm.Frpca)
    with pytest.raises(fb.NumericalError):
        fb.run_csr(fb.SparseMatrixCsr.from_triplets(6, 6, []), fb.PcaConfig(k=2, oversample=1, passes=4))


# ---- deferred errors (Ctx::dflag): retries and messages --------------------

def test_eig_noconv_retry_with_cusolver(fb, orc, monkeypatch):
    """A small-eigensolver non-convergence is recorded on the device and read
    once at the end of the call, which then re-runs with cuSOLVER: same
    answer as FRPCA_EIG=cusolver; FRPCA_EIG=strict turns it into an error."""
    oA = powerlaw_csr(orc, 3000, 800, 60000, 3)
    A = to_fb(fb, oA)
    c = cfg(fb, 20, 20, 4)
    monkeypatch.setenv("FRPCA_EIG", "cusolver")
    ref = fb.frpcat(A, c)
    monkeypatch.delenv("FRPCA_EIG")
    monkeypatch.setenv("FRPCA_TEST_EIG_NOCONV", "1")
    st = fb.RunStats()
    r = fb.frpcat(A, c, st)
    assert np.array_equal(r.S, ref.S) and np.array_equal(r.U, ref.U) and np.array_equal(r.V, ref.V)
    assert st.passes_over_matrix == 4
    monkeypatch.setenv("FRPCA_EIG", "strict")
    with pytest.raises(Exception, match="did not converge"):
        fb.frpcat(A, c)


def test_omega_shortfall_retry(fb, orc, monkeypatch):
    """The single-batch Omega defers its shortfall test to the end of the
    call; a shortfall re-runs the call with the host-checked batch loop."""
    oA = orc.Csr.random_sparse(600, 300, 0.05, 1234)
    A = to_fb(fb, oA)
    for q in (3, 4):
        ref = fb.frpcat(A, cfg(fb, 10, 10, q, seed=3))
        monkeypatch.setenv("FRPCA_TEST_OMEGA_SHORT", "1")
        r = fb.frpcat(A, cfg(fb, 10, 10, q, seed=3))
        monkeypatch.delenv("FRPCA_TEST_OMEGA_SHORT")
        assert np.array_equal(r.S, ref.S) and np.array_equal(r.U, ref.U)
    g0 = fb.gaussian_matrix(5000, 7, 9)
    monkeypatch.setenv("FRPCA_TEST_OMEGA_SHORT", "1")
    assert np.array_equal(fb.gaussian_matrix(5000, 7, 9), g0)


@pytest.mark.parametrize("log2s", ["6", "8", "10", "13"])
def test_omega_segment_length(fb, orc, monkeypatch, log2s):
    """The device stream does not depend on how it is cut into jump-ahead
    segments (FRPCA_OMEGA_LOG2S): bitwise equal to the default cut, and to
    the oracle's std::mt19937_64 + normal_distribution stream."""
    g0 = fb.gaussian_matrix(30000, 40, 5)
    monkeypatch.setenv("FRPCA_OMEGA_LOG2S", log2s)
    g1 = fb.gaussian_matrix(30000, 40, 5)
    assert np.array_equal(g0, g1)
    o = orc.gaussian_matrix(30000, 40, 5)
    assert np.array_equal(g1, o)


def test_deferred_error_then_clean_call(fb, orc):
    """A failed call (zero pivot / rank deficiency, reported at its end) leaves
    no state behind: the next call on the same context succeeds."""
    Z = fb.SparseMatrixCsr.from_triplets(50, 20, [])
    with pytest.raises(fb.NumericalError):
        fb.frpcat(Z, cfg(fb, 3, 2, 4))
    with pytest.raises(fb.NumericalError):
        fb.frpcat(Z, cfg(fb, 3, 2, 3))
    oA = orc.Csr.random_sparse(600, 300, 0.05, 1234)
    r = fb.frpcat(to_fb(fb, oA), cfg(fb, 10, 10, 4, seed=3))
    o = orc.pca(oA, orc.FRPCAT, 10, 10, 4, seed=3)
    assert_parity(r, o)
