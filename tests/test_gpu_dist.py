"""The library's sharded path on one GPU: a group of ranks on the
same device exchanging through the host-staged loopback collective
(csrc/comm.cu), so every sharded code path of the library runs -- the shard
plan (csrc/group.cu), frpca_dmat_upload_shard, the row/column-sharded drivers
(csrc/driver.cu: Omega slices, the n x l / m x l partial allreduce, the Gram
allreduce of the rank-local final W, rank-local output rows) -- exactly as it
does over NCCL on several GPUs, only the transport differs.

Reference loops these shard: randsvd.hpp:255-258 (frpca), :307-310 (frpcat).
Bars: the sharded result against the unsharded run of the same library
(sigma 1e-10 relative, subspaces 1e-8), and against the oracle."""
import ctypes as C
import threading

import numpy as np
import pytest

from metrics import SIGMA_TOL, SUBSPACE_TOL, sigma_rel, subspace_dist

pytestmark = pytest.mark.gpu


def _matrix(fb, shape, seed=7, density=0.02):
    import oracle
    m, n = shape
    A = oracle.Csr.random_sparse(m, n, density, seed)
    rp, ci, va = A.arrays()
    return fb.SparseMatrixCsr(m, n, rp, ci, va), A


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("algo,shape", [("frpcat", (3000, 800)), ("frpca", (800, 3000))])
@pytest.mark.parametrize("q", [2, 3, 4, 5])
def test_group_loopback_matches_unsharded(fb, orc, ctx, world, algo, shape, q):
    A, oA = _matrix(fb, shape)
    cfg = fb.PcaConfig(k=12, oversample=8, passes=q, seed=3)
    one = (fb.frpcat if algo == "frpcat" else fb.frpca)(A, cfg)
    g = fb.Group([0] * world)
    try:
        st = fb.RunStats()
        r, disp = g.run(A, cfg, fb.PcaAlgorithm.Frpcat if algo == "frpcat" else fb.PcaAlgorithm.Frpca, st)
    finally:
        g.close()
    assert disp == (fb.PcaAlgorithm.Frpcat if algo == "frpcat" else fb.PcaAlgorithm.Frpca)
    assert st.passes_over_matrix == q
    assert sigma_rel(r.S, one.S) <= SIGMA_TOL
    assert subspace_dist(one.U, r.U) <= SUBSPACE_TOL and subspace_dist(one.V, r.V) <= SUBSPACE_TOL
    o = orc.pca(oA, orc.FRPCAT if algo == "frpcat" else orc.FRPCA, 12, 8, q, seed=3)
    assert sigma_rel(r.S, o["S"]) <= SIGMA_TOL
    assert subspace_dist(o["U"], r.U) <= SUBSPACE_TOL and subspace_dist(o["V"], r.V) <= SUBSPACE_TOL


def test_group_auto_dispatch_and_synth_law(fb, orc):
    """C1's law at reduced size through auto dispatch, 2 ranks on one GPU."""
    from paper_1810_06825_b200 import synth
    m, n, rp, ci, va = synth.generate("C1", scale=0.05)
    A = fb.SparseMatrixCsr(m, n, rp, ci, va)
    cfg = fb.PcaConfig(k=20, oversample=20, passes=4, seed=0)
    one = fb.frpcat(A, cfg)
    g = fb.Group([0, 0])
    try:
        r, disp = g.run(A, cfg)
    finally:
        g.close()
    assert disp == fb.PcaAlgorithm.Frpcat
    assert sigma_rel(r.S, one.S) <= SIGMA_TOL
    assert subspace_dist(one.U, r.U) <= SUBSPACE_TOL and subspace_dist(one.V, r.V) <= SUBSPACE_TOL


def test_per_rank_api_equals_group_run(fb):
    """The one-process-per-GPU API (frpca_dmat_upload_shard + frpca_run on each
    rank's context, what bench.py does under torchrun) gives bitwise the
    group run's result: same shards, same exchanges."""
    from paper_1810_06825_b200 import _lib, shard
    A, _ = _matrix(fb, (2500, 700), seed=11)
    cfg = fb.PcaConfig(k=10, oversample=10, passes=4, seed=1)
    world = 2
    g = fb.Group([0] * world)
    try:
        ref, _ = g.run(A, cfg, fb.PcaAlgorithm.Frpcat)
        L = _lib.load()
        m, n = A.rows(), A.cols()
        rp, ci, va = A.rowPtr(), A.colIdx(), A.values()
        U = np.zeros((m, cfg.k), order="F")
        S = np.zeros(cfg.k)
        V = np.zeros((n, cfg.k), order="F")
        errs = [None] * world
        ccfg = cfg.to_c()

        def rank_main(r):
            try:
                h = g.context_handle(r)
                r0, r1, lrp, lci, lva = shard.shard_rows(rp, ci, va, world, r)
                dm = C.c_void_p()
                _lib.check(L.frpca_dmat_upload_shard(h, m, n, 0, r0, r1 - r0, n, int(lrp[-1]), lrp.ctypes.data,
                                                     lci.ctypes.data, lva.ctypes.data, C.byref(dm)))
                Ul = np.zeros((r1 - r0, cfg.k), order="F")
                Sl = np.zeros(cfg.k)
                Vl = np.zeros((n, cfg.k), order="F")
                try:
                    _lib.check(L.frpca_run(h, dm, _lib.ALGO_FRPCAT, C.byref(ccfg), None, 0, 0, Ul.ctypes.data,
                                           Sl.ctypes.data, Vl.ctypes.data, None, None, None))
                finally:
                    L.frpca_dmat_destroy(dm)
                U[r0:r1] = Ul
                if r == 0:
                    S[:] = Sl
                    V[:] = Vl
            except Exception as e:  # noqa: BLE001
                errs[r] = e

        th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert errs == [None] * world, errs
    finally:
        g.close()
    assert np.array_equal(U, ref.U) and np.array_equal(S, ref.S) and np.array_equal(V, ref.V)


def test_group_errors_reach_every_rank(fb):
    """Preconditions and numerical errors surface with the reference's
    messages (randsvd.hpp:286, dense_kernels.hpp:81 / :167) from a sharded run,
    and the group stays usable afterwards."""
    g = fb.Group([0, 0])
    try:
        A, _ = _matrix(fb, (600, 200))
        with pytest.raises(ValueError, match="k \\+ oversample must be <= cols"):
            g.run(A, fb.PcaConfig(k=150, oversample=60, passes=3), fb.PcaAlgorithm.Frpcat)
        Z = fb.SparseMatrixCsr(600, 200, np.zeros(601, dtype=np.int64), [], [])
        with pytest.raises(fb.NumericalError):
            g.run(Z, fb.PcaConfig(k=5, oversample=5, passes=3), fb.PcaAlgorithm.Frpcat)
        r, _ = g.run(A, fb.PcaConfig(k=5, oversample=5, passes=3), fb.PcaAlgorithm.Frpcat)
        assert np.all(np.isfinite(r.S))
    finally:
        g.close()


def test_group_rejects_nccl_on_one_device(fb):
    from paper_1810_06825_b200 import _lib
    with pytest.raises(ValueError, match="NCCL needs distinct devices"):
        fb.Group([0, 0], comm=_lib.COMM_NCCL)


@pytest.mark.parametrize("rows,cols,r0,r1", [(1000, 7, 0, 1000), (1000, 7, 250, 600), (5000, 40, 4999, 5000),
                                             (3, 100000, 1, 2), (20000, 12, 0, 1), (300000, 40, 0, 300000),
                                             (300000, 41, 12345, 200001)])
def test_sketch_window_is_the_stream_slice(fb, ctx, rows, cols, r0, r1):
    """A rank's slice of the sketch (rows [r0, r1) of a column-major rows x
    cols Omega, or a contiguous run) is bitwise the corresponding part of the
    full stream (dense_kernels.hpp:19-28): only the emitted positions change."""
    import ctypes as C
    from paper_1810_06825_b200 import _lib
    seed = fb.mix_seed(9, fb.kSketchStreamTag)
    full = fb.gaussian_matrix(rows, cols, seed)
    L = _lib.load()
    win = np.empty((r1 - r0) * cols)
    _lib.check(L.frpca_gaussian_window(ctx._h, rows * cols, rows, r0, r1, seed, win.ctypes.data))
    assert np.array_equal(win.reshape(cols, r1 - r0).T, full[r0:r1])
    # the same rows, row-major (the layout the products read; rng.cu k_place_rm)
    rm = np.full((r1 - r0) * cols, np.nan)
    _lib.check(L.frpca_gaussian_window_rows(ctx._h, (cols - 1) * rows + r1, rows, r0, r1, seed, rm.ctypes.data))
    assert np.array_equal(rm.reshape(r1 - r0, cols), full[r0:r1])
    # a contiguous run of columns [1, cols - 1), generated only up to its end
    run = np.empty((cols - 2) * rows) if cols > 2 else None
    if run is not None:
        cnt = (cols - 1) * rows
        _lib.check(L.frpca_gaussian_window(ctx._h, cnt, cnt, rows, cnt, seed, run.ctypes.data))
        assert np.array_equal(run, full[:, 1:cols - 1].ravel(order="F"))
