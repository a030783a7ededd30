"""Multi-rank path on the CPU (world_size 2, gloo): the same shard helpers the
GPU bench uses (paper_1810_06825_b200/shard.py) and the same exchange steps
the library performs with NCCL (allreduce of the A^T*Y / A*X partials and of
the Gram partials, csrc/driver.cu), executed with the oracle's kernels. The
sharded frpcat / frpca must reproduce the unsharded oracle within the parity
bars (the only difference is the summation order of the partials)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from metrics import SIGMA_TOL, SUBSPACE_TOL, sigma_rel, subspace_dist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(x: np.ndarray) -> np.ndarray:
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    dist.all_reduce(t)
    return t.numpy()


def _eig_factor(orc, W_loc, l):
    """Gram partial -> allreduce -> eig -> rank check (dense_kernels.hpp:156-167)."""
    B = _allreduce(orc.gram_lower(W_loc))
    V, D = orc.eig_sym(B)
    if D[-1] <= 0 or D[0] <= l * np.finfo(float).eps * D[-1]:
        raise orc.NumericalError("eig_svd: input does not have full numerical column rank")
    return V, np.sqrt(D)


def sharded_frpcat(orc, shard, m, n, k, s, q, seed):
    """frpcat (randsvd.hpp:278-328) over a row shard [r0, r1)."""
    from paper_1810_06825_b200 import shard as sh
    r0, r1, rp, ci, va = shard
    A = orc.Csr.create(r1 - r0, n, rp, ci, va)
    l = k + s
    loops = (q - 1) // 2
    om_seed = orc.mix_seed(seed, 0xA11CE)
    if q % 2 == 0:
        Om = orc.gaussian_matrix(l, m, om_seed)               # every rank draws the stream
        Z = _allreduce(orc.spmm_transpose(A, Om.T[r0:r1]))   # (Omega A)^T partial
        Q = orc.eig_svd(Z)[0] if q == 2 else orc.lu_basis(Z)
    else:
        Q = orc.gaussian_matrix(n, l, om_seed)
    for i in range(1, loops + 1):
        Z = _allreduce(orc.spmm_transpose(A, orc.spmm(A, Q)))
        Q = orc.eig_svd(Z)[0] if i == loops else orc.lu_basis(Z)
    W = orc.spmm(A, Q)                                        # local rows of A Q
    V, S = _eig_factor(orc, W, l)
    ind = np.arange(s + k - 1, s - 1, -1)
    U_loc = W @ (V[:, ind] / S[ind])
    Vout = Q @ V[:, ind]
    _ = sh
    return U_loc, S[ind], Vout


def sharded_frpca(orc, shard, m, n, k, s, q, seed):
    """frpca (randsvd.hpp:224-276) over a column shard [c0, c1)."""
    c0, c1, rp, ci, va = shard
    A = orc.Csr.create(m, c1 - c0, rp, ci, va)
    l = k + s
    loops = (q - 1) // 2
    om_seed = orc.mix_seed(seed, 0xA11CE)
    if q % 2 == 0:
        Om = orc.gaussian_matrix(n, l, om_seed)
        Y = _allreduce(orc.spmm(A, Om[c0:c1]))
        Q = orc.lu_basis(Y) if q > 2 else orc.eig_svd(Y)[0]
    else:
        Q = orc.gaussian_matrix(m, l, om_seed)
    for i in range(1, loops + 1):
        Y = _allreduce(orc.spmm(A, orc.spmm_transpose(A, Q)))
        Q = orc.eig_svd(Y)[0] if i == loops else orc.lu_basis(Y)
    W = orc.spmm_transpose(A, Q)                               # local rows of A^T Q
    V, S = _eig_factor(orc, W, l)
    ind = np.arange(s + k - 1, s - 1, -1)
    Uout = Q @ V[:, ind]
    V_loc = W @ (V[:, ind] / S[ind])
    return Uout, S[ind], V_loc


def _worker(rank, world, port, algo, shape, q, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as orc
        from paper_1810_06825_b200 import shard as sh
        m, n = shape
        A = orc.Csr.random_sparse(m, n, 0.05, 321)
        rp, ci, va = A.arrays()
        k, s = 6, 4
        if algo == "frpcat":
            shard = sh.shard_rows(rp, ci, va, world, rank)
            U, S, V = sharded_frpcat(orc, shard, m, n, k, s, q, seed=5)
            parts = (shard[0], U)
        else:
            shard = sh.shard_cols(rp, ci, va, n, world, rank)
            U, S, V = sharded_frpca(orc, shard, m, n, k, s, q, seed=5)
            parts = (shard[0], V)
        out_q.put((rank, parts, S, U if algo == "frpca" else V))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("algo,shape", [("frpcat", (400, 150)), ("frpca", (150, 400))])
@pytest.mark.parametrize("q", [3, 4])
def test_sharded_matches_unsharded(orc, algo, shape, q):
    world = 2
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, algo, shape, q, out_q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [out_q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    # replicated factor and S identical on both ranks (same reductions)
    assert np.array_equal(res[0][2], res[1][2])
    assert np.array_equal(res[0][3], res[1][3])
    local = np.concatenate([r[1][1] for r in res], axis=0)  # rank-local factor rows
    m, n = shape
    A = orc.Csr.random_sparse(m, n, 0.05, 321)
    o = orc.pca(A, orc.FRPCAT if algo == "frpcat" else orc.FRPCA, 6, 4, q, seed=5)
    assert sigma_rel(res[0][2], o["S"]) <= SIGMA_TOL
    if algo == "frpcat":
        assert subspace_dist(o["U"], local) <= SUBSPACE_TOL
        assert subspace_dist(o["V"], res[0][3]) <= SUBSPACE_TOL
    else:
        assert subspace_dist(o["V"], local) <= SUBSPACE_TOL
        assert subspace_dist(o["U"], res[0][3]) <= SUBSPACE_TOL


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_shard_partitions_cover_and_balance(world):
    from paper_1810_06825_b200 import shard as sh
    from paper_1810_06825_b200 import synth
    m, n, rp, ci, va = synth.generate("C1", scale=0.02)
    cuts = sh.row_cuts(rp, world)
    assert cuts[0] == 0 and cuts[-1] == m and all(a <= b for a, b in zip(cuts, cuts[1:]))
    w = [int(rp[b] - rp[a]) + (b - a) for a, b in zip(cuts, cuts[1:])]
    assert max(w) <= 1.1 * (sum(w) / world) + 2000
    nnz = 0
    for r in range(world):
        c0, c1, lrp, lci, lva = sh.shard_cols(rp, ci, va, n, world, r)
        assert lrp[-1] == lci.size and (lci.size == 0 or (lci.min() >= 0 and lci.max() < c1 - c0))
        nnz += lci.size
    assert nnz == rp[-1]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_library_shard_plan_matches_balance_rule(world):
    """The library's shard plan (csrc/group.cu through the C ABI) is the
    balance rule stated in numpy: row cut r = first row whose prefix weight
    (nnz + rows) reaches r/world of the total; column cut r = first column
    whose prefix weight (column nnz + 1) reaches r/world."""
    from paper_1810_06825_b200 import shard as sh
    from paper_1810_06825_b200 import synth
    m, n, rp, ci, va = synth.generate("C1", scale=0.02)
    w = rp.astype(np.float64) + np.arange(m + 1)
    rows = [0] + [int(np.searchsorted(w, w[-1] * r / world)) for r in range(1, world)] + [m]
    assert sh.row_cuts(rp, world) == rows
    pref = np.concatenate([[0.0], np.cumsum(np.bincount(ci, minlength=n).astype(np.float64) + 1.0)])
    cols = [0] + [int(np.searchsorted(pref, pref[-1] * r / world)) for r in range(1, world)] + [n]
    assert sh.col_cuts(rp, ci, n, world) == cols
    # the extracted column blocks are the columns' entries, in row order
    c0, c1 = cols[world // 2], cols[world // 2 + 1]
    _, _, lrp, lci, lva = sh.shard_cols(rp, ci, va, n, world, world // 2)
    keep = (ci >= c0) & (ci < c1)
    assert np.array_equal(lci, ci[keep] - c0) and np.array_equal(lva, va[keep])
    assert np.array_equal(np.diff(lrp), np.add.reduceat(keep.astype(np.int64), rp[:-1]) * (np.diff(rp) > 0))
