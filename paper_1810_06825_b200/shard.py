"""Host-side sharding of the sparse matrix across GPUs.

The plan is the library's own (csrc/group.cu through the C ABI: the same code
the single-process group run uses), so the one-process-per-GPU launch and
frpca_group_run_csr shard identically.

frpcat (rows >= cols): row-block shards, contiguous, balanced by nnz + rows
(the SpMM work of a row is its nnz plus one output-row write); the n x l
A^T*Y partials and the l x l Gram partials are summed across ranks.

frpca (rows <= cols): column-block shards (a row-block sharding of A^T),
balanced by column nnz + 1, shipped as local CSRs with local column ids; the
m x l A*X partials and the Gram partials are summed across ranks.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib


def _cuts(row_ptr, col_idx, ncols: int, world: int, col_shard: int) -> list[int]:
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    out = np.empty(world + 1, dtype=np.int64)
    _lib.check(_lib.load().frpca_shard_cuts(rp.size - 1, ncols, rp.ctypes.data, ci.ctypes.data, col_shard, world,
                                             out.ctypes.data))
    return [int(x) for x in out]


def row_cuts(row_ptr: np.ndarray, world: int, ncols: int = 0) -> list[int]:
    return _cuts(row_ptr, np.zeros(1, dtype=np.int64), ncols, world, 0)


def shard_rows(row_ptr, col_idx, values, world: int, rank: int):
    """This rank's row block [r0, r1) as a local CSR (global column ids)."""
    cuts = row_cuts(row_ptr, world)
    r0, r1 = cuts[rank], cuts[rank + 1]
    p0, p1 = int(row_ptr[r0]), int(row_ptr[r1])
    rp = np.ascontiguousarray(row_ptr[r0:r1 + 1] - row_ptr[r0])
    return r0, r1, rp, np.ascontiguousarray(col_idx[p0:p1]), np.ascontiguousarray(values[p0:p1])


def col_cuts(row_ptr, col_idx: np.ndarray, ncols: int, world: int) -> list[int]:
    return _cuts(row_ptr, col_idx, ncols, world, 1)


def shard_cols(row_ptr, col_idx, values, ncols: int, world: int, rank: int):
    """This rank's column block [c0, c1) as a local CSR (local column ids)."""
    cuts = col_cuts(row_ptr, col_idx, ncols, world)
    c0, c1 = cuts[rank], cuts[rank + 1]
    L = _lib.load()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    va = np.ascontiguousarray(values, dtype=np.float64)
    m = rp.size - 1
    nl = C.c_int64()
    _lib.check(L.frpca_shard_cols_count(m, rp.ctypes.data, ci.ctypes.data, c0, c1, C.byref(nl)))
    lrp = np.empty(m + 1, dtype=np.int64)
    lci = np.empty(max(nl.value, 1), dtype=np.int64)
    lva = np.empty(max(nl.value, 1), dtype=np.float64)
    _lib.check(L.frpca_shard_cols(m, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, c0, c1, lrp.ctypes.data,
                                  lci.ctypes.data, lva.ctypes.data))
    return c0, c1, lrp, lci[:nl.value], lva[:nl.value]
