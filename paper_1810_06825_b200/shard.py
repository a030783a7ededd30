"""Host-side sharding of the sparse matrix across GPUs.

frpcat (rows >= cols): row-block shards, contiguous, balanced by nnz + rows
(the SpMM work of a row is its nnz plus one output-row write); the n x l
A^T*Y partials and the l x l Gram partials are summed across ranks.

frpca (rows <= cols): column-block shards (a row-block sharding of A^T),
balanced by column nnz + 1, shipped as local CSRs with local column ids; the
m x l A*X partials and the Gram partials are summed across ranks.
"""
from __future__ import annotations

import numpy as np


def row_cuts(row_ptr: np.ndarray, world: int) -> list[int]:
    m = row_ptr.size - 1
    w = row_ptr.astype(np.float64) + np.arange(m + 1)
    total = w[-1]
    cuts = [0] + [int(np.searchsorted(w, total * r / world)) for r in range(1, world)] + [m]
    return cuts


def shard_rows(row_ptr, col_idx, values, world: int, rank: int):
    """This rank's row block [r0, r1) as a local CSR (global column ids)."""
    cuts = row_cuts(row_ptr, world)
    r0, r1 = cuts[rank], cuts[rank + 1]
    p0, p1 = int(row_ptr[r0]), int(row_ptr[r1])
    rp = np.ascontiguousarray(row_ptr[r0:r1 + 1] - row_ptr[r0])
    return r0, r1, rp, np.ascontiguousarray(col_idx[p0:p1]), np.ascontiguousarray(values[p0:p1])


def col_cuts(col_idx: np.ndarray, ncols: int, world: int) -> list[int]:
    counts = np.bincount(col_idx, minlength=ncols).astype(np.float64) + 1.0
    pref = np.concatenate([[0.0], np.cumsum(counts)])
    return [0] + [int(np.searchsorted(pref, pref[-1] * r / world)) for r in range(1, world)] + [ncols]


def shard_cols(row_ptr, col_idx, values, ncols: int, world: int, rank: int):
    """This rank's column block [c0, c1) as a local CSR (local column ids)."""
    cuts = col_cuts(col_idx, ncols, world)
    c0, c1 = cuts[rank], cuts[rank + 1]
    keep = (col_idx >= c0) & (col_idx < c1)
    rowid = np.repeat(np.arange(row_ptr.size - 1), np.diff(row_ptr))
    rp = np.zeros(row_ptr.size, dtype=np.int64)
    np.add.at(rp, rowid[keep] + 1, 1)
    rp = np.cumsum(rp)
    return c0, c1, rp, np.ascontiguousarray(col_idx[keep] - c0), np.ascontiguousarray(values[keep])
