"""B200-native frPCA / frPCAt hot path (arXiv 1810.06825) — Python host mirror.

Mirrors the reference's operator interface for this path
(/root/reference/proj/include/frpca/randsvd.hpp, sparse_matrix.hpp,
dense_kernels.hpp): same names, argument meaning and error behaviour, so the
parity tests read like the reference's own doctest suites. Every numerical
operation runs on the GPU through the C ABI of libfrpca_b200.so
(include/frpca_b200.h); nothing here computes on the CPU except host-side
CSR construction (from_triplets / validate), exactly as in the reference.

Dense matrices are numpy arrays; results come back column-major (Fortran
order) like the reference's Eigen matrices.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
import threading

import numpy as np

from . import _lib
from ._lib import NumericalError, CudaError, IoError  # noqa: F401

__all__ = [
    "SparseMatrixCsr", "PcaConfig", "RunStats", "SvdResult", "AutoPcaResult", "PcaAlgorithm",
    "NumericalError", "CudaError", "Context", "default_context",
    "spmm", "spmm_transpose", "transpose", "gaussian_matrix", "lu_basis", "orth", "eig_svd",
    "frpca", "frpcat", "auto_pca", "basic_rpca", "basic_rpcat", "mix_seed", "kSketchStreamTag",
    "read_matrix_market", "load_matrix_market", "write_matrix_market", "IoError",
    "run_csr", "ErrorNorm", "low_rank_error", "best_rank_k_error", "pc_correlation", "projector_distance",
    "AccuracyReport", "make_accuracy_report", "kDefaultOracleEntryLimit", "Group",
]

kSketchStreamTag = 0xA11CE  # randsvd.hpp:63


def mix_seed(seed: int, tag: int) -> int:
    """detail::mix_seed, types.hpp:52-57 (SplitMix64 step)."""
    M = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (tag + 1)) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


class PcaAlgorithm(enum.IntEnum):
    """randsvd.hpp:14 (eig_svds, the dense Gram baseline, is not provided)."""
    Frpca = _lib.ALGO_FRPCA
    Frpcat = _lib.ALGO_FRPCAT
    Auto = _lib.ALGO_AUTO
    BasicRpca = _lib.ALGO_BASIC_RPCA
    BasicRpcat = _lib.ALGO_BASIC_RPCAT


@dataclasses.dataclass
class PcaConfig:
    """randsvd.hpp:28-40."""
    k: int = 0
    oversample: int = 5
    passes: int = 2
    power: int = 0
    seed: int = 0
    deterministic: bool = False
    host_omega: bool = False  # draw Omega with the host libstdc++ generator

    def sketch_width(self) -> int:
        return self.k + self.oversample

    def to_c(self, device_io: bool = False) -> _lib.FrpcaConfig:
        flags = (_lib.FLAG_DEVICE_IO if device_io else 0) | (_lib.FLAG_HOST_OMEGA if self.host_omega else 0)
        return _lib.FrpcaConfig(self.k, self.oversample, self.passes, self.power,
                                self.seed & ((1 << 64) - 1), int(self.deterministic), flags)


@dataclasses.dataclass
class RunStats:
    """randsvd.hpp:42-53."""
    sketch_seconds: float = 0.0
    power_seconds: float = 0.0
    finalize_seconds: float = 0.0
    passes_over_matrix: int = 0
    capture_basis: bool = False
    basis: np.ndarray | None = None


@dataclasses.dataclass
class SvdResult:
    """types.hpp:34-41: U m x k, S k (descending), V n x k."""
    U: np.ndarray
    S: np.ndarray
    V: np.ndarray

    def rank(self) -> int:
        return int(self.S.size)


@dataclasses.dataclass
class AutoPcaResult:
    """randsvd.hpp:331-334."""
    svd: SvdResult
    dispatched: PcaAlgorithm = PcaAlgorithm.Auto


class Context:
    """Device context (stream, cuSOLVER handle, optional NCCL communicator)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        L = _lib.load()
        h = C.c_void_p()
        if world > 1:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _lib.check(L.frpca_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        else:
            _lib.check(L.frpca_ctx_create(device, C.byref(h)))
        self._h = h
        self.device, self.rank, self.world = device, rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _lib.check(_lib.load().frpca_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().frpca_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        _lib.check(_lib.load().frpca_ctx_sync(self._h))

    # per-kernel device timings of profiled launches
    def profile(self, enable: bool = True):
        _lib.check(_lib.load().frpca_profile_enable(self._h, int(enable)))

    def profile_reset(self):
        _lib.check(_lib.load().frpca_profile_reset(self._h))

    def profile_report(self) -> dict:
        L = _lib.load()
        n = C.c_int()
        _lib.check(L.frpca_profile_count(self._h, C.byref(n)))
        out = {}
        for i in range(n.value):
            name = C.c_char_p()
            la, ms, by, fl = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            _lib.check(L.frpca_profile_get(self._h, i, C.byref(name), C.byref(la), C.byref(ms),
                                           C.byref(by), C.byref(fl)))
            out[name.value.decode()] = dict(launches=la.value, ms=ms.value, bytes=by.value, flops=fl.value)
        return out


class Group:
    """Single-process multi-GPU (frpca_group_*): one context (rank)
    per listed device. Distinct devices exchange the A^T*Y / A*X and Gram
    partials through NCCL; a device listed more than once selects the
    host-staged loopback collective, which runs the sharded path on one GPU
    (tests). `run` shards a host CSR (row blocks for frpcat, column blocks for
    frpca) and returns the full SvdResult."""

    def __init__(self, devices, comm: int = _lib.COMM_AUTO):
        L = _lib.load()
        dv = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _lib.check(L.frpca_group_create(dv, len(devices), comm, C.byref(h)))
        self._h = h
        self.devices = list(devices)

    def __len__(self):
        return len(self.devices)

    def context_handle(self, rank: int) -> C.c_void_p:
        """The rank's C context (owned by the group)."""
        h = C.c_void_p()
        _lib.check(_lib.load().frpca_group_ctx(self._h, rank, C.byref(h)))
        return h

    def run(self, A: "SparseMatrixCsr", cfg: PcaConfig, algorithm: "PcaAlgorithm" = None,
            stats: RunStats | None = None) -> tuple[SvdResult, int]:
        algo = _lib.ALGO_AUTO if algorithm is None else int(algorithm)
        m, n = A.rows(), A.cols()
        k = max(int(cfg.k), 0)
        U = np.empty((m, k), order="F")
        S = np.empty(k)
        V = np.empty((n, k), order="F")
        st = _lib.FrpcaStats()
        disp = C.c_int(-1)
        ccfg = cfg.to_c()
        rp = np.ascontiguousarray(A.rowPtr(), dtype=np.int64)
        ci = np.ascontiguousarray(A.colIdx(), dtype=np.int64)
        va = np.ascontiguousarray(A.values(), dtype=np.float64)
        _lib.check(_lib.load().frpca_group_run_csr(self._h, m, n, int(rp[-1]), _ptr(rp), _ptr(ci), _ptr(va), algo,
                                                   C.byref(ccfg), _ptr(U), _ptr(S), _ptr(V), C.byref(st),
                                                   C.byref(disp)))
        if stats is not None:
            stats.sketch_seconds, stats.power_seconds = st.sketch_seconds, st.power_seconds
            stats.finalize_seconds = st.finalize_seconds
            stats.passes_over_matrix = int(st.passes_over_matrix)
        return SvdResult(U, S, V), disp.value

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().frpca_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = None
_default_lock = threading.Lock()


def default_context() -> Context:
    global _default
    with _default_lock:
        if _default is None:
            _default = Context(0)
        return _default


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class SparseMatrixCsr:
    """SparseMatrixCsr<double> (sparse_matrix.hpp:19-150).

    Host arrays follow the reference exactly (int64 row_ptr / col_idx, double
    values); the constructor validates with validate()'s checks and messages.
    The device copy (CSR + transposed CSR + work lists) is built on first use
    and cached; the pass counter lives with it (passCount / resetPassCount).
    """

    class Triplet(tuple):
        pass

    def __init__(self, rows: int = 0, cols: int = 0, row_ptr=None, col_idx=None, values=None,
                 validate: bool = True):
        self._rows, self._cols = int(rows), int(cols)
        self.row_ptr = np.ascontiguousarray(row_ptr if row_ptr is not None else [0], dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx if col_idx is not None else [], dtype=np.int64)
        self.vals = np.ascontiguousarray(values if values is not None else [], dtype=np.float64)
        if validate:
            self._validate()
        self._dmat = None
        self._ctx = None

    # -- construction ---------------------------------------------------------
    def _validate(self):
        """validate(), sparse_matrix.hpp:125-142 (same checks, same messages)."""
        m, n = self._rows, self._cols
        rp, ci = self.row_ptr, self.col_idx
        if m < 0 or n < 0:
            raise ValueError("csr: negative dimension")
        if rp.size != m + 1:
            raise ValueError("csr: row_ptr length must be rows + 1")
        if rp[0] != 0:
            raise ValueError("csr: row_ptr[0] must be 0")
        if rp[-1] != self.vals.size:
            raise ValueError("csr: row_ptr[rows] must equal nnz")
        if ci.size != self.vals.size:
            raise ValueError("csr: col_idx/values length mismatch")
        if m == 0:
            return
        bad_rp = np.flatnonzero(rp[:-1] > rp[1:])
        first_rp = bad_rp[0] if bad_rp.size else m
        valid_nnz = rp[first_rp]
        c = ci[:valid_nnz]
        rowid = np.repeat(np.arange(first_rp), np.diff(rp[:first_rp + 1]))
        bad_range = (c < 0) | (c >= n)
        start = np.zeros(valid_nnz, dtype=bool)
        if valid_nnz:
            start[rp[:first_rp][rp[:first_rp] < valid_nnz]] = True
        bad_inc = np.zeros(valid_nnz, dtype=bool)
        if valid_nnz > 1:
            bad_inc[1:] = (~start[1:]) & ~(c[:-1] < c[1:])
        # the reference reports the first failure in (row, position) order
        cand = []
        if bad_range.any():
            cand.append((int(np.flatnonzero(bad_range)[0]), 0, "csr: column index out of range"))
        if bad_inc.any():
            cand.append((int(np.flatnonzero(bad_inc)[0]), 1,
                         "csr: column indices must be strictly increasing within a row"))
        if cand:
            raise ValueError(min(cand)[2])
        if first_rp < m:
            raise ValueError("csr: row_ptr must be non-decreasing")
        _ = rowid

    @classmethod
    def from_triplets(cls, rows: int, cols: int, entries, device: bool = False,
                      ctx: "Context | None" = None) -> "SparseMatrixCsr":
        """sparse_matrix.hpp:62-95: sort by (row, col), sum duplicates in order,
        drop entries that sum to exactly zero. device=True builds the CSR on
        the GPU (frpca_csr_from_triplets: radix sort, run sums, compaction)."""
        if rows < 0 or cols < 0:
            raise ValueError("from_triplets: negative dimension")
        if isinstance(entries, tuple) and len(entries) == 3 and hasattr(entries[0], "__len__"):
            r, c, v = (np.asarray(entries[0], dtype=np.int64), np.asarray(entries[1], dtype=np.int64),
                       np.asarray(entries[2], dtype=np.float64))
        else:
            ent = list(entries)
            r = np.array([e[0] for e in ent], dtype=np.int64)
            c = np.array([e[1] for e in ent], dtype=np.int64)
            v = np.array([e[2] for e in ent], dtype=np.float64)
        if device:
            ctx = ctx or default_context()
            r, c, v = np.ascontiguousarray(r), np.ascontiguousarray(c), np.ascontiguousarray(v)
            n = r.size
            row_ptr = np.empty(rows + 1, dtype=np.int64)
            col = np.empty(max(n, 1), dtype=np.int64)
            val = np.empty(max(n, 1), dtype=np.float64)
            nnz = C.c_int64(0)
            _lib.check(_lib.load().frpca_csr_from_triplets(
                ctx._h, rows, cols, n, _ptr(r), _ptr(c), _ptr(v), C.byref(nnz), _ptr(row_ptr), _ptr(col),
                _ptr(val)))
            k = nnz.value
            return cls(rows, cols, row_ptr, col[:k].copy(), val[:k].copy(), validate=False)
        if r.size and ((r < 0).any() or (r >= rows).any() or (c < 0).any() or (c >= cols).any()):
            raise ValueError("from_triplets: entry out of bounds")
        order = np.lexsort((c, r))  # stable: duplicates keep input order
        r, c, v = r[order], c[order], v[order]
        if r.size:
            key_change = np.ones(r.size, dtype=bool)
            key_change[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
            starts = np.flatnonzero(key_change)
            # sequential sums in sorted order (reduceat adds left to right)
            sums = np.add.reduceat(v, starts) if starts.size else v
            if starts.size:
                # np.add.reduceat is pairwise for long runs: redo runs > 1 sequentially
                lens = np.diff(np.append(starts, r.size))
                for idx in np.flatnonzero(lens > 2):
                    s0 = starts[idx]
                    acc = 0.0
                    for t in range(lens[idx]):
                        acc += v[s0 + t]
                    sums[idx] = acc
            rr, cc = r[starts], c[starts]
            keep = sums != 0.0
            rr, cc, sums = rr[keep], cc[keep], sums[keep]
        else:
            rr, cc, sums = r, c, v
        row_ptr = np.zeros(rows + 1, dtype=np.int64)
        np.add.at(row_ptr, rr + 1, 1)
        np.cumsum(row_ptr, out=row_ptr)
        return cls(rows, cols, row_ptr, cc, sums)

    # -- accessors (sparse_matrix.hpp:97-118) ----------------------------------
    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def nonZeros(self) -> int:
        return int(self.vals.size)

    def rowPtr(self) -> np.ndarray:
        return self.row_ptr

    def colIdx(self) -> np.ndarray:
        return self.col_idx

    def values(self) -> np.ndarray:
        return self.vals

    def toDense(self) -> np.ndarray:
        D = np.zeros((self._rows, self._cols), order="F")
        rowid = np.repeat(np.arange(self._rows), np.diff(self.row_ptr))
        D[rowid, self.col_idx] = self.vals
        return D

    # -- device copy -----------------------------------------------------------
    def device(self, ctx: Context | None = None):
        ctx = ctx or default_context()
        if self._dmat is None or self._ctx is not ctx:
            self.release()
            h = C.c_void_p()
            _lib.check(_lib.load().frpca_dmat_upload(
                ctx._h, self._rows, self._cols, self.nonZeros(), _ptr(self.row_ptr),
                _ptr(self.col_idx), _ptr(self.vals), C.byref(h)))
            self._dmat, self._ctx = h, ctx
        return self._dmat

    def release(self):
        if self._dmat is not None:
            _lib.load().frpca_dmat_destroy(self._dmat)
            self._dmat = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass

    def passCount(self) -> int:
        if self._dmat is None:
            return 0
        v = C.c_uint64()
        _lib.check(_lib.load().frpca_dmat_pass_count(self._dmat, C.byref(v)))
        return int(v.value)

    def resetPassCount(self):
        if self._dmat is not None:
            _lib.check(_lib.load().frpca_dmat_reset_pass_count(self._dmat))


def _colmajor(X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim == 1:
        X = X.reshape(-1, 1)
    return np.asfortranarray(X)


def read_matrix_market(path: str):
    """The parse of load_matrix_market (matrix_market.hpp:27-93): returns
    (rows, cols, r, c, v) with 0-based triplets in file order, symmetric
    storage expanded. Host code (no GPU needed). Errors: IoError."""
    L = _lib.load()
    h = C.c_void_p()
    rows, cols, n = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    _lib.check(L.frpca_mtx_read(os.fsencode(path), C.byref(h), C.byref(rows), C.byref(cols), C.byref(n)))
    try:
        r = np.empty(n.value, dtype=np.int64)
        c = np.empty(n.value, dtype=np.int64)
        v = np.empty(n.value, dtype=np.float64)
        _lib.check(L.frpca_mtx_entries(h, _ptr(r), _ptr(c), _ptr(v)))
    finally:
        L.frpca_mtx_free(h)
    return rows.value, cols.value, r, c, v


def load_matrix_market(path: str, ctx: Context | None = None) -> SparseMatrixCsr:
    """matrix_market.hpp:27-93: parse on the host, from_triplets on the GPU."""
    rows, cols, r, c, v = read_matrix_market(path)
    return SparseMatrixCsr.from_triplets(rows, cols, (r, c, v), device=True, ctx=ctx)


def write_matrix_market(path: str, A: SparseMatrixCsr) -> None:
    """matrix_market.hpp:95-116: general coordinate, %.17g values."""
    rp = np.ascontiguousarray(A.rowPtr(), dtype=np.int64)
    ci = np.ascontiguousarray(A.colIdx(), dtype=np.int64)
    va = np.ascontiguousarray(A.values(), dtype=np.float64)
    _lib.check(_lib.load().frpca_mtx_write(os.fsencode(path), A.rows(), A.cols(), _ptr(rp), _ptr(ci), _ptr(va)))


def spmm(A: SparseMatrixCsr, X, ctx: Context | None = None) -> np.ndarray:
    """Y = A * X (sparse_matrix.hpp:177-206); one pass over A."""
    X = _colmajor(X)
    if X.shape[0] != A.cols():
        raise ValueError("spmm: inner dimensions do not match")
    ctx = ctx or default_context()
    h = A.device(ctx)
    Y = np.empty((A.rows(), X.shape[1]), order="F")
    _lib.check(_lib.load().frpca_spmm(ctx._h, h, 0, _ptr(X), max(X.shape[0], 1), X.shape[1], _ptr(Y)))
    return Y


def spmm_transpose(A: SparseMatrixCsr, Y, ctx: Context | None = None) -> np.ndarray:
    """Z = A^T * Y (sparse_matrix.hpp:208-240), served from the device transposed CSR."""
    Y = _colmajor(Y)
    if Y.shape[0] != A.rows():
        raise ValueError("spmm_transpose: inner dimensions do not match")
    ctx = ctx or default_context()
    h = A.device(ctx)
    Z = np.empty((A.cols(), Y.shape[1]), order="F")
    _lib.check(_lib.load().frpca_spmm(ctx._h, h, 1, _ptr(Y), max(Y.shape[0], 1), Y.shape[1], _ptr(Z)))
    return Z


def transpose(A: SparseMatrixCsr, ctx: Context | None = None) -> SparseMatrixCsr:
    """sparse_matrix.hpp:242-267, via the transposed CSR the device built at load."""
    ctx = ctx or default_context()
    h = A.device(ctx)
    rp = np.empty(A.cols() + 1, dtype=np.int64)
    ci = np.empty(A.nonZeros(), dtype=np.int64)
    va = np.empty(A.nonZeros(), dtype=np.float64)
    _lib.check(_lib.load().frpca_dmat_get_transpose(h, _ptr(rp), _ptr(ci), _ptr(va)))
    return SparseMatrixCsr(A.cols(), A.rows(), rp, ci, va)


def gaussian_matrix(rows: int, cols: int, seed: int, ctx: Context | None = None) -> np.ndarray:
    """dense_kernels.hpp:16-28, drawn on the device (bit-compatible stream)."""
    ctx = ctx or default_context()
    out = np.empty((rows, cols), order="F") if rows >= 1 and cols >= 1 else np.empty((0, 0))
    _lib.check(_lib.load().frpca_gaussian_matrix(ctx._h, rows, cols, seed & ((1 << 64) - 1), _ptr(out)))
    return out


def lu_basis(M, ctx: Context | None = None) -> np.ndarray:
    """dense_kernels.hpp:50-116: P^T L of a row-pivoted LU of tall M."""
    M = _colmajor(M)
    ctx = ctx or default_context()
    X = np.empty(M.shape, order="F")
    _lib.check(_lib.load().frpca_lu_basis(ctx._h, M.shape[0], M.shape[1], _ptr(M), _ptr(X)))
    return X


def orth(M, ctx: Context | None = None) -> np.ndarray:
    """dense_kernels.hpp:30-48: Householder-QR basis of range(M) (tall M);
    raises NumericalError when |diag R| <= m eps max|diag R|."""
    M = _colmajor(M)
    ctx = ctx or default_context()
    m, l = M.shape
    Q = np.empty((m, l), order="F")
    _lib.check(_lib.load().frpca_orth(ctx._h, m, l, _ptr(M), _ptr(Q)))
    return Q


def eig_svd(A, ctx: Context | None = None):
    """dense_kernels.hpp:145-174: returns (U, S ascending, V) of tall full-rank A."""
    A = _colmajor(A)
    ctx = ctx or default_context()
    m, n = A.shape
    U = np.empty((m, n), order="F")
    S = np.empty(n)
    V = np.empty((n, n), order="F")
    _lib.check(_lib.load().frpca_eig_svd(ctx._h, m, n, _ptr(A), _ptr(U), _ptr(S), _ptr(V)))
    return U, S, V


def _run(algo: int, A: SparseMatrixCsr, cfg: PcaConfig, stats: RunStats | None, omega,
         ctx: Context | None) -> tuple[SvdResult, int]:
    ctx = ctx or default_context()
    h = A.device(ctx)
    k = max(int(cfg.k), 0)
    l = cfg.k + cfg.oversample
    m, n = A.rows(), A.cols()
    eff = algo if algo != _lib.ALGO_AUTO else (_lib.ALGO_FRPCA if m < n else _lib.ALGO_FRPCAT)
    U = np.empty((m, k), order="F")
    S = np.empty(k)
    V = np.empty((n, k), order="F")
    basis = None
    if stats is not None and stats.capture_basis and l >= 1:
        basis = np.empty((m if eff in (_lib.ALGO_FRPCA, _lib.ALGO_BASIC_RPCA) else n, l), order="F")
    om = None if omega is None else _colmajor(omega)
    st = _lib.FrpcaStats()
    disp = C.c_int(-1)
    ccfg = cfg.to_c()
    _lib.check(_lib.load().frpca_run(
        ctx._h, h, algo, C.byref(ccfg), _ptr(om), 0 if om is None else om.shape[0],
        0 if om is None else om.shape[1], _ptr(U), _ptr(S), _ptr(V), _ptr(basis), C.byref(st),
        C.byref(disp)))
    if stats is not None:
        stats.sketch_seconds = st.sketch_seconds
        stats.power_seconds = st.power_seconds
        stats.finalize_seconds = st.finalize_seconds
        stats.passes_over_matrix = int(st.passes_over_matrix)
        if stats.capture_basis:
            stats.basis = basis
    return SvdResult(U, S, V), disp.value


def run_csr(A: SparseMatrixCsr, cfg: PcaConfig, algorithm: "PcaAlgorithm" = None, stats: RunStats | None = None,
            ctx: Context | None = None) -> tuple[SvdResult, int]:
    """One-shot run from the host CSR (frpca_run_csr): upload, run, release,
    with the sketch generated on a second stream during the upload. Returns
    (result, dispatched algorithm)."""
    ctx = ctx or default_context()
    algo = _lib.ALGO_AUTO if algorithm is None else int(algorithm)
    m, n = A.rows(), A.cols()
    eff = algo if algo != _lib.ALGO_AUTO else (_lib.ALGO_FRPCA if m < n else _lib.ALGO_FRPCAT)
    k = max(int(cfg.k), 0)
    l = cfg.k + cfg.oversample
    U = np.empty((m, k), order="F")
    S = np.empty(k)
    V = np.empty((n, k), order="F")
    basis = None
    if stats is not None and stats.capture_basis and l >= 1:
        basis = np.empty((m if eff in (_lib.ALGO_FRPCA, _lib.ALGO_BASIC_RPCA) else n, l), order="F")
    st = _lib.FrpcaStats()
    disp = C.c_int(-1)
    ccfg = cfg.to_c()
    rp = np.ascontiguousarray(A.rowPtr(), dtype=np.int64)
    ci = np.ascontiguousarray(A.colIdx(), dtype=np.int64)
    va = np.ascontiguousarray(A.values(), dtype=np.float64)
    _lib.check(_lib.load().frpca_run_csr(ctx._h, m, n, int(rp[-1]), _ptr(rp), _ptr(ci), _ptr(va), algo,
                                         C.byref(ccfg), None, 0, 0, _ptr(U), _ptr(S), _ptr(V), _ptr(basis),
                                         C.byref(st), C.byref(disp)))
    if stats is not None:
        stats.sketch_seconds, stats.power_seconds = st.sketch_seconds, st.power_seconds
        stats.finalize_seconds = st.finalize_seconds
        stats.passes_over_matrix = int(st.passes_over_matrix)
        if stats.capture_basis:
            stats.basis = basis
    return SvdResult(U, S, V), disp.value


def frpca(A: SparseMatrixCsr, cfg: PcaConfig, stats: RunStats | None = None, omega=None,
          ctx: Context | None = None) -> SvdResult:
    """Alg. 5 (randsvd.hpp:224-276), rows <= cols."""
    return _run(_lib.ALGO_FRPCA, A, cfg, stats, omega, ctx)[0]


def frpcat(A: SparseMatrixCsr, cfg: PcaConfig, stats: RunStats | None = None, omega=None,
           ctx: Context | None = None) -> SvdResult:
    """Alg. 6 (randsvd.hpp:278-328), rows >= cols."""
    return _run(_lib.ALGO_FRPCAT, A, cfg, stats, omega, ctx)[0]


def basic_rpca(A: SparseMatrixCsr, cfg: PcaConfig, stats: RunStats | None = None, omega=None,
               ctx: Context | None = None) -> SvdResult:
    """Baseline randomized PCA, sketch on the right (randsvd.hpp:95-134):
    Householder QR after every product, 2p + 2 passes (cfg.power = p)."""
    return _run(_lib.ALGO_BASIC_RPCA, A, cfg, stats, omega, ctx)[0]


def basic_rpcat(A: SparseMatrixCsr, cfg: PcaConfig, stats: RunStats | None = None, omega=None,
                ctx: Context | None = None) -> SvdResult:
    """Baseline with the sketch on the left (randsvd.hpp:136-175)."""
    return _run(_lib.ALGO_BASIC_RPCAT, A, cfg, stats, omega, ctx)[0]


def auto_pca(A: SparseMatrixCsr, cfg: PcaConfig, stats: RunStats | None = None,
             ctx: Context | None = None) -> AutoPcaResult:
    """randsvd.hpp:336-351: frpca when rows < cols, else frpcat (square -> frpcat)."""
    svd, d = _run(_lib.ALGO_AUTO, A, cfg, stats, None, ctx)
    return AutoPcaResult(svd, PcaAlgorithm(d))


# ---- validation metrics (validation.hpp:125-332) -------------------
kDefaultOracleEntryLimit = 4_000_000  # validation.hpp:26


class ErrorNorm(enum.IntEnum):
    """validation.hpp:17."""
    Frobenius = 0
    Spectral = 1


def low_rank_error(A: SparseMatrixCsr, r: SvdResult, norm: ErrorNorm,
                   entry_limit: int = kDefaultOracleEntryLimit, ctx: Context | None = None) -> float:
    """validation.hpp:170-203 on the GPU: |A - U diag(S) V^T| (spectral by
    matrix-free power iteration through the SpMM kernels)."""
    U, S, V = _colmajor(r.U), np.ascontiguousarray(r.S, dtype=np.float64), _colmajor(r.V)
    if U.shape[0] != A.rows() or V.shape[0] != A.cols():
        raise ValueError("low_rank_error: shape mismatch")
    if U.shape[1] != S.size or V.shape[1] != S.size:
        raise ValueError("low_rank_error: inconsistent factor widths")
    ctx = ctx or default_context()
    out = C.c_double(0.0)
    _lib.check(_lib.load().frpca_low_rank_error(ctx._h, A.device(ctx), S.size, _ptr(U), _ptr(S), _ptr(V),
                                                int(norm), int(entry_limit), C.byref(out)))
    return out.value


def best_rank_k_error(singular_values, k: int, norm: ErrorNorm) -> float:
    """validation.hpp:207-215 (host): sigma_{k+1} (spectral) or the root of
    the tail sum of squares (Frobenius)."""
    if k < 0:
        raise ValueError("best_rank_k_error: negative k")
    s = np.asarray(singular_values, dtype=np.float64)
    if k >= s.size:
        return 0.0
    return float(s[k]) if norm == ErrorNorm.Spectral else float(np.sqrt(np.sum(s[k:] ** 2)))


def pc_correlation(U_test, U_ref, ctx: Context | None = None) -> np.ndarray:
    """validation.hpp:228-246 on the GPU: |Pearson correlation| per column."""
    A, B = _colmajor(U_test), _colmajor(U_ref)
    if A.shape != B.shape:
        raise ValueError("pc_correlation: shape mismatch")
    if A.shape[0] < 2:
        raise ValueError("pc_correlation: need at least two samples")
    ctx = ctx or default_context()
    corr = np.empty(A.shape[1])
    _lib.check(_lib.load().frpca_pc_correlation(ctx._h, A.shape[0], A.shape[1], _ptr(A), _ptr(B), _ptr(corr)))
    return corr


def projector_distance(Q1, Q2, ctx: Context | None = None) -> float:
    """validation.hpp:264-282 on the GPU: |Q1 Q1^T - Q2 Q2^T|_2."""
    A, B = _colmajor(Q1), _colmajor(Q2)
    if A.shape[0] != B.shape[0]:
        raise ValueError("projector_distance: row mismatch")
    ctx = ctx or default_context()
    out = C.c_double(0.0)
    _lib.check(_lib.load().frpca_projector_distance(ctx._h, A.shape[0], A.shape[1], _ptr(A), B.shape[1], _ptr(B),
                                                    C.byref(out)))
    return out.value


@dataclasses.dataclass
class AccuracyReport:
    """validation.hpp:287-294 (field order = to_json's key order, :321-330)."""
    singular_value_rel_err: list
    recon_err_frobenius: float
    recon_err_spectral: float
    best_rank_k_err: float
    eps_equivalent: float
    pc_correlations: list

    def to_json(self) -> dict:
        return dataclasses.asdict(self)


def make_accuracy_report(A: SparseMatrixCsr, r: SvdResult, oracle_S, oracle_U,
                         ctx: Context | None = None) -> AccuracyReport:
    """validation.hpp:297-319, with the oracle's singular values / left
    vectors supplied by the caller (the metrics run on the GPU)."""
    k = r.S.size
    oS = np.asarray(oracle_S, dtype=np.float64)
    if oS.size < k:
        raise ValueError("make_accuracy_report: oracle has fewer values than k")
    rel = [abs(float(r.S[i])) if oS[i] == 0.0 else abs(float(r.S[i]) - float(oS[i])) / float(oS[i])
           for i in range(k)]
    fro = low_rank_error(A, r, ErrorNorm.Frobenius, ctx=ctx)
    spec = low_rank_error(A, r, ErrorNorm.Spectral, ctx=ctx)
    best = best_rank_k_error(oS, k, ErrorNorm.Spectral)
    eps = 0.0 if best == 0.0 else spec / best - 1.0
    corr = pc_correlation(r.U, np.asarray(oracle_U)[:, :k], ctx=ctx)
    return AccuracyReport(rel, fro, spec, best, eps, corr.tolist())
