"""ctypes binding of libfrpca_b200.so (include/frpca_b200.h).

The CUDA library is the only compute path: if it is missing this module raises
instead of falling back to anything else.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libfrpca_b200.so")

OK, ERR_INVALID, ERR_IO, ERR_NUMERICAL, ERR_CUDA = 0, 2, 3, 4, 5
ALGO_FRPCA, ALGO_FRPCAT, ALGO_AUTO, ALGO_BASIC_RPCA, ALGO_BASIC_RPCAT = 0, 1, 2, 3, 4
FLAG_DEVICE_IO, FLAG_HOST_OMEGA = 1, 2
COMM_AUTO, COMM_NCCL, COMM_LOOPBACK = 0, 1, 2

_i64, _u64, _i32, _u32 = C.c_int64, C.c_uint64, C.c_int32, C.c_uint32
_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)
_vp = C.c_void_p


class FrpcaConfig(C.Structure):
    _fields_ = [("k", _i64), ("oversample", _i64), ("passes", _i64), ("power", _i64),
                ("seed", _u64), ("deterministic", _i32), ("flags", _u32)]


class FrpcaStats(C.Structure):
    _fields_ = [("sketch_seconds", C.c_double), ("power_seconds", C.c_double),
                ("finalize_seconds", C.c_double), ("passes_over_matrix", _u64)]


# every symbol declared in include/frpca_b200.h, with its ctypes signature
SIGNATURES = {
    "frpca_last_error": (C.c_char_p, []),
    "frpca_version": (C.c_int, []),
    "frpca_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "frpca_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "frpca_ctx_create_dist": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(_vp)]),
    "frpca_ctx_destroy": (C.c_int, [_vp]),
    "frpca_group_create": (C.c_int, [C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(_vp)]),
    "frpca_group_size": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "frpca_group_ctx": (C.c_int, [_vp, C.c_int, C.POINTER(_vp)]),
    "frpca_group_destroy": (C.c_int, [_vp]),
    "frpca_group_run_csr": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, C.c_int, C.POINTER(FrpcaConfig),
                                      _vp, _vp, _vp, C.POINTER(FrpcaStats), C.POINTER(C.c_int)]),
    "frpca_shard_cuts": (C.c_int, [_i64, _i64, _vp, _vp, _i32, _i32, _vp]),
    "frpca_shard_cols_count": (C.c_int, [_i64, _vp, _vp, _i64, _i64, _lp]),
    "frpca_shard_cols": (C.c_int, [_i64, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "frpca_ctx_sync": (C.c_int, [_vp]),
    "frpca_host_alloc": (C.c_int, [_u64, C.POINTER(_vp)]),
    "frpca_host_free": (C.c_int, [_vp]),
    "frpca_dmat_upload": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, C.POINTER(_vp)]),
    "frpca_dmat_upload_shard": (C.c_int, [_vp, _i64, _i64, _i32, _i64, _i64, _i64, _i64,
                                          _vp, _vp, _vp, C.POINTER(_vp)]),
    "frpca_dmat_destroy": (C.c_int, [_vp]),
    "frpca_mtx_read": (C.c_int, [C.c_char_p, C.POINTER(_vp), _lp, _lp, _lp]),
    "frpca_mtx_entries": (C.c_int, [_vp, _vp, _vp, _vp]),
    "frpca_mtx_free": (None, [_vp]),
    "frpca_mtx_write": (C.c_int, [C.c_char_p, _i64, _i64, _vp, _vp, _vp]),
    "frpca_csr_from_triplets": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, _lp, _vp, _vp, _vp]),
    "frpca_run_csr": (C.c_int, [_vp, _i64, _i64, _i64, _vp, _vp, _vp, C.c_int, C.POINTER(FrpcaConfig), _vp,
                                _i64, _i64, _vp, _vp, _vp, _vp, C.POINTER(FrpcaStats), C.POINTER(C.c_int)]),
    "frpca_low_rank_error": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _vp, C.c_int, _u64, _dp]),
    "frpca_pc_correlation": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "frpca_projector_distance": (C.c_int, [_vp, _i64, _i64, _vp, _i64, _vp, _dp]),
    "frpca_dmat_info": (C.c_int, [_vp, _lp, _lp, _lp]),
    "frpca_dmat_pass_count": (C.c_int, [_vp, C.POINTER(_u64)]),
    "frpca_dmat_reset_pass_count": (C.c_int, [_vp]),
    "frpca_dmat_get_transpose": (C.c_int, [_vp, _vp, _vp, _vp]),
    "frpca_spmm": (C.c_int, [_vp, _vp, C.c_int, _vp, _i64, _i64, _vp]),
    "frpca_gaussian_matrix": (C.c_int, [_vp, _i64, _i64, _u64, _vp]),
    "frpca_gaussian_window": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _u64, _vp]),
    "frpca_gaussian_window_rows": (C.c_int, [_vp, _i64, _i64, _i64, _i64, _u64, _vp]),
    "frpca_lu_basis": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "frpca_orth": (C.c_int, [_vp, _i64, _i64, _vp, _vp]),
    "frpca_eig_svd": (C.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "frpca_run": (C.c_int, [_vp, _vp, C.c_int, C.POINTER(FrpcaConfig), _vp, _i64, _i64,
                            _vp, _vp, _vp, _vp, C.POINTER(FrpcaStats), C.POINTER(C.c_int)]),
    "frpca_profile_enable": (C.c_int, [_vp, C.c_int]),
    "frpca_profile_count": (C.c_int, [_vp, C.POINTER(C.c_int)]),
    "frpca_profile_get": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_char_p), _lp,
                                    _dp, _dp, _dp]),
    "frpca_profile_reset": (C.c_int, [_vp]),
    "frpca_timer_begin": (C.c_int, [_vp]),
    "frpca_timer_end": (C.c_int, [_vp, _dp]),
    "frpca_launch_count": (C.c_int, [C.POINTER(_u64)]),
}

_lib = None


def load():
    """Loads the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class NumericalError(RuntimeError):
    """frpca::NumericalError (types.hpp:27-30): rank deficiency, non-convergence."""


class CudaError(RuntimeError):
    """CUDA / NCCL / cuSOLVER failure (status 5)."""


class IoError(OSError):
    """frpca::IoError (types.hpp:19-22): file I/O and Matrix Market format errors."""


def check(status: int):
    if status == OK:
        return
    msg = load().frpca_last_error().decode()
    if status == ERR_INVALID:
        raise ValueError(msg)  # std::invalid_argument
    if status == ERR_NUMERICAL:
        raise NumericalError(msg)
    if status == ERR_IO:
        raise IoError(msg)
    raise CudaError(msg)
