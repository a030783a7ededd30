"""Seeded synthetic inputs for BASELINE.json's configs.

`generate(name)` returns (rows, cols, row_ptr, col_idx, values) as numpy
arrays in the reference CSR format (int64 / int64 / float64). `scale` shrinks
rows, cols and nnz proportionally for parity tests at oracle-friendly sizes.
Buffers can be allocated by the caller (e.g. pinned memory for e2e timing).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import functools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(os.path.dirname(_HERE), "lib", "libfrpca_synth.so")


class SynthSpec(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("row_law", C.c_int32),
                ("col_law", C.c_int32), ("val_law", C.c_int32), ("pad", C.c_int32),
                ("row_p", C.c_double), ("row_a", C.c_double), ("row_lo", C.c_double),
                ("row_hi", C.c_double), ("row_scale", C.c_double), ("row_lambda", C.c_double),
                ("col_a", C.c_double), ("seed", C.c_uint64)]


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config: matrix law + PcaConfig (k, s, q) + entry point."""
    name: str
    rows: int
    cols: int
    nnz_target: int
    row_law: int          # 0 Bernoulli(p), 1 Zipf(row_a) scaled+clipped, 2 Poisson(row_lambda)
    row_a: float = 0.0
    row_hi: float = 0.0
    row_p: float = 0.0
    row_lambda: float = 0.0
    col_law: int = 0      # 0 uniform, 1 Zipf(col_a) over a seeded permutation
    col_a: float = 0.0
    val_law: int = 0      # 0 U(0,1), 1 lognormal(0,1), 2 Poisson(1)+1, 3 1.0|U(1,5) 10%, 4 N(0,1)
    k: int = 100
    s: int = 100
    q: int = 4
    seed: int = 0
    algorithm: str = "frpcat"


# BASELINE.json "configs", in order (seed = config index, PcaConfig::seed = 0).
CONFIGS = {
    "C0": Config("C0", 20000, 5000, 500000, row_law=0, row_p=0.005, val_law=0,
                 k=20, s=20, q=3, seed=0, algorithm="frpcat"),
    "C1": Config("C1", 1000000, 100000, 10000000, row_law=1, row_a=2.0, row_hi=2000,
                 col_law=1, col_a=1.1, val_law=1, k=100, s=100, q=4, seed=1, algorithm="frpcat"),
    "C2": Config("C2", 5000000, 500000, 100000000, row_law=1, row_a=2.0, row_hi=2000,
                 col_law=1, col_a=1.1, val_law=2, k=100, s=50, q=5, seed=2, algorithm="frpcat"),
    "C3": Config("C3", 12869521, 323899, 400000000, row_law=1, row_a=1.8, row_hi=5000,
                 col_law=1, col_a=1.05, val_law=3, k=100, s=100, q=3, seed=3, algorithm="frpcat"),
    "C4": Config("C4", 200000, 20000000, 400000000, row_law=2, row_lambda=2000.0,
                 col_law=1, col_a=1.2, val_law=4, k=100, s=100, q=4, seed=4, algorithm="frpca"),
}


@functools.lru_cache(maxsize=None)
def _lib():
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} missing: run paper_1810_06825_b200/build.py")
    L = C.CDLL(_SO)
    L.synth_solve_scale.restype = C.c_double
    L.synth_solve_scale.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double]
    L.synth_expected_degree.restype = C.c_double
    L.synth_expected_degree.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double]
    L.synth_degrees.argtypes = [C.POINTER(SynthSpec), C.c_int, C.c_void_p]
    L.synth_fill.argtypes = [C.POINTER(SynthSpec), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    return L


@functools.lru_cache(maxsize=None)
def _scale_for(a: float, hi: float, mean: float) -> float:
    return float(_lib().synth_solve_scale(a, 1.0, hi, mean))


def spec(cfg: Config, scale: float = 1.0) -> SynthSpec:
    rows = max(1, int(round(cfg.rows * scale)))
    cols = max(1, int(round(cfg.cols * scale)))
    sp = SynthSpec()
    sp.rows, sp.cols = rows, cols
    sp.row_law, sp.col_law, sp.val_law = cfg.row_law, cfg.col_law, cfg.val_law
    sp.row_p = cfg.row_p
    sp.row_a = cfg.row_a
    sp.row_lo = 1.0
    sp.row_hi = min(cfg.row_hi, cols) if cfg.row_hi else 0.0
    sp.row_lambda = min(cfg.row_lambda, cols / 4.0)
    sp.col_a = cfg.col_a
    sp.seed = cfg.seed
    if cfg.row_law == 1:
        mean = cfg.nnz_target / cfg.rows
        sp.row_scale = _scale_for(cfg.row_a, sp.row_hi, mean)
    return sp


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def generate(name: str, scale: float = 1.0, threads: int | None = None, alloc=None):
    """Returns (rows, cols, row_ptr, col_idx, values). `alloc(shape, dtype)` may
    supply the output arrays (e.g. pinned host memory)."""
    cfg = CONFIGS[name]
    sp = spec(cfg, scale)
    t = threads or default_threads()
    alloc = alloc or (lambda n, dt: np.empty(n, dtype=dt))
    row_ptr = alloc(sp.rows + 1, np.int64)
    _lib().synth_degrees(C.byref(sp), t, row_ptr.ctypes.data)
    nnz = int(row_ptr[-1])
    col_idx = alloc(nnz, np.int64)
    values = alloc(nnz, np.float64)
    _lib().synth_fill(C.byref(sp), t, row_ptr.ctypes.data, col_idx.ctypes.data, values.ctypes.data)
    return sp.rows, sp.cols, row_ptr, col_idx, values
