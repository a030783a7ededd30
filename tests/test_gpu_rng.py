"""Device Omega generator vs the libstdc++ stream the reference draws
(dense_kernels.hpp:19-28): golden vectors (tests/golden/omega_stream.json, made
by g++ from std::mt19937_64 + std::normal_distribution) and the oracle's
gaussian_matrix at sizes that cross many jump-ahead segments. Accept/reject
decisions are exact (they only use r2), so every value sits at its reference
position, and the device log is glibc's restated (glibc_log.cuh), so every
value is bitwise equal to the host's libstdc++ stream."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "omega_stream.json")))


def ulp_diff(a, b):
    ia = a.view(np.int64)
    ib = b.view(np.int64)
    return np.abs(ia - ib)


@pytest.mark.parametrize("case", range(len(GOLD["cases"])))
def test_device_stream_matches_golden(fb, ctx, case):
    c = GOLD["cases"][case]
    got = fb.gaussian_matrix(c["rows"], c["cols"], c["seed"]).ravel(order="F")
    want = np.array([float.fromhex(h) for h in c["values_hex"]])
    d = ulp_diff(got, want)
    assert d.max() == 0, f"{int((d != 0).sum())} values differ, max {d.max()} ulp"


@pytest.mark.parametrize("rows,cols,seed", [(1000, 7, 1), (100000, 40, 2), (2000000, 3, 3),
                                            (12345, 200, 0xA11CE)])
def test_device_stream_matches_host(fb, orc, rows, cols, seed):
    got = fb.gaussian_matrix(rows, cols, seed)
    want = orc.gaussian_matrix(rows, cols, seed)
    d = ulp_diff(got.ravel(order="F"), want.ravel(order="F"))
    assert d.max() == 0, f"{int((d != 0).sum())} values differ, max {d.max()} ulp"


def test_device_stream_deterministic(fb, ctx):
    a = fb.gaussian_matrix(50000, 10, 99)
    b = fb.gaussian_matrix(50000, 10, 99)
    assert np.array_equal(a, b)


def test_device_stream_moments(fb, ctx):  # test_dense_kernels.cpp:23-29
    g = fb.gaussian_matrix(10000, 1, 7).ravel()
    assert abs(g.mean()) < 0.05 and abs(g.var(ddof=1) - 1.0) < 0.1
