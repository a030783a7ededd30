"""SURVEY §8 row f2 (the load step), host side: the library's Matrix Market
reader (csrc/mtx.cpp, parallel chunks) against the oracle's line-by-line
restatement of load_matrix_market (matrix_market.hpp:27-93, istream
extraction): same triplets in the same order, bitwise values, same error
messages; and write_matrix_market (:95-116) round trips exactly."""
import os

import numpy as np
import pytest

BANNER = "%%MatrixMarket matrix coordinate real general\n"


def both(fb, orc, path):
    """(library result or its exception message, oracle result or message)."""
    out = []
    for f, exc in ((fb.read_matrix_market, fb.IoError), (orc.read_matrix_market, OSError)):
        try:
            out.append(f(str(path)))
        except exc as e:
            out.append(str(e))
    return out


def same(a, b):
    if isinstance(a, str) or isinstance(b, str):
        return a == b
    return a[0] == b[0] and a[1] == b[1] and all(np.array_equal(x, y) for x, y in zip(a[2:], b[2:]))


CASES = {
    "general": BANNER + "3 4 4\n1 1 1.5\n3 4 -2\n2 2 1e-3\n1 4 7\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 2.0\n2 1 -1.5\n3 2 4e-3\n",
    "integer_upper": "%%MatrixMarket MATRIX Coordinate Integer General\n2 2 2\n1 2 3\n2 1 -4\n",
    "upper_tag": "%%MATRIXMARKET matrix coordinate real general\n1 1 0\n",
    "comments_blanks": BANNER + "% c1\n\n%c2\n2 2 2\n% mid\n\n1 1 1\n%x\n2 2 2\n",
    "extra_lines_ignored": BANNER + "2 2 1\n1 1 1\n2 2 garbage here\n",
    "crlf": BANNER.replace("\n", "\r\n") + "2 2 2\r\n1 1 1.25\r\n2 2 2.5\r\n",
    "crlf_blank": BANNER + "2 2 2\n1 1 1\n\r\n2 2 2\n",
    "numbers": BANNER + "1 6 6\n1 1 +1.5\n1 2 .5\n1 3 5.\n1 4 1E-3\n1 5 -0\n1 6 0x10\n",
    "trailing_text": BANNER + "2 2 1\n1 2 3.5abc\n",
    "duplicates": BANNER + "2 2 4\n1 1 1\n1 1 2\n2 2 3\n1 1 -3\n",
    "empty_matrix": BANNER + "4 5 0\n",
    "no_final_newline": BANNER + "2 2 1\n2 1 9",
    # errors
    "missing_banner": "%MatrixMarket matrix coordinate real general\n1 1 0\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 0\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 0\n",
    "empty": "",
    "missing_size": BANNER + "% only comments\n",
    "bad_size": BANNER + "2 x 1\n",
    "negative_size": BANNER + "2 -2 1\n",
    "sym_not_square": "%%MatrixMarket matrix coordinate real symmetric\n2 3 0\n",
    "out_of_range": BANNER + "2 2 1\n3 1 1\n",
    "zero_index": BANNER + "2 2 1\n0 1 1\n",
    "malformed_entry": BANNER + "2 2 1\n1 1\n",
    "inf_value": BANNER + "2 2 1\n1 1 inf\n",
    "float_index": BANNER + "2 2 1\n1.0 1 1\n",
    "early_eof": BANNER + "2 2 3\n1 1 1\n% c\n",
    "error_after_count_ignored": BANNER + "2 2 1\n1 1 1\n0 0 x\n",
}


ERRORS = {"missing_banner", "upper_tag", "array", "complex", "pattern", "hermitian", "empty", "missing_size", "bad_size",
          "negative_size", "sym_not_square", "out_of_range", "zero_index", "malformed_entry", "inf_value",
          "float_index", "early_eof", "crlf_blank"}


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_matches_reference_restatement(fb, orc, tmp_path, name):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(CASES[name].encode())
    a, b = both(fb, orc, p)
    assert same(a, b), (a, b)
    assert isinstance(a, str) == (name in ERRORS), a


def test_missing_file(fb, orc, tmp_path):
    a, b = both(fb, orc, tmp_path / "nope.mtx")
    assert isinstance(a, str) and a == b and "cannot open" in a


def _big(tmp_path, rng, symmetric, n, m, nnz, err_at=None):
    lines = ["%%MatrixMarket matrix coordinate real " + ("symmetric" if symmetric else "general"), "% big"]
    lines.append(f"{n} {m} {nnz}")
    i = rng.integers(1, n + 1, nnz)
    j = rng.integers(1, m + 1, nnz)
    if symmetric:
        i, j = np.maximum(i, j), np.minimum(i, j)
    v = rng.standard_normal(nnz) * 10.0 ** rng.integers(-5, 5, nnz)
    for t in range(nnz):
        if t % 997 == 0:
            lines.append("% interleaved comment")
        if t % 1499 == 0:
            lines.append("")
        if err_at is not None and t == err_at:
            lines.append(f"{i[t]} {j[t]} not-a-number")
            continue
        lines.append(f"{i[t]} {j[t]} {float(v[t])!r}")
    p = tmp_path / "big.mtx"
    p.write_text("\n".join(lines) + "\n")
    return p


@pytest.mark.parametrize("symmetric", [False, True])
def test_reader_big_file_parallel_chunks(fb, orc, tmp_path, symmetric):
    """Several MB, so the library parses in parallel chunks; interleaved
    comments and blank lines; order and values must match exactly."""
    rng = np.random.default_rng(7 + symmetric)
    p = _big(tmp_path, rng, symmetric, 5000, 5000 if symmetric else 3000, 200000)
    assert os.path.getsize(p) > (1 << 21)
    a, b = both(fb, orc, p)
    assert not isinstance(a, str), a
    assert same(a, b)
    assert a[2].size == (200000 if not symmetric else 200000 + int(np.count_nonzero(a[2] != a[3]) // 2))


@pytest.mark.parametrize("err_at", [3, 120000, 199999])
def test_reader_big_file_first_error(fb, orc, tmp_path, err_at):
    rng = np.random.default_rng(11)
    p = _big(tmp_path, rng, False, 5000, 3000, 200000, err_at=err_at)
    a, b = both(fb, orc, p)
    assert isinstance(a, str) and a == b


def test_write_read_round_trip(fb, orc, tmp_path):
    A = orc.Csr.random_sparse(300, 200, 0.05, 5)
    rp, ci, va = A.arrays()
    va = va * 10.0 ** np.random.default_rng(1).integers(-12, 12, va.size)
    B = fb.SparseMatrixCsr(300, 200, rp, ci, va)
    p = tmp_path / "w.mtx"
    fb.write_matrix_market(str(p), B)
    rows, cols, r, c, v = fb.read_matrix_market(str(p))
    assert (rows, cols) == (300, 200)
    C = fb.SparseMatrixCsr.from_triplets(rows, cols, (r, c, v))
    assert np.array_equal(C.rowPtr(), rp) and np.array_equal(C.colIdx(), ci) and np.array_equal(C.values(), va)
    assert p.read_text().startswith("%%MatrixMarket matrix coordinate real general\n300 200 ")
