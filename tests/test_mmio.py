"""MatrixMarket ingestion (reference io.cpp:71-191).

CPU: our host parser + the reference's own assembly reproduce the
reference's read_matrix_market bit for bit, and every error case raises the
same class with the same message (line numbers included).  GPU: the full
read (host parse + device assembly) matches the reference."""
import numpy as np
import pytest

from paper_2011_08879_b200 import larch as lk

GOOD = {
    "general_real": """%%MatrixMarket matrix coordinate real general
% a comment

4 5 6
1 1 1.5
4 5 -2e-3
2 3 7
1 1 0.25
3 2 0
4 1 1e300
""",
    "symmetric_int": """%%MatrixMarket matrix coordinate integer symmetric
3 3 4
1 1 2
2 1 -1
3 2 -1
3 3 2
""",
    "pattern_upper": """%%MATRIXMARKET Matrix Coordinate Pattern General
2 2 3
1 2
2 1
2 2
""",
    "empty": """%%MatrixMarket matrix coordinate real general
3 3 0
""",
    "crlf_and_spaces": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n  1   1   3.0  \r\n2 2 4\r\n",
    "crlf_comments": "%%MatrixMarket matrix coordinate real general\r\n% c\r\n%\r\n2 2 1\r\n1 1 3.0\r\n",
    "crlf_pattern": "%%MatrixMarket matrix coordinate pattern general\r\n2 2 1\r\n1 1\r\n",
}

BAD = {
    "no_banner": "MatrixMarket matrix coordinate real general\n1 1 0\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1\n",
    "vector": "%%MatrixMarket vector coordinate real general\n2 1\n1 1\n",
    "short_size": "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "bad_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n",
    "bad_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0abc\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "missing_value": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n",
    "negative": "%%MatrixMarket matrix coordinate real general\n-2 2 0\n",
    "empty_file": "",
    # a CRLF blank line is "\r" to std::getline: not empty, so the reference
    # parses it as the size / an entry line and fails
    "crlf_blank_before_size": "%%MatrixMarket matrix coordinate real general\r\n\r\n2 2 1\r\n1 1 3.0\r\n",
    "crlf_blank_between": "%%MatrixMarket matrix coordinate real general\r\n2 2 2\r\n1 1 3.0\r\n\r\n2 2 4\r\n",
    "cr_only": "%%MatrixMarket matrix coordinate real general\r2 2 1\r1 1 3.0\r",
}


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(text.encode())
    return str(p)


@pytest.mark.parametrize("name", sorted(GOOD))
def test_parse_matches_reference(R, tmp_path, name):
    O = R
    path = _write(tmp_path, name, GOOD[name])
    nr, nc, rows, cols, vals = O.ref_read_mm(path)
    mr, mc, er, ec, ev = lk.read_matrix_market_entries(path)
    assert (mr, mc) == (nr, nc)
    ro, co, vo = O.ref_coo_from_entries(mr, mc, er, ec, ev)
    assert np.array_equal(ro, rows) and np.array_equal(co, cols) and np.array_equal(vo, vals)


@pytest.mark.parametrize("name", sorted(BAD))
def test_errors_match_reference(R, tmp_path, name):
    O = R
    path = _write(tmp_path, name, BAD[name])
    with pytest.raises(O.OracleError) as ref_err:
        O.ref_read_mm(path)
    with pytest.raises(lk.FormatError) as ours:
        lk.read_matrix_market_entries(path)
    want_unsupported = ref_err.value.status == 11
    assert isinstance(ours.value, lk.UnsupportedFormatError) == want_unsupported
    assert str(ours.value) == ref_err.value.msg


def test_missing_file():
    with pytest.raises(lk.FormatError):
        lk.read_matrix_market_entries("/nonexistent/file.mtx")


def test_stencil_roundtrip_matches_reference(R, tmp_path):
    """A 5-pt stencil written as symmetric MatrixMarket (lower triangle)."""
    O = R
    A = O.stencil("5pt", 20)
    lines = []
    for r in range(A.nrows):
        for k in range(A.row_ptr[r], A.row_ptr[r + 1]):
            if A.cols[k] <= r:
                lines.append(f"{r + 1} {A.cols[k] + 1} {float(A.vals[k])!r}")
    text = "%%MatrixMarket matrix coordinate real symmetric\n" + \
        f"{A.nrows} {A.ncols} {len(lines)}\n" + "\n".join(lines) + "\n"
    path = _write(tmp_path, "st5", text)
    nr, nc, rows, cols, vals = O.ref_read_mm(path)
    mr, mc, er, ec, ev = lk.read_matrix_market_entries(path)
    ro, co, vo = O.ref_coo_from_entries(mr, mc, er, ec, ev)
    assert np.array_equal(ro, rows) and np.array_equal(co, cols) and np.array_equal(vo, vals)
    assert np.array_equal(co, A.cols) and np.array_equal(vo, A.vals)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["general_real", "symmetric_int", "pattern_upper", "empty"])
def test_device_read_matches_reference(R, ex, tmp_path, name):
    O = R
    path = _write(tmp_path, name, GOOD[name])
    nr, nc, rows, cols, vals = O.ref_read_mm(path)
    M = lk.read_matrix_market(ex, path)
    assert (M.nrows, M.ncols) == (nr, nc)
    assert np.array_equal(M.row_idx.cpu().numpy(), rows)
    assert np.array_equal(M.col_idx.cpu().numpy(), cols)
    assert np.array_equal(M.vals.cpu().numpy(), vals)


def test_hostile_nnz_header(tmp_path):
    """an nnz near INT64_MAX in the size line (symmetric: 2*nnz
    would overflow) is a FormatError from the short entry list, not an
    exception escaping the C ABI."""
    path = _write(tmp_path, "huge", "%%MatrixMarket matrix coordinate real symmetric\n"
                  "2 2 9223372036854775000\n1 1 1.0\n")
    with pytest.raises(lk.FormatError):
        lk.read_matrix_market_entries(path)
