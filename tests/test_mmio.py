"""Matrix Market reader / writer (csrc/mmio.cpp) against the reference's
read_matrix_market / write_matrix_market (matrix_market.cpp:29-110),
compiled in oracle/_ref.

CPU: every malformed input fails before any device work, with the
reference's status code and message (line numbers included) -- a corpus of
header, size-line and entry-line defects, blank and comment lines, early
end of file, entries after the nnz-th that must be ignored, and a large
file so the parallel chunked tokeniser is exercised.  GPU: valid inputs
(general, symmetric, duplicates in and out of order, CRLF, tabs, trailing
text) give the reference's CSR bit for bit, and the writer's bytes equal
the reference's.
"""
import numpy as np
import pytest

HDR = "%%MatrixMarket matrix coordinate real general\n"
SYM = "%%MatrixMarket matrix coordinate real symmetric\n"

BAD = {
    "empty": "",
    "no_banner": "not a banner\n3 3 0\n",
    "array": "%%MatrixMarket matrix array real general\n3 3\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n",
    "short_header": "%%MatrixMarket matrix coordinate\n",
    "no_size": HDR + "% only a comment\n\n",
    "bad_size": HDR + "3 x 3\n",
    "size_float": HDR + "3.5 3 1\n",
    "rect": HDR + "2 3 0\n",
    "bad_entry": HDR + "3 3 2\n1 1 1.0\n2 two 1.0\n",
    "entry_two_tokens": HDR + "3 3 1\n1 1\n",
    "entry_range": HDR + "3 3 2\n1 1 1.0\n4 1 1.0\n",
    "entry_zero_index": HDR + "3 3 1\n0 1 1.0\n",
    "entry_inf_text": HDR + "3 3 1\n1 1 inf\n",
    "entry_overflow": HDR + "3 3 1\n1 1 1e400\n",
    "entry_exp_only": HDR + "3 3 1\n1 1 1e\n",
    "comment_in_entries": HDR + "3 3 2\n1 1 1.0\n% comment\n2 2 1.0\n",
    "eof_in_entries": HDR + "3 3 3\n1 1 1.0\n\n2 2 1.0\n",
    "eof_after_blank": HDR + "%c\n\n3 3 2\n\n1 1 1.0\n   \n",
    "vtab_line": HDR + "3 3 1\n\v\n",
    "neg_dim": HDR + "-2 -2 0\n",
    "index_overflow": HDR + "3 3 1\n99999999999999999999 1 1.0\n",
}

GOOD = {
    "general": HDR + "3 3 4\n1 1 2.0\n3 1 -1.5\n2 2 4\n3 3 1e-3\n",
    "dups": HDR + "3 3 5\n2 1 1.0\n1 1 0.1\n2 1 2.0\n2 1 0.3\n1 1 -0.1\n",
    "symmetric": SYM + "4 4 5\n1 1 4.0\n2 1 -1.0\n3 2 -1.0\n4 4 2.0\n4 1 0.5\n",
    "crlf_tabs": "%%MatrixMarket\tmatrix coordinate REAL General\r\n%x\r\n3 3 2\r\n\t1\t2\t+3.25\r\n\r\n3 3 .5e1 trailing\r\n",
    "extra_after_nnz": HDR + "3 3 1\n1 1 1.0\nthis line is never read\n",
    "plus_sign_and_hex": HDR + "2 2 2\n+1 +1 0x10\n2 2 -0.0\n",
    "zero_nnz": HDR + "3 3 0\n",
    "denormal": HDR + "2 2 1\n1 1 1e-320\n",
    "no_trailing_newline": HDR + "2 2 2\n1 1 1\n2 2 2",
}


def big_text(n=40000, seed=0, bad_at=None):
    rng = np.random.default_rng(seed)
    rows = rng.integers(1, n + 1, 6 * n)
    cols = rng.integers(1, n + 1, 6 * n)
    vals = rng.standard_normal(6 * n)
    lines = [f"{int(r)} {int(c)} {float(v)!r}" for r, c, v in zip(rows, cols, vals)]
    for k in range(0, len(lines), 997):
        lines.insert(k, "")  # blank lines inside the entry list
    if bad_at is not None:
        lines[bad_at] = "1 1 nan"
    nnz = sum(1 for x in lines if x)
    return HDR + f"% generated\n{n} {n} {nnz}\n" + "\n".join(lines) + "\n"


def write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(text.encode())
    return str(p)


@pytest.mark.parametrize("name", sorted(BAD))
def test_parse_errors_match_reference(P, ref, tmp_path, name):
    path = write(tmp_path, name, BAD[name])
    with pytest.raises(Exception) as er:
        ref.read_matrix_market(path)
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.read_matrix_market(path)
    assert e.value.status == er.value.status, (name, e.value.message, er.value.message)
    assert e.value.message == er.value.message, name


@pytest.mark.parametrize("bad_at", [5, 150000, 239000])
def test_parse_errors_large_file(P, ref, tmp_path, bad_at):
    """Above 4 MB the entry section is tokenised in parallel chunks: the
    first bad line must still be the one reported."""
    path = write(tmp_path, "big", big_text(bad_at=bad_at))
    with pytest.raises(Exception) as er:
        ref.read_matrix_market(path)
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.read_matrix_market(path)
    assert (e.value.status, e.value.message) == (er.value.status, er.value.message)


def test_missing_entries_large_file(P, ref, tmp_path):
    lines = big_text().split("\n")
    n, _, nnz = lines[2].split()
    lines[2] = f"{n} {n} {int(nnz) + 7}"
    path = write(tmp_path, "short", "\n".join(lines))
    with pytest.raises(Exception) as er:
        ref.read_matrix_market(path)
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.read_matrix_market(path)
    assert (e.value.status, e.value.message) == (er.value.status, er.value.message)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOOD) + ["big"])
def test_read_matches_reference(P, ref, tmp_path, name):
    path = write(tmp_path, name, big_text() if name == "big" else GOOD[name])
    rp, ci, v = ref.read_matrix_market(path)
    A = P.Matrix.read_matrix_market(path)
    grp, gci, gv = A.csr()
    assert np.array_equal(grp, rp) and np.array_equal(gci, ci)
    assert np.array_equal(gv.view(np.uint64), v.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["general", "dups", "symmetric", "big"])
def test_write_bytes_match_reference(P, ref, tmp_path, name):
    src = write(tmp_path, name, big_text() if name == "big" else GOOD[name])
    csr = ref.read_matrix_market(src)
    ours, theirs = tmp_path / "ours.mtx", tmp_path / "theirs.mtx"
    P.Matrix.from_csr(*csr).write_matrix_market(str(ours))
    ref.write_matrix_market(csr, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
