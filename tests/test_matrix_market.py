"""Matrix Market ingestion: the B200 reader against the reference's own
read_matrix_market (oracle/_ref, matrix_market.cpp:26-91) on the same files -- identical CSR
arrays, identical IngestionError texts.  Host-only code, so these run without a GPU; the device
operator built from a file is checked in the gpu-marked test at the end.
"""
import numpy as np
import pytest

from oracle import ref
from paper_2506_08355_b200 import bosp

needs_ref = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def ours(path):
    out = bosp.read_matrix_market(path)
    if isinstance(out, tuple):
        return out
    return out.n, out.n, out.rowptr, out.colidx, out.vals


def same(path):
    a = ours(path)
    b = ref.read_matrix_market(path)
    assert a[0] == b[0] and a[1] == b[1]
    for u, v in zip(a[2:], b[2:]):
        assert np.array_equal(np.asarray(u), np.asarray(v)), (u, v)
    return a


GENERAL = """%%MatrixMarket matrix coordinate real general
% a comment
%another
4 4 7

3 1 -2.5
1 1 4.0
1 2 1e-3
4 4 +2
3 1 0.5
2 2 7
1 4 -1.25E+1
"""

SYMMETRIC = """%%MatrixMarket MATRIX Coordinate Real Symmetric
5 5 6
1 1 2
2 1 -1
2 2 2
3 2 -1
5 3 0.25
5 5 3
"""


@needs_ref
def test_general_with_comments_duplicates_and_empty_rows(tmp_path):
    n, m, rp, ci, vv = same(write(tmp_path, "g.mtx", GENERAL))
    assert (n, m) == (4, 4)
    assert list(rp) == [0, 3, 4, 5, 6]  # row 3 (index 2) holds the summed duplicate
    assert vv[4] == -2.0


@needs_ref
def test_symmetric_expansion(tmp_path):
    n, _, rp, ci, vv = same(write(tmp_path, "s.mtx", SYMMETRIC))
    dense = np.zeros((n, n))
    for r in range(n):
        dense[r, ci[rp[r]:rp[r + 1]]] = vv[rp[r]:rp[r + 1]]
    assert np.array_equal(dense, dense.T)
    assert dense[2, 4] == 0.25 and dense[4, 2] == 0.25


@needs_ref
def test_rectangular_and_random_large(tmp_path):
    same(write(tmp_path, "r.mtx", "%%MatrixMarket matrix coordinate real general\n3 5 2\n1 5 1.0\n3 2 -1.0\n"))
    rng = np.random.default_rng(3)
    n, k = 3000, 40000
    i = rng.integers(1, n + 1, k)
    j = rng.integers(1, n + 1, k)
    v = rng.standard_normal(k)
    lines = ["%%MatrixMarket matrix coordinate real general", f"{n} {n} {k}"]
    lines += [f"{int(a)} {int(b)} {float(c)!r}" for a, b, c in zip(i, j, v)]
    same(write(tmp_path, "big.mtx", "\n".join(lines) + "\n"))


BAD = {
    "empty": "",
    "banner": "%%MatrixMarkt matrix coordinate real general\n1 1 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n1 1\n1\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "nosize": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "badsize": "%%MatrixMarket matrix coordinate real general\n3 x 2\n",
    "badentry": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 two 3\n",
    "bounds0": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n",
    "bounds": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 3 1.0\n",
    "eof": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(BAD))
def test_malformed_files_same_error(tmp_path, case):
    path = write(tmp_path, case + ".mtx", BAD[case])
    with pytest.raises(bosp.IngestionError) as ours_err:
        bosp.read_matrix_market(path)
    with pytest.raises(ref.RefError) as ref_err:
        ref.read_matrix_market(path)
    assert ref_err.value.kind == "IngestionError"
    assert str(ref_err.value).split(": ", 1)[1] in str(ours_err.value)


def test_missing_file(tmp_path):
    with pytest.raises(bosp.IngestionError, match="cannot open file"):
        bosp.read_matrix_market(str(tmp_path / "nope.mtx"))


@pytest.mark.gpu
def test_operator_from_file_applies(tmp_path):
    from paper_2506_08355_b200 import problems as P
    t = P.t_matrix(500, -1.0)
    rows, cols = np.repeat(np.arange(500), np.diff(t.rowptr)), t.colidx
    body = "\n".join(f"{int(r) + 1} {int(c) + 1} {float(v)!r}" for r, c, v in zip(rows, cols, t.vals))
    path = write(tmp_path, "t.mtx", f"%%MatrixMarket matrix coordinate real general\n500 500 {len(t.vals)}\n{body}\n")
    op = bosp.LinearOperator.from_matrix_market(path)
    x = np.random.default_rng(0).standard_normal((500, 3))
    assert np.allclose(op.apply(x), t.scipy() @ x, rtol=0, atol=1e-13)
