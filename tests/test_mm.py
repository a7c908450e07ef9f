"""Matrix Market ingestion (F4, spec-only in the reference)
and make_rhs.  Host code: checked on CPU against scipy's
independent reader, the spec's examples and round trips."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def write(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_spec_minimal_identity(S, tmp_path):
    p = write(tmp_path, "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 1.0")
    m = S.mm_read(p)
    assert (m.nrows, m.ncols) == (2, 2)
    assert list(m.row_ptr) == [0, 1, 2] and list(m.col_idx) == [0, 1] and list(m.values) == [1.0, 1.0]


def test_symmetric_expansion_matches_scipy(S, tmp_path):
    import scipy.io
    import scipy.sparse as sp

    rng = np.random.default_rng(1)
    n = 300
    a = sp.random(n, n, density=0.02, random_state=2, format="coo")
    a = sp.tril(a + a.T).tocoo()
    a.data = rng.uniform(-3, 3, a.nnz)
    a = (a + sp.diags(rng.uniform(5, 6, n))).tocoo()
    p = tmp_path / "sym.mtx"
    scipy.io.mmwrite(str(p), a, symmetry="symmetric", precision=17)
    m = S.mm_read(p)
    ref = sp.csr_matrix(scipy.io.mmread(str(p), spmatrix=False))
    ref.sum_duplicates()
    ref.sort_indices()
    assert np.array_equal(m.row_ptr, ref.indptr) and np.array_equal(m.col_idx, ref.indices)
    assert np.array_equal(m.values.view(np.uint64), ref.data.view(np.uint64))
    full = m.nnz()
    assert full == 2 * a.nnz - n  # off-diagonals mirrored, the diagonal once


def test_general_with_comments_integer_and_duplicates(S, tmp_path):
    text = (
        "%%MatrixMarket matrix coordinate integer general\n"
        "% a comment\n"
        "%\n"
        "3 4 5\n"
        "3 4 7\n"
        "1 2 1\n"
        "\n"
        "1 2 2\n"  # duplicate of (1, 2): summed in file order
        "2 1 -4\n"
        "1 1 5\n"
    )
    m = S.mm_read(write(tmp_path, text))
    assert (m.nrows, m.ncols) == (3, 4)
    assert list(m.row_ptr) == [0, 2, 3, 4]
    assert list(m.col_idx) == [0, 1, 0, 3]
    assert list(m.values) == [5.0, 3.0, -4.0, 7.0]


def test_round_trip_bitwise(S, tmp_path):
    from paper_2106_12836_b200 import CsrMatrix

    rng = np.random.default_rng(7)
    a = S.convdiff_2d(40)
    vals = a.values * rng.uniform(0.1, 10, a.nnz()) + rng.standard_normal(a.nnz()) * 1e-300
    vals[3] = np.inf
    vals[5] = -0.0
    m = CsrMatrix(a.nrows, a.ncols, a.row_ptr, a.col_idx, vals)
    p = tmp_path / "rt.mtx"
    S.mm_write(p, m)
    r = S.mm_read(p)
    assert np.array_equal(r.row_ptr, m.row_ptr) and np.array_equal(r.col_idx, m.col_idx)
    assert np.array_equal(r.values.view(np.uint64), m.values.view(np.uint64))


@pytest.mark.parametrize(
    "text,err",
    [
        ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "line 1: format 'array'"),
        ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "line 1: field 'complex' not supported"),
        ("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n", "line 1: field 'pattern' not supported"),
        ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n", "line 1: symmetry 'hermitian'"),
        ("%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1\n", "line 1: missing %%MatrixMarket banner"),
        ("%%MatrixMarket matrix coordinate real general\n% c\n2 2\n", "line 3: malformed size line"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 2.0\n", "line 4: index (3, 1) out of bounds for 2x2"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n0 1 2.0\n", "line 4: index (0, 1) out of bounds"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 x\n", "line 3: malformed entry value"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n", "line 4: file ends after 2 of 3 entries"),
        ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n2 2 1\n", "line 4: more entries than the size line states"),
        ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 1\n", "line 3: symmetric file has an entry above"),
        ("", "line 1: empty file"),
    ],
)
def test_parse_errors_name_the_line(S, tmp_path, text, err):
    with pytest.raises(S.SaitInvalidArgument, match="^mm_read: " + err.replace("(", r"\(").replace(")", r"\)")):
        S.mm_read(write(tmp_path, text))


def test_missing_file(S, tmp_path):
    with pytest.raises(S.SaitInvalidArgument, match="cannot open"):
        S.mm_read(tmp_path / "nope.mtx")


def test_make_rhs_spec_examples(S):
    from paper_2106_12836_b200 import CsrMatrix

    eye = CsrMatrix(4, 4, np.arange(5), np.arange(4), np.ones(4))
    assert np.array_equal(S.make_rhs(eye, "ones-solution"), np.ones(4))
    a = S.laplacian_3d(2)
    b = S.make_rhs(a, "ones-solution")
    nbrs = np.diff(a.row_ptr) - 1
    assert np.array_equal(b, 6.0 - nbrs)
    r1 = S.make_rhs(a, "seeded-random", 11)
    r2 = S.make_rhs(a, "seeded-random", 11)
    assert np.array_equal(r1.view(np.uint64), r2.view(np.uint64))
    assert abs(np.linalg.norm(r1) - 1.0) < 1e-15
    with pytest.raises(S.SaitInvalidArgument):
        S.make_rhs(a, "zeros")
