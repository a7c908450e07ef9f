"""Edge cases the reference handles: empty matrices, 1x1, a single dense row,
identity / diagonal inputs, all-dropped off-diagonals, exact zeros kept by
spgemm (kernels.hpp:18-20), and vectors of length zero."""
import numpy as np
import pytest

from helpers import bitwise_equal, bitwise_equal_csr, to_oracle, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def test_empty_matrix_everything(S, port):
    e = S.CsrMatrix(0, 0, [0], [], [])
    for lower in (True, False):
        kind = S.lower_triangular if lower else S.upper_triangular
        m = S.sait_thr(e, kind, S.SaitThrParams(0.1, 3))
        assert m.nrows == 0 and m.nnz() == 0
        assert S.sait_pat(e, kind, S.SaitPatParams(2, 2)).nnz() == 0
    pair = S.SaitPairPreconditioner(e, e)
    z = np.empty(0)
    pair.apply(np.empty(0), z)
    assert S.spgemm(e, e).nnz() == 0
    assert S.transpose(e).nnz() == 0


def test_one_by_one(S, port):
    t = S.CsrMatrix(1, 1, [0, 1], [0], [4.0])
    m = S.sait_thr(t, S.lower_triangular, S.SaitThrParams(0.5, 5))
    assert list(m.values) == [0.25]
    pair = S.SaitPairPreconditioner(m, m)
    z = np.empty(1)
    pair.apply(np.array([8.0]), z)
    assert z[0] == 0.5
    with pytest.raises(S.SaitRuntimeError, match="zero diagonal at row 0"):
        S.sait_thr(S.CsrMatrix(1, 1, [0, 1], [0], [0.0]), S.lower_triangular, S.SaitThrParams(0.5, 1))


def test_dense_last_row_and_exact_zeros(S, port):
    """A lower T whose last row is dense (a long row for every kernel), with
    values chosen so some products cancel to exactly 0.0 (kept, not dropped,
    when tau = 0)."""
    n = 3000
    rows, cols, vals = [], [], []
    rng = np.random.default_rng(1)
    for i in range(n):
        rows.append(i); cols.append(i); vals.append(2.0)
        if i == n - 1:
            for j in range(i):
                rows.append(i); cols.append(j); vals.append(float(rng.choice([-1.0, 1.0])))
        elif i > 0:
            rows.append(i); cols.append(i - 1); vals.append(1.0)
    import scipy.sparse as sp

    T = S.CsrMatrix.from_scipy(sp.csr_matrix((vals, (rows, cols)), shape=(n, n)))
    for tau, k in ((0.0, 4), (0.3, 6)):
        got = S.sait_thr(T, S.lower_triangular, S.SaitThrParams(tau, k))
        assert bitwise_equal_csr(got, port.sait_thr(to_oracle(T), True, tau, k))
    M = S.sait_thr(T, S.lower_triangular, S.SaitThrParams(0.0, 4))
    pair = S.SaitPairPreconditioner(M, S.transpose(M))
    r = rng.standard_normal(n)
    z = np.empty(n)
    pair.apply(r, z)
    assert bitwise_equal(z, port.pair_apply(to_oracle(M), to_oracle(S.transpose(M)), r))


def test_diagonal_and_identity_inputs(S):
    d = S.CsrMatrix(5, 5, np.arange(6), np.arange(5), [1.0, 2.0, 4.0, 8.0, -16.0])
    m = S.sait_thr(d, S.upper_triangular, S.SaitThrParams(0.9, 7))
    assert list(m.values) == [1.0, 0.5, 0.25, 0.125, -0.0625]
    assert list(S.sait_pat_capture_pattern(d, S.lower_triangular, 3).col_idx) == list(range(5))


def test_everything_dropped_but_diagonal(S, port):
    from oracle import oracle as O

    T = O.synthetic_lower(500, 4, 0.1, seed=3)
    got = S.sait_thr(to_product(T), S.lower_triangular, S.SaitThrParams(0.999, 3))
    exp = port.sait_thr(T, True, 0.999, 3)
    assert bitwise_equal_csr(got, exp) and got.nnz() == 500


def test_nonfinite_values_in_build(S, port):
    """NaN entries are dropped by a positive threshold (|NaN| >= tau is false)
    unless diagonal, kept when tau == 0 — exactly as drop_by_threshold."""
    import scipy.sparse as sp

    n = 50
    a = sp.tril(sp.random(n, n, density=0.2, random_state=2), k=-1).tolil()
    a[10, 3] = np.nan
    a = (a + 3 * sp.eye(n)).tocsr()
    a.sort_indices()
    T = S.CsrMatrix.from_scipy(a)
    for tau in (0.0, 0.05):
        got = S.sait_thr(T, S.lower_triangular, S.SaitThrParams(tau, 3))
        exp = port.sait_thr(to_oracle(T), True, tau, 3)
        assert np.array_equal(got.row_ptr, exp.row_ptr) and np.array_equal(got.col_idx, exp.col_idx)
        assert np.array_equal(np.isnan(got.values), np.isnan(exp.values))
        fin = ~np.isnan(exp.values)
        assert bitwise_equal(got.values[fin], exp.values[fin])


def test_device_pool_reserve():
    """sait_device_pool_reserve grows the pool; negative sizes are invalid"""
    import paper_2106_12836_b200 as S

    S.reserve_device_pool(64 << 20)
    S.reserve_device_pool(0)
    with pytest.raises(S.SaitInvalidArgument):
        S.reserve_device_pool(-1)


@pytest.mark.parametrize("fmt", ["csr", "sell32_int32", "sell32_int16", "sell32_dict"])
def test_forced_formats_on_tiny_and_empty(S, port, fmt):
    """Every forced apply format on an empty pair, a 1x1 pair and a 33-row
    pair (one full slice + one 1-row slice); the format reports its storage."""
    e = S.CsrMatrix(0, 0, [0], [], [])
    pe = S.SaitPairPreconditioner(e, e, format=fmt)
    pe.apply(np.empty(0), np.empty(0))
    t = S.CsrMatrix(1, 1, [0, 1], [0], [2.0])
    p1 = S.SaitPairPreconditioner(t, t, format=fmt)
    z = np.empty(1)
    p1.apply(np.array([3.0]), z)
    assert z[0] == 12.0
    n = 33
    A = S.laplacian_2d(6)  # 36 rows
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(0.0, 2))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(0.0, 2))
    pair = S.SaitPairPreconditioner(ML, MU, format=fmt)
    r = S.uniform_pm1(9, A.nrows)
    z = np.empty(A.nrows)
    pair.apply(r, z)
    assert bitwise_equal(z, port.pair_apply(to_oracle(ML), to_oracle(MU), r))
    assert pair.factor_format(0)["nnz"] == ML.nnz()
    del n


def test_spmm_edge_widths(S, port):
    """sait_spmm (dense.hpp:41 block product): widths 0, 1, 7, 9, 17 on the
    device are each column's spmv bitwise; an empty matrix is a no-op."""
    import torch

    from paper_2106_12836_b200 import _native as N

    A = S.laplacian_2d(20)
    Ao = to_oracle(A)
    d = S.DeviceCsr.upload(A)
    n = A.nrows
    for w in (0, 1, 7, 9, 17):
        X = torch.from_numpy(np.concatenate([S.uniform_pm1(70 + c, n) for c in range(w)]) if w else np.zeros(0)).cuda()
        Y = torch.empty(max(1, n * w), dtype=torch.float64, device="cuda")
        N.check(N.lib.sait_spmm(d.handle, X.data_ptr() if w else 0, Y.data_ptr(), w, None))
        torch.cuda.synchronize()
        if w:
            want = np.concatenate([port.spmv(Ao, S.uniform_pm1(70 + c, n)) for c in range(w)])
            assert bitwise_equal(Y.cpu().numpy()[: n * w], want)
    e = S.DeviceCsr.upload(S.CsrMatrix(0, 0, [0], [], []))
    N.check(N.lib.sait_spmm(e.handle, 0, 0, 3, None))


def test_assemble_rows_edge_cases(S):
    """sait_csr_assemble_rows with no pieces (an all-empty row block) and
    with pieces whose rows are all empty; sait_csr_col_span of an empty block."""
    import ctypes as C

    import torch

    from paper_2106_12836_b200 import _native as N
    from paper_2106_12836_b200.dist import assemble_row_block, row_block_span

    blk = assemble_row_block({}, [0, 5], 4, 5)
    h = blk.to_host()
    assert h.nrows == 4 and h.nnz() == 0 and list(h.row_ptr) == [0, 0, 0, 0, 0]
    assert row_block_span(blk, 0, 4) == (0, 0)
    rp = torch.zeros(5, dtype=torch.int32, device="cuda")
    ci = torch.zeros(1, dtype=torch.int32, device="cuda")
    v = torch.zeros(1, dtype=torch.float64, device="cuda")
    blk2 = assemble_row_block({0: {"rp": rp, "ci": ci, "v": v, "nnz": 0, "nrows": 4}}, [0, 5], 4, 5)
    assert blk2.to_host().nnz() == 0
    with pytest.raises(S.SaitInvalidArgument):
        N.check(N.lib.sait_csr_assemble_rows(-1, None, 4, 5, None, C.byref(C.c_void_p())))
