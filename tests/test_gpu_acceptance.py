"""The reference's acceptance criteria, run on the device
path.  #7 needs SuiteSparse files (set SAIT_SUITESPARSE_DIR to a directory
holding thermomech_TC.mtx); everything else is synthetic."""
import os

import numpy as np
import pytest

from helpers import bitwise_equal, to_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def _random_triangular(rng, n, density, lower=True, dominant=True):
    import scipy.sparse as sp

    from paper_2106_12836_b200 import CsrMatrix

    m = sp.random(n, n, density=density, random_state=rng.integers(1 << 31), format="csr",
                  data_rvs=lambda k: rng.uniform(-1, 1, k))
    m = sp.tril(m, -1) if lower else sp.triu(m, 1)
    d = np.abs(m).sum(axis=1).A1 + 1.0 if dominant else np.ones(n)
    t = (m + sp.diags(d * rng.uniform(1.0, 2.0, n))).tocsr()
    t.sort_indices()
    return t, CsrMatrix(n, n, t.indptr.astype(np.int64), t.indices.astype(np.int64), t.data.copy())


def _csr_scipy(m):
    import scipy.sparse as sp

    return sp.csr_matrix((m.values, m.col_idx, m.row_ptr), shape=(m.nrows, m.ncols))


def test_1_exact_series_property(S):
    """sait_thr(T, 0, n - 1) is T^-1: ||T M - I||_inf <= 1e-10 (50 matrices)."""
    import scipy.sparse as sp

    rng = np.random.default_rng(1)
    for q in range(50):
        n = (5, 20, 64)[q % 3]
        lower = q % 2 == 0
        t, tp = _random_triangular(rng, n, 0.3, lower)
        kind = S.lower_triangular if lower else S.upper_triangular
        m = _csr_scipy(S.sait_thr(tp, kind, S.SaitThrParams(0.0, n - 1)))
        err = np.abs((t @ m - sp.identity(n)).toarray()).sum(axis=1).max()
        assert err <= 1e-10, (q, n, err)


@pytest.mark.parametrize("m", [1, 3, 7])
def test_2_jacobi_equivalence(S, m):
    """jacobi_sweeps_apply(T, b, m + 1) == spmv(sait_thr(T, 0, m), b) to 1e-12."""
    rng = np.random.default_rng(2 + m)
    for lower in (True, False):
        _, tp = _random_triangular(rng, 100, 0.05, lower)
        kind = S.lower_triangular if lower else S.upper_triangular
        b = rng.uniform(-1, 1, 100)
        x1 = S.jacobi_sweeps_apply(tp, kind, b, m + 1)
        x2 = S.spmv(S.sait_thr(tp, kind, S.SaitThrParams(0.0, m)), b)
        assert np.linalg.norm(x1 - x2) <= 1e-12 * np.linalg.norm(x2)


def test_3_pattern_theorem(S):
    """sait_pat's captured pattern at step p = structural pattern of
    sum_{i <= p} tT^i (brute-force boolean powers), p = 0..3, 20 matrices."""
    import scipy.sparse as sp

    rng = np.random.default_rng(3)
    for q in range(20):
        lower = q % 2 == 0
        t, tp = _random_triangular(rng, 200, 0.01, lower)
        off = (sp.tril(t, -1) if lower else sp.triu(t, 1)).astype(bool).astype(np.int64)
        acc = sp.identity(200, dtype=np.int64, format="csr")
        power = sp.identity(200, dtype=np.int64, format="csr")
        kind = S.lower_triangular if lower else S.upper_triangular
        for p in range(4):
            if p:
                power = (power @ off).astype(bool).astype(np.int64)
                acc = (acc + power).astype(bool).astype(np.int64)
            pat = S.sait_pat_capture_pattern(tp, kind, p)
            got = sp.csr_matrix((np.ones(len(pat.col_idx)), pat.col_idx, pat.row_ptr), shape=(200, 200))
            assert (got.astype(bool) != acc.astype(bool)).nnz == 0, (q, p)


def test_4_ilu0_exact_on_pattern(S):
    """Device ILU(0) of laplacian_3d(20): LU = A on pattern(A) to 1e-12 ||A||_inf,
    pattern(L) U pattern(U) = pattern(A) U diag."""
    A = S.laplacian_3d(20)
    f = S.ilu0_device(A)
    L, U = _csr_scipy(f.lower.to_host()), _csr_scipy(f.upper.to_host())
    a = _csr_scipy(A)
    lu = (L @ U).tocsr()
    pa = a.astype(bool)
    diff = (lu - a).multiply(pa)
    assert np.abs(diff).max() <= 1e-12 * np.abs(a).sum(axis=1).max()
    import scipy.sparse as sp

    union = (L.astype(bool) + U.astype(bool)).astype(bool)
    want = (pa + sp.identity(a.shape[0], dtype=bool)).astype(bool)
    assert (union != want).nnz == 0


def _pcg_iters(S, A, M, b, tol=1e-10):
    _, st = S.pcg(A, M, b, tol, 5000)
    assert st.converged
    return st.iterations


def _pair(S, f, tau, k):
    return S.SaitPairPreconditioner(S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(tau, k)),
                                    S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(tau, k)))


def test_5_laplacian_ordering(S):
    """laplacian_3d(32), ILU(0), PCG to 1e-10 with b = A 1:
    iter(none) > iter(SAIT 0.05) >= iter(SAIT 0.01) >= iter(exact) > 0."""
    A = S.laplacian_3d(32)
    b = S.make_rhs(A, "ones-solution")
    f = S.ilu0_device(A)
    it_none = _pcg_iters(S, A, None, b)
    it_05 = _pcg_iters(S, A, _pair(S, f, 0.05, 10), b)
    it_01 = _pcg_iters(S, A, _pair(S, f, 0.01, 10), b)
    it_ex = _pcg_iters(S, A, S.ExactIluPreconditioner(f), b)
    assert it_none > it_05 >= it_01 >= it_ex > 0, (it_none, it_05, it_01, it_ex)


def test_6_paper_scale_table(S):
    """laplacian_3d(100), ILU(0), SAIT_Thr(tau, 10): nnz ratio and PCG
    iterations within 15 % of the paper (1.74 / 189, 4.92 / 154), exact ILU
    within 10 % of 145.  RHS ~ U[-1, 1] (seed 1): SURVEY.md §4 measured that
    b = A 1 lands outside the published band (154 vs 189)."""
    A = S.laplacian_3d(100)
    f = S.ilu0_device(A)
    b = S.uniform_pm1(1, A.nrows)
    nnz_lu = f.lower.nnz() + f.upper.nnz()
    for tau, ratio, iters in ((0.05, 1.74, 189), (0.01, 4.92, 154)):
        P = _pair(S, f, tau, 10)
        assert abs(P.nnz() / nnz_lu - ratio) <= 0.15 * ratio, (tau, P.nnz() / nnz_lu)
        it = _pcg_iters(S, A, P, b)
        assert abs(it - iters) <= 0.15 * iters, (tau, it)
    it_ex = _pcg_iters(S, A, S.ExactIluPreconditioner(f), b)
    assert abs(it_ex - 145) <= 0.10 * 145, it_ex


@pytest.mark.skipif(not os.environ.get("SAIT_SUITESPARSE_DIR"), reason="needs SuiteSparse .mtx files")
def test_7_suitesparse_thermomech_tc(S):
    path = os.path.join(os.environ["SAIT_SUITESPARSE_DIR"], "thermomech_TC.mtx")
    A = S.mm_read(path)
    b = S.make_rhs(A, "ones-solution")
    f = S.ilu0_device(A)
    assert abs(_pcg_iters(S, A, None, b, 1e-8) - 89) <= 9
    assert abs(_pcg_iters(S, A, S.ExactIluPreconditioner(f), b, 1e-8) - 10) <= 3
    P = _pair(S, f, 0.06, 10)
    assert abs(_pcg_iters(S, A, P, b, 1e-8) - 11) <= 3
    assert abs(P.nnz() / (f.lower.nnz() + f.upper.nnz()) - 1.01) <= 0.1


def test_8_jacobi_plateau(S):
    """laplacian_3d(32), ILU(0): PCG iterations with k Jacobi sweeps per factor
    are non-increasing in k (+-2) for k = 1..10, and k = 10 is within 2 of the
    exact solves.  k sweeps == sait_thr(T, 0, k - 1) (acceptance #2; one
    sweep is D^-1), so the device PCG runs the sweeps as that SAIT pair."""
    A = S.laplacian_3d(32)
    b = S.make_rhs(A, "ones-solution")
    f = S.ilu0_device(A)

    def sweeps(k):
        if k > 1:
            return _pair(S, f, 0.0, k - 1)
        # one sweep is D^-1: the diagonal pattern (sait_pat with p = 0)
        return S.SaitPairPreconditioner(S.sait_pat(f.lower, S.lower_triangular, S.SaitPatParams(0, 1)),
                                        S.sait_pat(f.upper, S.upper_triangular, S.SaitPatParams(0, 1)))

    its = [_pcg_iters(S, A, sweeps(k), b) for k in range(1, 11)]
    assert all(its[i + 1] <= its[i] + 2 for i in range(9)), its
    it_ex = _pcg_iters(S, A, S.ExactIluPreconditioner(f), b)
    assert abs(its[-1] - it_ex) <= 2, (its, it_ex)


def test_9_lobpcg_analytic_exact_and_sait(S, port):
    """laplacian_3d(20), nev = 4: eigenvalues equal the analytic spectrum to
    1e-8 with ExactIlu and with SAIT_Thr(0.03, 10); SAIT needs at most 3x the
    exact run's iterations; the exact run is bitwise the oracle's."""
    m = 20
    A = S.laplacian_3d(m)
    f = S.ilu0_device(A)
    h = 1.0 / (m + 1)
    sn = np.sin(np.pi * np.arange(1, m + 1) * h / 2) ** 2
    lam = np.sort((4 * (sn[:, None, None] + sn[None, :, None] + sn[None, None, :])).ravel())[:4]
    E = S.ExactIluPreconditioner(f)
    r_ex = S.lobpcg(A, E, 4, 1e-6, 500, 5)
    r_sait = S.lobpcg(A, _pair(S, f, 0.03, 10), 4, 1e-6, 500, 5)
    for r in (r_ex, r_sait):
        assert np.max(np.abs(r.eigenvalues - lam) / lam) <= 1e-8
    assert r_sait.iterations <= 3 * r_ex.iterations
    ev, _, it, hist = __import__("oracle.oracle", fromlist=["lobpcg"]).lobpcg(
        to_oracle(A), to_oracle(f.lower.to_host()), to_oracle(f.upper.to_host()), 4, 1e-6, 500, 5, exact=True)
    assert it == r_ex.iterations and bitwise_equal(ev, r_ex.eigenvalues)
    assert bitwise_equal(np.asarray(hist).ravel(), np.asarray(r_ex.residual_history).ravel())


def test_10_determinism(S):
    """Two executions of runs #5 and #9 give bit-identical results."""
    A = S.laplacian_3d(24)
    f = S.ilu0_device(A)
    b = S.make_rhs(A, "ones-solution")
    P = _pair(S, f, 0.05, 10)
    x1, s1 = S.pcg(A, P, b, 1e-10, 1000)
    x2, s2 = S.pcg(A, P, b, 1e-10, 1000)
    assert bitwise_equal(x1, x2) and bitwise_equal(s1.history, s2.history)
    r1 = S.lobpcg(A, P, 4, 1e-6, 300, 5)
    r2 = S.lobpcg(A, P, 4, 1e-6, 300, 5)
    assert bitwise_equal(r1.eigenvalues, r2.eigenvalues) and bitwise_equal(r1.eigenvectors, r2.eigenvectors)


def test_spd_experiment_from_matrix_market(S, tmp_path):
    """F4 end to end (the paper's SPD experiment): a
    symmetric-stored Matrix Market file (lower triangle, like SuiteSparse's
    SPD matrices) -> mm_read -> device ILU(0) -> SAIT_Thr(0.05, 10) -> PCG.
    The file round-trips to the original matrix, and SAIT needs more
    iterations than the exact solves but fewer than no preconditioner."""
    import sys

    from conftest import ROOT

    A = S.laplacian_3d(20)
    rows = np.repeat(np.arange(A.nrows), np.diff(A.row_ptr))
    low = A.col_idx <= rows
    p = tmp_path / "lap20_sym.mtx"
    with open(p, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real symmetric\n% 3-D Laplacian 20^3, lower triangle\n")
        fh.write(f"{A.nrows} {A.ncols} {int(low.sum())}\n")
        for i, j, v in zip(rows[low], A.col_idx[low], A.values[low]):
            fh.write(f"{i + 1} {j + 1} {float(v)!r}\n")
    B = S.mm_read(p)
    assert np.array_equal(B.row_ptr, A.row_ptr) and np.array_equal(B.col_idx, A.col_idx)
    assert bitwise_equal(B.values, A.values)
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import run_spd_table

    row = run_spd_table.run_one("lap20_sym.mtx", B, 0.05, 0, [2], 1e-8, 5000)
    assert row["exact"] < row["sait"] < row["no_pc"], row
    assert 1.0 < row["ratio"] < 3.0
