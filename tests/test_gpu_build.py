"""GPU parity of the SAIT builder against the reference (golden fixtures made
by the compiled reference) and the C restatement (oracle port).  Bitwise:
the device recursion performs the reference's exact operation sequence."""
import numpy as np
import pytest

from conftest import golden_csr
from helpers import bitwise_equal, bitwise_equal_csr, to_product

pytestmark = pytest.mark.gpu

THR_CASES = [(0.0, 1), (0.0, 5), (0.01, 3), (0.05, 10), (0.2, 4), (0.0, 250)]
PAT_CASES = [(0, 1), (1, 3), (2, 2), (3, 5)]
CAP_CASES = [(0.01, 3, 3.0), (0.0, 4, 1.5), (0.05, 6, 1.0)]
NAMES = [("syn_lower", True), ("syn_upper", False)]


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def kind(S, lower):
    return S.lower_triangular if lower else S.upper_triangular


@pytest.mark.parametrize("name,lower", NAMES)
@pytest.mark.parametrize("tau,steps", THR_CASES)
def test_sait_thr_golden(S, golden, name, lower, tau, steps):
    t = to_product(golden_csr(golden, f"{name}/T"))
    m = S.sait_thr(t, kind(S, lower), S.SaitThrParams(tau, steps))
    assert bitwise_equal_csr(m, golden_csr(golden, f"{name}/thr_{tau}_{steps}"))


@pytest.mark.parametrize("name,lower", NAMES)
@pytest.mark.parametrize("p,m", PAT_CASES)
def test_sait_pat_golden(S, golden, name, lower, p, m):
    t = to_product(golden_csr(golden, f"{name}/T"))
    out = S.sait_pat(t, kind(S, lower), S.SaitPatParams(p, m))
    assert bitwise_equal_csr(out, golden_csr(golden, f"{name}/pat_{p}_{m}"))
    pat = S.sait_pat_capture_pattern(t, kind(S, lower), p)
    assert bitwise_equal_csr(pat, golden_csr(golden, f"{name}/patcap_{p}"))


@pytest.mark.parametrize("name,lower", NAMES)
@pytest.mark.parametrize("tau,steps,f", CAP_CASES)
def test_sait_cap_golden(S, golden, name, lower, tau, steps, f):
    t = to_product(golden_csr(golden, f"{name}/T"))
    m = S.sait_thr_cap(t, kind(S, lower), S.SaitThrParams(tau, steps), f)
    assert bitwise_equal_csr(m, golden_csr(golden, f"{name}/cap_{tau}_{steps}_{f}"))


def test_config1_factors(S, golden):
    """BASELINE config 1: 64x64 Poisson, ILU(0), tau=1e-2, k=4 (51,215 nnz per factor)."""
    L = to_product(golden_csr(golden, "c1/L"))
    U = to_product(golden_csr(golden, "c1/U"))
    st = []
    ML = S.sait_thr(L, S.lower_triangular, S.SaitThrParams(1e-2, 4), stats_out=st)
    MU = S.sait_thr(U, S.upper_triangular, S.SaitThrParams(1e-2, 4), stats_out=st)
    assert bitwise_equal_csr(ML, golden_csr(golden, "c1/ML"))
    assert bitwise_equal_csr(MU, golden_csr(golden, "c1/MU"))
    assert ML.nnz() == 51215 and MU.nnz() == 51215
    assert st[0].nnz_out == 51215 and st[0].steps_run == 4


@pytest.mark.parametrize("seed,n,lower", [(21, 300, True), (22, 300, False), (23, 1, True), (24, 2, False)])
@pytest.mark.parametrize("tau,steps", [(0.0, 3), (0.03, 6)])
def test_random_vs_oracle(S, port, seed, n, lower, tau, steps):
    from oracle import oracle as O

    t = O.synthetic_lower(n, 9, 0.02, seed=seed)
    if not lower:
        t = port.transpose(t)
    expect = port.sait_thr(t, lower, tau, steps)
    got = S.sait_thr(to_product(t), kind(S, lower), S.SaitThrParams(tau, steps))
    assert bitwise_equal_csr(got, expect)


def test_long_rows_use_global_tables(S, port):
    """tau = 0 on a dense-ish lower T: rows of M^T exceed the shared-memory
    tables (>2048 distinct columns) and take the global-memory path."""
    from oracle import oracle as O

    t = O.synthetic_lower(3000, 12, 0.3, seed=5)
    expect = port.sait_thr(t, True, 0.0, 40)
    got = S.sait_thr(to_product(t), S.lower_triangular, S.SaitThrParams(0.0, 40))
    assert bitwise_equal_csr(got, expect)


def test_exact_series_property(S, port):
    """SPEC acceptance #1: sait_thr(T, 0, n-1) is T^-1 (||T M - I||_inf small)."""
    from oracle import oracle as O

    for n in (5, 20, 64):
        t = O.synthetic_lower(n, 3, 0.3, seed=100 + n)
        m = S.sait_thr(to_product(t), S.lower_triangular, S.SaitThrParams(0.0, n - 1))
        tm = (t.to_scipy() @ m.to_scipy()).toarray() - np.eye(n)
        assert np.abs(tm).sum(axis=1).max() <= 1e-10


def test_errors_match_reference(S, golden):
    """Exception kinds and messages (sait.cpp:60,77,92; csr.cpp:132)."""
    t = to_product(golden_csr(golden, "syn_lower/T"))
    with pytest.raises(S.SaitInvalidArgument, match=r"sait_thr: threshold must be in \[0, 1\), got 1.500000"):
        S.sait_thr(t, S.lower_triangular, S.SaitThrParams(1.5, 3))
    with pytest.raises(S.SaitInvalidArgument, match="sait_polynomial: steps must be >= 1"):
        S.sait_thr(t, S.lower_triangular, S.SaitThrParams(0.1, 0))
    with pytest.raises(S.SaitInvalidArgument, match=r"check_triangular: entry \(1, 0\) outside stated triangle"):
        S.sait_thr(t, S.upper_triangular, S.SaitThrParams(0.1, 2))
    with pytest.raises(S.SaitInvalidArgument, match="sait_pat: refine_steps must be >= 1"):
        S.sait_pat(t, S.lower_triangular, S.SaitPatParams(1, 0))
    with pytest.raises(S.SaitInvalidArgument, match="sait_pat: pattern_steps must be >= 0"):
        S.sait_pat(t, S.lower_triangular, S.SaitPatParams(-1, 1))
    z = S.CsrMatrix(3, 3, [0, 1, 2, 4], [0, 1, 1, 2], [2.0, 0.0, 1.0, 3.0])
    with pytest.raises(S.SaitRuntimeError, match="jacobi_split: singular matrix, zero diagonal at row 1"):
        S.sait_thr(z, S.lower_triangular, S.SaitThrParams(0.1, 2))
    nd = S.CsrMatrix(3, 3, [0, 1, 1, 3], [0, 0, 2], [2.0, 1.0, 3.0])
    with pytest.raises(S.SaitRuntimeError, match="zero diagonal at row 1"):
        S.sait_thr(nd, S.lower_triangular, S.SaitThrParams(0.1, 2))
    rect = S.CsrMatrix(2, 3, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(S.SaitInvalidArgument, match="jacobi_split: matrix is not square"):
        S.sait_thr(rect, S.lower_triangular, S.SaitThrParams(0.1, 2))


@pytest.mark.parametrize("lower", [True, False])
@pytest.mark.parametrize("draws", [3, 30])
def test_jacobi_split_row_lengths(S, port, lower, draws):
    """The split's thread-per-row (short rows) and 8-lanes-per-row (>= 12
    entries per row on average) variants, both triangles: bitwise the oracle."""
    from oracle import oracle as O

    t = O.synthetic_lower(700, draws, 0.05, seed=31 + draws)
    if not lower:
        t = port.transpose(t)
    inv, tt = port.jacobi_split(t, lower)
    sp = S.jacobi_split(to_product(t), kind(S, lower))
    assert bitwise_equal(np.asarray(sp.inv_diag), inv)
    assert bitwise_equal_csr(sp.iteration_matrix, tt)


def test_spec_examples(S):
    """SPEC.md:217-238 examples for jacobi_split / sait_core / sait_thr."""
    t = S.CsrMatrix(2, 2, [0, 1, 3], [0, 0, 1], [2.0, 4.0, 2.0])
    sp = S.jacobi_split(t, S.lower_triangular)
    assert list(sp.inv_diag) == [0.5, 0.5]
    assert list(sp.iteration_matrix.row_ptr) == [0, 0, 1] and list(sp.iteration_matrix.values) == [-2.0]
    eye = S.CsrMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])
    m = S.sait_thr(eye, S.lower_triangular, S.SaitThrParams(0.3, 4))
    assert m == eye
    d = S.CsrMatrix(3, 3, [0, 1, 2, 3], [0, 1, 2], [2.0, 4.0, 8.0])
    m = S.sait_pat(d, S.upper_triangular, S.SaitPatParams(2, 3))
    assert list(m.values) == [0.5, 0.25, 0.125]


_STAGE_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2106_12836_b200 as S
from oracle import oracle as O
P = O.get("port")
T = O.synthetic_lower(20000, 15, 0.01, seed=4)
Tp = S.CsrMatrix(T.nrows, T.ncols, T.row_ptr, T.col_idx, T.values)
Tu = P.transpose(T)
Tup = S.CsrMatrix(Tu.nrows, Tu.ncols, Tu.row_ptr, Tu.col_idx, Tu.values)
cases = [(lambda: P.sait_thr(T, True, 1e-2, 3), lambda: S.sait_thr(Tp, S.lower_triangular, S.SaitThrParams(1e-2, 3))),
         (lambda: P.sait_thr(T, True, 0.0, 3), lambda: S.sait_thr(Tp, S.lower_triangular, S.SaitThrParams(0.0, 3))),
         (lambda: P.sait_thr_cap(T, True, 1e-2, 3, 1.0),
          lambda: S.sait_thr_cap(Tp, S.lower_triangular, S.SaitThrParams(1e-2, 3), 1.0)),
         (lambda: P.sait_thr(Tu, False, 1e-2, 3), lambda: S.sait_thr(Tup, S.upper_triangular, S.SaitThrParams(1e-2, 3))),
         (lambda: P.sait_pat(T, True, 2, 3), lambda: S.sait_pat(Tp, S.lower_triangular, S.SaitPatParams(2, 3))),
         (lambda: P.sait_thr_cap(Tu, False, 1e-2, 3, 1.0),
          lambda: S.sait_thr_cap(Tup, S.upper_triangular, S.SaitThrParams(1e-2, 3), 1.0))]
for ref, dev in cases:
    want, got = ref(), dev()
    ok = (np.array_equal(got.row_ptr, want.row_ptr) and np.array_equal(got.col_idx, want.col_idx)
          and np.array_equal(got.values.view(np.uint64), want.values.view(np.uint64)))
    print(int(ok))
"""


@pytest.mark.parametrize("steps", [1, 2, 5])
@pytest.mark.parametrize("case", ["diag_only", "golden_T", "zero_diag"])
def test_sait_polynomial_stored_diagonal(S, ref, golden, case, steps):
    """The generic sait_polynomial (sait.cpp:75-88) accepts any square
    iteration matrix: add_identity (kernels.cpp:104-134) adds 1.0 to a stored
    diagonal.  The device must not take the first-step filter pass (which
    assumes jacobi_split's diagonal-free tT) there; bitwise vs the reference,
    same step count."""
    from oracle.oracle import Csr

    if case == "diag_only":
        n = 64
        tt = Csr(n, n, np.arange(n + 1), np.arange(n), np.linspace(-0.5, 0.7, n))
    else:
        tt = golden_csr(golden, "syn_lower/T")
        if case == "zero_diag":
            vals = tt.values.copy() * 0.1
            for i in range(tt.nrows):
                for q in range(tt.row_ptr[i], tt.row_ptr[i + 1]):
                    if tt.col_idx[q] == i:
                        vals[q] = 0.0
            tt = Csr(tt.nrows, tt.ncols, tt.row_ptr, tt.col_idx, vals)
        else:
            tt = Csr(tt.nrows, tt.ncols, tt.row_ptr, tt.col_idx, tt.values * 0.1)
    want = ref.sait_polynomial_tt(tt, steps)
    st = []
    got = S.sait_polynomial(to_product(tt), steps, stats_out=st)
    assert bitwise_equal_csr(got, want)


@pytest.mark.parametrize("window", ["0", "1", "bitmap"])
@pytest.mark.parametrize("column_form", ["0", "1"])
@pytest.mark.parametrize("cap", ["none", "0", "1000", "200000"])
def test_hash_rows_staging_and_overflow(cap, column_form, window):
    """Hash-table and window rows (hundreds of products) stage their sorted
    survivors in the count pass; rows past the staging capacity are
    recomputed in the numeric pass.  Every split (all staged, none, a few,
    most) gives the oracle's bits, with the direct-addressed window rows on
    (default: the -0.0 window for tau > 0 threshold builds, the bitmap
    window for tau = 0 and pattern builds), the bitmap window for every
    epilogue (SAIT_WIN_ZERO=0), or off (SAIT_SPGEMM_WINDOW=0: hash tables
    only)."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, SAIT_BUILD_COLUMN_FORM=column_form, SAIT_SPGEMM_WINDOW="0" if window == "0" else "1")
    if window == "bitmap":
        env["SAIT_WIN_ZERO"] = "0"
    if cap == "none":
        env["SAIT_SPGEMM_NOSTAGE"] = "1"
    else:
        env["SAIT_SPGEMM_STAGE_CAP"] = cap
    out = subprocess.run([sys.executable, "-c", _STAGE_CHILD.format(root=ROOT)], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split() == ["1"] * 6


@pytest.mark.parametrize("column_form", ["0", "1"])
@pytest.mark.parametrize("slack", ["101", "400"])
def test_hash_table_load_factors(slack, column_form):
    """Hash tables sized at the minimum (slots just above the possible distinct
    columns: long linear probes, nearly full tables) and at 4x give the same
    bits as the oracle (SAIT_HASH_SLACK, percent; the default is 140), in
    both the row-form and the column-form recursion."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    env = dict(os.environ, SAIT_HASH_SLACK=slack, SAIT_BUILD_COLUMN_FORM=column_form)
    out = subprocess.run([sys.executable, "-c", _STAGE_CHILD.format(root=ROOT)], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split() == ["1"] * 6


def test_build_pair_concurrent_equals_separate(S, port):
    """sait_build_pair (both factors at once, M_U on a second stream/thread)
    is bitwise the two separate builds; errors of either factor surface."""
    from helpers import bitwise_equal_csr, to_oracle

    A = S.laplacian_3d(32)
    f = S.ilu_k(A, 0)
    st = []
    ML, MU = S.sait_thr_pair(f.lower, f.upper, S.SaitThrParams(5e-2, 3), stats_out=st)
    assert bitwise_equal_csr(ML, port.sait_thr(to_oracle(f.lower), True, 5e-2, 3))
    assert bitwise_equal_csr(MU, port.sait_thr(to_oracle(f.upper), False, 5e-2, 3))
    assert [x.steps_run for x in st] == [3, 3]
    bad = S.CsrMatrix(f.upper.nrows, f.upper.ncols, f.upper.row_ptr, f.upper.col_idx, f.upper.values.copy())
    bad.values[bad.row_ptr[5]] = 0.0  # U's diagonal of row 5
    with pytest.raises(S.SaitRuntimeError, match="zero diagonal at row 5"):
        S.sait_thr_pair(f.lower, bad, S.SaitThrParams(5e-2, 3))
