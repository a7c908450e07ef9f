"""The oracle (C restatement, oracle/sait_oracle.c) pinned against the
reference: golden fixtures produced by the compiled reference
(tests/golden/make_golden.py) and, where oracle/_ref is built, the reference
library itself.  CPU only."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_csr
from helpers import bitwise_equal, bitwise_equal_csr

THR_CASES = [(0.0, 1), (0.0, 5), (0.01, 3), (0.05, 10), (0.2, 4), (0.0, 250)]
PAT_CASES = [(0, 1), (1, 3), (2, 2), (3, 5)]
CAP_CASES = [(0.01, 3, 3.0), (0.0, 4, 1.5), (0.05, 6, 1.0)]
NAMES = [("syn_lower", True), ("syn_upper", False)]


@pytest.mark.parametrize("name,lower", NAMES)
def test_port_matches_golden_thr_pat_cap(port, golden, name, lower):
    t = golden_csr(golden, f"{name}/T")
    for tau, k in THR_CASES:
        assert bitwise_equal_csr(port.sait_thr(t, lower, tau, k), golden_csr(golden, f"{name}/thr_{tau}_{k}")), (tau, k)
    for p, m in PAT_CASES:
        assert bitwise_equal_csr(port.sait_pat(t, lower, p, m), golden_csr(golden, f"{name}/pat_{p}_{m}"))
        assert bitwise_equal_csr(port.sait_pat_capture_pattern(t, lower, p), golden_csr(golden, f"{name}/patcap_{p}"))
    for tau, k, f in CAP_CASES:
        assert bitwise_equal_csr(port.sait_thr_cap(t, lower, tau, k, f), golden_csr(golden, f"{name}/cap_{tau}_{k}_{f}"))


def test_port_matches_golden_config1(port, golden):
    A = golden_csr(golden, "c1/A")
    from oracle import oracle as O

    assert bitwise_equal_csr(O.laplacian_2d(64), A)
    L, U = port.ilu_k(A, 0)
    assert bitwise_equal_csr(L, golden_csr(golden, "c1/L")) and bitwise_equal_csr(U, golden_csr(golden, "c1/U"))
    ML = port.sait_thr(L, True, 1e-2, 4)
    MU = port.sait_thr(U, False, 1e-2, 4)
    assert bitwise_equal_csr(ML, golden_csr(golden, "c1/ML")) and bitwise_equal_csr(MU, golden_csr(golden, "c1/MU"))
    assert bitwise_equal(port.pair_apply(ML, MU, golden["c1/r"]), golden["c1/z"])
    assert bitwise_equal(port.pair_apply_block(ML, MU, golden["c1/R8"]), golden["c1/Z8"])
    assert bitwise_equal(O.uniform_pm1(1, 4096), golden["c1/r"])


def test_port_ilu1_golden(port, golden):
    from oracle import oracle as O

    L, U = port.ilu_k(O.laplacian_3d(12), 1)
    assert bitwise_equal_csr(L, golden_csr(golden, "lap12/L1")) and bitwise_equal_csr(U, golden_csr(golden, "lap12/U1"))


def test_ratio_table_fixture_matches_paper():
    """3-significant-figure nnz ratios, reproduced by the
    reference (fixture) — the known-answer test of the build path."""
    with open(os.path.join(GOLDEN, "ratio_table_100.json")) as f:
        t = json.load(f)
    paper = {
        "ilu0": {"thr_0.05_10": 1.74, "thr_0.02_10": 2.73, "thr_0.01_10": 4.92, "pat_1_10": 1.00, "pat_2_10": 2.48, "pat_3_10": 4.92},
        "ilu1": {"thr_0.05_10": 1.00, "thr_0.02_10": 3.37, "thr_0.01_10": 5.17, "pat_1_10": 1.00, "pat_2_10": 3.25, "pat_3_10": 7.54},
    }
    for lev, row in paper.items():
        for key, ratio in row.items():
            lo, up = t[lev][key]
            assert round(lo / t[lev]["L"], 2) == ratio, (lev, key)
            assert abs(up / t[lev]["U"] - ratio) < 0.01, (lev, key)


def test_spec_examples_port(port):
    """SPEC.md examples for the kernels (spmv :57-60, add_identity :75-78,
    drop_by_threshold :84-87, jacobi_split :217-220)."""
    from oracle.oracle import csr

    a = csr(2, 2, [0, 1, 3], [0, 0, 1], [2.0, 1.0, 3.0])
    assert list(port.spmv(a, np.ones(2))) == [2.0, 4.0]
    m = csr(2, 2, [0, 1, 1], [0], [-1.0])
    r = port.add_identity(m)
    assert list(r.col_idx) == [0, 1] and list(r.values) == [0.0, 1.0]
    m = csr(2, 2, [0, 2, 3], [0, 1, 1], [1.0, 0.005, 1.0])
    r = port.drop_by_threshold(m, 0.01)
    assert list(r.col_idx) == [0, 1] and list(r.row_ptr) == [0, 1, 2]
    t = csr(2, 2, [0, 1, 3], [0, 0, 1], [2.0, 4.0, 2.0])
    inv, tt = port.jacobi_split(t, True)
    assert list(inv) == [0.5, 0.5] and list(tt.values) == [-2.0] and list(tt.row_ptr) == [0, 0, 1]
    s = csr(4, 4, [0, 0, 1, 2, 3], [0, 1, 2], [1.0, 1.0, 1.0])  # strictly lower bidiagonal
    s2 = port.spgemm(s, s)
    assert list(s2.row_ptr) == [0, 0, 0, 1, 2] and list(s2.col_idx) == [0, 1]
    s4 = port.spgemm(s2, s2)
    assert s4.nnz == 0


def test_port_errors(port):
    from oracle.oracle import InvalidArgument, RuntimeErr, csr

    t = csr(3, 3, [0, 1, 2, 4], [0, 1, 1, 2], [2.0, 0.0, 1.0, 3.0])
    with pytest.raises(RuntimeErr, match="jacobi_split: singular matrix, zero diagonal at row 1"):
        port.sait_thr(t, True, 0.1, 2)
    with pytest.raises(InvalidArgument, match=r"sait_thr: threshold must be in \[0, 1\), got 1.500000"):
        port.sait_thr(t, True, 1.5, 2)
    with pytest.raises(InvalidArgument, match=r"check_triangular: entry \(2, 1\) outside stated triangle"):
        port.sait_thr(t, False, 0.1, 2)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_port_vs_reference_random(port, ref, seed):
    from oracle import oracle as O

    t = O.synthetic_lower(400, 7, 0.05, seed=seed)
    u = port.transpose(O.synthetic_lower(400, 7, 0.05, seed=seed + 10))
    for tau, k in [(0.0, 4), (0.02, 5), (0.1, 8)]:
        assert bitwise_equal_csr(port.sait_thr(t, True, tau, k), ref.sait_thr(t, True, tau, k))
        assert bitwise_equal_csr(port.sait_thr(u, False, tau, k), ref.sait_thr(u, False, tau, k))
    assert bitwise_equal_csr(port.sait_pat(t, True, 2, 4), ref.sait_pat(t, True, 2, 4))
    assert bitwise_equal_csr(port.sait_thr_cap(u, False, 0.01, 4, 2.0), ref.sait_thr_cap(u, False, 0.01, 4, 2.0))
    b = O.uniform_pm1(seed, 400)
    assert bitwise_equal(port.jacobi_sweeps_apply(t, True, b, 4), ref.jacobi_sweeps_apply(t, True, b, 4))
    A = O.convdiff_2d(20)
    L, U = port.ilu_k(A, 1)
    L2, U2 = ref.ilu_k(A, 1)
    assert bitwise_equal_csr(L, L2) and bitwise_equal_csr(U, U2)


def test_ref_kernels_match_port(port, ref):
    """The restated kernels (kernels.cpp) against the reference's own."""
    import scipy.sparse as sp

    from oracle.oracle import from_scipy

    a = from_scipy(sp.random(80, 60, density=0.1, random_state=1, format="csr"))
    b = from_scipy(sp.random(60, 70, density=0.1, random_state=2, format="csr"))
    assert bitwise_equal_csr(port.spgemm(a, b), ref.spgemm(a, b))
    assert bitwise_equal_csr(port.transpose(a), ref.transpose(a))
    sq = from_scipy(sp.random(50, 50, density=0.2, random_state=3, format="csr"))
    assert bitwise_equal_csr(port.add_identity(sq), ref.add_identity(sq))
    assert bitwise_equal_csr(port.drop_by_threshold(sq, 0.5), ref.drop_by_threshold(sq, 0.5))
    pat = from_scipy(sp.random(50, 50, density=0.2, random_state=4, format="csr")).pattern()
    assert bitwise_equal_csr(port.drop_by_pattern(sq, pat), ref.drop_by_pattern(sq, pat))
    d = np.linspace(-2, 3, 50)
    assert bitwise_equal_csr(port.scale_columns(sq, d), ref.scale_columns(sq, d))
    x = np.linspace(-1, 1, 60)
    assert bitwise_equal(port.spmv(a, x), ref.spmv(a, x))


@pytest.mark.parametrize("name,lower", NAMES)
def test_port_trisolve_golden(port, golden, name, lower):
    """trisolve (kernels.cpp:196-234) pinned on the reference's own output."""
    t = golden_csr(golden, f"{name}/T")
    assert bitwise_equal(port.trisolve(t, lower, golden[f"{name}/b"]), golden[f"{name}/x_tri"])


def test_port_exact_and_jacobi_golden(port, golden):
    """ExactIluPreconditioner / JacobiSweepsPreconditioner(3) on config 1."""
    L, U, r = golden_csr(golden, "c1/L"), golden_csr(golden, "c1/U"), golden["c1/r"]
    assert bitwise_equal(port.trisolve(U, False, port.trisolve(L, True, r)), golden["c1/z_exact"])
    z = port.jacobi_sweeps_apply(U, False, port.jacobi_sweeps_apply(L, True, r, 3), 3)
    assert bitwise_equal(z, golden["c1/z_jacobi3"])


def test_port_trisolve_nontriangular_and_errors(port, ref):
    """Entries on the wrong side of the diagonal read x as zero; the first
    zero/missing diagonal in solve order raises (reference wording)."""
    from oracle import oracle as O

    rng = np.random.default_rng(5)
    n = 60
    dense = rng.uniform(-1, 1, (n, n)) * (rng.random((n, n)) < 0.15)
    np.fill_diagonal(dense, rng.uniform(1, 2, n))
    import scipy.sparse as sp

    m = O.from_scipy(sp.csr_matrix(dense))
    b = rng.uniform(-1, 1, n)
    for lower in (True, False):
        assert bitwise_equal(port.trisolve(m, lower, b), ref.trisolve(m, lower, b))
    dense[7, 7] = 0.0
    dense[40, 40] = 0.0
    m = O.from_scipy(sp.csr_matrix(dense))
    for lower, row in ((True, 7), (False, 40)):
        with pytest.raises(Exception, match=f"zero diagonal at row {row}"):
            port.trisolve(m, lower, b)
        with pytest.raises(Exception, match=f"zero diagonal at row {row}"):
            ref.trisolve(m, lower, b)
