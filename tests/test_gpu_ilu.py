"""GPU parity of the device ILU(0) (F1; ilu.hpp:27, ilu.cpp:98-173 at level 0)
against the reference's own factors (golden) and the oracle port: bitwise,
since every row performs the reference's IKJ operation sequence."""
import numpy as np
import pytest

from conftest import golden_csr
from helpers import bitwise_equal_csr, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def test_ilu0_golden_config1(S, golden):
    A = to_product(golden_csr(golden, "c1/A"))
    f = S.ilu0_device(A)
    assert bitwise_equal_csr(f.lower.to_host(), golden_csr(golden, "c1/L"))
    assert bitwise_equal_csr(f.upper.to_host(), golden_csr(golden, "c1/U"))


def _random_matrix(n, density, seed, dominant=True):
    import scipy.sparse as sp
    from oracle import oracle as O

    rng = np.random.default_rng(seed)
    m = sp.random(n, n, density=density, random_state=seed, format="csr", data_rvs=lambda k: rng.uniform(-1, 1, k))
    d = rng.uniform(0.5, 1.5, n) * (np.abs(m).sum(axis=1).A1 + 1.0 if dominant else 1.0)
    m = (m + sp.diags(d)).tocsr()
    m.sort_indices()
    return O.from_scipy(m)


@pytest.mark.parametrize("case", ["lap3d_40", "convdiff_200", "random_5k", "random_weak_3k", "lap2d_1"])
def test_ilu0_vs_port(S, port, case):
    from oracle import oracle as O

    A = {
        "lap3d_40": lambda: O.laplacian_3d(40),
        "convdiff_200": lambda: O.convdiff_2d(200),
        "random_5k": lambda: _random_matrix(5000, 0.002, 3),
        "random_weak_3k": lambda: _random_matrix(3000, 0.003, 4, dominant=False),
        "lap2d_1": lambda: O.laplacian_2d(1),
    }[case]()
    L, U = port.ilu_k(A, 0)
    f = S.ilu0_device(to_product(A))
    assert bitwise_equal_csr(f.lower.to_host(), L)
    assert bitwise_equal_csr(f.upper.to_host(), U)


def test_ilu0_full_size_c2(S, port):
    """BASELINE config 2's factorization (128^3 Laplacian), bitwise."""
    from oracle import oracle as O

    A = O.laplacian_3d(128)
    L, U = port.ilu_k(A, 0)
    f = S.ilu0_device(to_product(A))
    assert bitwise_equal_csr(f.lower.to_host(), L)
    assert bitwise_equal_csr(f.upper.to_host(), U)


def test_ilu0_errors(S):
    from paper_2106_12836_b200 import CsrMatrix

    # structurally zero diagonal: row 1 has no (1, 1) entry
    a = CsrMatrix(3, 3, np.array([0, 1, 2, 4]), np.array([0, 0, 1, 2]), np.array([1.0, 1.0, 1.0, 1.0]))
    with pytest.raises(S.SaitInvalidArgument, match=r"^ilu_k: structurally zero diagonal at row 1$"):
        S.ilu0_device(a)
    # pivot breakdown: [[1, 1], [1, 1]] -> u_11 = 1 - 1 * 1 = 0
    b = CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([1.0, 1.0, 1.0, 1.0]))
    with pytest.raises(S.SaitRuntimeError, match=r"^ilu_k: pivot breakdown at row 1 \(\|pivot\| = 0\.000000\)$"):
        S.ilu0_device(b)
    # tiny pivot relative to max |a| (1e-14 * max): breakdown at row 2, |pivot| printed with %f
    c = CsrMatrix(3, 3, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.array([1e6, 2.0, 1e-9]))
    with pytest.raises(S.SaitRuntimeError, match=r"^ilu_k: pivot breakdown at row 2 \(\|pivot\| = 0\.000000\)$"):
        S.ilu0_device(c)
    rect = CsrMatrix(2, 3, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(S.SaitInvalidArgument, match="not square"):
        S.ilu0_device(rect)


def test_ilu0_error_messages_match_port(S, port):
    """Two breakdowns (rows 30 and 41): the first in row order is reported,
    with the port's exact message."""
    import scipy.sparse as sp
    from oracle import oracle as O

    d = np.diag(np.full(50, 2.0)) + np.diag(np.full(49, -1.0), 1) + np.diag(np.full(49, -1.0), -1)
    for r in (29, 40):  # decoupled [[1, 1], [1, 1]] blocks on rows r, r + 1
        d[r - 1 : r + 3, r - 1 : r + 3] = 0.0
        d[r - 1, r - 1] = d[r + 2, r + 2] = 2.0
        d[r : r + 2, r : r + 2] = 1.0
    A = O.from_scipy(sp.csr_matrix(d))
    with pytest.raises(Exception) as want:
        port.ilu_k(A, 0)
    with pytest.raises(S.SaitRuntimeError) as got:
        S.ilu0_device(to_product(A))
    assert str(got.value) == str(want.value)
    assert "row 30" in str(got.value)


def test_ilu0_empty(S):
    from paper_2106_12836_b200 import CsrMatrix

    f = S.ilu0_device(CsrMatrix(0, 0, np.array([0]), np.array([], dtype=np.int64), np.array([])))
    assert f.lower.to_host().nrows == 0 and f.upper.to_host().nnz() == 0


def test_ilu0_feeds_sait(S, port):
    """Device ILU(0) -> device SAIT build -> pair: bitwise the host chain."""
    from oracle import oracle as O

    A = O.laplacian_3d(24)
    L, U = port.ilu_k(A, 0)
    want_l = port.sait_thr(L, True, 5e-2, 3)
    f = S.ilu0_device(to_product(A))
    ml = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    assert bitwise_equal_csr(ml.to_host() if hasattr(ml, "to_host") else ml, want_l)


@pytest.mark.parametrize("case", ["golden_lap12", "lap3d_40", "convdiff_150", "random_4k", "lap2d_2"])
def test_ilu1_device_vs_port(S, port, golden, case):
    """Device ILU(1): the level-1 pattern from the structural product
    (tril(A,-1) + I)(triu(A,1) + I), the reference's IKJ numeric on it —
    bitwise the reference's ilu_k(a, 1) (golden) and the port."""
    from conftest import golden_csr
    from oracle import oracle as O

    A = {
        "golden_lap12": lambda: O.laplacian_3d(12),
        "lap3d_40": lambda: O.laplacian_3d(40),
        "convdiff_150": lambda: O.convdiff_2d(150),
        "random_4k": lambda: _random_matrix(4000, 0.002, 7),
        "lap2d_2": lambda: O.laplacian_2d(2),
    }[case]()
    L, U = port.ilu_k(A, 1)
    if case == "golden_lap12":
        assert bitwise_equal_csr(L, golden_csr(golden, "lap12/L1"))
        assert bitwise_equal_csr(U, golden_csr(golden, "lap12/U1"))
    f = S.ilu_device(to_product(A), 1)
    assert bitwise_equal_csr(f.lower.to_host(), L)
    assert bitwise_equal_csr(f.upper.to_host(), U)


def test_ilu_device_levels_beyond_one_are_refused(S):
    with pytest.raises(S.SaitInvalidArgument, match="fill levels 0 and 1"):
        S.ilu_device(S.laplacian_2d(8), 2)
    with pytest.raises(S.SaitInvalidArgument, match="negative fill level"):
        S.ilu_device(S.laplacian_2d(8), -1)
