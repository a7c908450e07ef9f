"""GPU parity of the exact triangular solve (kernels.cpp:196-234) and of the
two comparator preconditioners built on the reference's factors:
ExactIluPreconditioner (preconditioner.cpp:25-32) and
JacobiSweepsPreconditioner (preconditioner.cpp:51-63).  Bitwise against the
reference's own outputs (golden) and the oracle port: each row is summed
sequentially in stored order, products rounded before the subtraction."""
import numpy as np
import pytest

from conftest import golden_csr
from helpers import bitwise_equal, to_product

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


@pytest.mark.parametrize("name,lower", [("syn_lower", True), ("syn_upper", False)])
def test_trisolve_golden(S, golden, name, lower):
    t = to_product(golden_csr(golden, f"{name}/T"))
    kind = S.lower_triangular if lower else S.upper_triangular
    x = S.trisolve(t, kind, golden[f"{name}/b"])
    assert bitwise_equal(x, golden[f"{name}/x_tri"])


def test_exact_ilu_golden(S, golden):
    f = S.IluFactors(to_product(golden_csr(golden, "c1/L")), to_product(golden_csr(golden, "c1/U")))
    p = S.ExactIluPreconditioner(f)
    assert p.name() == "exact" and p.nnz() == f.lower.nnz() + f.upper.nnz()
    z = np.empty(4096)
    p.apply(golden["c1/r"], z)
    assert bitwise_equal(z, golden["c1/z_exact"])
    # device vectors, repeated applies (epoch-tagged flags are reused)
    import torch

    r = torch.from_numpy(golden["c1/r"]).cuda()
    zd = torch.empty_like(r)
    for _ in range(3):
        zd.zero_()
        p.apply(r, zd)
        torch.cuda.synchronize()
        assert bitwise_equal(zd.cpu().numpy(), golden["c1/z_exact"])


def test_jacobi_sweeps_golden(S, golden):
    f = S.IluFactors(to_product(golden_csr(golden, "c1/L")), to_product(golden_csr(golden, "c1/U")))
    p = S.JacobiSweepsPreconditioner(f, 3)
    assert p.name() == "jacobi" and p.sweeps() == 3
    z = np.empty(4096)
    p.apply(golden["c1/r"], z)
    assert bitwise_equal(z, golden["c1/z_jacobi3"])
    with pytest.raises(S.SaitInvalidArgument, match="sweeps must be >= 1"):
        S.JacobiSweepsPreconditioner(f, 0)


@pytest.mark.parametrize("case", ["lap3d_40", "convdiff_300", "syn_lower_50k", "ilu1_lap3d_24"])
def test_exact_ilu_vs_port(S, port, case):
    """Long dependency chains (2D/3D stencils), irregular rows (synthetic),
    ILU(1) fill: both solves bitwise equal to the port."""
    from oracle import oracle as O

    if case == "lap3d_40":
        A = O.laplacian_3d(40)
        L, U = port.ilu_k(A, 0)
    elif case == "convdiff_300":
        A = O.convdiff_2d(300)
        L, U = port.ilu_k(A, 0)
    elif case == "ilu1_lap3d_24":
        A = O.laplacian_3d(24)
        L, U = port.ilu_k(A, 1)
    else:
        L = O.synthetic_lower(50000, 15, 0.01, seed=4)
        U = port.transpose(O.synthetic_lower(50000, 15, 0.01, seed=5))
    n = L.nrows
    r = O.uniform_pm1(21, n)
    want_y = port.trisolve(L, True, r)
    want_z = port.trisolve(U, False, want_y)
    y = S.trisolve(to_product(L), S.unit_lower_triangular, r)
    assert bitwise_equal(y, want_y)
    p = S.ExactIluPreconditioner(S.IluFactors(to_product(L), to_product(U)))
    z = np.empty(n)
    p.apply(r, z)
    assert bitwise_equal(z, want_z)


def test_trisolve_nontriangular_reads_zero(S, port):
    """Entries on the wrong side of the diagonal see x = 0 (the reference's
    zero-initialised vector), including the -0.0 / NaN products that implies."""
    import scipy.sparse as sp
    from oracle import oracle as O

    rng = np.random.default_rng(9)
    n = 3000
    m = sp.random(n, n, density=0.002, random_state=3, format="csr")
    m = (m + sp.diags(rng.uniform(1, 2, n))).tocsr()
    m.sort_indices()
    m.data[5] = -m.data[5]
    t = O.from_scipy(m)
    b = rng.uniform(-1, 1, n)
    b[::7] = -0.0
    for lower, kind in ((True, S.lower_triangular), (False, S.upper_triangular)):
        assert bitwise_equal(S.trisolve(to_product(t), kind, b), port.trisolve(t, lower, b))


def test_trisolve_errors(S):
    import scipy.sparse as sp

    from paper_2106_12836_b200 import CsrMatrix

    d = np.array([[2.0, 0, 0], [1, 0, 0], [1, 1, 3]])
    m = sp.csr_matrix(d)
    t = CsrMatrix(3, 3, m.indptr, m.indices, m.data)
    with pytest.raises(S.SaitError, match="zero diagonal at row 1"):
        S.trisolve(t, S.lower_triangular, np.ones(3))
    # explicit stored zero on the diagonal, upper solve order (row 2 first)
    t2 = CsrMatrix(3, 3, np.array([0, 1, 2, 3]), np.array([0, 1, 2]), np.array([1.0, 0.0, 0.0]))
    with pytest.raises(S.SaitError, match="zero diagonal at row 2"):
        S.trisolve(t2, S.upper_triangular, np.ones(3))
    with pytest.raises(S.SaitInvalidArgument, match="right-hand side length mismatch"):
        S.trisolve(t, S.lower_triangular, np.ones(4))
    rect = CsrMatrix(2, 3, np.array([0, 1, 2]), np.array([0, 1]), np.array([1.0, 1.0]))
    with pytest.raises(S.SaitInvalidArgument, match="not square"):
        S.trisolve(rect, S.lower_triangular, np.ones(2))


def test_exact_ilu_concurrent_streams(S, port):
    """Two streams applying the same preconditioner at once (per-stream flags)."""
    import torch
    from oracle import oracle as O

    A = O.laplacian_3d(32)
    L, U = port.ilu_k(A, 0)
    p = S.ExactIluPreconditioner(S.IluFactors(to_product(L), to_product(U)))
    n = A.nrows
    rs = [O.uniform_pm1(40 + i, n) for i in range(2)]
    want = [port.trisolve(U, False, port.trisolve(L, True, r)) for r in rs]
    streams = [torch.cuda.Stream() for _ in range(2)]
    rd = [torch.from_numpy(r).cuda() for r in rs]
    zd = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    torch.cuda.synchronize()
    import threading

    def run(i):
        with torch.cuda.stream(streams[i]):
            for _ in range(3):
                p.apply(rd[i], zd[i])

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    for i in range(2):
        assert bitwise_equal(zd[i].cpu().numpy(), want[i])
