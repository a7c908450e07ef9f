"""Row-sharded PCG / GMRES (dist_solvers.py) against the single-GPU device
solvers: with 2048-aligned shards the gathered canonical dot partials fold to
the single-GPU values, so iteration counts, residual histories and solutions
are bitwise equal.  Several ranks run inside one process on one GPU (every
stage issued for all ranks before the next: no cross-rank waiting)."""
import numpy as np
import pytest

from helpers import bitwise_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2106_12836_b200 as S

    return S


def _pair(S, A, tau, k):
    f = S.ilu_k(A, 0)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(tau, k))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(tau, k))
    return ML, MU


def _shards(b, ctxs):
    import torch

    bd = torch.from_numpy(b).cuda()
    return [bd[c.own[0] : c.own[1]].clone() for c in ctxs]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("precond", [True, False])
def test_dist_pcg_bitwise(S, world, precond):
    import torch

    from paper_2106_12836_b200 import dist_solvers as DS

    A = S.laplacian_3d(24)
    ML, MU = _pair(S, A, 5e-2, 10) if precond else (None, None)
    b = S.make_rhs(A, "ones-solution")
    P = S.SaitPairPreconditioner(ML, MU) if precond else None
    x1, st1 = S.pcg(A, P, b, 1e-10, 1000)
    ctxs = DS.make_contexts_local(A, ML, MU, world)
    xs, st = DS.pcg(ctxs, DS.LocalComm(), _shards(b, ctxs), 1e-10, 1000)
    torch.cuda.synchronize()
    x = torch.cat(xs).cpu().numpy()
    assert st.converged and st.iterations == st1.iterations
    assert bitwise_equal(st.history, st1.history)
    assert bitwise_equal(x, x1)
    assert st.true_relres == st1.true_relres


@pytest.mark.parametrize("world", [2, 3])
def test_dist_gmres_bitwise(S, world):
    import torch

    from paper_2106_12836_b200 import dist_solvers as DS

    A = S.convdiff_2d(100)
    ML, MU = _pair(S, A, 2e-2, 4)
    b = S.uniform_pm1(3, A.nrows)
    P = S.SaitPairPreconditioner(ML, MU)
    for restart in (5, 30):
        x1, st1 = S.gmres(A, P, b, restart, 1e-8, 400)
        ctxs = DS.make_contexts_local(A, ML, MU, world)
        xs, st = DS.gmres(ctxs, DS.LocalComm(), _shards(b, ctxs), restart, 1e-8, 400)
        torch.cuda.synchronize()
        x = torch.cat(xs).cpu().numpy()
        assert st.iterations == st1.iterations and st.converged == st1.converged
        assert bitwise_equal(st.history, st1.history)
        assert bitwise_equal(x, x1)


@pytest.mark.parametrize("world,nev,precond", [(2, 4, True), (3, 8, True), (2, 3, False)])
def test_dist_lobpcg_bitwise(S, world, nev, precond):
    import torch

    from paper_2106_12836_b200 import dist_solvers as DS

    A = S.laplacian_3d(24)
    ML, MU = _pair(S, A, 5e-2, 3) if precond else (None, None)
    P = S.SaitPairPreconditioner(ML, MU) if precond else None
    r1 = S.lobpcg(A, P, nev, 1e-6, 40, 5)
    ctxs = DS.make_contexts_local(A, ML, MU, world)
    r = DS.lobpcg(ctxs, DS.LocalComm(), nev, 1e-6, 40, 5)
    torch.cuda.synchronize()
    assert r.iterations == r1.iterations
    assert bitwise_equal(r.eigenvalues, r1.eigenvalues)
    assert bitwise_equal(np.asarray(r.residual_history).ravel(), np.asarray(r1.residual_history).ravel())
    X = np.concatenate([x.cpu().numpy().reshape(nev, -1) for x in r.eigenvectors], axis=1)  # (nev, n)
    X1 = np.asarray(r1.eigenvectors)
    X1 = X1.T if X1.shape[0] != nev else X1
    assert bitwise_equal(X, X1)
