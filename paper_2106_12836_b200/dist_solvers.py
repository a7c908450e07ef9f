"""Row-sharded solver loops: PCG and GMRES(m) over ranks that
each own a 2048-aligned row block of A, the SAIT pair and the vectors.

The loops restate `sait_pcg` / `sait_gmres` (csrc/solvers.cu) operation by
operation on top of the same device kernels (`sait_vec_*`, `sait_dot_*`):
  * A x and M r run as PeerRowOperator / PeerShardedPair (halos read over
    peer memory inside the SpMVs);
  * a dot is the canonical per-2048-block partials on every rank, all ranks'
    partials gathered in rank order, then the canonical fold — so every dot,
    and therefore every iterate, is bitwise the single-GPU solver's;
  * the small host work (alpha/beta, Givens rotations, back substitution) is
    the same IEEE double arithmetic, replicated on every rank.

The code is SPMD over a list of rank contexts: a multi-process job passes its
one context and a TorchComm (all_gather over torch.distributed); the single-GPU
tests pass several contexts living in one process and a LocalComm, and every
stage is issued for all of them before the next (so no kernel waits on a flag
that is not yet published).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .dist import PeerRowOperator, PeerShardedPair

ALIGN = 2048  # the canonical dot block: shards must not split one


@dataclass
class RankContext:
    A: PeerRowOperator
    M: PeerShardedPair | None

    @property
    def own(self):
        return self.A.own

    @property
    def nloc(self):
        return self.A.own[1] - self.A.own[0]


class LocalComm:
    """All ranks in this process: gathering is concatenation."""

    def gather(self, parts):
        return parts


class TorchComm:
    """One rank per process: all_gather of the (padded) partials."""

    def __init__(self, world: int, group=None):
        self.world, self.group = world, group

    def gather(self, parts):
        import torch
        import torch.distributed as dist

        (mine,) = parts
        m, nb = mine.shape
        sizes = [torch.zeros(1, dtype=torch.int64, device=mine.device) for _ in range(self.world)]
        dist.all_gather(sizes, torch.tensor([nb], dtype=torch.int64, device=mine.device), group=self.group)
        nbs = [int(x.item()) for x in sizes]
        pad = torch.zeros((m, max(nbs)), dtype=mine.dtype, device=mine.device)
        pad[:, :nb] = mine
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad.contiguous(), group=self.group)
        return [b[:, :k] for b, k in zip(bufs, nbs)]


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


class _Dots:
    """Canonical dots across ranks: local partials, gather, fold."""

    def __init__(self, ctxs, comm):
        import torch

        self.ctxs, self.comm = ctxs, comm
        self.nb = [int(N.lib.sait_dot_blocks(c.nloc)) for c in ctxs]
        self.out = torch.empty(64, dtype=torch.float64, device="cuda")

    def __call__(self, xs, Vs, m=1, ld=None, sqrt=False):
        """xs[q] . V_j[q] for j < m (V column-major with leading dimension ld,
        default the local length); returns m host doubles."""
        import torch

        s = _stream()
        parts = []
        for c, x, V, nb in zip(self.ctxs, xs, Vs, self.nb):
            p = torch.empty((m, nb), dtype=torch.float64, device="cuda")
            N.check(N.lib.sait_dot_partials(x.data_ptr(), V.data_ptr(), ld or c.nloc, m, c.nloc, p.data_ptr(), s))
            parts.append(p)
        # (contexts own >= 1 row: PeerRowOperator refuses empty row blocks)
        allp = torch.cat([p.reshape(m, -1) for p in self.comm.gather(parts)], dim=1).contiguous()
        N.check(N.lib.sait_dot_fold(allp.data_ptr(), allp.shape[1], m, self.out.data_ptr(), int(sqrt), s))
        return self.out[:m].cpu().numpy().tolist()


def _apply_A(ctxs, xs, ys):
    s = _stream()
    for c in ctxs:
        c.A.epoch += 1
    for c, x in zip(ctxs, xs):
        c.A.stage_input(x, c.A.epoch, s)
    for c, y in zip(ctxs, ys):
        c.A.stage_spmv(y, c.A.epoch, s)


def _apply_M(ctxs, rs, zs):
    s = _stream()
    if ctxs[0].M is None:
        for r, z in zip(rs, zs):
            z.copy_(r)
        return
    for c in ctxs:
        c.M.epoch += 1
    for c, r in zip(ctxs, rs):
        c.M.stage_input(r, c.M.epoch, s)
    for c in ctxs:
        c.M.stage_lower(c.M.epoch, s)
    for c, z in zip(ctxs, zs):
        c.M.stage_upper(z, c.M.epoch, s)


def _vec(op, a, xs, ys):
    s = _stream()
    for x, y in zip(xs, ys):
        N.check(N.lib.sait_vec_update(op, y.numel(), float(a), x.data_ptr(), y.data_ptr(), s))


@dataclass
class DistSolveStats:
    iterations: int
    converged: bool
    relres_estimate: float
    true_relres: float
    seconds: float
    history: np.ndarray


def pcg(ctxs, comm, bs, tol=1e-10, maxit=10000):
    """Row-sharded PCG (restates sait_pcg, solvers.cu): returns (x_locals, stats)."""
    import torch

    t0 = time.perf_counter()
    dot = _Dots(ctxs, comm)
    xs = [torch.zeros_like(b) for b in bs]
    rs = [b.clone() for b in bs]
    zs = [torch.empty_like(b) for b in bs]
    ps = [torch.empty_like(b) for b in bs]
    qs = [torch.empty_like(b) for b in bs]
    bnorm = dot(bs, bs, sqrt=True)[0]
    rel, its = 1.0, 0
    conv, breakdown = bnorm == 0.0, False
    hist = [1.0]
    if not conv:
        _apply_M(ctxs, rs, zs)
        for p, z in zip(ps, zs):
            p.copy_(z)
        rz = dot(rs, zs)[0]
        while its < maxit:
            _apply_A(ctxs, ps, qs)
            pq = dot(ps, qs)[0]
            if not (pq > 0.0):
                breakdown = True
                break
            alpha = rz / pq
            _vec(0, alpha, ps, xs)
            _vec(0, -alpha, qs, rs)
            its += 1
            rel = dot(rs, rs, sqrt=True)[0] / bnorm
            hist.append(rel)
            if rel <= tol:
                conv = True
                break
            _apply_M(ctxs, rs, zs)
            rz2 = dot(rs, zs)[0]
            beta = rz2 / rz
            rz = rz2
            _vec(1, beta, zs, ps)  # p = z + beta p
    _apply_A(ctxs, xs, qs)
    _vec(2, 0.0, bs, qs)  # q = b - A x
    tr = dot(qs, qs, sqrt=True)[0]
    if breakdown:
        raise N.SaitRuntimeError(f"pcg: breakdown, p'Ap <= 0 at iteration {its}")
    st = DistSolveStats(its, conv, 0.0 if bnorm == 0.0 else rel, 0.0 if bnorm == 0.0 else tr / bnorm,
                        time.perf_counter() - t0, np.array(hist))
    return xs, st


def gmres(ctxs, comm, bs, restart=30, tol=1e-8, maxit=10000):
    """Row-sharded right-preconditioned GMRES(m) with CGS2 (restates
    sait_gmres, solvers.cu): returns (x_locals, stats)."""
    import torch

    t0 = time.perf_counter()
    m = restart
    s = _stream()
    dot = _Dots(ctxs, comm)
    Vs = [torch.empty((m + 1) * c.nloc, dtype=torch.float64, device="cuda") for c in ctxs]
    ws = [torch.empty_like(b) for b in bs]
    zs = [torch.empty_like(b) for b in bs]
    us = [torch.empty_like(b) for b in bs]
    xs = [torch.zeros_like(b) for b in bs]
    dsc = torch.empty(m + 2, dtype=torch.float64, device="cuda")  # device scalars: norm, h

    def col(V, c, i):
        return V[i * c.nloc : (i + 1) * c.nloc]

    def div_into(src, dst_fn, value):
        dsc[0:1].fill_(value)
        for c, w, V in zip(ctxs, src, Vs):
            N.check(N.lib.sait_vec_div(c.nloc, w.data_ptr(), dsc.data_ptr(), dst_fn(c, V).data_ptr(), s))

    H = np.zeros((m + 1) * m)
    cs, sn = [0.0] * m, [0.0] * m
    bnorm = dot(bs, bs, sqrt=True)[0]
    its, conv, est, beta = 0, False, 1.0, bnorm
    hist = [1.0]
    if bnorm == 0.0:
        conv, est = True, 0.0
    for w, b in zip(ws, bs):
        w.copy_(b)
    while not conv and its < maxit:
        div_into(ws, lambda c, V: col(V, c, 0), beta)  # v0 = r / beta
        g = [0.0] * (m + 1)
        g[0] = beta
        k = 0
        for i in range(m):
            if its >= maxit:
                break
            _apply_M(ctxs, [col(V, c, i) for c, V in zip(ctxs, Vs)], zs)
            _apply_A(ctxs, zs, ws)
            h1 = dot(ws, Vs, m=i + 1)  # CGS2, pass 1
            dh = torch.tensor(h1, dtype=torch.float64, device="cuda")
            for c, w, V in zip(ctxs, ws, Vs):
                N.check(N.lib.sait_vec_cgs(c.nloc, w.data_ptr(), V.data_ptr(), c.nloc, i + 1, dh.data_ptr(), s))
            h2 = dot(ws, Vs, m=i + 1)  # pass 2
            dh2 = torch.tensor(h2, dtype=torch.float64, device="cuda")
            for c, w, V in zip(ctxs, ws, Vs):
                N.check(N.lib.sait_vec_cgs(c.nloc, w.data_ptr(), V.data_ptr(), c.nloc, i + 1, dh2.data_ptr(), s))
            nrm = dot(ws, ws, sqrt=True)[0]
            h = [h1[j] + h2[j] for j in range(i + 1)] + [nrm]
            if nrm != 0.0:
                div_into(ws, lambda c, V, i=i: col(V, c, i + 1), nrm)
            for j in range(i):  # previous rotations
                t0_ = cs[j] * h[j] + sn[j] * h[j + 1]
                t1_ = -sn[j] * h[j] + cs[j] * h[j + 1]
                h[j], h[j + 1] = t0_, t1_
            den = math.sqrt(h[i] * h[i] + h[i + 1] * h[i + 1])
            if den == 0.0:
                cs[i], sn[i] = 1.0, 0.0
            else:
                cs[i], sn[i] = h[i] / den, h[i + 1] / den
            h[i], h[i + 1] = den, 0.0
            g[i + 1] = -sn[i] * g[i]
            g[i] = cs[i] * g[i]
            for j in range(i + 1):
                H[j * m + i] = h[j]
            its += 1
            k = i + 1
            est = abs(g[i + 1]) / bnorm
            hist.append(est)
            if est <= tol:
                conv = True
                break
        y = [0.0] * m
        for ii in range(k - 1, -1, -1):  # back substitution
            t = g[ii]
            for jj in range(ii + 1, k):
                t = t - H[ii * m + jj] * y[jj]
            y[ii] = t / H[ii * m + ii]
        yd = torch.tensor(y[:k], dtype=torch.float64, device="cuda")
        for c, V, u in zip(ctxs, Vs, us):
            N.check(N.lib.sait_vec_lincomb(c.nloc, V.data_ptr(), c.nloc, k, yd.data_ptr(), u.data_ptr(), s))
        _apply_M(ctxs, us, zs)
        _vec(3, 0.0, zs, xs)  # x += M (V y)
        _apply_A(ctxs, xs, zs)
        _vec(2, 0.0, bs, zs)  # z = b - A x
        for w, z in zip(ws, zs):
            w.copy_(z)
        beta = dot(ws, ws, sqrt=True)[0]
        if beta == 0.0:
            conv = True
    st = DistSolveStats(its, conv, est, 0.0 if bnorm == 0.0 else beta / bnorm, time.perf_counter() - t0,
                        np.array(hist))
    return xs, st


@dataclass
class DistEigResult:
    eigenvalues: np.ndarray
    eigenvectors: list  # this process's row blocks (n_local x nev, column-major), one per context
    iterations: int
    residual_history: np.ndarray


def lobpcg(ctxs, comm, nev, tol=1e-6, maxit=1000, seed=5):
    """Row-sharded block LOBPCG (restates sait_lobpcg, solvers.cu): every Gram
    block is the canonical partials of all ranks folded in rank order, the
    small dense algebra is the library's own (sait_dense_*), so eigenvalues,
    residual histories and the eigenvector blocks are bitwise the single-GPU
    solver's."""
    import torch

    k = nev
    if not 1 <= k <= 16:
        raise N.SaitInvalidArgument("lobpcg: block size must be in [1, 16]")
    s = _stream()
    dot = _Dots(ctxs, comm)
    nl = [c.nloc for c in ctxs]
    kw = dict(dtype=torch.float64, device="cuda")
    S = [torch.empty(3 * k * n_, **kw) for n_ in nl]   # [X W P], column-major
    AS = [torch.empty(3 * k * n_, **kw) for n_ in nl]
    R = [torch.empty(k * n_, **kw) for n_ in nl]
    tmp = [torch.empty(4 * k * n_, **kw) for n_ in nl]

    def blk(lst, i, cols=1):  # block i (of k columns) of each rank's stacked array
        return [t[i * k * n_ : (i + cols) * k * n_] for t, n_ in zip(lst, nl)]

    def column(lst, j):
        return [t[j * n_ : (j + 1) * n_] for t, n_ in zip(lst, nl)]

    def block_A(src, dst):  # column by column (bitwise the block SpMM)
        for j in range(k):
            _apply_A(ctxs, column(src, j), column(dst, j))

    def block_M(src, dst):
        for j in range(k):
            _apply_M(ctxs, column(src, j), column(dst, j))

    def gram(A_, ka, B_, kb):
        parts = []
        for c, a_, b_ in zip(ctxs, A_, B_):
            p = torch.empty((ka * kb, int(N.lib.sait_dot_blocks(c.nloc))), **kw)
            N.check(N.lib.sait_gram_partials(a_.data_ptr(), ka, b_.data_ptr(), kb, c.nloc, p.data_ptr(), s))
            parts.append(p)
        allp = torch.cat([p.reshape(ka * kb, -1) for p in comm.gather(parts)], dim=1).contiguous()
        out = torch.empty(ka * kb, **kw)
        N.check(N.lib.sait_dot_fold(allp.data_ptr(), allp.shape[1], ka * kb, out.data_ptr(), 0, s))
        return out.cpu().numpy().astype(np.float64)

    def lincomb(in_, kin, Cm, kout, out_):
        dC = torch.from_numpy(np.ascontiguousarray(Cm, dtype=np.float64)).cuda()
        for n_, a_, o_ in zip(nl, in_, out_):
            N.check(N.lib.sait_block_lincomb(n_, a_.data_ptr(), kin, dC.data_ptr(), kout, o_.data_ptr(), s))

    def copy(dst, src):
        for d_, s_ in zip(dst, src):
            d_.copy_(s_)

    def cholqr(Y, AY):
        G = gram(Y, k, Y, k)
        L = np.zeros(k * k)
        Li = np.zeros(k * k)
        if not N.lib.sait_dense_chol_lower(G.ctypes.data_as(N.PD), k, L.ctypes.data_as(N.PD)):
            return False
        N.lib.sait_dense_tri_lower_inv(L.ctypes.data_as(N.PD), k, Li.ctypes.data_as(N.PD))
        Ri = Li.reshape(k, k).T.copy().ravel()
        lincomb(Y, k, Ri, k, blk(tmp, 0))
        copy(Y, blk(tmp, 0))
        if AY is not None:
            lincomb(AY, k, Ri, k, blk(tmp, 0))
            copy(AY, blk(tmp, 0))
        return True

    def rr(GA, GB, m):
        Cm = np.zeros(m * k)
        lam_ = np.zeros(k)
        ok = N.lib.sait_dense_rayleigh_ritz(GA.ctypes.data_as(N.PD), GB.ctypes.data_as(N.PD), m, k,
                                            Cm.ctypes.data_as(N.PD), lam_.ctypes.data_as(N.PD))
        return bool(ok), Cm, lam_

    X, W, P = blk(S, 0), blk(S, 1), blk(S, 2)
    AX, AW, AP = blk(AS, 0), blk(AS, 1), blk(AS, 2)
    for c, x in zip(ctxs, X):  # X0 column j from seed * 1000 + j over the global row index
        for j in range(k):
            N.check(N.lib.sait_fill_uniform_pm1_device(seed * 1000 + j, c.nloc, c.own[0],
                                                       x[j * c.nloc :].data_ptr(), s))
    block_A(X, AX)
    GB = gram(X, k, X, k)
    GA = gram(X, k, AX, k)
    ok, Cm, lam = rr(GA, GB, k)
    if not ok:
        raise N.SaitRuntimeError("lobpcg: initial block is rank deficient")
    lincomb(X, k, Cm, k, blk(tmp, 0))
    copy(X, blk(tmp, 0))
    lincomb(AX, k, Cm, k, blk(tmp, 0))
    copy(AX, blk(tmp, 0))
    hist = []
    have_p = False
    it = 0
    failed = None
    while True:
        dl = torch.from_numpy(lam.copy()).cuda()
        for n_, ax, x, r_ in zip(nl, AX, X, R):
            N.check(N.lib.sait_block_residual(n_, k, ax.data_ptr(), x.data_ptr(), dl.data_ptr(), r_.data_ptr(), s))
        norms = [dot(column(R, j), column(R, j), sqrt=True)[0] for j in range(k)]
        hist.append(norms)
        conv = all(v <= tol for v in norms)
        if conv or it == maxit:
            break
        if ctxs[0].M is not None:
            block_M(R, W)
        else:
            copy(W, R)
        G1 = gram(X, k, W, k)
        dG = torch.from_numpy(G1).cuda()
        for n_, x, w in zip(nl, X, W):
            N.check(N.lib.sait_block_sub_lincomb(n_, x.data_ptr(), k, dG.data_ptr(), w.data_ptr(), s))
        if not cholqr(W, None):
            failed = "lobpcg: preconditioned residual block is rank deficient"
            break
        block_A(W, AW)
        use_p = have_p and cholqr(P, AP)
        m = 3 * k if use_p else 2 * k
        ok = False
        while True:
            Sm = [t[: m * n_] for t, n_ in zip(S, nl)]
            ASm = [t[: m * n_] for t, n_ in zip(AS, nl)]
            GB = gram(Sm, m, Sm, m)
            GA = gram(Sm, m, ASm, m)
            for i in range(m):
                for j in range(i + 1, m):
                    s2 = 0.5 * (GA[i * m + j] + GA[j * m + i])
                    GA[i * m + j] = s2
                    GA[j * m + i] = s2
            ok, Cm, lam_new = rr(GA, GB, m)
            if ok:
                lam = lam_new
                break
            if m == 3 * k:
                m = 2 * k
                continue
            break
        if not ok:
            failed = "lobpcg: Gram matrix not positive definite"
            break
        Wm = [t[k * n_ : m * n_] for t, n_ in zip(S, nl)]     # [W P] of the subspace used
        AWm = [t[k * n_ : m * n_] for t, n_ in zip(AS, nl)]
        Sm = [t[: m * n_] for t, n_ in zip(S, nl)]
        ASm = [t[: m * n_] for t, n_ in zip(AS, nl)]
        lincomb(Wm, m - k, Cm[k * k :], k, blk(tmp, 0))
        lincomb(AWm, m - k, Cm[k * k :], k, blk(tmp, 1))
        lincomb(Sm, m, Cm, k, blk(tmp, 2))
        lincomb(ASm, m, Cm, k, blk(tmp, 3))
        copy(P, blk(tmp, 0))
        copy(AP, blk(tmp, 1))
        copy(X, blk(tmp, 2))
        copy(AX, blk(tmp, 3))
        have_p = True
        it += 1
    if failed:
        raise N.SaitRuntimeError(failed)
    return DistEigResult(np.array(lam[:k]), [x.clone() for x in X], it, np.array(hist))


def make_contexts_local(A, ML, MU, world: int):
    """`world` rank contexts in this process (one GPU), wired to each other."""
    ctx = {}
    rA = lambda q: ctx[q].A.buf.ptr  # noqa: E731
    rM = lambda q, f: ctx[q].M.bufs[f].ptr  # noqa: E731
    for q in range(world):
        a = PeerRowOperator(A, q, world, resolve=rA, align=ALIGN)
        m = PeerShardedPair(ML, MU, q, world, resolve=rM, align=ALIGN) if ML is not None else None
        ctx[q] = RankContext(a, m)
    return [ctx[q] for q in range(world)]


def make_context_distributed(A, ML, MU, rank: int, world: int, group=None):
    """This process's rank context of a torch.distributed job (IPC-wired)."""
    a = PeerRowOperator.distributed(A, rank, world, group, align=ALIGN)
    m = PeerShardedPair.distributed(ML, MU, rank, world, group, align=ALIGN) if ML is not None else None
    return RankContext(a, m)


del C
