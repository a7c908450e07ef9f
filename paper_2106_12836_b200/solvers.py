"""Device-resident solver loops driving the SAIT apply (north_star (3)).

``gmres`` (right-preconditioned GMRES(m), CGS2 Arnoldi) and ``pcg``
 run entirely on the GPU; only control scalars come back
per iteration.  ``M`` is a SaitPairPreconditioner, an ExactIluPreconditioner
(the comparator: two device triangular solves) or None (identity).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .csr import CsrMatrix, DeviceCsr, _stream_handle


@dataclass
class SolveStats:
    iterations: int
    converged: bool
    relres_estimate: float
    true_relres: float
    seconds: float
    history: np.ndarray
    precond_seconds: float = 0.0  # device time of the preconditioner applies (the paper's split)
    precond_applies: int = 0


def _prep(A, b, stream):
    import torch

    dA = A if isinstance(A, DeviceCsr) else DeviceCsr.upload(A, stream)
    on_dev = isinstance(b, torch.Tensor) and b.is_cuda
    bd = b if on_dev else torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).cuda()
    x = torch.empty_like(bd)
    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    return dA, bd, x, on_dev, s


def _finish(rc, st, hist, x, on_dev):
    N.check(rc)
    its = st.iterations
    stats = SolveStats(its, bool(st.converged), st.relres_estimate, st.true_relres, st.seconds, hist[: its + 1].copy(),
                       st.precond_seconds, st.precond_applies)
    return (x if on_dev else x.cpu().numpy()), stats


def _precond(M, pair_fn, exact_fn):
    from .preconditioner import ExactIluPreconditioner

    if M is None:
        return None, pair_fn
    if isinstance(M, ExactIluPreconditioner):
        return M._h, exact_fn
    return M.handle, pair_fn


def gmres(A, M, b, restart: int = 30, tol: float = 1e-8, maxit: int = 10000, stream=None):
    dA, bd, x, on_dev, s = _prep(A, b, stream)
    hist = np.zeros(maxit + 1)
    st = N.SolveStats()
    mh, fn = _precond(M, N.lib.sait_gmres, N.lib.sait_gmres_exact)
    rc = fn(dA.handle, mh, bd.data_ptr(), x.data_ptr(), bd.numel(), int(restart), float(tol), int(maxit),
                          hist.ctypes.data_as(N.PD), C.byref(st), s)
    return _finish(rc, st, hist, x, on_dev)


def pcg(A, M, b, tol: float = 1e-10, maxit: int = 10000, stream=None):
    dA, bd, x, on_dev, s = _prep(A, b, stream)
    hist = np.zeros(maxit + 1)
    st = N.SolveStats()
    mh, fn = _precond(M, N.lib.sait_pcg, N.lib.sait_pcg_exact)
    rc = fn(dA.handle, mh, bd.data_ptr(), x.data_ptr(), bd.numel(), float(tol), int(maxit),
                        hist.ctypes.data_as(N.PD), C.byref(st), s)
    return _finish(rc, st, hist, x, on_dev)


@dataclass
class EigResult:
    """SPEC.md EigResult: eigenvalues ascending, eigenvectors (n, nev)."""

    eigenvalues: np.ndarray
    eigenvectors: object
    iterations: int
    residual_history: np.ndarray
    stats: SolveStats | None = None  # seconds + preconditioner share (SAIT pair only)


def lobpcg(A, M, nev: int, tol: float = 1e-6, maxit: int = 1000, seed: int = 5, stream=None, host_vectors=True,
           gram: str = "canonical"):
    """Block LOBPCG.  gram="canonical" (default) is bitwise
    the restatement; gram="tensor" uses FP64 tensor-core Grams
    (sait_lobpcg_opt): faster, deterministic, within +-1 iteration of it."""
    import torch

    dA = A if isinstance(A, DeviceCsr) else DeviceCsr.upload(A, stream)
    n = dA.nrows
    evals = np.zeros(nev)
    vecs = torch.empty((nev, n), dtype=torch.float64, device="cuda")  # column-major n x nev
    res = np.zeros((maxit + 1) * nev)
    its = C.c_int()
    s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
    mh, fn = _precond(M, N.lib.sait_lobpcg, N.lib.sait_lobpcg_exact)
    st = None
    if gram not in ("canonical", "tensor"):
        raise ValueError(f"unknown gram mode {gram!r}")
    if fn is N.lib.sait_lobpcg:
        st = N.SolveStats()
        N.check(N.lib.sait_lobpcg_opt(dA.handle, mh, int(nev), float(tol), int(maxit), int(seed),
                                      1 if gram == "tensor" else 0, evals.ctypes.data_as(N.PD), vecs.data_ptr(),
                                      res.ctypes.data_as(N.PD), C.byref(its), C.byref(st), s))
    else:
        N.check(fn(dA.handle, mh, int(nev), float(tol), int(maxit), int(seed), evals.ctypes.data_as(N.PD),
                   vecs.data_ptr(), res.ctypes.data_as(N.PD), C.byref(its), s))
    it = its.value
    v = vecs.T
    hist = res[: (it + 1) * nev].reshape(it + 1, nev)
    stats = None
    if st is not None:
        stats = SolveStats(it, bool(st.converged), 0.0, 0.0, st.seconds, hist, st.precond_seconds, st.precond_applies)
    return EigResult(evals, v.cpu().numpy() if host_vectors else v, it, hist, stats)
