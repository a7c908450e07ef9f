"""ctypes bindings for the test oracle (TEST INFRASTRUCTURE ONLY).

Two backends with one Python surface:

* ``Oracle("port")`` — ``oracle/liboracle.so``, the C restatement
  (``oracle/sait_oracle.c``), every function citing the reference file:line.
* ``Oracle("reference")`` — ``oracle/_ref/libsaitref.so``, the unmodified
  reference sources compiled by ``oracle/Makefile`` plus ``ref_wrapper.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module, and only as
the checker or the timed CPU baseline — never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsaitref.so")


class OracleError(Exception):
    pass


class InvalidArgument(OracleError, ValueError):
    """Mirror of std::invalid_argument."""


class RuntimeErr(OracleError, RuntimeError):
    """Mirror of std::runtime_error."""


class _CCsr(C.Structure):
    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("row_ptr", C.POINTER(C.c_int64)),
        ("col_idx", C.POINTER(C.c_int64)),
        ("values", C.POINTER(C.c_double)),
    ]


@dataclass
class Csr:
    """Host CSR with the reference's layout (int64 row_ptr/col_idx, fp64 values)."""

    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray | None

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_scipy(self):
        import scipy.sparse as sp

        vals = self.values if self.values is not None else np.ones(self.nnz)
        return sp.csr_matrix((vals, self.col_idx, self.row_ptr), shape=(self.nrows, self.ncols))

    def pattern(self) -> "Csr":
        return Csr(self.nrows, self.ncols, self.row_ptr.copy(), self.col_idx.copy(), None)

    def same(self, other: "Csr") -> bool:
        """Bitwise equality (pattern and value bits)."""
        if (self.nrows, self.ncols) != (other.nrows, other.ncols):
            return False
        if not np.array_equal(self.row_ptr, other.row_ptr) or not np.array_equal(self.col_idx, other.col_idx):
            return False
        if (self.values is None) != (other.values is None):
            return False
        if self.values is None:
            return True
        return np.array_equal(self.values.view(np.uint64), other.values.view(np.uint64))


def csr(nrows, ncols, row_ptr, col_idx, values=None) -> Csr:
    return Csr(
        int(nrows),
        int(ncols),
        np.ascontiguousarray(row_ptr, dtype=np.int64),
        np.ascontiguousarray(col_idx, dtype=np.int64),
        None if values is None else np.ascontiguousarray(values, dtype=np.float64),
    )


def from_scipy(m) -> Csr:
    m = m.tocsr()
    m.sort_indices()
    return csr(m.shape[0], m.shape[1], m.indptr, m.indices, m.data)


_P64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)


def _in(m: Csr) -> _CCsr:
    c = _CCsr()
    c.nrows, c.ncols = m.nrows, m.ncols
    c.row_ptr = m.row_ptr.ctypes.data_as(_P64)
    c.col_idx = m.col_idx.ctypes.data_as(_P64)
    c.values = m.values.ctypes.data_as(_PD) if m.values is not None else _PD()
    c._keep = m  # keep arrays alive
    return c


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_PD)


class Oracle:
    def __init__(self, backend: str = "port"):
        self.backend = backend
        path = PORT_SO if backend == "port" else REF_SO
        if not os.path.exists(path):
            raise OSError(f"oracle backend {backend!r} not built: {path} missing (run oracle/Makefile)")
        self.lib = C.CDLL(path)
        self.p = "orc_" if backend == "port" else "ref_"
        L = self.lib
        self._err = getattr(L, self.p + "last_error")
        self._err.restype = C.c_char_p
        self._free = getattr(L, self.p + "free")
        self._free.argtypes = [C.c_void_p]
        self._csr_free = getattr(L, self.p + "csr_free")
        self._csr_free.argtypes = [C.POINTER(_CCsr)]

    # -- plumbing
    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc == 0:
            return
        msg = self._err().decode()
        if rc == 1:
            raise InvalidArgument(msg)
        if rc == 2:
            raise RuntimeErr(msg)
        raise OracleError(msg)

    def _out(self, c: _CCsr) -> Csr:
        n = c.nrows
        nnz = c.row_ptr[n] if n >= 0 else 0
        rp = np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(c.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
        vals = None
        if bool(c.values):
            vals = np.ctypeslib.as_array(c.values, shape=(max(nnz, 1),))[:nnz].copy()
        self._csr_free(C.byref(c))
        return Csr(int(c.nrows), int(c.ncols), rp, ci, vals)

    def _call_csr(self, name, *args) -> Csr:
        out = _CCsr()
        self._check(self._fn(name)(*args, C.byref(out)))
        return self._out(out)

    # -- kernels.cpp
    def spmv(self, a: Csr, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(a.nrows)
        self._check(self._fn("spmv")(C.byref(_in(a)), _dptr(x), C.c_int64(len(x)), _dptr(y), C.c_int64(len(y))))
        return y

    def spgemm(self, a: Csr, b: Csr) -> Csr:
        return self._call_csr("spgemm", C.byref(_in(a)), C.byref(_in(b)))

    def add_identity(self, a: Csr) -> Csr:
        return self._call_csr("add_identity", C.byref(_in(a)))

    def drop_by_threshold(self, a: Csr, tau: float) -> Csr:
        return self._call_csr("drop_by_threshold", C.byref(_in(a)), C.c_double(tau))

    def drop_by_pattern(self, a: Csr, s: Csr) -> Csr:
        return self._call_csr("drop_by_pattern", C.byref(_in(a)), C.byref(_in(s)))

    def scale_columns(self, a: Csr, d: np.ndarray) -> Csr:
        d = np.ascontiguousarray(d, dtype=np.float64)
        return self._call_csr("scale_columns", C.byref(_in(a)), _dptr(d), C.c_int64(len(d)))

    def transpose(self, a: Csr) -> Csr:
        return self._call_csr("transpose", C.byref(_in(a)))

    # -- sait.cpp
    def jacobi_split(self, t: Csr, lower: bool):
        inv = _PD()
        out = _CCsr()
        self._check(self._fn("jacobi_split")(C.byref(_in(t)), C.c_int(int(lower)), C.byref(inv), C.byref(out)))
        d = np.ctypeslib.as_array(inv, shape=(max(t.nrows, 1),))[: t.nrows].copy()
        self._free(inv)
        return d, self._out(out)

    def sait_thr(self, t: Csr, lower: bool, tau: float, steps: int) -> Csr:
        if self.backend == "port":
            return self._thr_port(t, lower, tau, steps)[0]
        return self._call_csr("sait_thr", C.byref(_in(t)), C.c_int(int(lower)), C.c_double(tau), C.c_int(steps))

    def _thr_port(self, t, lower, tau, steps):
        out = _CCsr()
        sr = C.c_int()
        self._check(self.lib.orc_sait_thr(C.byref(_in(t)), C.c_int(int(lower)), C.c_double(tau), C.c_int(steps), C.byref(out), C.byref(sr)))
        return self._out(out), sr.value

    def sait_polynomial_tt(self, tt: Csr, steps: int) -> Csr:
        """sait_polynomial(split, steps, {}) on the iteration matrix tt as given
        (reference only: sait.cpp:75-88)."""
        return self._call_csr("sait_polynomial_tt", C.byref(_in(tt)), C.c_int(steps))

    def sait_thr_steps(self, t: Csr, lower: bool, tau: float, steps: int):
        """(M, steps actually run) — port only."""
        return self._thr_port(t, lower, tau, steps)

    def sait_pat(self, t: Csr, lower: bool, p: int, m: int) -> Csr:
        if self.backend == "port":
            out = _CCsr()
            sr = C.c_int()
            self._check(self.lib.orc_sait_pat(C.byref(_in(t)), C.c_int(int(lower)), C.c_int(p), C.c_int(m), C.byref(out), C.byref(sr)))
            return self._out(out)
        return self._call_csr("sait_pat", C.byref(_in(t)), C.c_int(int(lower)), C.c_int(p), C.c_int(m))

    def sait_pat_capture_pattern(self, t: Csr, lower: bool, p: int) -> Csr:
        return self._call_csr("sait_pat_capture_pattern", C.byref(_in(t)), C.c_int(int(lower)), C.c_int(p))

    def sait_thr_cap(self, t: Csr, lower: bool, tau: float, steps: int, cap_factor: float) -> Csr:
        if self.backend == "port":
            out = _CCsr()
            sr = C.c_int()
            self._check(self.lib.orc_sait_thr_cap(C.byref(_in(t)), C.c_int(int(lower)), C.c_double(tau), C.c_int(steps), C.c_double(cap_factor), C.byref(out), C.byref(sr)))
            return self._out(out)
        return self._call_csr("sait_thr_cap", C.byref(_in(t)), C.c_int(int(lower)), C.c_double(tau), C.c_int(steps), C.c_double(cap_factor))

    def jacobi_sweeps_apply(self, t: Csr, lower: bool, b: np.ndarray, sweeps: int) -> np.ndarray:
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(t.nrows)
        self._check(self._fn("jacobi_sweeps_apply")(C.byref(_in(t)), C.c_int(int(lower)), _dptr(b), C.c_int(sweeps), _dptr(x)))
        return x

    def trisolve(self, t: Csr, lower: bool, b: np.ndarray) -> np.ndarray:
        """kernels.cpp:196-234 (x starts at zero, as the reference's vector)."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(t.nrows)
        self._check(self._fn("trisolve")(C.byref(_in(t)), C.c_int(int(lower)), _dptr(b), _dptr(x)))
        return x

    # -- ilu.cpp
    def ilu_k(self, a: Csr, level: int):
        lo, up = _CCsr(), _CCsr()
        self._check(self._fn("ilu_k")(C.byref(_in(a)), C.c_int(level), C.byref(lo), C.byref(up)))
        return self._out(lo), self._out(up)

    # -- preconditioner.cpp
    def pair_apply(self, ml: Csr, mu: Csr, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.empty(mu.nrows)
        self._check(self._fn("pair_apply")(C.byref(_in(ml)), C.byref(_in(mu)), _dptr(r), _dptr(z)))
        return z

    def pair_apply_block(self, ml: Csr, mu: Csr, r: np.ndarray) -> np.ndarray:
        """r: (n, nvec) array; returns (n, nvec).  Column-major like DenseMatrix."""
        nvec = r.shape[1]
        rc = np.asfortranarray(r, dtype=np.float64)
        z = np.empty((mu.nrows, nvec), order="F")
        self._check(self._fn("pair_apply_block")(C.byref(_in(ml)), C.byref(_in(mu)), rc.ctypes.data_as(_PD), C.c_int64(nvec), z.ctypes.data_as(_PD)))
        return z


_singletons: dict[str, Oracle] = {}


def get(backend: str = "port") -> Oracle:
    if backend not in _singletons:
        _singletons[backend] = Oracle(backend)
    return _singletons[backend]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ---- port-only helpers (generators, solvers) --------------------------------

def _port():
    return get("port")


def laplacian_2d(nx: int) -> Csr:
    return _port()._call_csr("laplacian_2d", C.c_int64(nx))


def laplacian_3d(n: int) -> Csr:
    return _port()._call_csr("laplacian_3d", C.c_int64(n))


def convdiff_2d(nx: int, bx: float = 20.0, by: float = -10.0) -> Csr:
    return _port()._call_csr("convdiff_2d", C.c_int64(nx), C.c_double(bx), C.c_double(by))


def synthetic_lower(n: int, draws: int = 15, p: float = 0.01, seed: int = 4) -> Csr:
    return _port()._call_csr("synthetic_lower", C.c_int64(n), C.c_int64(draws), C.c_double(p), C.c_uint64(seed))


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    L = _port().lib
    L.orc_fill_uniform_pm1.argtypes = [C.c_uint64, C.c_int64, _PD]
    L.orc_fill_uniform_pm1(C.c_uint64(seed), C.c_int64(n), _dptr(out))
    return out


class _SolveStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_relres", C.c_double), ("true_relres", C.c_double)]


def _solver(name, a, ml, mu, b, *args, exact=False):
    L = _port().lib
    L.orc_solver_precond_exact(C.c_int(int(exact)))
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(a.nrows)
    maxit = args[-1].value
    hist = np.zeros(maxit + 1)
    st = _SolveStats()
    pm = C.byref(_in(ml)) if ml is not None else None
    pu = C.byref(_in(mu)) if mu is not None else None
    fn = getattr(L, name)
    try:
        rc = fn(C.byref(_in(a)), pm, pu, _dptr(b), *args, _dptr(x), _dptr(hist), C.byref(st))
    finally:
        L.orc_solver_precond_exact(C.c_int(0))
    _port()._check(rc)
    its = st.iterations
    return x, {"iterations": its, "converged": bool(st.converged), "relres": st.final_relres,
               "true_relres": st.true_relres, "history": hist[: its + 1].copy()}


def gmres(a, ml, mu, b, restart=30, tol=1e-8, maxit=10000, exact=False):
    """Restated right-preconditioned GMRES(m) (oracle/solvers.c); exact=True
    preconditions with the ILU factors (ml = L, mu = U) by two trisolves."""
    return _solver("orc_gmres", a, ml, mu, b, C.c_int(restart), C.c_double(tol), C.c_int(maxit), exact=exact)


def pcg(a, ml, mu, b, tol=1e-10, maxit=10000, exact=False):
    """Restated PCG (oracle/solvers.c); exact as in gmres."""
    return _solver("orc_pcg", a, ml, mu, b, C.c_double(tol), C.c_int(maxit), exact=exact)


def dot(a, b):
    L = _port().lib
    L.orc_dot.restype = C.c_double
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return L.orc_dot(_dptr(a), _dptr(b), C.c_int64(len(a)))


def lobpcg(a, ml, mu, nev, tol=1e-6, maxit=500, seed=5, exact=False):
    """Restated block LOBPCG (oracle/solvers.c).  Returns (evals, evecs (n, nev)
    column-major, iterations, residual-norm history (iters+1, nev)); exact=True
    preconditions with the ILU factors (ml = L, mu = U) by two trisolves."""
    L = _port().lib
    L.orc_solver_precond_exact(C.c_int(int(exact)))
    n = a.nrows
    evals = np.zeros(nev)
    evecs = np.zeros((nev, n))  # row j = column j of the n x nev block
    res = np.zeros((maxit + 1) * nev)
    its = C.c_int()
    pm = C.byref(_in(ml)) if ml is not None else None
    pu = C.byref(_in(mu)) if mu is not None else None
    try:
        rc = L.orc_lobpcg(C.byref(_in(a)), pm, pu, C.c_int(nev), C.c_double(tol), C.c_int(maxit), C.c_uint64(seed),
                          _dptr(evals), evecs.ctypes.data_as(_PD), C.byref(its), _dptr(res))
    finally:
        L.orc_solver_precond_exact(C.c_int(0))
    _port()._check(rc)
    it = its.value
    return evals, evecs.T, it, res[: (it + 1) * nev].reshape(it + 1, nev)
