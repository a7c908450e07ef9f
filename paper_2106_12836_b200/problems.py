"""Inputs of the SAIT path: ILU(k) factors (ilu.hpp:27) and the seeded
synthetic problems of BASELINE.json.  Host code in
libsait_b200.so."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .csr import CsrMatrix, _from_c


@dataclass
class IluFactors:
    """ilu.hpp:12-16"""

    lower: CsrMatrix
    upper: CsrMatrix
    level: int = 0


def ilu_k(a: CsrMatrix, level: int) -> IluFactors:
    lo, up = N.HostCsr(), N.HostCsr()
    N.check(N.lib.sait_ilu_k(C.byref(a._as_c()), int(level), C.byref(lo), C.byref(up)))
    return IluFactors(_from_c(lo), _from_c(up), int(level))


def ilu_device(a, level: int = 0, stream=None) -> IluFactors:
    """ilu_k(a, level) computed on the GPU for level 0 or 1 (sait_ilu_device):
    bitwise the same factors, returned as DeviceCsr (``.to_host()`` for
    CsrMatrix).  ``a`` is a CsrMatrix (uploaded) or a DeviceCsr."""
    from .csr import DeviceCsr, _stream_handle

    da = a if isinstance(a, DeviceCsr) else DeviceCsr.upload(a, stream)
    lo, up = C.c_void_p(), C.c_void_p()
    N.check(N.lib.sait_ilu_device(da.handle, int(level), _stream_handle(stream), C.byref(lo), C.byref(up)))
    return IluFactors(DeviceCsr(lo.value), DeviceCsr(up.value), int(level))


def ilu0_device(a, stream=None) -> IluFactors:
    """ilu_k(a, 0) on the GPU (sait_ilu0)."""
    return ilu_device(a, 0, stream)


def mm_read(path) -> CsrMatrix:
    """SPEC.md:373-381 mm_read: Matrix Market coordinate real/integer,
    general or symmetric (expanded), duplicates summed in file order."""
    out = N.HostCsr()
    N.check(N.lib.sait_mm_read(str(path).encode(), C.byref(out)))
    return _from_c(out)


def mm_write(path, m: CsrMatrix) -> None:
    """General coordinate form with %.17g values (mm_read round-trips it bit for bit)."""
    N.check(N.lib.sait_mm_write(str(path).encode(), C.byref(m._as_c())))


def make_rhs(a: CsrMatrix, mode: str = "ones-solution", seed: int = 0) -> np.ndarray:
    """'ones-solution' b = A 1, or 'seeded-random' unit vector."""
    modes = {"ones-solution": 0, "seeded-random": 1}
    if mode not in modes:
        raise N.SaitInvalidArgument(f"make_rhs: unknown mode {mode!r}")
    b = np.empty(a.nrows)
    N.check(N.lib.sait_make_rhs(C.byref(a._as_c()), modes[mode], int(seed), b.ctypes.data_as(N.PD)))
    return b


def _gen(fn, *args) -> CsrMatrix:
    out = N.HostCsr()
    N.check(fn(*args, C.byref(out)))
    return _from_c(out)


def laplacian_2d(nx: int) -> CsrMatrix:
    """5-point, diag 4, lexicographic x-fastest, Dirichlet."""
    return _gen(N.lib.sait_problem_laplacian_2d, C.c_int64(nx))


def laplacian_3d(n: int) -> CsrMatrix:
    """7-point, diag 6."""
    return _gen(N.lib.sait_problem_laplacian_3d, C.c_int64(n))


def convdiff_2d(nx: int, bx: float = 20.0, by: float = -10.0) -> CsrMatrix:
    """9-point diffusion + first-order upwind convection (BASELINE config 3)."""
    return _gen(N.lib.sait_problem_convdiff_2d, C.c_int64(nx), C.c_double(bx), C.c_double(by))


def synthetic_lower(n: int, draws: int = 15, p: float = 0.01, seed: int = 4) -> CsrMatrix:
    """BASELINE config 4's random lower-triangular T."""
    return _gen(N.lib.sait_problem_synthetic_lower, C.c_int64(n), C.c_int64(draws), C.c_double(p), C.c_uint64(seed))


def uniform_pm1(seed: int, n: int) -> np.ndarray:
    out = np.empty(n)
    N.lib.sait_fill_uniform_pm1(C.c_uint64(seed), C.c_int64(n), out.ctypes.data_as(N.PD))
    return out
