"""Preconditioner interface and the SAIT pair (preconditioner.hpp:17-101).

``SaitPairPreconditioner(lower_inverse, upper_inverse)`` owns the two
approximate inverses on the GPU and applies ``z = M_U (M_L r)`` with the
device SpMV pair.  ``apply`` accepts host numpy arrays (copies inside, like a
reference caller holding std::vector) or torch CUDA tensors (device-resident
solver loops; enqueued on torch's current stream, no synchronisation).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .csr import CsrMatrix, DeviceCsr, _stream_handle


class Preconditioner:
    """preconditioner.hpp:17-30"""

    def apply(self, r, z) -> None:
        raise NotImplementedError

    def apply_block(self, r):
        """Column by column unless a variant can do better (preconditioner.cpp:13-19)."""
        r = np.asarray(r, dtype=np.float64)
        z = np.empty_like(r, order="F")
        for j in range(r.shape[1]):
            zj = np.empty(r.shape[0])
            self.apply(np.ascontiguousarray(r[:, j]), zj)
            z[:, j] = zj
        return z

    def name(self) -> str:
        raise NotImplementedError

    def nnz(self) -> int:
        return 0


class IdentityPreconditioner(Preconditioner):
    """preconditioner.hpp:33-37"""

    def apply(self, r, z) -> None:
        z[...] = r

    def name(self) -> str:
        return "none"


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


class SaitPairPreconditioner(Preconditioner):
    """preconditioner.hpp:54-68; preconditioner.cpp:34-49."""

    def __init__(self, lower_inverse, upper_inverse, stream=None, format: str = "auto"):
        """``format`` (not in the reference): the factors' apply storage --
        "auto" (default), "csr", "sell32_int32", "sell32_int16", "sell32_dict";
        every format gives the same bits (sait_pair_create_ex)."""
        fmt = {v: k for k, v in N.FORMAT_NAMES.items()}.get(format)
        if fmt is None:
            raise ValueError(f"unknown apply format {format!r}")
        self._host_l = lower_inverse if isinstance(lower_inverse, CsrMatrix) else None
        self._host_u = upper_inverse if isinstance(upper_inverse, CsrMatrix) else None
        dl = lower_inverse if isinstance(lower_inverse, DeviceCsr) else DeviceCsr.upload(lower_inverse, stream)
        du = upper_inverse if isinstance(upper_inverse, DeviceCsr) else DeviceCsr.upload(upper_inverse, stream)
        h = C.c_void_p()
        N.check(N.lib.sait_pair_create_ex(dl.handle, du.handle, 1, fmt, C.byref(h)))
        dl.release()
        du.release()  # the pair owns both factors now (the reference ctor moves them in)
        self._h = h
        n, nnz = C.c_int64(), C.c_int64()
        N.check(N.lib.sait_pair_info(self._h, C.byref(n), C.byref(nnz)))
        self.n = n.value
        self._nnz = nnz.value

    def factor_format(self, which: int) -> dict:
        """Apply storage of M_L (which=0) or M_U (which=1): format name, whether
        the rows were length-sorted within 1024-row windows (``row_sorted``),
        stored slots, slices, dictionary size and ``stream_bytes`` (what one
        SpMV must move in that format: the roofline denominator)."""
        f = N.FactorFormat()
        N.check(N.lib.sait_pair_format(self._h, int(which), C.byref(f)))
        return {"format": N.FORMAT_NAMES[f.format], "row_sorted": bool(f.row_sorted), "nrows": f.nrows, "nnz": f.nnz,
                "stored_slots": f.stored_slots, "nslices": f.nslices, "dict_elems": f.dict_elems,
                "stream_bytes": f.stream_bytes}

    # -- interface
    def name(self) -> str:
        return "sait"

    def nnz(self) -> int:
        return self._nnz

    def apply(self, r, z, stream=None) -> None:
        if _is_cuda_tensor(r):
            import torch

            s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
            N.check(N.lib.sait_pair_apply(self._h, r.data_ptr(), r.numel(), z.data_ptr(), z.numel(), s))
            return
        rh = np.ascontiguousarray(r, dtype=np.float64)
        if not (isinstance(z, np.ndarray) and z.dtype == np.float64 and z.flags.c_contiguous):
            raise TypeError("apply: z must be a contiguous float64 numpy array or a CUDA tensor")
        N.check(N.lib.sait_pair_apply_host(self._h, rh.ctypes.data_as(N.PD), rh.size, z.ctypes.data_as(N.PD), z.size, _stream_handle(stream)))

    def apply_block(self, r, z=None, layout: str = "col", stream=None):
        """Z = M_U (M_L R) for an (n, nvec) block; the matrices are read once
        per 8 vectors (the reference's spmm re-reads them per column)."""
        if _is_cuda_tensor(r):
            import torch

            s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
            if z is None:
                z = torch.empty_like(r)
            n, nvec = (r.shape[0], r.shape[1]) if r.dim() == 2 else (r.numel(), 1)
            lay = 1 if layout == "row" else 0
            N.check(N.lib.sait_pair_apply_block(self._h, r.data_ptr(), z.data_ptr(), n, nvec, lay, s))
            return z
        # host block: column-major (each vector contiguous); the copies
        # overlap the device work vector by vector (pinned buffers for full
        # overlap, e.g. torch pin_memory() views)
        r = np.asarray(r, dtype=np.float64)
        n, nvec = r.shape
        rf = np.asfortranarray(r)
        if z is None:
            zf = np.empty((n, nvec), order="F")
        else:
            if not (isinstance(z, np.ndarray) and z.dtype == np.float64 and z.shape == (n, nvec) and z.flags.f_contiguous):
                raise TypeError("apply_block: z must be an F-contiguous float64 (n, nvec) numpy array")
            zf = z
        N.check(N.lib.sait_pair_apply_block_host(self._h, rf.ctypes.data_as(N.PD), zf.ctypes.data_as(N.PD), n, nvec, 0, _stream_handle(stream)))
        return zf

    def _factor(self, which: int) -> DeviceCsr:
        a, b = C.c_void_p(), C.c_void_p()
        N.check(N.lib.sait_pair_factors(self._h, C.byref(a), C.byref(b)))
        return DeviceCsr((a if which == 0 else b).value, owned=False)

    def lower_inverse(self) -> CsrMatrix:
        if self._host_l is None:
            self._host_l = self._factor(0).to_host()
        return self._host_l

    def upper_inverse(self) -> CsrMatrix:
        if self._host_u is None:
            self._host_u = self._factor(1).to_host()
        return self._host_u

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if self._h:
            N.lib.sait_pair_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ExactIluPreconditioner(Preconditioner):
    """preconditioner.hpp:39-49 / preconditioner.cpp:25-32: z = U^-1 (L^-1 r),
    the sequential baseline SAIT replaces, as two device triangular solves
    (sait_exact_ilu_*).  ``factors`` is an IluFactors (host CsrMatrix or
    DeviceCsr lower/upper)."""

    def __init__(self, factors, stream=None):
        lo, up = factors.lower, factors.upper
        dl = lo if isinstance(lo, DeviceCsr) else DeviceCsr.upload(lo, stream)
        du = up if isinstance(up, DeviceCsr) else DeviceCsr.upload(up, stream)
        h = C.c_void_p()
        N.check(N.lib.sait_exact_ilu_create(dl.handle, du.handle, 1, C.byref(h)))
        dl.release()
        du.release()
        self._h = h
        n, nnz = C.c_int64(), C.c_int64()
        N.check(N.lib.sait_exact_ilu_info(self._h, C.byref(n), C.byref(nnz)))
        self.n, self._nnz = n.value, nnz.value

    def name(self) -> str:
        return "exact"

    def nnz(self) -> int:
        return self._nnz

    def apply(self, r, z, stream=None) -> None:
        import torch

        if _is_cuda_tensor(r):
            s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
            N.check(N.lib.sait_exact_ilu_apply(self._h, r.data_ptr(), r.numel(), z.data_ptr(), z.numel(), s))
            return
        rd = torch.from_numpy(np.ascontiguousarray(r, dtype=np.float64)).cuda()
        zd = torch.empty(len(z), dtype=torch.float64, device="cuda")
        N.check(N.lib.sait_exact_ilu_apply(self._h, rd.data_ptr(), rd.numel(), zd.data_ptr(), zd.numel(), None))
        z[...] = zd.cpu().numpy()

    def close(self) -> None:
        if self._h:
            N.lib.sait_exact_ilu_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class JacobiSweepsPreconditioner(Preconditioner):
    """preconditioner.hpp:72-83 / preconditioner.cpp:51-60: ``sweeps`` Jacobi
    sweeps on the L-system, then on the U-system (the paper's section 4.3
    comparison), on the device."""

    def __init__(self, factors, sweeps: int, stream=None):
        if sweeps < 1:
            raise N.SaitInvalidArgument("JacobiSweepsPreconditioner: sweeps must be >= 1")
        self._l = factors.lower if isinstance(factors.lower, DeviceCsr) else DeviceCsr.upload(factors.lower, stream)
        self._u = factors.upper if isinstance(factors.upper, DeviceCsr) else DeviceCsr.upload(factors.upper, stream)
        self._sweeps = int(sweeps)

    def name(self) -> str:
        return "jacobi"

    def nnz(self) -> int:
        return self._l.nnz() + self._u.nnz()

    def sweeps(self) -> int:
        return self._sweeps

    def apply(self, r, z, stream=None) -> None:
        from .csr import unit_lower_triangular, upper_triangular
        from .sait import jacobi_sweeps_apply

        y = jacobi_sweeps_apply(self._l, unit_lower_triangular, r, self._sweeps, stream)
        out = jacobi_sweeps_apply(self._u, upper_triangular, y, self._sweeps, stream)
        if _is_cuda_tensor(r):
            z.copy_(out)
        else:
            z[...] = out


def apply_precond(p: Preconditioner, r):
    """preconditioner.hpp:101"""
    z = np.empty(len(r))
    p.apply(np.ascontiguousarray(r, dtype=np.float64), z)
    return z
