"""SAIT construction and the sparse kernels it is built from.

Python mirror of sait.hpp:14-74 and kernels.hpp:12-40.  Functions take a
host ``CsrMatrix`` (returning a host ``CsrMatrix``, like the reference) or a
``DeviceCsr`` (returning a ``DeviceCsr``, for device pipelines).  All
arithmetic runs in libsait_b200.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .csr import CsrMatrix, DeviceCsr, TriangularKind, _kind_lower, _stream_handle


@dataclass
class SaitThrParams:
    """sait.hpp:14-17"""

    threshold: float = 0.0
    steps: int = 1


@dataclass
class SaitPatParams:
    """sait.hpp:24-27"""

    pattern_steps: int = 1
    refine_steps: int = 1


@dataclass
class BuildStats:
    steps_run: int
    stabilized: bool
    nnz_out: int
    products: int
    seconds: float


def _dev(m, stream):
    """(DeviceCsr, was_host) for a host or device input."""
    if isinstance(m, DeviceCsr):
        return m, False
    if isinstance(m, CsrMatrix):
        return DeviceCsr.upload(m, stream), True
    raise TypeError(f"expected CsrMatrix or DeviceCsr, got {type(m).__name__}")


def _out(h: C.c_void_p, host: bool, stream):
    d = DeviceCsr(h.value)
    if not host:
        return d
    m = d.to_host(stream)
    d.free()
    return m


def build(t, kind, spec: N.DropSpec, stream=None, stats_out: list | None = None):
    """sait_build: the common entry of sait_thr / sait_pat / the fill cap."""
    dt, host = _dev(t, stream)
    h = C.c_void_p()
    st = N.BuildStats()
    N.check(N.lib.sait_build(dt.handle, _kind_lower(kind), C.byref(spec), _stream_handle(stream), C.byref(h), C.byref(st)))
    if stats_out is not None:
        stats_out.append(BuildStats(st.steps_run, bool(st.stabilized), st.nnz_out, st.products, st.seconds))
    return _out(h, host, stream)


def build_pair(lower, upper, spec: N.DropSpec, stream=None, stats_out: list | None = None):
    """sait_build_pair: M_L = build(lower) and M_U = build(upper) with the same
    drop spec, the two recursions running concurrently on the device."""
    dl, host_l = _dev(lower, stream)
    du, host_u = _dev(upper, stream)
    hl, hu = C.c_void_p(), C.c_void_p()
    st = (N.BuildStats * 2)()
    N.check(N.lib.sait_build_pair(dl.handle, du.handle, C.byref(spec), _stream_handle(stream), C.byref(hl), C.byref(hu),
                                  st))
    if stats_out is not None:
        for x in st:
            stats_out.append(BuildStats(x.steps_run, bool(x.stabilized), x.nnz_out, x.products, x.seconds))
    return _out(hl, host_l, stream), _out(hu, host_u, stream)


def sait_thr_pair(lower, upper, params: SaitThrParams, stream=None, stats_out=None):
    """sait_thr of both ILU factors (lower, upper) at once."""
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, float(params.threshold), int(params.steps), 0, 0, 0.0)
    return build_pair(lower, upper, spec, stream, stats_out)


def sait_thr(t, kind: TriangularKind, params: SaitThrParams, stream=None, stats_out=None):
    """sait.hpp:58 / sait.cpp:90-101"""
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD, float(params.threshold), int(params.steps), 0, 0, 0.0)
    return build(t, kind, spec, stream, stats_out)


def sait_pat(t, kind: TriangularKind, params: SaitPatParams, stream=None, stats_out=None):
    """sait.hpp:69 / sait.cpp:113-136"""
    spec = N.DropSpec(N.SAIT_DROP_PATTERN, 0.0, 0, int(params.pattern_steps), int(params.refine_steps), 0.0)
    return build(t, kind, spec, stream, stats_out)


def sait_thr_cap(t, kind: TriangularKind, params: SaitThrParams, cap_factor: float, stream=None, stats_out=None):
    """sait_thr with BASELINE config 4's per-column fill cap."""
    spec = N.DropSpec(N.SAIT_DROP_THRESHOLD_CAP, float(params.threshold), int(params.steps), 0, 0, float(cap_factor))
    return build(t, kind, spec, stream, stats_out)


def sait_polynomial_nodrop(t, kind: TriangularKind, steps: int, stream=None, stats_out=None):
    """sait_polynomial(split, steps, {}) followed by M D^-1 (sait.cpp:75-88)."""
    spec = N.DropSpec(N.SAIT_DROP_NONE, 0.0, int(steps), 0, 0, 0.0)
    return build(t, kind, spec, stream, stats_out)


def sait_polynomial(tt, steps: int, stream=None, stats_out=None):
    """sait.hpp:53 / sait.cpp:75-88 with an empty DropRule: the unit-diagonal
    recursion M <- tt M + I on the iteration matrix ``tt`` as given (any square
    matrix; a stored diagonal gets 1.0 added by add_identity), no scaling."""
    dt, host = _dev(tt, stream)
    h = C.c_void_p()
    st = N.BuildStats()
    N.check(N.lib.sait_polynomial(dt.handle, int(steps), _stream_handle(stream), C.byref(h), C.byref(st)))
    if stats_out is not None:
        stats_out.append(BuildStats(st.steps_run, bool(st.stabilized), st.nnz_out, st.products, st.seconds))
    return _out(h, host, stream)


def sait_pat_capture_pattern(t, kind: TriangularKind, pattern_steps: int, stream=None):
    """sait.hpp:64 / sait.cpp:103-111 (returns a pattern: values None)."""
    dt, host = _dev(t, stream)
    h = C.c_void_p()
    N.check(N.lib.sait_pat_capture_pattern(dt.handle, _kind_lower(kind), int(pattern_steps), _stream_handle(stream), C.byref(h)))
    return _out(h, host, stream)


@dataclass
class JacobiSplit:
    """sait.hpp:32-36"""

    inv_diag: np.ndarray
    iteration_matrix: CsrMatrix
    kind: TriangularKind


def jacobi_split(t: CsrMatrix, kind: TriangularKind, stream=None) -> JacobiSplit:
    """sait.hpp:40 / sait.cpp:32-73 (host in, host out)."""
    import torch

    dt, _ = _dev(t, stream)
    inv = torch.empty(max(t.nrows, 1), dtype=torch.float64, device="cuda")
    h = C.c_void_p()
    N.check(N.lib.sait_jacobi_split(dt.handle, _kind_lower(kind), inv.data_ptr(), _stream_handle(stream), C.byref(h)))
    tt = _out(h, True, stream)
    return JacobiSplit(inv[: t.nrows].cpu().numpy(), tt, kind)


# ------------------------------------------------------------ kernels.hpp

def _binary(fn, *handles_and_args, host, stream):
    h = C.c_void_p()
    N.check(fn(*handles_and_args, _stream_handle(stream), C.byref(h)))
    return _out(h, host, stream)


def spgemm(a, b, stream=None):
    """kernels.hpp:21 / kernels.cpp:34-102"""
    da, ha = _dev(a, stream)
    db, _ = _dev(b, stream)
    return _binary(N.lib.sait_spgemm, da.handle, db.handle, host=ha, stream=stream)


def add_identity(m, stream=None):
    """kernels.hpp:25 / kernels.cpp:104-134"""
    dm, hm = _dev(m, stream)
    return _binary(N.lib.sait_add_identity, dm.handle, host=hm, stream=stream)


def drop_by_threshold(m, tau: float, stream=None):
    """kernels.hpp:30 / kernels.cpp:136-160"""
    dm, hm = _dev(m, stream)
    return _binary(N.lib.sait_drop_by_threshold, dm.handle, C.c_double(tau), host=hm, stream=stream)


def drop_by_pattern(m, s, stream=None):
    """kernels.hpp:33 / kernels.cpp:162-194"""
    dm, hm = _dev(m, stream)
    if isinstance(s, CsrMatrix) and s.values is None:
        s = CsrMatrix(s.nrows, s.ncols, s.row_ptr, s.col_idx, np.zeros(s.nnz()))
    ds, _ = _dev(s, stream)
    return _binary(N.lib.sait_drop_by_pattern, dm.handle, ds.handle, host=hm, stream=stream)


def transpose(m, stream=None):
    """csr.hpp:84 / csr.cpp:72-92"""
    dm, hm = _dev(m, stream)
    return _binary(N.lib.sait_transpose, dm.handle, host=hm, stream=stream)


def scale_columns(m, d, stream=None):
    """kernels.hpp:40 / kernels.cpp:236-246"""
    import torch

    dm, hm = _dev(m, stream)
    dd = torch.as_tensor(np.ascontiguousarray(d, dtype=np.float64)).cuda() if not isinstance(d, torch.Tensor) else d
    return _binary(N.lib.sait_scale_columns, dm.handle, dd.data_ptr(), C.c_int64(dd.numel()), host=hm, stream=stream)


def spmv(a, x, y=None, stream=None):
    """kernels.hpp:14-15 / kernels.cpp:10-32.

    Host numpy x -> host numpy y (synchronous); torch CUDA tensors -> device
    call on ``stream`` (default: torch's current stream)."""
    import torch

    da, _ = _dev(a, stream)
    if isinstance(x, torch.Tensor) and x.is_cuda:
        if y is None:
            y = torch.empty(da.nrows, dtype=torch.float64, device=x.device)
        s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
        N.check(N.lib.sait_spmv(da.handle, x.data_ptr(), x.numel(), y.data_ptr(), y.numel(), s))
        return y
    xh = np.ascontiguousarray(x, dtype=np.float64)
    xd = torch.from_numpy(xh).cuda()
    yd = torch.empty(da.nrows if y is None else len(y), dtype=torch.float64, device="cuda")
    N.check(N.lib.sait_spmv(da.handle, xd.data_ptr(), xd.numel(), yd.data_ptr(), yd.numel(), None))
    out = yd.cpu().numpy()
    if y is not None:
        y[:] = out
        return y
    return out


def _vector_call(fn, da, x, out_len, stream, *args):
    """Run fn(da.handle, *args(x_ptr, y_ptr), stream) on CUDA tensors, or on
    host numpy via device copies (synchronous)."""
    import torch

    if isinstance(x, torch.Tensor) and x.is_cuda:
        y = torch.empty(out_len, dtype=torch.float64, device=x.device)
        s = _stream_handle(stream) if stream is not None else torch.cuda.current_stream().cuda_stream
        N.check(fn(x, y, s))
        return y
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    yd = torch.empty(out_len, dtype=torch.float64, device="cuda")
    N.check(fn(xd, yd, None))
    return yd.cpu().numpy()


def trisolve(t, kind: TriangularKind, b, stream=None):
    """kernels.hpp:36 / kernels.cpp:196-234: x = T^-1 b by substitution on the
    device (synchronization-free row scheduling), bitwise the reference's x."""
    dt, _ = _dev(t, stream)
    lower = int(_kind_lower(kind))
    return _vector_call(lambda x, y, s: N.lib.sait_trisolve(dt.handle, lower, x.data_ptr(), x.numel(), y.data_ptr(), s),
                        dt, b, dt.nrows, stream)


def jacobi_sweeps_apply(t, kind: TriangularKind, b, sweeps: int, stream=None):
    """sait.hpp:73 / sait.cpp:138-159: ``sweeps`` Jacobi sweeps on T x = b from 0."""
    dt, _ = _dev(t, stream)
    lower = int(_kind_lower(kind))
    return _vector_call(lambda x, y, s: N.lib.sait_jacobi_sweeps_apply(dt.handle, lower, x.data_ptr(), int(sweeps), y.data_ptr(), s),
                        dt, b, dt.nrows, stream)
