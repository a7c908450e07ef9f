"""Host and device CSR types (mirror of csr.hpp:12-98).

``CsrMatrix`` is the reference's host value type (int64 ``row_ptr`` /
``col_idx``, fp64 ``values``); ``DeviceCsr`` owns a matrix resident on the
GPU (int32 indices, fp64 values) behind a ``sait_dcsr_t`` handle.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N


@dataclass(frozen=True)
class TriangularKind:
    """csr.hpp:64-73.  Unit diagonals are stored explicitly."""

    side: str = "lower"  # "lower" | "upper"
    unit_diagonal: bool = False

    @property
    def lower(self) -> bool:
        return self.side == "lower"


lower_triangular = TriangularKind("lower", False)
unit_lower_triangular = TriangularKind("lower", True)
upper_triangular = TriangularKind("upper", False)
unit_upper_triangular = TriangularKind("upper", True)


def _kind_lower(kind) -> int:
    if isinstance(kind, TriangularKind):
        return int(kind.lower)
    if kind in ("lower", "upper"):
        return int(kind == "lower")
    return int(bool(kind))


@dataclass(eq=False)
class CsrMatrix:
    """Compressed sparse row matrix, reference layout (csr.hpp:24-43)."""

    nrows: int = 0
    ncols: int = 0
    row_ptr: np.ndarray = field(default_factory=lambda: np.zeros(1, dtype=np.int64))
    col_idx: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.int64))
    values: np.ndarray | None = field(default_factory=lambda: np.zeros(0, dtype=np.float64))

    def __post_init__(self):
        self.nrows, self.ncols = int(self.nrows), int(self.ncols)
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        if self.values is not None:
            self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0

    def row_cols(self, i: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[i] : self.row_ptr[i + 1]]

    def row_vals(self, i: int) -> np.ndarray:
        return self.values[self.row_ptr[i] : self.row_ptr[i + 1]]

    def __eq__(self, other) -> bool:  # defaulted operator== (csr.hpp:42): elementwise ==
        if not isinstance(other, CsrMatrix):
            return NotImplemented
        if (self.nrows, self.ncols) != (other.nrows, other.ncols):
            return False
        if not (np.array_equal(self.row_ptr, other.row_ptr) and np.array_equal(self.col_idx, other.col_idx)):
            return False
        if self.values is None or other.values is None:
            return self.values is None and other.values is None
        return bool(np.array_equal(self.values, other.values))

    def bitwise_equal(self, other: "CsrMatrix") -> bool:
        if not self.same_pattern(other):
            return False
        if self.values is None or other.values is None:
            return self.values is None and other.values is None
        return bool(np.array_equal(self.values.view(np.uint64), other.values.view(np.uint64)))

    def same_pattern(self, other: "CsrMatrix") -> bool:
        return (
            (self.nrows, self.ncols) == (other.nrows, other.ncols)
            and np.array_equal(self.row_ptr, other.row_ptr)
            and np.array_equal(self.col_idx, other.col_idx)
        )

    def pattern(self) -> "CsrMatrix":
        """pattern_of (csr.cpp:141-148): positions only."""
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr.copy(), self.col_idx.copy(), None)

    def to_scipy(self):
        import scipy.sparse as sp

        vals = self.values if self.values is not None else np.ones(self.nnz())
        return sp.csr_matrix((vals, self.col_idx, self.row_ptr), shape=(self.nrows, self.ncols))

    @staticmethod
    def from_scipy(m) -> "CsrMatrix":
        m = m.tocsr()
        m.sort_indices()
        return CsrMatrix(m.shape[0], m.shape[1], m.indptr, m.indices, m.data)

    # ---- ctypes plumbing
    def _as_c(self) -> N.HostCsr:
        c = N.HostCsr()
        c.nrows, c.ncols = self.nrows, self.ncols
        c.row_ptr = self.row_ptr.ctypes.data_as(N.P64)
        c.col_idx = self.col_idx.ctypes.data_as(N.P64)
        c.values = self.values.ctypes.data_as(N.PD) if self.values is not None else N.PD()
        return c


SparsityPattern = CsrMatrix  # a CsrMatrix with values=None (csr.hpp:46-60)


def _from_c(c: N.HostCsr) -> CsrMatrix:
    """Copy a library-filled HostCsr into numpy and release it."""
    n = c.nrows
    rp = np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)).copy()
    nnz = int(rp[-1])
    ci = np.ctypeslib.as_array(c.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    vals = np.ctypeslib.as_array(c.values, shape=(max(nnz, 1),))[:nnz].copy() if bool(c.values) else None
    N.lib.sait_host_csr_free(C.byref(c))
    return CsrMatrix(int(c.nrows), int(c.ncols), rp, ci, vals)


def _stream_handle(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(getattr(stream, "cuda_stream", stream))


class DeviceCsr:
    """A CSR matrix resident on the current GPU (int32 indices, fp64 values)."""

    __slots__ = ("_h", "nrows", "ncols", "_owned")

    def __init__(self, handle: int, owned: bool = True):
        self._h = C.c_void_p(handle)
        self._owned = owned
        nr, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        N.check(N.lib.sait_csr_info(self._h, C.byref(nr), C.byref(nc), C.byref(nz)))
        self.nrows, self.ncols = nr.value, nc.value

    @classmethod
    def upload(cls, m: CsrMatrix, stream=None) -> "DeviceCsr":
        h = C.c_void_p()
        N.check(N.lib.sait_csr_upload(C.byref(m._as_c()), _stream_handle(stream), C.byref(h)))
        return cls(h.value)

    def nnz(self) -> int:
        nz = C.c_int64()
        N.check(N.lib.sait_csr_info(self._h, None, None, C.byref(nz)))
        return nz.value

    def to_host(self, stream=None) -> CsrMatrix:
        """Download into freshly allocated int64 / fp64 arrays (sait_csr_download:
        pinned, chunked, widened on the host cores)."""
        nz = self.nnz()
        vp = C.c_void_p()
        N.check(N.lib.sait_csr_device_arrays(self._h, None, None, C.byref(vp)))
        rp = np.empty(self.nrows + 1, dtype=np.int64)
        ci = np.empty(nz, dtype=np.int64)
        vals = np.empty(nz, dtype=np.float64) if vp.value else None
        N.check(N.lib.sait_csr_download(self._h, rp.ctypes.data_as(N.P64), ci.ctypes.data_as(N.P64),
                                        vals.ctypes.data_as(N.PD) if vals is not None else N.PD(),
                                        _stream_handle(stream)))
        return CsrMatrix(self.nrows, self.ncols, rp, ci, vals)

    def device_arrays(self):
        """(row_ptr, col_idx, values) device pointers (int32, int32, fp64)."""
        rp, ci, v = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(N.lib.sait_csr_device_arrays(self._h, C.byref(rp), C.byref(ci), C.byref(v)))
        return rp.value, ci.value, v.value

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def release(self) -> C.c_void_p:
        """Hand ownership of the handle to the caller (e.g. a pair)."""
        self._owned = False
        return self._h

    def free(self) -> None:
        if self._owned and self._h:
            N.lib.sait_csr_free(self._h)
        self._h = C.c_void_p()
        self._owned = False

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
