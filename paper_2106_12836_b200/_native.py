"""ctypes binding of the C ABI (include/sait_c.h) exported by libsait_b200.so.

The shared library is built in-tree (``make`` / ``__graft_entry__.build()``).
There is no fallback: if the library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SAIT_CHECKED=1 loads the bounds-checked build (make checked: every device
# index the kernels derive is range-checked and traps with a message) --
# the stand-in for compute-sanitizer, which this GPU pool does not allow.
# SAIT_LIB_VARIANT=<subdir> loads an experimental build from that subdirectory
# (kernel A/B measurements, tools/*_time.py).
_sub = "checked" if os.environ.get("SAIT_CHECKED") == "1" else os.environ.get("SAIT_LIB_VARIANT", "")
LIB_PATH = os.path.join(HERE, _sub, "libsait_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first (make, or __graft_entry__.build()); "
        "there is no CPU fallback"
    )

lib = C.CDLL(LIB_PATH)

SAIT_OK = 0
SAIT_ERR_INVALID_ARGUMENT = 1
SAIT_ERR_RUNTIME = 2
SAIT_ERR_CUDA = 3
SAIT_ERR_NOMEM = 4

SAIT_DROP_THRESHOLD = 1
SAIT_DROP_PATTERN = 2
SAIT_DROP_THRESHOLD_CAP = 3
SAIT_DROP_NONE = 4

P64 = C.POINTER(C.c_int64)
PD = C.POINTER(C.c_double)
VP = C.c_void_p


class Halo(C.Structure):
    """sait_halo_t"""

    _fields_ = [
        ("own_lo", C.c_int64),
        ("own_hi", C.c_int64),
        ("lo_src", C.c_void_p),
        ("lo_shift", C.c_int64),
        ("hi_src", C.c_void_p),
        ("hi_shift", C.c_int64),
        ("lo_flag", C.c_void_p),
        ("hi_flag", C.c_void_p),
        ("epoch", C.c_int),
    ]


class FactorFormat(C.Structure):
    """sait_factor_format (include/sait_c.h)"""

    _fields_ = [("format", C.c_int), ("row_sorted", C.c_int), ("nrows", C.c_int64), ("nnz", C.c_int64),
                ("stored_slots", C.c_int64), ("nslices", C.c_int64), ("dict_elems", C.c_int64),
                ("stream_bytes", C.c_int64)]


SAIT_FMT_AUTO, SAIT_FMT_CSR, SAIT_FMT_SELL_I32, SAIT_FMT_SELL_I16, SAIT_FMT_SELL_DICT = range(5)
FORMAT_NAMES = {0: "auto", 1: "csr", 2: "sell32_int32", 3: "sell32_int16", 4: "sell32_dict"}


class RowPiece(C.Structure):
    """sait_row_piece (include/sait_c.h)"""

    _fields_ = [("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p), ("col_offset", C.c_int64)]


class PeerFactorDesc(C.Structure):
    """sait_peer_factor_desc (include/sait_c.h)"""

    _fields_ = [("ext", C.c_void_p * 2), ("flag", C.c_void_p), ("ext_len", C.c_int64), ("own_offset", C.c_int64),
                ("own_len", C.c_int64), ("send_a0", C.c_int64), ("send_n0", C.c_int64), ("send_a1", C.c_int64),
                ("send_n1", C.c_int64), ("halo", Halo * 2)]


class HostCsr(C.Structure):
    _fields_ = [
        ("nrows", C.c_int64),
        ("ncols", C.c_int64),
        ("row_ptr", P64),
        ("col_idx", P64),
        ("values", PD),
    ]


class DropSpec(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("tau", C.c_double),
        ("steps", C.c_int),
        ("pattern_steps", C.c_int),
        ("refine_steps", C.c_int),
        ("cap_factor", C.c_double),
    ]


class BuildStats(C.Structure):
    _fields_ = [
        ("steps_run", C.c_int),
        ("stabilized", C.c_int),
        ("nnz_out", C.c_int64),
        ("products", C.c_int64),
        ("seconds", C.c_double),
    ]


class SolveStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("relres_estimate", C.c_double),
        ("true_relres", C.c_double),
        ("seconds", C.c_double),
        ("precond_seconds", C.c_double),
        ("precond_applies", C.c_int64),
    ]


# Every symbol include/sait_c.h declares, with its prototype.
PROTOTYPES = {
    "sait_last_error": (C.c_char_p, []),
    "sait_abi_version": (C.c_int, []),
    "sait_host_csr_free": (None, [C.POINTER(HostCsr)]),
    "sait_csr_upload": (C.c_int, [C.POINTER(HostCsr), VP, C.POINTER(VP)]),
    "sait_csr_info": (C.c_int, [VP, P64, P64, P64]),
    "sait_csr_download": (C.c_int, [VP, P64, P64, PD, VP]),
    "sait_csr_to_host": (C.c_int, [VP, VP, C.POINTER(HostCsr)]),
    "sait_csr_device_arrays": (C.c_int, [VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(VP)]),
    "sait_csr_free": (None, [VP]),
    "sait_lobpcg_opt": (C.c_int, [VP, VP, C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_int, PD, VP, PD,
                                  C.POINTER(C.c_int), C.POINTER(SolveStats), VP]),
    "sait_spmm": (C.c_int, [VP, VP, VP, C.c_int64, VP]),
    "sait_lobpcg_ex": (C.c_int, [VP, VP, C.c_int, C.c_double, C.c_int, C.c_uint64, PD, VP, PD, C.POINTER(C.c_int),
                                 C.POINTER(SolveStats), VP]),
    "sait_peer_pair_create": (C.c_int, [VP, VP, C.POINTER(PeerFactorDesc), C.POINTER(VP)]),
    "sait_peer_pair_apply": (C.c_int, [VP, VP, VP, VP]),
    "sait_peer_pair_destroy": (None, [VP]),
    "sait_csr_assemble_rows": (C.c_int, [C.c_int, C.POINTER(RowPiece), C.c_int64, C.c_int64, VP, C.POINTER(VP)]),
    "sait_csr_col_span": (C.c_int, [VP, P64, P64, VP]),
    "sait_csr_shift_cols": (C.c_int, [VP, C.c_int64, C.c_int64, VP]),
    "sait_csr_row_ptr_at": (C.c_int, [VP, P64, C.c_int, P64, VP]),
    "sait_column_work": (C.c_int, [VP, VP, VP]),
    "sait_spmv": (C.c_int, [VP, VP, C.c_int64, VP, C.c_int64, VP]),
    "sait_spgemm": (C.c_int, [VP, VP, VP, C.POINTER(VP)]),
    "sait_add_identity": (C.c_int, [VP, VP, C.POINTER(VP)]),
    "sait_drop_by_threshold": (C.c_int, [VP, C.c_double, VP, C.POINTER(VP)]),
    "sait_drop_by_pattern": (C.c_int, [VP, VP, VP, C.POINTER(VP)]),
    "sait_scale_columns": (C.c_int, [VP, VP, C.c_int64, VP, C.POINTER(VP)]),
    "sait_transpose": (C.c_int, [VP, VP, C.POINTER(VP)]),
    "sait_build_session_create": (C.c_int, [VP, C.c_int, C.POINTER(DropSpec), C.c_int64, C.c_int64, VP, C.POINTER(VP)]),
    "sait_build_session_remaining": (C.c_int, [VP]),
    "sait_build_session_step": (C.c_int, [VP, C.POINTER(C.c_int)]),
    "sait_build_session_stop": (C.c_int, [VP]),
    "sait_build_session_finish": (C.c_int, [VP, C.c_int, C.POINTER(VP), C.POINTER(BuildStats)]),
    "sait_build_session_destroy": (None, [VP]),
    "sait_operator_create": (C.c_int, [VP, C.c_int, C.POINTER(VP)]),
    "sait_operator_apply": (C.c_int, [VP, VP, C.c_int64, VP, C.c_int64, VP]),
    "sait_operator_destroy": (None, [VP]),
    "sait_operator_apply_halo": (C.c_int, [VP, VP, C.c_int64, C.POINTER(Halo), VP, C.c_int64, VP]),
    "sait_publish_epoch": (C.c_int, [VP, C.c_int, VP]),
    "sait_ipc_handle": (C.c_int, [VP, VP]),
    "sait_ipc_open": (C.c_int, [VP, C.POINTER(VP)]),
    "sait_ipc_close": (C.c_int, [VP]),
    "sait_jacobi_split": (C.c_int, [VP, C.c_int, VP, VP, C.POINTER(VP)]),
    "sait_build_pair": (C.c_int, [VP, VP, C.POINTER(DropSpec), VP, C.POINTER(VP), C.POINTER(VP), C.POINTER(BuildStats)]),
    "sait_build": (C.c_int, [VP, C.c_int, C.POINTER(DropSpec), VP, C.POINTER(VP), C.POINTER(BuildStats)]),
    "sait_polynomial": (C.c_int, [VP, C.c_int, VP, C.POINTER(VP), C.POINTER(BuildStats)]),
    "sait_pat_capture_pattern": (C.c_int, [VP, C.c_int, C.c_int, VP, C.POINTER(VP)]),
    "sait_jacobi_sweeps_apply": (C.c_int, [VP, C.c_int, VP, C.c_int, VP, VP]),
    "sait_mm_read": (C.c_int, [C.c_char_p, C.POINTER(HostCsr)]),
    "sait_mm_write": (C.c_int, [C.c_char_p, C.POINTER(HostCsr)]),
    "sait_make_rhs": (C.c_int, [C.POINTER(HostCsr), C.c_int, C.c_uint64, VP]),
    "sait_ilu0": (C.c_int, [VP, VP, C.POINTER(VP), C.POINTER(VP)]),
    "sait_ilu_device": (C.c_int, [VP, C.c_int, VP, C.POINTER(VP), C.POINTER(VP)]),
    "sait_trisolve": (C.c_int, [VP, C.c_int, VP, C.c_int64, VP, VP]),
    "sait_exact_ilu_create": (C.c_int, [VP, VP, C.c_int, C.POINTER(VP)]),
    "sait_exact_ilu_info": (C.c_int, [VP, P64, P64]),
    "sait_exact_ilu_apply": (C.c_int, [VP, VP, C.c_int64, VP, C.c_int64, VP]),
    "sait_exact_ilu_destroy": (None, [VP]),
    "sait_pair_create": (C.c_int, [VP, VP, C.c_int, C.POINTER(VP)]),
    "sait_pair_create_ex": (C.c_int, [VP, VP, C.c_int, C.c_int, C.POINTER(VP)]),
    "sait_pair_format": (C.c_int, [VP, C.c_int, C.POINTER(FactorFormat)]),
    "sait_pair_info": (C.c_int, [VP, P64, P64]),
    "sait_pair_apply": (C.c_int, [VP, VP, C.c_int64, VP, C.c_int64, VP]),
    "sait_pair_apply_host": (C.c_int, [VP, PD, C.c_int64, PD, C.c_int64, VP]),
    "sait_pair_apply_block": (C.c_int, [VP, VP, VP, C.c_int64, C.c_int64, C.c_int, VP]),
    "sait_pair_apply_block_host": (C.c_int, [VP, PD, PD, C.c_int64, C.c_int64, C.c_int, VP]),
    "sait_pair_spmv_factor": (C.c_int, [VP, C.c_int, VP, VP, VP]),
    "sait_pair_factors": (C.c_int, [VP, C.POINTER(VP), C.POINTER(VP)]),
    "sait_pair_destroy": (None, [VP]),
    "sait_gmres": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_int, C.c_double, C.c_int, PD, C.POINTER(SolveStats), VP]),
    "sait_pcg": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_double, C.c_int, PD, C.POINTER(SolveStats), VP]),
    "sait_gmres_exact": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_int, C.c_double, C.c_int, PD, C.POINTER(SolveStats), VP]),
    "sait_dot_blocks": (C.c_int64, [C.c_int64]),
    "sait_dot_partials": (C.c_int, [VP, VP, C.c_int64, C.c_int, C.c_int64, VP, VP]),
    "sait_dot_fold": (C.c_int, [VP, C.c_int64, C.c_int, VP, C.c_int, VP]),
    "sait_vec_update": (C.c_int, [C.c_int, C.c_int64, C.c_double, VP, VP, VP]),
    "sait_vec_cgs": (C.c_int, [C.c_int64, VP, VP, C.c_int64, C.c_int, VP, VP]),
    "sait_vec_div": (C.c_int, [C.c_int64, VP, VP, VP, VP]),
    "sait_vec_lincomb": (C.c_int, [C.c_int64, VP, C.c_int64, C.c_int, VP, VP, VP]),
    "sait_gram_partials": (C.c_int, [VP, C.c_int, VP, C.c_int, C.c_int64, VP, VP]),
    "sait_block_lincomb": (C.c_int, [C.c_int64, VP, C.c_int, VP, C.c_int, VP, VP]),
    "sait_block_sub_lincomb": (C.c_int, [C.c_int64, VP, C.c_int, VP, VP, VP]),
    "sait_block_residual": (C.c_int, [C.c_int64, C.c_int, VP, VP, VP, VP, VP]),
    "sait_fill_uniform_pm1_device": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, VP, VP]),
    "sait_dense_chol_lower": (C.c_int, [PD, C.c_int, PD]),
    "sait_dense_tri_lower_inv": (None, [PD, C.c_int, PD]),
    "sait_dense_rayleigh_ritz": (C.c_int, [PD, PD, C.c_int, C.c_int, PD, PD]),
    "sait_pcg_exact": (C.c_int, [VP, VP, VP, VP, C.c_int64, C.c_double, C.c_int, PD, C.POINTER(SolveStats), VP]),
    "sait_lobpcg": (C.c_int, [VP, VP, C.c_int, C.c_double, C.c_int, C.c_uint64, PD, VP, PD, C.POINTER(C.c_int), VP]),
    "sait_lobpcg_exact": (C.c_int, [VP, VP, C.c_int, C.c_double, C.c_int, C.c_uint64, PD, VP, PD, C.POINTER(C.c_int), VP]),
    "sait_ilu_k": (C.c_int, [C.POINTER(HostCsr), C.c_int, C.POINTER(HostCsr), C.POINTER(HostCsr)]),
    "sait_problem_laplacian_2d": (C.c_int, [C.c_int64, C.POINTER(HostCsr)]),
    "sait_problem_laplacian_3d": (C.c_int, [C.c_int64, C.POINTER(HostCsr)]),
    "sait_problem_convdiff_2d": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.POINTER(HostCsr)]),
    "sait_problem_synthetic_lower": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.POINTER(HostCsr)]),
    "sait_fill_uniform_pm1": (None, [C.c_uint64, C.c_int64, PD]),
    "sait_device_synchronize": (C.c_int, []),
    "sait_device_alloc": (C.c_int, [C.c_size_t, C.POINTER(VP)]),
    "sait_device_free": (None, [VP]),
    "sait_memcpy": (C.c_int, [VP, VP, C.c_size_t, C.c_int]),
    "sait_stream_create": (C.c_int, [C.POINTER(VP)]),
    "sait_stream_destroy": (None, [VP]),
    "sait_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(VP)]),
    "sait_host_free": (None, [VP]),
    "sait_kernel_launch_count": (C.c_int64, []),
    "sait_device_pool_reserve": (C.c_int, [C.c_int, C.c_int64]),
}

for _name, (_res, _args) in PROTOTYPES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class SaitError(Exception):
    code = -1


class SaitInvalidArgument(SaitError, ValueError):
    """std::invalid_argument in the reference."""

    code = SAIT_ERR_INVALID_ARGUMENT


class SaitRuntimeError(SaitError, RuntimeError):
    """std::runtime_error in the reference."""

    code = SAIT_ERR_RUNTIME


class SaitCudaError(SaitError, RuntimeError):
    code = SAIT_ERR_CUDA


class SaitOutOfMemory(SaitError, MemoryError):
    code = SAIT_ERR_NOMEM


_EXC = {
    SAIT_ERR_INVALID_ARGUMENT: SaitInvalidArgument,
    SAIT_ERR_RUNTIME: SaitRuntimeError,
    SAIT_ERR_CUDA: SaitCudaError,
    SAIT_ERR_NOMEM: SaitOutOfMemory,
}


def check(rc: int) -> None:
    if rc != SAIT_OK:
        msg = lib.sait_last_error().decode()
        raise _EXC.get(rc, SaitError)(msg)


def launch_count() -> int:
    return int(lib.sait_kernel_launch_count())


def reserve_device_pool(nbytes: int, device: int | None = None) -> None:
    """sait_device_pool_reserve: grow the library's device pool up front."""
    if device is None:
        import torch

        device = torch.cuda.current_device()
    check(lib.sait_device_pool_reserve(int(device), int(nbytes)))
