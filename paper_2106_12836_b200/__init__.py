"""B200-native SAIT: sparse approximate inverses of triangular (ILU) factors
from the truncated Jacobi series, built and applied by hand-written sm_100a
kernels (libsait_b200.so, C ABI in include/sait_c.h).

Python surface mirrors the reference's saitprec:: C++ API
(/root/reference/proj/core/include/saitprec/*.hpp).  There is no CPU
fallback: importing this package fails if the CUDA library is not built.
"""
from . import _native  # noqa: F401  (raises ImportError if the .so is missing)
from ._native import (
    SaitCudaError,
    SaitError,
    SaitInvalidArgument,
    SaitOutOfMemory,
    SaitRuntimeError,
    launch_count,
    reserve_device_pool,
)
from .csr import (
    CsrMatrix,
    DeviceCsr,
    SparsityPattern,
    TriangularKind,
    lower_triangular,
    unit_lower_triangular,
    unit_upper_triangular,
    upper_triangular,
)
from .preconditioner import (
    ExactIluPreconditioner,
    IdentityPreconditioner,
    JacobiSweepsPreconditioner,
    Preconditioner,
    SaitPairPreconditioner,
    apply_precond,
)
from .problems import (
    IluFactors,
    convdiff_2d,
    ilu0_device,
    ilu_device,
    ilu_k,
    laplacian_2d,
    laplacian_3d,
    make_rhs,
    mm_read,
    mm_write,
    synthetic_lower,
    uniform_pm1,
)
from .solvers import EigResult, SolveStats, gmres, lobpcg, pcg
from .sait import (
    BuildStats,
    JacobiSplit,
    SaitPatParams,
    SaitThrParams,
    add_identity,
    build,
    drop_by_pattern,
    drop_by_threshold,
    jacobi_split,
    sait_pat,
    sait_pat_capture_pattern,
    sait_polynomial,
    sait_polynomial_nodrop,
    sait_thr,
    sait_thr_cap,
    sait_thr_pair,
    build_pair,
    scale_columns,
    spgemm,
    spmv,
    transpose,
    trisolve,
    jacobi_sweeps_apply,
)

__all__ = [n for n in dir() if not n.startswith("_")]
