"""Time the comparator preconditioners on the device at BASELINE config 2
(128^3 Laplacian, ILU(0)): ExactIlu (two synchronization-free trisolves),
JacobiSweeps(k), and the SAIT pair (tau=5e-2, k=3), device vectors.

    python tools/prof_exact.py [n]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    A = S.laplacian_3d(n)
    t0 = time.perf_counter()
    f = S.ilu_k(A, 0)
    s_host_ilu = time.perf_counter() - t0
    Ad = S.DeviceCsr.upload(A)
    ms_dev_ilu = timed(lambda: S.ilu0_device(Ad), 3)
    N = A.nrows
    r = torch.from_numpy(S.uniform_pm1(1000, N)).cuda()
    z = torch.empty_like(r)
    E = S.ExactIluPreconditioner(f)
    ms_exact = timed(lambda: E.apply(r, z), 10)
    ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
    MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
    P = S.SaitPairPreconditioner(ML, MU)
    ms_pair = timed(lambda: P.apply(r, z), 50)
    J = S.JacobiSweepsPreconditioner(f, 3)
    ms_jac = timed(lambda: J.apply(r, z), 10)
    # single triangular solve, L only
    Ld = S.DeviceCsr.upload(f.lower)
    y = torch.empty_like(r)
    ms_l = timed(lambda: S.trisolve(Ld, S.unit_lower_triangular, r), 10)
    t0 = time.perf_counter()
    E.apply(r, z)
    torch.cuda.synchronize()
    print(f"n={n}^3 rows={N} nnz(L+U)={E.nnz()} nnz(ML+MU)={P.nnz()}")
    print(f"ilu(0) host       {s_host_ilu * 1e3:8.1f} ms   device {ms_dev_ilu:8.2f} ms")
    print(f"exact ilu apply   {ms_exact:8.3f} ms  ({8 * 2 * E.nnz() / ms_exact / 1e6:.1f} GB/s of CSR values+idx est.)")
    print(f"trisolve L only   {ms_l:8.3f} ms")
    print(f"jacobi sweeps(3)  {ms_jac:8.3f} ms")
    print(f"sait pair apply   {ms_pair:8.3f} ms   speedup over exact {ms_exact / ms_pair:.1f}x")
    del y


if __name__ == "__main__":
    main()
