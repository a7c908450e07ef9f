"""Run BASELINE.json configs 1, 3, 4, 5 at full size on one GPU and print a
JSON line per config (setup, build, solve).  Usage:
  python tools/run_configs.py [c1 c3 c4 c5] [--c5-maxit N]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402


def log(d):
    print(json.dumps(d), flush=True)


def build_pair(A, tau, k):
    """ILU(0) on the device (F1, bitwise the reference's factors), then the
    two SAIT builds; --host-ilu also times the host ilu_k for comparison."""
    dA = S.DeviceCsr.upload(A)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = S.ilu0_device(dA)
    torch.cuda.synchronize()
    t_ilu = time.perf_counter() - t0
    extra = {}
    if "--host-ilu" in sys.argv:
        t0 = time.perf_counter()
        S.ilu_k(A, 0)
        extra["ilu_host_s"] = time.perf_counter() - t0
    st = []
    L, U = f.lower, f.upper
    ML = S.sait_thr(L, S.lower_triangular, S.SaitThrParams(tau, k), stats_out=st)
    MU = S.sait_thr(U, S.upper_triangular, S.SaitThrParams(tau, k), stats_out=st)
    info = {"ilu_device_s": t_ilu, **extra, "nnz_L": L.nnz(), "nnz_U": U.nnz(), "nnz_ML": ML.nnz(), "nnz_MU": MU.nnz(),
            "build_s": st[0].seconds + st[1].seconds, "steps": [st[0].steps_run, st[1].steps_run],
            "built_nnz_per_s": (ML.nnz() + MU.nnz()) / (st[0].seconds + st[1].seconds)}
    return S.SaitPairPreconditioner(ML, MU), info


def gmres_cfg(name, A, tau, k, seed):
    pair, info = build_pair(A, tau, k)
    b = torch.from_numpy(S.uniform_pm1(seed, A.nrows)).cuda()
    dA = S.DeviceCsr.upload(A)
    x, st = S.gmres(dA, pair, b, 30, 1e-8, 20000)
    info.update({"config": name, "n": A.nrows, "nnz_A": A.nnz(), "gmres_iters": st.iterations,
                 "converged": st.converged, "true_relres": st.true_relres, "solve_s": st.seconds})
    log(info)


def main():
    which = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c1", "c3", "c4", "c5"]
    if "c1" in which:
        gmres_cfg("c1", S.laplacian_2d(64), 1e-2, 4, 1)
    if "c3" in which:
        t0 = time.perf_counter()
        A = S.convdiff_2d(2048, 20.0, -10.0)
        gen = time.perf_counter() - t0
        gmres_cfg("c3", A, 2e-2, 4, 3)
        log({"c3_generate_s": gen})
    if "c4" in which:
        t0 = time.perf_counter()
        T = S.synthetic_lower(16777216, 15, 0.01, 4)
        gen = time.perf_counter() - t0
        dT = S.DeviceCsr.upload(T)
        for cap in (None, 3.0):
            secs = []
            for rep in range(4):  # one warm-up build (pool growth), then the median of 3
                st = []
                if cap is None:
                    M = S.sait_thr(dT, S.lower_triangular, S.SaitThrParams(1e-2, 3), stats_out=st)
                else:
                    M = S.sait_thr_cap(dT, S.lower_triangular, S.SaitThrParams(1e-2, 3), cap, stats_out=st)
                if rep:
                    secs.append(st[0].seconds)
                if rep < 3:
                    M.free()
            t_b = sorted(secs)[1]
            log({"config": "c4", "cap": cap, "n": T.nrows, "nnz_T": T.nnz(), "generate_s": gen, "nnz_M": M.nnz(),
                 "ratio": M.nnz() / T.nnz(), "build_s": t_b, "build_samples_s": secs, "steps": st[0].steps_run,
                 "products": st[0].products, "built_nnz_per_s": M.nnz() / t_b})
            M.free()
    if "c5" in which:
        maxit = 2000
        for a in sys.argv:
            if a.startswith("--c5-maxit="):
                maxit = int(a.split("=")[1])
        A = S.laplacian_3d(256)
        pair, info = build_pair(A, 5e-2, 3)
        dA = S.DeviceCsr.upload(A)
        t0 = time.perf_counter()
        gram = os.environ.get("SAIT_LOBPCG_GRAM", "canonical")
        r = S.lobpcg(dA, pair, 8, 1e-6, maxit, 5, host_vectors=False, gram=gram)
        m = 256
        h = 1.0 / (m + 1)
        sn = np.sin(np.pi * np.arange(1, m + 1) * h / 2) ** 2
        lam = np.sort((4 * (sn[:, None, None] + sn[None, :, None] + sn[None, None, :])).ravel())[:8]
        info.update({"config": "c5", "gram": gram, "n": A.nrows, "lobpcg_iters": r.iterations, "lobpcg_s": time.perf_counter() - t0,
                     "final_resnorm_max": float(r.residual_history[-1].max()),
                     "eig_rel_err_max": float(np.max(np.abs(r.eigenvalues - lam) / lam))})
        log(info)


if __name__ == "__main__":
    main()
