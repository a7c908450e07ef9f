"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Run in the build container (where /root/reference exists and oracle/Makefile
has built oracle/_ref/libsaitref.so from the unmodified reference sources):

    make -C oracle && python tests/golden/make_golden.py

Every matrix below is produced by the reference's own saitprec:: functions
(sait_thr, sait_pat, sait_pat_capture_pattern, ilu_k, trisolve,
jacobi_sweeps_apply, SaitPairPreconditioner::apply / apply_block) through oracle/ref_wrapper.cpp.  Inputs come from the
oracle's seeded generators (oracle/sait_oracle.c), which the reference lacks
(SPEC.md:353-408 is spec-only).  The fixtures travel with the repo; the GPU
box never needs /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle as O  # noqa: E402


def put(store, key, m):
    store[key + "/shape"] = np.array([m.nrows, m.ncols], dtype=np.int64)
    store[key + "/row_ptr"] = m.row_ptr
    store[key + "/col_idx"] = m.col_idx
    if m.values is not None:
        store[key + "/values"] = m.values


THR_CASES = [(0.0, 1), (0.0, 5), (0.01, 3), (0.05, 10), (0.2, 4), (0.0, 250)]
PAT_CASES = [(0, 1), (1, 3), (2, 2), (3, 5)]
CAP_CASES = [(0.01, 3, 3.0), (0.0, 4, 1.5), (0.05, 6, 1.0)]


def small_inputs():
    lo = O.synthetic_lower(200, 6, 0.05, seed=11)
    up = O.get("port").transpose(O.synthetic_lower(200, 6, 0.05, seed=12))
    return {"syn_lower": (lo, True), "syn_upper": (up, False)}


def main():
    R = O.get("reference")
    store = {}
    # 1. small seeded triangular matrices, every drop rule
    for name, (t, lower) in small_inputs().items():
        put(store, f"{name}/T", t)
        for tau, k in THR_CASES:
            put(store, f"{name}/thr_{tau}_{k}", R.sait_thr(t, lower, tau, k))
        for p, m in PAT_CASES:
            put(store, f"{name}/pat_{p}_{m}", R.sait_pat(t, lower, p, m))
            put(store, f"{name}/patcap_{p}", R.sait_pat_capture_pattern(t, lower, p))
        for tau, k, f in CAP_CASES:
            put(store, f"{name}/cap_{tau}_{k}_{f}", R.sait_thr_cap(t, lower, tau, k, f))
        b = O.uniform_pm1(77, t.nrows)
        store[f"{name}/b"] = b
        store[f"{name}/x_tri"] = R.trisolve(t, lower, b)  # kernels.cpp:196-234
    # 2. BASELINE config 1: 64x64 Poisson, ILU(0), SAIT tau=1e-2 k=4, r ~ U[-1,1] seed 1
    A = O.laplacian_2d(64)
    L, U = R.ilu_k(A, 0)
    ML = R.sait_thr(L, True, 1e-2, 4)
    MU = R.sait_thr(U, False, 1e-2, 4)
    r = O.uniform_pm1(1, A.nrows)
    put(store, "c1/A", A)
    put(store, "c1/L", L)
    put(store, "c1/U", U)
    put(store, "c1/ML", ML)
    put(store, "c1/MU", MU)
    store["c1/r"] = r
    store["c1/z"] = R.pair_apply(ML, MU, r)
    # ExactIluPreconditioner (preconditioner.cpp:28-32) and
    # JacobiSweepsPreconditioner with 3 sweeps (preconditioner.cpp:58-63)
    store["c1/z_exact"] = R.trisolve(U, False, R.trisolve(L, True, r))
    store["c1/z_jacobi3"] = R.jacobi_sweeps_apply(U, False, R.jacobi_sweeps_apply(L, True, r, 3), 3)
    blk = np.stack([O.uniform_pm1(500 + c, A.nrows) for c in range(8)], axis=1)
    store["c1/R8"] = blk
    store["c1/Z8"] = R.pair_apply_block(ML, MU, blk)
    # ILU(1) of a small 3D Laplacian (pins the level-of-fill restatement)
    A3 = O.laplacian_3d(12)
    L1, U1 = R.ilu_k(A3, 1)
    put(store, "lap12/L1", L1)
    put(store, "lap12/U1", U1)
    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **store)

    # 3. the paper's nnz-ratio table on the 100^3 Laplacian,
    #    reproduced by the reference: exact nnz counts per factor.
    if "--ratios" in sys.argv:
        A = O.laplacian_3d(100)
        table = {}
        for lev in (0, 1):
            L, U = R.ilu_k(A, lev)
            table[f"ilu{lev}"] = {"L": L.nnz, "U": U.nnz}
            for tau in (0.05, 0.02, 0.01):
                table[f"ilu{lev}"][f"thr_{tau}_10"] = [R.sait_thr(L, True, tau, 10).nnz, R.sait_thr(U, False, tau, 10).nnz]
            for p in (1, 2, 3):
                table[f"ilu{lev}"][f"pat_{p}_10"] = [R.sait_pat(L, True, p, 10).nnz, R.sait_pat(U, False, p, 10).nnz]
        with open(os.path.join(HERE, "ratio_table_100.json"), "w") as f:
            json.dump(table, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
