"""The paper's SPD experiment (tables SPD_Thr / SPD_Pat) on
the device: for each matrix, PCG iteration counts with no preconditioner, the
exact ILU(k) solves, and SAIT_Thr(tau, 10) / SAIT_Pat(p, 10) built from the
same factors, plus device times.  The right-hand side is SPEC.md's
"ones-solution" b = A 1; stop at ||r|| / ||b|| <= 1e-8 (the paper's choice
is not stated; DESIGN.md records this reading).

    python tools/run_spd_table.py [file.mtx ...] [--tau 0.05] [--level 0] [--json out.json]

The SuiteSparse files are not in this container (SPEC.md: user-supplied
paths); without files it runs on seeded stand-ins (3-D Laplacians).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402


def run_one(name, A, tau, level, pat, tol, maxit):
    b = S.make_rhs(A, "ones-solution")
    row = {"matrix": name, "rows": A.nrows, "nnz": A.nnz(), "level": level, "tau": tau}
    _, st = S.pcg(A, None, b, tol, maxit)
    row["no_pc"] = st.iterations
    t0 = time.perf_counter()
    if level <= 1:
        f = S.ilu_device(A, level)
        torch.cuda.synchronize()
        row["ilu_device_ms"] = (time.perf_counter() - t0) * 1e3
        L, U = f.lower, f.upper
    else:
        f = S.ilu_k(A, level)
        row["ilu_host_ms"] = (time.perf_counter() - t0) * 1e3
        L, U = S.DeviceCsr.upload(f.lower), S.DeviceCsr.upload(f.upper)
    nnz_lu = L.nnz() + U.nnz()
    E = S.ExactIluPreconditioner(S.IluFactors(L, U))
    _, st = S.pcg(A, E, b, tol, maxit)
    row["exact"] = st.iterations
    row["exact_s"] = st.seconds
    stats = []
    t0 = time.perf_counter()
    ML = S.sait_thr(L, S.lower_triangular, S.SaitThrParams(tau, 10), stats_out=stats)
    MU = S.sait_thr(U, S.upper_triangular, S.SaitThrParams(tau, 10), stats_out=stats)
    torch.cuda.synchronize()
    row["sait_build_ms"] = (time.perf_counter() - t0) * 1e3
    P = S.SaitPairPreconditioner(ML, MU)
    row["ratio"] = round(P.nnz() / nnz_lu, 2)
    _, st = S.pcg(A, P, b, tol, maxit)
    row["sait"] = st.iterations
    row["sait_s"] = st.seconds
    row["increase"] = f"{100.0 * (row['sait'] - row['exact']) / max(row['exact'], 1):.1f}%"
    for p in pat:
        MLp = S.sait_pat(L, S.lower_triangular, S.SaitPatParams(p, 10))
        MUp = S.sait_pat(U, S.upper_triangular, S.SaitPatParams(p, 10))
        Pp = S.SaitPairPreconditioner(MLp, MUp)
        _, st = S.pcg(A, Pp, b, tol, maxit)
        row[f"pat{p}_ratio"] = round(Pp.nnz() / nnz_lu, 2)
        row[f"pat{p}"] = st.iterations
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("files", nargs="*")
    ap.add_argument("--tau", type=float, default=0.05)
    ap.add_argument("--level", type=int, default=0)
    ap.add_argument("--pat", type=int, nargs="*", default=[2, 3])
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--maxit", type=int, default=30000)
    ap.add_argument("--json")
    args = ap.parse_args()
    inputs = [(os.path.basename(f), lambda f=f: S.mm_read(f)) for f in args.files]
    if not inputs:
        inputs = [(f"laplacian_3d({n})", lambda n=n: S.laplacian_3d(n)) for n in (32, 64)]
    rows = []
    for name, load in inputs:
        row = run_one(name, load(), args.tau, args.level, args.pat, args.tol, args.maxit)
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.json:
        with open(args.json, "w") as fh:
            json.dump(rows, fh, indent=1)


if __name__ == "__main__":
    main()
