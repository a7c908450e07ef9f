"""Generate the full-size parity fixtures (TEST INFRASTRUCTURE: run here, in
the container that has /root/reference; the outputs are committed).

For BASELINE configs 3, 4 and 5 at their full sizes, the CPU side runs once:
  * the factors: the reference's own ilu_k (ILU(0)) and sait_thr
    (oracle/_ref = the reference sources compiled by oracle/Makefile;
    sait.cpp:90-101), C4 through the reference's DropRule hook with the fill
    cap (ref_wrapper.cpp), optionally cross-checked against the C restatement;
  * two seeded pair applies (preconditioner.cpp:42-45) and, for C5, the
    block-8 apply (preconditioner.cpp:47-49);
  * the solvers of oracle/solvers.c: C3 GMRES(30) to 1e-8 from the seed-3
    rhs; C5 block LOBPCG (8 pairs, tol 1e-6, seed 5) for its first
    C5_PREFIX iterations (the whole 570-iteration run would take ~9 h here).
Only digests (SHA-256 of int64 row_ptr / col_idx and the fp64 value bits),
sizes, step/iteration counts and the (short) residual histories are stored:
tests/golden/fullsize.json and tests/golden/fullsize_hist.npz.  The -m gpu
test tests/test_gpu_fullsize_c345.py rebuilds everything on the device and
compares.

Usage: python tests/golden/make_fullsize.py [c3] [c4] [c5] [--cross-port]
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

OUT_JSON = os.path.join(HERE, "fullsize.json")
C5_PREFIX = 12  # LOBPCG iterations pinned at config-5 size (see c5)
OUT_NPZ = os.path.join(HERE, "fullsize_hist.npz")


def csr_digest(m) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(m.row_ptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(m.col_idx, dtype=np.int64).tobytes())
    if m.values is not None:
        h.update(np.ascontiguousarray(m.values, dtype=np.float64).view(np.uint64).tobytes())
    return h.hexdigest()


def vec_digest(v) -> str:
    return hashlib.sha256(np.ascontiguousarray(v, dtype=np.float64).view(np.uint64).tobytes()).hexdigest()


def load():
    rec = json.load(open(OUT_JSON)) if os.path.exists(OUT_JSON) else {}
    hist = dict(np.load(OUT_NPZ)) if os.path.exists(OUT_NPZ) else {}
    return rec, hist


def save(rec, hist):
    with open(OUT_JSON, "w") as f:
        json.dump(rec, f, indent=1, sort_keys=True)
    np.savez_compressed(OUT_NPZ, **hist)


def log(*a):
    print(*a, flush=True)


def factors(R, P, A, tau, k, cross):
    t0 = time.perf_counter()
    L, U = R.ilu_k(A, 0)
    log(f"  ilu_k {time.perf_counter() - t0:.1f} s  nnz L {L.nnz} U {U.nnz}")
    t0 = time.perf_counter()
    ML = R.sait_thr(L, True, tau, k)
    MU = R.sait_thr(U, False, tau, k)
    log(f"  reference sait_thr x2 {time.perf_counter() - t0:.1f} s  nnz {ML.nnz} {MU.nnz}")
    out = {"nnz_L": int(L.nnz), "nnz_U": int(U.nnz), "nnz_ML": int(ML.nnz), "nnz_MU": int(MU.nnz),
           "digest_L": csr_digest(L), "digest_U": csr_digest(U),
           "digest_ML": csr_digest(ML), "digest_MU": csr_digest(MU)}
    if cross:
        t0 = time.perf_counter()
        pl, sl = P.sait_thr_steps(L, True, tau, k)
        pu, su = P.sait_thr_steps(U, False, tau, k)
        assert csr_digest(pl) == out["digest_ML"] and csr_digest(pu) == out["digest_MU"], "port != reference"
        out["steps_run"] = [int(sl), int(su)]
        out["port_cross_checked"] = True
        log(f"  port sait_thr x2 {time.perf_counter() - t0:.1f} s (bitwise the reference), steps {sl} {su}")
    return L, U, ML, MU, out


def applies(R, ML, MU, n, seeds):
    out = {}
    for s in seeds:
        r = O.uniform_pm1(s, n)
        z = R.pair_apply(ML, MU, r)
        out[str(s)] = {"digest": vec_digest(z), "norm2": float(np.linalg.norm(z))}
    return out


def c3(rec, hist, cross):
    log("C3: convdiff 2048^2, ILU(0), tau 2e-2, k 4, GMRES(30) 1e-8, rhs seed 3")
    R, P = O.get("reference"), O.get("port")
    A = O.convdiff_2d(2048, 20.0, -10.0)
    L, U, ML, MU, d = factors(R, P, A, 2e-2, 4, cross)
    d["n"] = int(A.nrows)
    d["nnz_A"] = int(A.nnz)
    d["digest_A"] = csr_digest(A)
    d["apply"] = applies(R, ML, MU, A.nrows, (3000, 3001))
    b = O.uniform_pm1(3, A.nrows)
    t0 = time.perf_counter()
    x, st = O.gmres(A, ML, MU, b, restart=30, tol=1e-8, maxit=20000)
    t = time.perf_counter() - t0
    log(f"  oracle GMRES(30): {st['iterations']} its, converged {st['converged']}, true relres {st['true_relres']:.3e}, {t:.0f} s")
    d["gmres"] = {"restart": 30, "tol": 1e-8, "maxit": 20000, "rhs_seed": 3, "iterations": int(st["iterations"]),
                  "converged": bool(st["converged"]), "relres": float(st["relres"]),
                  "true_relres": float(st["true_relres"]), "x_digest": vec_digest(x), "cpu_seconds": t,
                  "cpu_threads": os.cpu_count()}
    hist["c3_gmres_history"] = st["history"]
    rec["c3"] = d
    save(rec, hist)


def c4(rec, hist, cross, log2n=22):
    log(f"C4: synthetic lower n=2^{log2n}, tau 1e-2, k 3, cap 3x")
    R, P = O.get("reference"), O.get("port")
    n = 1 << log2n
    T = O.synthetic_lower(n, 15, 0.01, 4)
    t0 = time.perf_counter()
    M = R.sait_thr_cap(T, True, 1e-2, 3, 3.0)
    t = time.perf_counter() - t0
    log(f"  reference capped build {t:.1f} s, nnz {M.nnz}")
    d = {"log2n": log2n, "n": n, "nnz_T": int(T.nnz), "digest_T": csr_digest(T), "nnz_M": int(M.nnz),
         "digest_M": csr_digest(M), "cpu_seconds": t}
    if cross:
        pm = P.sait_thr_cap(T, True, 1e-2, 3, 3.0)
        assert csr_digest(pm) == d["digest_M"], "port != reference"
        d["port_cross_checked"] = True
    rec[f"c4_2^{log2n}"] = d
    save(rec, hist)


def c5(rec, hist, cross):
    log("C5: laplacian 256^3, ILU(0), tau 5e-2, k 3, LOBPCG block 8 tol 1e-6 seed 5")
    R, P = O.get("reference"), O.get("port")
    A = O.laplacian_3d(256)
    L, U, ML, MU, d = factors(R, P, A, 5e-2, 3, cross)
    n = A.nrows
    d["n"] = int(n)
    d["nnz_A"] = int(A.nnz)
    d["apply"] = applies(R, ML, MU, n, (5000, 5001))
    Rb = np.stack([O.uniform_pm1(5100 + j, n) for j in range(8)], axis=1)  # (n, 8), column j = seed 5100 + j
    Zb = R.pair_apply_block(ML, MU, Rb)
    # digest of the column-major (n, 8) block = the 8 columns one after the other
    d["apply_block8"] = {"seeds": [5100 + j for j in range(8)], "digest": vec_digest(np.asfortranarray(Zb).T)}
    del Rb, Zb
    # the restatement's LOBPCG costs ~1 min per iteration at this size on
    # this host (570 iterations: ~9 h), so the fixture pins a prefix: the
    # first C5_PREFIX iterations' residual-norm history, Ritz values and
    # block, bitwise (the device's canonical mode is the same arithmetic)
    prefix = C5_PREFIX
    t0 = time.perf_counter()
    ev, X, its, res = O.lobpcg(A, ML, MU, 8, tol=1e-6, maxit=prefix, seed=5)
    t = time.perf_counter() - t0
    log(f"  oracle LOBPCG prefix: {its} its, evals {ev}, max res {res[-1].max():.3e}, {t:.0f} s")
    d["lobpcg_prefix"] = {"nev": 8, "tol": 1e-6, "maxit": prefix, "seed": 5, "iterations": int(its),
                          "evals": [float(v) for v in ev], "evals_digest": vec_digest(ev),
                          "evecs_digest": vec_digest(X.T), "cpu_seconds": t, "cpu_threads": os.cpu_count()}
    hist["c5_lobpcg_prefix_resnorms"] = res
    rec["c5"] = d
    save(rec, hist)


def main():
    which = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c3", "c4", "c5"]
    cross = "--cross-port" in sys.argv
    rec, hist = load()
    if "c3" in which:
        c3(rec, hist, cross)
    if "c4" in which:
        c4(rec, hist, cross)
    if "c5" in which:
        c5(rec, hist, cross)


if __name__ == "__main__":
    main()
