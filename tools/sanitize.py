"""Small end-to-end workload for compute-sanitizer (memcheck /
racecheck on the device paths): every builder bin (tiny, shared-memory and
global hash tables, staging overflow), the pair apply (device, chunked host,
block), the solvers, ILU(0)/ILU(1), the exact triangular solves and the
peer-halo SpMV with virtual ranks.  Checks results against the oracle so a
silent corruption also fails.

    compute-sanitizer --tool memcheck python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py
    SAIT_CHECKED=1 python tools/sanitize.py   # the bounds-checked build (make checked)

Summaries of the round-2 runs: profiles/r02_sanitizer.txt.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ.setdefault("SAIT_PIPE_MB", "0.0625;0.125;0.0625")  # several host-apply chunks at this size

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2106_12836_b200 as S  # noqa: E402
from helpers import bitwise_equal, bitwise_equal_csr, to_oracle, to_product  # noqa: E402
from oracle import oracle as O  # noqa: E402

P = O.get("port")


def check(ok, what):
    if not ok:
        raise SystemExit(f"MISMATCH: {what}")
    print("ok", what, flush=True)


# builder: every bin
T = O.synthetic_lower(3000, 12, 0.3, seed=5)  # long rows -> hash tables / global tables
check(bitwise_equal_csr(S.sait_thr(to_product(T), S.lower_triangular, S.SaitThrParams(1e-2, 4)),
                        P.sait_thr(T, True, 1e-2, 4)), "build: hash/global bins")
A = O.laplacian_3d(16)
L, U = P.ilu_k(A, 0)
ML, MU = P.sait_thr(L, True, 5e-2, 3), P.sait_thr(U, False, 5e-2, 3)
mlp = S.sait_thr(to_product(L), S.lower_triangular, S.SaitThrParams(5e-2, 3))
check(bitwise_equal_csr(mlp, ML), "build: tiny bins")
check(bitwise_equal_csr(S.sait_thr_cap(to_product(T), S.lower_triangular, S.SaitThrParams(1e-2, 3), 1.5),
                        P.sait_thr_cap(T, True, 1e-2, 3, 1.5)), "build: fill cap")
check(bitwise_equal_csr(S.sait_pat(to_product(T), S.lower_triangular, S.SaitPatParams(2, 3)),
                        P.sait_pat(T, True, 2, 3)), "build: pattern")
# window rows (config-4 shape: -0.0 windows of every span bin, the row-form
# cap pass, the staging chunks), both factors' orientations
T4 = O.synthetic_lower(20000, 15, 0.01, seed=4)
T4u = P.transpose(T4)
check(bitwise_equal_csr(S.sait_thr(to_product(T4), S.lower_triangular, S.SaitThrParams(1e-2, 3)),
                        P.sait_thr(T4, True, 1e-2, 3)), "build: window rows")
check(bitwise_equal_csr(S.sait_thr(to_product(T4u), S.upper_triangular, S.SaitThrParams(1e-2, 3)),
                        P.sait_thr(T4u, False, 1e-2, 3)), "build: window rows (upper)")
for f in (1.0, 3.0):
    check(bitwise_equal_csr(S.sait_thr_cap(to_product(T4), S.lower_triangular, S.SaitThrParams(1e-2, 3), f),
                            P.sait_thr_cap(T4, True, 1e-2, 3, f)), f"build: row-form cap pass (f = {f})")

# apply: device, host (chunked), block
pair = S.SaitPairPreconditioner(to_product(ML), to_product(MU))
r = O.uniform_pm1(3, A.nrows)
want = P.pair_apply(ML, MU, r)
z = np.empty(A.nrows)
pair.apply(r, z)
check(bitwise_equal(z, want), "apply: host vectors")
rd = torch.from_numpy(r).cuda()
zd = torch.empty_like(rd)
pair.apply(rd, zd)
torch.cuda.synchronize()
check(bitwise_equal(zd.cpu().numpy(), want), "apply: device vectors")
R = np.stack([O.uniform_pm1(10 + c, A.nrows) for c in range(8)], axis=1)
Z = pair.apply_block(R)
check(bitwise_equal(np.asfortranarray(Z).ravel(order="F"),
                    np.asfortranarray(P.pair_apply_block(ML, MU, R)).ravel(order="F")), "apply: block of 8")

for fmt in ("csr", "sell32_int32", "sell32_int16", "sell32_dict"):
    pf = S.SaitPairPreconditioner(to_product(ML), to_product(MU), format=fmt)
    zf = torch.empty_like(rd)
    pf.apply(rd, zf)
    torch.cuda.synchronize()
    check(bitwise_equal(zf.cpu().numpy(), want), f"apply: format {fmt}")
    del pf
Md = S.DeviceCsr.upload(to_product(ML))
Xb = torch.from_numpy(np.asfortranarray(R).ravel(order="F").copy()).cuda()
Yb = torch.empty(A.nrows * 8, dtype=torch.float64, device="cuda")
from paper_2106_12836_b200 import _native as NN  # noqa: E402

NN.check(NN.lib.sait_spmm(Md.handle, Xb.data_ptr(), Yb.data_ptr(), 8, None))
torch.cuda.synchronize()
check(bitwise_equal(Yb.cpu().numpy(), np.concatenate([P.spmv(ML, R[:, c]) for c in range(8)])), "spmm (block of 8)")

# solvers
b = O.uniform_pm1(4, A.nrows)
xo, so = O.pcg(A, ML, MU, b, 1e-10, 300)
x, st = S.pcg(to_product(A), pair, b, 1e-10, 300)
check(st.iterations == so["iterations"] and bitwise_equal(x, xo), "pcg")
xo, so = O.gmres(A, ML, MU, b, 10, 1e-8, 300)
x, st = S.gmres(to_product(A), pair, b, 10, 1e-8, 300)
check(st.iterations == so["iterations"] and bitwise_equal(x, xo), "gmres")
ev, _, it, _ = O.lobpcg(A, ML, MU, 4, 1e-6, 20, 5)
res = S.lobpcg(to_product(A), pair, 4, 1e-6, 20, 5)
check(res.iterations == it and bitwise_equal(res.eigenvalues, ev), "lobpcg")
ev8, _, it8, _ = O.lobpcg(A, ML, MU, 8, 1e-6, 200, 5)
rt = S.lobpcg(to_product(A), pair, 8, 1e-6, 200, 5, gram="tensor")  # deferred W, fused norms, upper-tile Grams
check(abs(rt.iterations - it8) <= 1 and np.max(np.abs(rt.eigenvalues - ev8) / np.abs(ev8)) < 1e-12,
      "lobpcg: tensor-core Grams")

# ILU(0)/(1), trisolve, exact preconditioner
for lev in (0, 1):
    Lw, Uw = P.ilu_k(A, lev)
    f = S.ilu_device(to_product(A), lev)
    check(bitwise_equal_csr(f.lower.to_host(), Lw) and bitwise_equal_csr(f.upper.to_host(), Uw), f"ilu({lev})")
E = S.ExactIluPreconditioner(S.IluFactors(to_product(L), to_product(U)))
ze = np.empty(A.nrows)
E.apply(r, ze)
check(bitwise_equal(ze, P.trisolve(U, False, P.trisolve(L, True, r))), "exact ilu apply")

# peer-halo SpMV, three virtual ranks
from paper_2106_12836_b200.dist import PeerShardedPair  # noqa: E402

ranks = {}
for q in range(3):
    ranks[q] = PeerShardedPair(to_product(ML), to_product(MU), q, 3, resolve=lambda qq, ff: ranks[qq].bufs[ff].ptr,
                               align=256)
s = torch.cuda.current_stream().cuda_stream
for q in range(3):
    a0, a1 = ranks[q].own
    ranks[q].stage_input(rd[a0:a1], 1, s)
for q in range(3):
    ranks[q].stage_lower(1, s)
zs = []
for q in range(3):
    a0, a1 = ranks[q].own
    zq = torch.empty(a1 - a0, dtype=torch.float64, device="cuda")
    ranks[q].stage_upper(zq, 1, s)
    zs.append(zq)
torch.cuda.synchronize()
check(bitwise_equal(torch.cat(zs).cpu().numpy(), want), "peer-halo pair, 3 virtual ranks")
for q in range(3):
    ranks[q].close()

# column-sharded build of 3 virtual ranks -> device redistribution to row blocks
import ctypes as C  # noqa: E402

from paper_2106_12836_b200.dist import column_bounds_by_work, redistribute_local, row_bounds  # noqa: E402

dL = S.DeviceCsr.upload(to_product(L))
cb = column_bounds_by_work(dL, 3)
spec = NN.DropSpec(NN.SAIT_DROP_THRESHOLD, 5e-2, 3, 0, 0, 0.0)
sess = []
for q in range(3):
    h = C.c_void_p()
    NN.check(NN.lib.sait_build_session_create(dL.handle, 1, C.byref(spec), cb[q], cb[q + 1], None, C.byref(h)))
    sess.append(h)
while NN.lib.sait_build_session_remaining(sess[0]) > 0:
    fl = []
    for h in sess:
        ch = C.c_int(1)
        NN.check(NN.lib.sait_build_session_step(h, C.byref(ch)))
        fl.append(ch.value)
    if max(fl) == 0:
        for h in sess:
            NN.check(NN.lib.sait_build_session_stop(h))
blocks = []
for h in sess:
    out = C.c_void_p()
    NN.check(NN.lib.sait_build_session_finish(h, 0, C.byref(out), None))
    NN.lib.sait_build_session_destroy(h)
    blocks.append(S.DeviceCsr(out.value))
rb = row_bounds(A.nrows, 3)
rows = redistribute_local(blocks, cb, rb)
got = [rows[q].to_host() for q in range(3)]
okr = all(np.array_equal(got[q].col_idx, ML.col_idx[ML.row_ptr[rb[q]]:ML.row_ptr[rb[q + 1]]]) and
          bitwise_equal(got[q].values, ML.values[ML.row_ptr[rb[q]]:ML.row_ptr[rb[q + 1]]]) for q in range(3))
check(okr, "column-sharded build -> row blocks (3 virtual ranks)")
print("SANITIZE WORKLOAD DONE")
