"""Host block apply (sait_pair_apply_block_host) on the C2 workload: 100 pinned
host vectors in, 100 out, per call; prints GB/s of PCIe traffic and the
pipelined-vs-serial times.  SAIT_BLK_SLOTS selects the slot count.

    python tools/blk_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402

A = S.laplacian_3d(128)
f = S.ilu_device(A, 0)
ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
P = S.SaitPairPreconditioner(ML, MU)
n, nv = A.nrows, 100
Rh = torch.empty((nv, n), dtype=torch.float64).pin_memory()
Rh.uniform_(-1, 1)
Zh = torch.empty((nv, n), dtype=torch.float64).pin_memory()
Rn, Zn = Rh.numpy(), Zh.numpy()


def timed(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


t = timed(lambda: P.apply_block(Rn.T, Zn.T))
print(f"slots={os.environ.get('SAIT_BLK_SLOTS', '3')} block: {t * 1e3:.2f} ms  "
      f"{2 * nv * n * 8 / t / 1e9:.1f} GB/s PCIe (both directions)", flush=True)
if os.environ.get("BLK_PROBE_ALL"):
    os.environ["SAIT_BLOCK_HOST_PIPELINE"] = "0"
    t = timed(lambda: P.apply_block(Rn.T, Zn.T), 2)
    print(f"serial block: {t * 1e3:.2f} ms", flush=True)
    os.environ["SAIT_BLOCK_HOST_PIPELINE"] = "1"
    t = timed(lambda: [P.apply(Rn[i], Zn[i]) for i in range(nv)], 2)
    print(f"per-vector: {t * 1e3:.2f} ms", flush=True)
    # copy engines alone on the same buffers
    d = torch.empty((nv, n), dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        with torch.cuda.stream(s1):
            d[: nv // 2].copy_(Rh[: nv // 2], non_blocking=True)
        with torch.cuda.stream(s2):
            Zh[nv // 2:].copy_(d[nv // 2:], non_blocking=True)
        torch.cuda.synchronize()

    def h2d():
        d.copy_(Rh, non_blocking=True)
        torch.cuda.synchronize()

    def d2h():
        Zh.copy_(d, non_blocking=True)
        torch.cuda.synchronize()

    for nm, fn, by in (("H2D", h2d, nv * n * 8), ("D2H", d2h, nv * n * 8), ("H2D||D2H", both, nv * n * 8)):
        t = timed(fn, 3)
        print(f"{nm}: {by / t / 1e9:.1f} GB/s", flush=True)
