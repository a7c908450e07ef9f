"""C2 builds: serial sait_thr of both factors vs sait_thr_pair (concurrent),
median wall of N reps.  python tools/build_probe.py [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12836_b200 as S  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 15
A = S.laplacian_3d(128)
f = S.ilu_device(A, 0)
L, U = f.lower, f.upper
P = S.SaitThrParams(5e-2, 3)


def serial():
    a = S.sait_thr(L, S.lower_triangular, P)
    b = S.sait_thr(U, S.upper_triangular, P)
    torch.cuda.synchronize()
    a.free()
    b.free()


def pair():
    a, b = S.sait_thr_pair(L, U, P)
    torch.cuda.synchronize()
    a.free()
    b.free()


for name, fn in (("serial", serial), ("pair", pair), ("serial", serial), ("pair", pair)):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: median {np.median(ts) * 1e3:.3f} ms  min {min(ts) * 1e3:.3f} ms", flush=True)
