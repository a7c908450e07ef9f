import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12836_b200 as S
m = int(sys.argv[1]) if len(sys.argv) > 1 else 96
its = int(sys.argv[2]) if len(sys.argv) > 2 else 5
A = S.laplacian_3d(m)
f = S.ilu_k(A, 0)
ML = S.sait_thr(f.lower, S.lower_triangular, S.SaitThrParams(5e-2, 3))
MU = S.sait_thr(f.upper, S.upper_triangular, S.SaitThrParams(5e-2, 3))
pair = S.SaitPairPreconditioner(ML, MU)
dA = S.DeviceCsr.upload(A)
r = S.lobpcg(dA, pair, 8, 1e-6, its, 5, host_vectors=False)
print("iters", r.iterations)
