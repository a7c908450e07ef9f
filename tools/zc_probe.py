import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12836_b200 as S
from paper_2106_12836_b200 import _native as N
f = N.lib.sait_debug_zero_copy_ms
f.restype = ctypes.c_double
f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int]
n = 2097152
h = torch.empty(n, dtype=torch.float64).pin_memory()
for d in (0, 1):
    for v in (1, 2):
        ms = f(h.data_ptr(), n, d, v)
        print("dir", "D2H-store" if d == 0 else "H2D-load", "vec", v, f"{ms:.3f} ms", f"{n*8/ms/1e6:.1f} GB/s")
