import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12836_b200 as S
from paper_2106_12836_b200 import _native as N
N.lib.sait_debug_pointer_type.argtypes = [ctypes.c_void_p]
t = torch.empty(1 << 20, dtype=torch.float64).pin_memory()
u = torch.empty(1 << 20, dtype=torch.float64)
p = ctypes.c_void_p()
N.check(N.lib.sait_host_alloc(8 << 20, ctypes.byref(p)))
print("torch pinned ->", N.lib.sait_debug_pointer_type(t.data_ptr()), " pageable ->", N.lib.sait_debug_pointer_type(u.data_ptr()), " sait_host_alloc ->", N.lib.sait_debug_pointer_type(p.value))
n = 2097152
src = torch.randn(n, dtype=torch.float64).pin_memory()
dst = torch.empty(n, dtype=torch.float64).pin_memory()
out = (ctypes.c_double * 3)()
N.lib.sait_debug_copy_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
for ch in (1, 2, 4, 8, 16, 64, -4, -16):
    N.lib.sait_debug_copy_probe(src.data_ptr(), dst.data_ptr(), n, ch, out)
    print("chunks", ch, "h2d %.3f ms d2h %.3f ms both %.3f ms" % tuple(x * 1e3 for x in out))
