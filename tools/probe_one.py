import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
rp, c, v = O.gen_stencil_3d(200); n = rp.shape[0] - 1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
ctx = _lib.context()
f = ctx.lib.lmpk_probe_tile_compute
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
y = torch.zeros(2, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
t = K.Tiling(b, 8, tile_nnz=9600, slots=1, mode_flags=_lib.FLAG_MODE_STREAM)
out = ctypes.c_double()
rc = f(ctx.handle, t.handle, ctypes.c_void_p(y.data_ptr()), n, 20, int(os.environ.get("THREADS", "800")), int(os.environ.get("CPS", "1")), ctypes.byref(out))
print("ns per 1K nnz", out.value, rc)
