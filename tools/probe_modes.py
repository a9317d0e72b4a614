"""Compute-probe variants on cfg2 tiles: mode 0 = the real tile kernel, 1 =
gathers confined to 8 KB, 2 = perfectly coalesced gathers, 3 = no gathers
(modes 1-3: width-7 full slices only, single-slice path)."""
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
for mode in (0, 1, 2, 3):
    for threads in (768,):
        for exact in (1,):
            out = ctypes.c_double()
            rc = f(ctx.handle, t.handle, ctypes.c_void_p(y.data_ptr()), n, 200, threads, 1 | (0x100 if exact else 0) | (mode << 12), ctypes.byref(out))
            print(f"mode {mode} threads {threads:4d} exact {exact}: {out.value:7.1f} ns per 1K nnz per SM rc={rc}", flush=True)
