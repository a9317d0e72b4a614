import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
rp, c, v = O.gen_stencil_3d(int(os.environ.get("N", "200"))); n = rp.shape[0] - 1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
ctx = _lib.context()
f = ctx.lib.lmpk_probe_tile_compute
f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
y = torch.zeros(2, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
for tile in (9600, 4800, 2400):
    t = K.Tiling(b, 8, tile_nnz=tile, slots=1 if tile > 5000 else 2, mode_flags=_lib.FLAG_MODE_STREAM)
    for exact in (0, 1):
        for threads, cps in ((512, 1), (800, 1), (1024, 1), (256, 2), (512, 2), (256, 4), (128, 8)):
            if tile * 12 * cps > 225000: continue
            out = ctypes.c_double()
            rc = f(ctx.handle, t.handle, ctypes.c_void_p(y.data_ptr()), n, 20, threads, cps | (0x100 if exact else 0), ctypes.byref(out))
            print(f"tile {tile:5d} exact {exact} threads {threads:4d} ctas/sm {cps}: {out.value:7.1f} ns per 1K nnz per SM  rc={rc}", flush=True)
