"""Per-SM rate of the row kernel alone (lmpk_probe_tile_compute) on cfg2
tiles: plain vs compressed blocks, probe gather variants (MODE 0 real,
1 confined to 8 KB, 2 coalesced, 3 none)."""
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
for comp, slots in ((0, 2), (1, 2), (1, 1)):
    t = K.Tiling(b, 8, slots=slots, mode_flags=_lib.FLAG_MODE_STREAM | (_lib.FLAG_COMPRESS if comp else 0))
    for exact in (1, 0):
        for mode in (0, 1, 2, 3):
            for threads in (768, 1024):
                out = ctypes.c_double()
                rc = f(ctx.handle, t.handle, ctypes.c_void_p(y.data_ptr()), n, 10, threads, 1 | (0x100 if exact else 0) | (mode << 12), ctypes.byref(out))
                print(f"comp {comp} R {slots} tiles {t.info['n_tiles']} exact {exact} probe {mode} threads {threads}: {out.value:7.1f} ns/1K nnz/SM rc={rc}", flush=True)
