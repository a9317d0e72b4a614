"""Small driver for ncu: cfg2 (7-pt 200^3, level order), one mode, few launches."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
mode = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 200
tile = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0] - 1; k = 8
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
fl = {"sweep": _lib.FLAG_MODE_STREAM, "stream": _lib.FLAG_MODE_STREAM, "res": _lib.FLAG_MODE_RESIDENT}[mode]
t = K.Tiling(b, k, tile_nnz=tile, ctas_per_sm=cps, threads=512, mode_flags=fl, slots=int(os.environ.get("SLOTS", "2")))
y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
cfg = K.mpk_power_cfg(k)
for _ in range(2):
    K.mpk_run(t, y, cfg, flags=_lib.FLAG_SWEEP if mode == "sweep" else 0)
torch.cuda.synchronize(); print("done", t.info)
