"""ncu driver: cfg2 (7-pt 200^3, level order), MPK with env-selected tiling
(COMP=1 compressed blocks, SLOTS, Q, TILE); a few launches."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
N = int(os.environ.get("N", "200")); k = 8
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0] - 1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
q = int(os.environ.get("Q", "1"))
fl = (_lib.FLAG_MODE_RESIDENT if q == k else _lib.FLAG_MODE_STREAM) | (_lib.FLAG_COMPRESS if os.environ.get("COMP", "1") == "1" else 0)
t = K.Tiling(b, k, tile_nnz=int(os.environ.get("TILE", "0")), mode_flags=fl, slots=int(os.environ.get("SLOTS", "1")), group=q, queue_slack=int(os.environ.get("SLACK", "0")))
y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
cfg = K.mpk_power_cfg(k)
for _ in range(int(os.environ.get("REPS", "3"))):
    K.mpk_run(t, y, cfg, flags=(_lib.FLAG_SWEEP if os.environ.get("SWEEP") else 0) | (int(os.environ.get("POL", "0")) << 8))
torch.cuda.synchronize(); print("done", t.info)
