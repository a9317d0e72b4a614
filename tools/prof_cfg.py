"""ncu driver for one BASELINE shape: CASE=cfg3|cfg5 [K=8], default tiling, 3 MPK launches."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K, _lib
case = os.environ.get("CASE", "cfg5"); k = int(os.environ.get("K", "8"))
a = {"cfg3": lambda: lm.gen_stencil_3d27pt(160, seed=1), "cfg5": lambda: lm.gen_anderson_3d(128, seed=2)}[case]()
_, perm = lm.bfs_levels(a, 0)
ap = lm.permute_symmetric(a, perm)
d = ap.device()
t = K.Tiling(d, k, mode_flags=int(os.environ.get("MODE_FLAGS", "0")))
y = torch.zeros(k + 1, a.n_rows, dtype=torch.float64, device="cuda"); y[0] = 1.0
cfg = K.mpk_power_cfg(k)
for _ in range(3):
    K.mpk_run(t, y, cfg)
torch.cuda.synchronize(); print("done", t.info)
