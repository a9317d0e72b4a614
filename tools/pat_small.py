import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
from oracle import levelmpk_oracle as O, cpu as C
a = lm.gen_stencil_3d(int(os.environ.get("N","20")), 2)
perm, _ = C.bfs_levels(a.row_ptr, a.col, 0)
rp, c, v = C.permute_symmetric(a.row_ptr, a.col, a.val, perm)
d = K.DeviceCsr.from_host(rp, c, v)
print("building", flush=True)
t = K.Tiling(d, 4)
torch.cuda.synchronize()
print("tiling", t.info, flush=True)
x = np.random.default_rng(0).uniform(-1,1,a.n_rows)
y = torch.zeros((5, a.n_rows), dtype=torch.float64, device="cuda"); y[0] = torch.from_numpy(x)
K.mpk_run(t, y, K.mpk_power_cfg(4), exact=True)
print("ran", flush=True)
ref = O.mpk_powers(rp, c, v, x, 4)
print("bitwise", np.array_equal(y.cpu().numpy(), ref), flush=True)
