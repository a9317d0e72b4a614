import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K
from oracle import levelmpk_oracle as O
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0]-1
a = K.DeviceCsr.from_host(rp, c, v); torch.cuda.synchronize(); print("h2d ok", flush=True)
y = torch.zeros(9, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
K.mpk_baseline(a, y, 8); torch.cuda.synchronize(); print("baseline natural ok", flush=True)
perm, inv, lp = K.bfs_levels(a, 0); torch.cuda.synchronize(); print("bfs ok", len(lp), flush=True)
b = K.permute_symmetric(a, perm, inv); torch.cuda.synchronize(); print("permute ok", flush=True)
K.mpk_baseline(b, y, 8); torch.cuda.synchronize(); print("baseline perm ok", flush=True)
