import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K
from oracle import levelmpk_oracle as O
N, P, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0]-1
a = K.DeviceCsr.from_host(rp, c, v)
y = torch.zeros(P + 1, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
if mode == "base":
    K.mpk_baseline(a, y, P); torch.cuda.synchronize(); print("ok", flush=True)
else:
    for p in range(1, P + 1):
        K.spmv_rows(a, y[p - 1], y[p], 0, n); torch.cuda.synchronize()
    print("ok", flush=True)
