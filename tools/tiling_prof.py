"""Host-side phase times of lmpk_tiling_create on cfg2 (LMPK_TILING_PROF=1)."""
import os, sys, time
os.environ["LMPK_TILING_PROF"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
a = lm.gen_stencil_3d(int(os.environ.get("N", "200")), 2, device=True)
lm.warmup()
d = a.device()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    perm, inv, lp = K.bfs_levels(d, 0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    b = K.permute_symmetric(d, perm, inv)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"--- pass {i}: bfs {1e3*(t1-t0):.2f} ms permute {1e3*(t2-t1):.2f} ms", file=sys.stderr, flush=True)
    t = K.Tiling(b, 8)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"--- tiling total {1e3*(t3-t2):.2f} ms", file=sys.stderr, flush=True)
    t.close()
