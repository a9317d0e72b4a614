import sys, os, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
n = 200_000
rng = np.random.default_rng(3)
for ln in (97_280, 48_640, 20_000):
    cols = np.sort(rng.choice(n, ln, replace=False))
    rp = np.zeros(n + 1, dtype=np.int32); rp[8:] = ln
    a = lm.CsrMatrix(n, rp, cols.astype(np.int32), rng.standard_normal(ln))
    x = torch.from_numpy(rng.uniform(-1, 1, n)).cuda()
    out = torch.zeros(n, dtype=torch.float64, device="cuda")
    d = a.device()
    for _ in range(3): K.spmv_rows(d, x, out, 0, n)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): K.spmv_rows(d, x, out, 0, n)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(ln, "ms", round(ms, 4), "ns/entry", round(ms * 1e6 / ln, 2), "cycles@1.965", round(ms * 1e6 / ln * 1.965, 2))
