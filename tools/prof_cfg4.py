import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
a = lm.gen_rmat(int(os.environ.get("SCALE", "22")))
pre = lm.prepare(a, "lb_lg_p2p", 6, 126e6)
d = pre.a.device()
y = torch.zeros(7, a.n_rows, dtype=torch.float64, device="cuda"); y[0] = 1.0
for _ in range(2): K.mpk_baseline(d, y, 6)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); K.mpk_baseline(d, y, 6); e1.record(); e1.synchronize()
print("crs 6 powers ms", e0.elapsed_time(e1))
lens = np.diff(pre.a.row_ptr); print("rows >128:", int((lens > 128).sum()), "nnz in them", int(lens[lens > 128].sum()))
