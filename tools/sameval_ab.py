"""A/B of the fast units / same-value pairs of the lean walk on cfg2 (LMPK_NO_FAST=1, LMPK_NO_SAMEVAL=1),
alternating tilings on one box; bitwise against the CRS baseline."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
a = lm.gen_stencil_3d(int(os.environ.get("N", "200")), 2, device=True)
k = 8
d = a.device()
perm, inv, lp = K.bfs_levels(d, 0)
b = K.permute_symmetric(d, perm, inv)
n = b.n
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
cfg = K.mpk_power_cfg(k)
yb = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); yb[0] = x
K.mpk_baseline(b, yb, k)
til = {}
for name, env in (("fast", {}), ("fast_novrow", {"LMPK_NO_VROW": "1"}), ("sameval_only", {"LMPK_NO_FAST": "1"}), ("off", {"LMPK_NO_SAMEVAL": "1"})):
    for kk in ("LMPK_NO_SAMEVAL", "LMPK_NO_FAST", "LMPK_NO_VROW"): os.environ.pop(kk, None)
    os.environ.update(env)
    til[name] = K.Tiling(b, k)
for kk in ("LMPK_NO_SAMEVAL", "LMPK_NO_FAST", "LMPK_NO_VROW"): os.environ.pop(kk, None)
y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = x
res = {kk: [] for kk in til}
for rnd in range(6):
    for name, t in til.items():
        for _ in range(3): K.mpk_run(t, y, cfg, check_errors=False)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): K.mpk_run(t, y, cfg, check_errors=False)
        e1.record(); e1.synchronize()
        res[name].append(e0.elapsed_time(e1) / 50)
        assert torch.equal(y, yb), name
print(json.dumps({kk: [round(v, 4) for v in vs] for kk, vs in res.items()}))
