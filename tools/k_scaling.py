"""MPK time vs k on cfg2 (q = 1 walk) against k tiled sweeps and k CRS SpMVs."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
rp, c, v = O.gen_stencil_3d(int(os.environ.get("N", "200"))); n = rp.shape[0] - 1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1) / reps
for k in (1, 2, 4, 8, 16):
    t = K.Tiling(b, k)
    cfg = K.mpk_power_cfg(k)
    y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
    tm = ev(lambda: K.mpk_run(t, y, cfg, check_errors=False))
    ts = ev(lambda: K.mpk_run(t, y, cfg, flags=_lib.FLAG_SWEEP, check_errors=False))
    tc = ev(lambda: K.mpk_baseline(b, y, k))
    print(f"k={k:2d}: MPK {tm:.3f} ms ({tm/k*1e3:.0f} us/power)  sweep {ts:.3f}  CRS {tc:.3f}  slack {t.info['queue_slack']} D {t.info['max_fwd_reach']}", flush=True)
