"""MPK vs k x CRS SpMV on the other BASELINE shapes (reduced sizes that keep
the per-row structure): cfg3 27-point perturbed, cfg5 Anderson periodic."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
def ev(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); e1.synchronize(); return e0.elapsed_time(e1) / reps
cases = [("cfg3 27pt 128^3", lambda: lm.gen_stencil_3d27pt(128, seed=1), (2, 4, 8, 16)),
         ("cfg5 anderson 128^3", lambda: lm.gen_anderson_3d(128, seed=2), (8,)),
         ("cfg1 5pt 256^2", lambda: lm.gen_laplace_2d5pt(256, 256), (4,))]
for name, gen, ks in cases:
    t0 = time.time(); a = gen(); tg = time.time() - t0
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    d = ap.device()
    for k in ks:
        t = K.Tiling(d, k)
        cfg = K.mpk_power_cfg(k)
        y = torch.zeros(k + 1, a.n_rows, dtype=torch.float64, device="cuda"); y[0] = 1.0
        tm = ev(lambda: K.mpk_run(t, y, cfg, check_errors=False))
        tc = ev(lambda: K.mpk_baseline(d, y, k))
        print(f"{name}: nnz {a.n_nz/1e6:.1f}M k={k:2d}: MPK {tm*1e3:8.1f} us  {2*a.n_nz*k/tm/1e6:6.0f} GF/s   "
              f"k x CRS {tc*1e3:8.1f} us  speedup {tc/tm:.2f}  (tiles {t.info['n_tiles']}, D {t.info['max_fwd_reach']}, gen {tg:.0f}s)", flush=True)
