"""cfg2 timing of the MPK modes for the library selected by LMPK_LIB."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
N = int(os.environ.get("N", "200")); k = int(os.environ.get("K", "8"))
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0] - 1; nnz = int(rp[-1])
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
Q_ro = 12 * nnz + 4 * (n + 1) + 8 * n * (k + 1); F = 2 * nnz * k
def ev_time(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts), sum(ts) / len(ts)
ref = None
specs = json.loads(os.environ.get("SPECS", '[["res",2,0],["stream",2,0],["sweep",2,0]]'))
for mode, slots, tile in specs:
    fl = _lib.FLAG_MODE_RESIDENT if mode == "res" else _lib.FLAG_MODE_STREAM
    try:
        t = K.Tiling(b, k, tile_nnz=tile, slots=slots, mode_flags=fl)
        cfg = K.mpk_power_cfg(k)
        y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = x
        f = _lib.FLAG_SWEEP if mode == "sweep" else 0
        tmin, tmean = ev_time(lambda: K.mpk_run(t, y, cfg, flags=f, check_errors=False))
        K.mpk_run(t, y, cfg, flags=f)
        if ref is None: ref = y.clone()
        print(json.dumps(dict(lib=os.path.basename(os.environ.get("LMPK_LIB", "default")), mode=mode, slots=slots,
              tile=t.info["tile_nnz_cap"], n_tiles=t.info["n_tiles"], ms=round(tmin, 4), ms_mean=round(tmean, 4),
              gflops=round(F / tmin / 1e6), ro_frac=round(Q_ro / (tmin * 1e-3) / 6531.6e9, 4),
              bitwise=bool(torch.equal(y, ref)))), flush=True)
    except Exception as e:
        print(json.dumps(dict(mode=mode, slots=slots, err=str(e)[:200])), flush=True)
