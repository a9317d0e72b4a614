"""cfg2 timing of MPK plans: SPECS is a JSON list of
[q, slots, tile_nnz, slack, policy, exact, no_tma, ready_queue, compress, ring]; q = 0 -> sweep."""
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
specs = json.loads(os.environ.get("SPECS", '[[1,2,0,0,0,0],[2,2,0,0,0,0],[8,2,0,0,0,0],[0,2,0,0,0,0]]'))
for spec in specs:
    q, slots, tile, slack, polf, exact, notma, ko, comp, ring = (list(spec) + [0] * 10)[:10]
    try:
        fl = (_lib.FLAG_MODE_RESIDENT if q == k else _lib.FLAG_MODE_STREAM) | (_lib.FLAG_NO_TMA if notma else 0) | (_lib.FLAG_COMPRESS if comp else 0) | (_lib.FLAG_RING if ring else 0)
        t = K.Tiling(b, k, tile_nnz=tile, slots=slots, mode_flags=fl, queue_slack=slack, group=max(q, 1))
        cfg = K.mpk_power_cfg(k)
        y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = x
        f = (_lib.FLAG_SWEEP if q == 0 else 0) | (polf << 8) | (_lib.FLAG_NO_TMA if notma else 0) | (_lib.FLAG_READY_QUEUE if ko else 0)
        run = lambda: K.mpk_run(t, y, cfg, flags=f, check_errors=False, exact=bool(exact))
        tmin, tmean = ev_time(run)
        K.mpk_run(t, y, cfg, flags=f, exact=True)
        if ref is None: ref = y.clone()
        K.mpk_run(t, y, cfg, flags=f, exact=bool(exact))
        err = float(max(((y[i] - ref[i]).norm() / ref[i].norm()).item() for i in range(1, k + 1)))
        print(json.dumps(dict(q=q, ring=ring, st=t.info['super_tiles'], ko=ko, comp=comp, xst=t.info["x_staged_tiles"], ctiles=t.info['compressed_tiles'], dtiles=t.info['dict_tiles'], mb=round(t.info['block_bytes']/1e6), notma=notma, slots=t.info["slots"], pol=polf, exact=exact, slack=t.info["queue_slack"],
              tile=t.info["tile_nnz_cap"], n_tiles=t.info["n_tiles"], D=t.info["max_fwd_reach"],
              ms=round(tmin, 4), ms_mean=round(tmean, 4), gflops=round(F / tmin / 1e6),
              ro_frac=round(Q_ro / (tmin * 1e-3) / 6531.6e9, 4), rel_err=err)), flush=True)
    except Exception as e:
        print(json.dumps(dict(spec=spec, err=str(e)[:300])), flush=True)
