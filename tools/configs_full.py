"""MPK on the BASELINE.json shapes at full size (cfg3 27-pt 160^3 perturbed,
cfg5 Anderson 128^3, cfg4 R-MAT scale 22 when CFG4=1, cfg1 5-pt 256^2):
the default plan (ring walk, compressed tiles) and the round-1 group walk on
plain blocks, against k x CRS SpMV on the same GPU; bitwise check vs CRS."""
import os, sys, time, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K, _lib
def ev(fn, reps=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
cases = [("cfg1 5pt 256^2", lambda: lm.gen_laplace_2d5pt(256, 256), (4,)),
         ("cfg5 anderson 128^3", lambda: lm.gen_anderson_3d(128, seed=2), (8,)),
         ("cfg3 27pt 160^3", lambda: lm.gen_stencil_3d27pt(160, seed=1), (2, 4, 8, 16))]
if os.environ.get("CFG4"):
    cases.append(("cfg4 rmat s22", lambda: lm.gen_rmat(22), (6,)))
for name, gen, ks in cases:
    t0 = time.time(); a = gen(); tg = time.time() - t0
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    d = ap.device()
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, a.n_rows)).cuda()
    for k in ks:
        cfg = K.mpk_power_cfg(k)
        yb = torch.zeros(k + 1, a.n_rows, dtype=torch.float64, device="cuda"); yb[0] = x
        tc = ev(lambda: K.mpk_baseline(d, yb, k))
        out = {"case": name, "nnz": a.n_nz, "k": k, "crs_us": round(tc * 1e3, 1), "gen_s": round(tg)}
        for plan, fl, rf in (("ring", 0, 0), ("ring_tiles_sweep", 0, _lib.FLAG_SWEEP),
                             ("group_plain", _lib.FLAG_MODE_STREAM, 0)):
            t = K.Tiling(d, k, mode_flags=fl, **({"queue_slack": int(os.environ["SLACK"])} if os.environ.get("SLACK") else {}),
                         **({"tile_nnz": int(os.environ["RUN"])} if os.environ.get("RUN") and fl == 0 else {}))
            y = torch.zeros_like(yb); y[0] = x
            tm = ev(lambda: K.mpk_run(t, y, cfg, flags=rf, check_errors=False))
            K.mpk_run(t, y, cfg, flags=rf)
            out[plan] = {"us": round(tm * 1e3, 1), "gflops": round(2 * a.n_nz * k / tm / 1e6),
                         "speedup_vs_crs": round(tc / tm, 2), "bitwise": bool(torch.equal(y, yb)),
                         "tiles": t.info["n_tiles"], "dict_tiles": t.info["dict_tiles"],
                         "block_MB": round(t.info["block_bytes"] / 1e6)}
            del t
        print(json.dumps(out), flush=True)
