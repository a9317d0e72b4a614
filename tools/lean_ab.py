"""A/B of the lean ring walk against the general ring kernel on BASELINE
shapes (cfg2 by default; CASES=cfg2,cfg5,cfg1): bitwise check against the CRS
k x SpMV baseline, CUDA-event timing (min / mean of REPS calls)."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K, _lib

REPS = int(os.environ.get("REPS", "20"))


def ev(fn, reps=REPS):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts), sum(ts) / len(ts)


gens = {"cfg2": (lambda: lm.gen_stencil_3d(200, 2, device=True), 8),
        "cfg5": (lambda: lm.gen_anderson_3d(128, seed=2), 8),
        "cfg1": (lambda: lm.gen_laplace_2d5pt(256, 256), 4),
        "small": (lambda: lm.gen_stencil_3d(40, 2), 8)}
for name in os.environ.get("CASES", "cfg2").split(","):
    gen, k = gens[name]
    a = gen()
    d = a.device()
    perm, inv, lp = K.bfs_levels(d, 0)
    b = K.permute_symmetric(d, perm, inv)
    n, nnz = b.n, b.nnz
    x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    cfg = K.mpk_power_cfg(k)
    yb = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); yb[0] = x
    K.mpk_baseline(b, yb, k)
    tc = ev(lambda: K.mpk_baseline(b, yb, k))
    for slack, qp in [(int(v.split(":")[0]), v.split(":")[1] if ":" in v else "") for v in os.environ.get("SLACKS", "0").split(",")]:
        if qp:
            os.environ["LMPK_PASS_POWERS"] = qp
        else:
            os.environ.pop("LMPK_PASS_POWERS", None)
        t = K.Tiling(b, k, queue_slack=slack)
        out = {"case": name, "n": n, "nnz": nnz, "k": k, "crs_ms": round(tc[0], 4), "tiles": t.info["n_tiles"],
               "lean_MB": round(t.info["lean_bytes"] / 1e6, 1), "pat_tiles": t.info["lean_pattern_tiles"], "block_MB": round(t.info["block_bytes"] / 1e6, 1),
               "slack": t.info["queue_slack"], "qp": qp, "D": t.info["max_fwd_reach"]}
        qro = 12 * nnz + 4 * (n + 1) + 8 * n * (k + 1)
        arms = (("ring", "1"), ("lean", None))
        if os.environ.get("ONLY"):
            arms = [a for a in arms if a[0] == os.environ["ONLY"]]
        for tag, env in arms:
            if env:
                os.environ["LMPK_NO_LEAN_RUN"] = env
            else:
                os.environ.pop("LMPK_NO_LEAN_RUN", None)
            for pol in [int(p) for p in os.environ.get("POLS", "0").split(",")]:
                y = torch.zeros_like(yb); y[0] = x
                f = pol << 8
                tm = ev(lambda: K.mpk_run(t, y, cfg, flags=f, check_errors=False, exact=True))
                y.zero_(); y[0] = x
                K.mpk_run(t, y, cfg, flags=f, exact=True)
                out[f"{tag}_p{pol}"] = {"ms": round(tm[0], 4), "mean": round(tm[1], 4),
                                        "frac": round(qro / (tm[0] * 1e-3) / 6440.7e9, 3),
                                        "bitwise": bool(torch.equal(y, yb))}
        os.environ.pop("LMPK_NO_LEAN_RUN", None)
        print(json.dumps(out), flush=True)
