"""Sweep of the staged lean walk's knobs on a BASELINE shape (CASE=cfg2|cfg5|cfg1|small):
each VARIANTS entry is a ';'-separated list of ENV=value settings applied
before the tiling is built; bitwise check against the CRS baseline and
CUDA-event timing (min / mean of REPS calls)."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K

REPS = int(os.environ.get("REPS", "30"))
KNOBS = ("LMPK_ACQ", "LMPK_XLEAN_CTAS", "LMPK_XLEAN", "LMPK_XP", "LMPK_XLEAN_PUB", "LMPK_NO_WORKLIST", "LMPK_LEAN_NP", "LMPK_NO_XP", "LMPK_XP_LIMIT", "LMPK_XP_RUN", "LMPK_NO_XLEAN", "LMPK_XLEAN_ROWS", "LMPK_XLEAN_NP", "LMPK_XLEAN_PAIR", "LMPK_SUPER_NNZ", "LMPK_LEAN_CARVE",
         "LMPK_PASS_POWERS", "LMPK_NO_PATTERN")


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
name = os.environ.get("CASE", "cfg2")
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
qro = 12 * nnz + 4 * (n + 1) + 8 * n * (k + 1)
for var in os.environ.get("VARIANTS", "LMPK_NO_XLEAN=1|").split("|"):
    for kn in KNOBS:
        os.environ.pop(kn, None)
    for kv in filter(None, var.split(";")):
        kk, vv = kv.split("=")
        os.environ[kk] = vv
    t = K.Tiling(b, k, queue_slack=int(os.environ.get("SLACK", "0")))
    y = torch.zeros_like(yb); y[0] = x
    tm = ev(lambda: K.mpk_run(t, y, cfg, check_errors=False, exact=True))
    y.zero_(); y[0] = x
    K.mpk_run(t, y, cfg, exact=True)
    i = t.info
    print(json.dumps({"case": name, "var": var, "ms": round(tm[0], 4), "mean": round(tm[1], 4),
                      "frac": round(qro / (tm[0] * 1e-3) / 6546.6e9, 3), "bitwise": bool(torch.equal(y, yb)),
                      "tiles": i["n_tiles"], "super": i["super_tiles"], "lean_MB": round(i["lean_bytes"] / 1e6, 1),
                      "xs": i["lean_xstaged"], "np": i["lean_ring"], "piece": i["lean_piece"], "slack": i["queue_slack"],
                      "D": i["max_fwd_reach"]}), flush=True)
    t.close()
