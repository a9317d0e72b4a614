"""cfg5 knob sweep: complex Chebyshev step (degree 64 = 8 x k=8) on Anderson
128^3 under ';'-separated ENV=value variants (VARIANTS, '|'-separated); every
result is compared bitwise with the first variant's."""
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200.cheb import ChebCoeffs, cheb_coeffs_schrodinger, gershgorin_bounds
KNOBS = ("LMPK_PASS_POWERS", "LMPK_SUPER_NNZ", "LMPK_SLOT_KB", "LMPK_XLEAN", "LMPK_XLEAN_ROWS", "LMPK_SCHEDULE",
         "LMPK_NO_LEAN", "LMPK_XLEAN_NP", "LMPK_NO_WORKLIST", "LMPK_NO_DP", "LMPK_DP_TILE_KB", "LMPK_DP_PAIR",
         "LMPK_RING_SLACK", "LMPK_LEAN_NP", "LMPK_LEAN_CARVE")
n = int(os.environ.get("N", "128"))
a = lm.gen_anderson_3d(n, seed=2)
lo, hi = gershgorin_bounds(a)
c = cheb_coeffs_schrodinger(8.0, lo, hi).c
c = np.resize(c, 65) if c.size < 65 else c[:65]
coeffs = ChebCoeffs(c=c.astype(np.complex128), dt=8.0, lam_min=lo, lam_max=hi, tol=1e-12)
psi = np.exp(2j * np.pi * np.random.default_rng(0).random(a.n_rows)) / np.sqrt(a.n_rows)
xd = torch.from_numpy(psi).cuda()
flops = 4.0 * a.n_nz * 64
ref = None
for var in os.environ.get("VARIANTS", "LMPK_SCHEDULE=walk|LMPK_SCHEDULE=sweep").split("|"):
    for kn in KNOBS:
        os.environ.pop(kn, None)
    for kv in filter(None, var.split(";")):
        kk, vv = kv.split("=")
        os.environ[kk] = vv
    try:
        prop = lm.ChebPropagator(a, 8.0, coeffs=coeffs, p_m_batch=8, cache_bytes=126e6)
        y = prop.step(xd); torch.cuda.synchronize()
        ts = []
        for _ in range(6):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); y = prop.step(xd); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
        if ref is None:
            ref = y
        til = prop._plan_for[8].tiling(complex_state=True)
        i = til.info if til is not None else {}
        print(json.dumps({"var": var, "ms": round(min(ts), 3), "gflops": round(flops / (min(ts) * 1e-3) / 1e9),
                          "bitwise": bool(torch.equal(y, ref)), "tiles": i.get("n_tiles"), "super": i.get("super_tiles"),
                          "block_MB": round(i.get("block_bytes", 0) / 1e6, 1), "lean_MB": round(i.get("lean_bytes", 0) / 1e6, 1),
                          "dp": i.get("dp_tiles"), "slack": i.get("queue_slack"), "D": i.get("max_fwd_reach"), "xs": i.get("lean_xstaged"), "np": i.get("lean_ring"), "piece": i.get("lean_piece"),
                          "sched": prop._plan_for[8].schedule_choice(True, False)}), flush=True)
        del prop
    except Exception as e:
        print(json.dumps({"var": var, "error": str(e)[:300]}), flush=True)
