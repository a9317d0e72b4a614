"""Does the recursively refined permutation (s_m >= 1, groups.py:192-366)
shrink the GPU walk's reuse window?  CASE=cfg3|cfg2, K=4: run_plan timing of
lb_lg_p2p (s_m = 0) against lb_lg_p2p_rec (s_m = 1, 2) with the schedule
forced to the walk, plus the CRS k x SpMV; all results compared bitwise after
undoing the permutations."""
import os, sys, json, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K, executor as E

case = os.environ.get("CASE", "cfg3"); k = int(os.environ.get("K", "4"))
C = float(os.environ.get("CACHE", "126e6"))
n3 = int(os.environ.get("N", "160"))
a = {"cfg3": lambda: lm.gen_stencil_3d27pt(n3, seed=1), "cfg2": lambda: lm.gen_stencil_3d(200, 2, device=True)}[case]()
x = np.random.default_rng(0).uniform(-1, 1, a.n_rows)
os.environ["LMPK_SCHEDULE"] = os.environ.get("SCHED", "walk")


def ev(fn, reps=5):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)


ref = None
for variant, sm in (("lb_lg_p2p", 0), ("lb_lg_p2p_rec", 1), ("lb_lg_p2p_rec", 2)):
    t0 = time.perf_counter()
    pre = lm.prepare(a, variant, k, C, s_m=sm)
    plan = lm.build_plan(pre, variant, 1)
    torch.cuda.synchronize(); tp = time.perf_counter() - t0
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    K.permute_vectors(pre.perm.device()[0], torch.from_numpy(x).cuda().unsqueeze(0), y[0:1])
    launch, sched = E.plan_launcher(plan, y)
    ms = ev(launch)
    til = plan.tiling()
    yb = y.clone(); tb = ev(lambda: K.mpk_baseline(plan.a.device(), yb, k))
    out = torch.empty_like(y); K.permute_vectors(pre.perm.device()[0], y, out, scatter=True)
    same = None if ref is None else bool(torch.equal(out, ref))
    if ref is None: ref = out
    flagged = len(pre.flagged_leaves()); spans = len(pre.tree.spans)
    print(json.dumps({"case": case, "k": k, "variant": variant, "s_m": sm, "walk_ms": round(ms, 4), "crs_ms": round(tb, 4),
                      "sched": sched, "prep_s": round(tp, 3), "items": plan.n_items, "spans": spans, "flagged_left": flagged,
                      "tiles": til.info["n_tiles"], "D": til.info["max_fwd_reach"], "equal_to_s0_after_undo": same}), flush=True)
