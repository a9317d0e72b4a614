"""BASELINE config 4 end to end on one GPU: R-MAT scale 22 (a=.57, b=c=.19,
d=.05, seed 1, 8 edges/vertex, symmetrised, self-loops, row-normalised),
device BFS levels + permutation, then run_mpk k=6 through the public API
(the plan runs as CRS sweeps: hub rows exceed the tile format)."""
import os, sys, time, json, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
scale = int(os.environ.get("SCALE", "22"))
t0 = time.time(); a = lm.gen_rmat(scale); tg = time.time() - t0
lm.warmup(); torch.cuda.synchronize()
t0 = time.perf_counter(); pre = lm.prepare(a, "lb_lg_p2p", 6, 126e6); torch.cuda.synchronize(); tp = time.perf_counter() - t0
plan = lm.build_plan(pre, "lb_lg_p2p", 1)
x = torch.from_numpy(np.random.default_rng(0).uniform(0, 1, a.n_rows)).cuda()
res = lm.run_plan(plan, x=x)
ts = [lm.run_plan(plan, x=x).seconds for _ in range(3)]
base = lm.run_baseline(pre.a, x, 6)
same = bool(torch.equal(res.y.data, base.y.data))
lens = np.diff(a.row_ptr)
print(json.dumps({"case": f"cfg4 rmat scale {scale}", "n": a.n_rows, "nnz": a.n_nz, "max_row": int(lens.max()),
                  "levels": int(pre.levels.n_levels), "gen_s": round(tg, 1), "prepare_s": round(tp, 3),
                  "mpk_ms": round(min(ts) * 1e3, 2), "gflops": round(2 * a.n_nz * 6 / min(ts) / 1e9, 1),
                  "tiling": "crs fallback" if plan.tiling() is None else "tiles",
                  "bitwise_vs_run_baseline": same}))
