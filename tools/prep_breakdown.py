"""Where cfg2 preprocessing time goes (GPU box): prepare (BFS, groups,
permutation), build_plan, tiling."""
import os, sys, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K
import cProfile, pstats
a = lm.gen_stencil_3d(int(os.environ.get("N", "200")), 2, device=bool(int(os.environ.get("DEV", "1"))))
lm.warmup(); torch.cuda.synchronize()
def run():
    t0 = time.perf_counter(); pre = lm.prepare(a, "lb_lg_p2p", 8, 126e6); torch.cuda.synchronize(); t1 = time.perf_counter()
    plan = lm.build_plan(pre, "lb_lg_p2p", 1); t2 = time.perf_counter()
    til = plan.tiling(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"prepare {t1-t0:.3f}s build_plan {t2-t1:.3f}s tiling {t3-t2:.3f}s", flush=True)
run()
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
