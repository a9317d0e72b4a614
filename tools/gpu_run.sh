export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
python - <<'PY'
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2205_01598_b200 as lm
for name, gen in (("cfg3", lambda: lm.gen_stencil_3d27pt(160, seed=1)), ("cfg2", lambda: lm.gen_stencil_3d(200, 2)), ("cfg5", lambda: lm.gen_anderson_3d(128, seed=2))):
    a = gen()
    pre = lm.prepare(a, "lb_lg_p2p", 8, 126e6)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    x = torch.rand(a.n_rows, dtype=torch.float64, device="cuda")
    res = lm.run_plan(plan, x=x)
    ts = [lm.run_plan(plan, x=x).seconds for _ in range(5)]
    print(name, "choice", plan.schedule_choice(False), "run_plan min s", round(min(ts) * 1e3, 3), "ms")
PY
