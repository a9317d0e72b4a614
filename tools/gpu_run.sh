export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,1,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -2
timeout 900 python tools/cheb_rate.py 2>&1 | tail -1
LMPK_NO_UNIFORM_KERNEL=1 timeout 900 python tools/cheb_rate.py 2>&1 | tail -1
timeout 600 python tools/configs_full.py 2>&1 | grep case | head -2 | tail -1
