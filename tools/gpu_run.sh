export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,0,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -3
