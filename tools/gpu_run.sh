export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|Error" | tail -3
SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,100,0,1,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -2
timeout 900 python tools/configs_full.py 2>&1 | grep case | head -4
