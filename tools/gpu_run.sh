export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SPECS='[[1,2,0,0,2,1,0,0,1,1],[1,3,0,0,2,1,0,0,1,1],[1,2,0,110,2,1,0,0,1],[1,2,0,160,2,1,0,0,1],[1,2,0,0,2,0,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -5
python tools/probe_c.py 2>&1 | grep "R 2" | head -8
