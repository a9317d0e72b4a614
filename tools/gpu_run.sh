export PYTHONDONTWRITEBYTECODE=1
SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,1,0,0,1,1],[1,3,0,0,0,1,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -3
