export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_compress.py -q -x 2>&1 | grep -E "passed|failed|Error|assert" | tail -4
SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,1,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -2
LMPK_SORT=1 SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,1,0,0,1,1],[1,3,0,0,0,1,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -3
