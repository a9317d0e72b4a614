export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_compress.py -x -q 2>&1 | tail -2
echo "== default slots"
SPECS='[[1,2,0,0,0,1,0,0,0],[1,2,0,0,0,1,0,0,1],[1,1,0,0,0,1,0,0,1],[1,1,0,0,1,1,0,0,1],[1,1,0,0,2,1,0,0,1],[8,1,0,0,0,1,0,0,1],[2,1,0,0,0,1,0,0,1],[0,1,0,0,0,1,0,0,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -8
for kb in 160 72; do echo "== slot $kb KB"
LMPK_SLOT_KB=$kb SPECS='[[1,1,0,0,0,1,0,0,1],[1,2,0,0,0,1,0,0,1],[1,3,0,0,0,1,0,0,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -3
done
