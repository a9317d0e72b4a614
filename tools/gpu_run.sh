export PYTHONDONTWRITEBYTECODE=1
for lib in liblmpk liblmpk_p28 liblmpk_p30; do echo "== $lib"
LMPK_LIB=$PWD/paper_2205_01598_b200/_lib/$lib.so SPECS='[[1,2,0,0,0,1,0,0,1,1],[1,2,0,0,0,1,0,0,1,1]]' timeout 300 python tools/bench_modes.py 2>&1 | tail -2
done
