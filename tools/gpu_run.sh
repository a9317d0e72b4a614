export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
timeout 600 python bench.py --steps 200 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
sed -i 's/regex:mpk_ring -s 4/regex:mpk_ring -s 4/' tools/profile_round.sh
bash tools/profile_round.sh > /dev/null 2>&1; echo prof done
timeout 900 python tools/configs_full.py 2>&1 | grep case
timeout 900 python tools/cheb_rate.py 2>&1 | tail -1
