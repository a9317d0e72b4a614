# scratch driver for gpurun: GPU tests, smoke, one bench line
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
python -c 'import __graft_entry__ as g; g.smoke()' 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['roofline']['frac'], d['kspmv_baseline'])"
