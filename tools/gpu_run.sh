export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
python tools/prof_cfg4.py 2>&1 | tail -2
SCALE=22 timeout 1500 python tools/cfg4_run.py 2>&1 | tail -1
timeout 600 python tools/configs_full.py 2>&1 | grep case | head -2
