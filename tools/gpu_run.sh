export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed" | tail -2
timeout 900 python tools/cheb_rate.py 2>&1 | tail -1
