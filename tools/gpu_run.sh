export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_cheb_scale.py -q -x 2>&1 | grep -E "passed|failed|Error|assert" | tail -4
