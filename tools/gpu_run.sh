export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_compress.py -x -q -k "oversize or hub or schedule" 2>&1 | grep -E "passed|failed|Error|assert" | tail -5
