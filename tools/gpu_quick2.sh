export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
for cfg in cfg4 cfg2; do
  timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/q_$cfg.json 2> gpurun_out/q_$cfg.err
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/q_$cfg.json').read().strip().splitlines()[-1])
  print('$cfg', 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['config'].get('schedule'), d.get('kspmv_baseline'), 'bit', d.get('bitwise_vs_baseline'), 'prep', d.get('preprocess'))
except Exception as e: print('ERR', e, open('gpurun_out/q_$cfg.err').read()[-1500:])
"
done
