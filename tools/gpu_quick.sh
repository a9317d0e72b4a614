# quick GPU loop: lean/walk parity tests + one bench line (cfg2 unless CFG is set)
export PYTHONDONTWRITEBYTECODE=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_walk.py tests/test_gpu_compress.py tests/test_gpu_parity.py tests/test_gpu_cheb_scale.py -m gpu -q -x 2>&1 | tail -8
for cfg in ${CFGS:-cfg2}; do
  timeout 600 python bench.py --config $cfg --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline > gpurun_out/q_$cfg.json 2> gpurun_out/q_$cfg.err
  python -c "
import json
try:
  d=json.loads(open('gpurun_out/q_$cfg.json').read().strip().splitlines()[-1])
  print('$cfg', 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['config'], d.get('kspmv_baseline'), 'bit', d.get('bitwise_vs_baseline'), 'prep', d.get('preprocess'))
except Exception as e: print('ERR', e, open('gpurun_out/q_$cfg.err').read()[-1500:])
"
done
