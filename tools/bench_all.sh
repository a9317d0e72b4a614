#!/bin/bash
# One bench line per BASELINE config (gpurun, 1 GPU): gpurun_out/bench_<cfg>.json
mkdir -p gpurun_out
STEPS=${STEPS:-50}
for cfg in ${CONFIGS:-cfg2 cfg1 cfg3 cfg4 cfg5 cfg3-k2 cfg3-k4 cfg3-k16}; do
  timeout 900 python bench.py --config $cfg --steps $STEPS --warmup 5 $EXTRA > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
  echo "$cfg rc=$? $(python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/bench_$cfg.json').read().strip().splitlines()[-1])
  print(round(d['value'],1), d['unit'], 'ms', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), 'sched', d['config'].get('schedule'), 'e2e', round(d['e2e']['value'],1), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'ks', (d.get('kspmv_baseline') or {}).get('speedup_vs_crs'), 'bit', d.get('bitwise_vs_baseline'), (d.get('cpu_baseline') or {}).get('bitwise_gpu_vs_cpu', (d.get('cpu_baseline') or {}).get('gpu_vs_cpu_rel_l2')))
except Exception as e: print('ERR', e, open('gpurun_out/bench_$cfg.err').read()[-600:])
")"
done
