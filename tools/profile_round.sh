#!/bin/bash
# ncu evidence for profiles/ (GPU box through gpurun; 1 GPU):
#   * launch list of the default bench command (cfg2)
#   * one `ncu --set full` capture of the dominant kernel of ONE steady-state
#     step per config (bench.py --profile-step + --profile-from-start off)
# then `python tools/summarize_profiles.py rNN` here.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
for cfg in ${PROF_CONFIGS:-cfg2 cfg5 cfg1 cfg3 cfg4}; do
  case $cfg in
    cfg4) K='regex:spmv_rows' ;;
    *) K='regex:mpk_(lean|ring|group)_kernel|spmv_rows_kernel' ;;
  esac
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k "$K" -c 1 -f \
      -o gpurun_out/prof_$cfg $CMD --config $cfg --profile-step > gpurun_out/ncu_full_$cfg.log 2>&1
  echo "ncu $cfg rc=$?"
done
