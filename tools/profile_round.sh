#!/bin/bash
# ncu evidence for profiles/: plain run, launch list, one full capture of the
# MPK kernel (run on the GPU box through gpurun; 1 GPU).
set -u
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-clocks"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -20 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 200 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mpk_ring -s 4 -c 1 -f \
    -o gpurun_out/prof_mpk $CMD > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
