export PYTHONDONTWRITEBYTECODE=1
for c in cfg3 cfg5; do
CASE=$c ncu --set full --clock-control none --import-source on -k regex:mpk_ring -s 2 -c 1 -f -o gpurun_out/prof_$c python tools/prof_cfg.py > gpurun_out/ncu_$c.log 2>&1; tail -1 gpurun_out/ncu_$c.log
done
