#!/bin/bash
# DRAM / L2 counters of the lean walk over slack x block-policy x y-policy (one GPU).
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for spec in "$@"; do
  IFS=: read slack pol ypol qp <<< "$spec"
  LMPK_PASS_POWERS=$qp LMPK_YPOL=$ypol CASES=cfg2 ONLY=lean REPS=1 SLACKS=$slack POLS=$pol timeout 300 \
    ncu --metrics $M --clock-control none -k regex:mpk_lean -s 4 -c 1 --csv python tools/lean_ab.py > gpurun_out/sw.csv 2>/dev/null
  python - "$spec" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/sw.csv")) if len(r) > 10 and (r[0] == "ID" or r[0].isdigit())]
h = rows[0]; d = {}
for r in rows[1:]:
    d[r[h.index("Metric Name")]] = (r[h.index("Metric Value")], r[h.index("Metric Unit")])
print(sys.argv[1], {k.split("__")[1][:40]: v for k, v in d.items()})
PY
done
