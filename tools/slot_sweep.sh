#!/bin/bash
# lean walk on cfg2 over slot sizes (KB) x slack: time, DRAM bytes, L1/L2 hit rates
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct
for spec in "$@"; do
  IFS=: read kb slack <<< "$spec"
  LMPK_SLOT_KB=$kb CASES=cfg2 ONLY=lean REPS=10 SLACKS=$slack POLS=0 timeout 300 python tools/lean_ab.py 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$spec', d['tiles'], d['lean_p0'])"
  LMPK_SLOT_KB=$kb CASES=cfg2 ONLY=lean REPS=1 SLACKS=$slack POLS=0 timeout 300 \
    ncu --metrics $M --clock-control none -k regex:mpk_lean -s 4 -c 1 --csv python tools/lean_ab.py > gpurun_out/sw.csv 2>/dev/null
  python - "$spec" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/sw.csv")) if len(r) > 10 and (r[0] == "ID" or r[0].isdigit())]
h = rows[0]; d = {}
for r in rows[1:]:
    d[r[h.index("Metric Name")]] = r[h.index("Metric Value")]
print("   ", {k.split("__")[1][:32]: v for k, v in d.items()})
PY
done
