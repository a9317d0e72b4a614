#!/bin/bash
# DRAM bytes and duration per Chebyshev batch launch of cfg5 under tiling knobs
# (ncu, three metrics; gpurun, 1 GPU).  Usage: bash tools/dp_traffic.sh "VAR1" "VAR2" ...
mkdir -p gpurun_out
for v in "$@"; do
  tag=$(echo "$v" | tr -c 'A-Za-z0-9=\n' '_')
  VARIANTS="$v" timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:mpk_ -s 16 -c 24 --csv --log-file gpurun_out/traffic_$tag.csv \
    python tools/cfg5_sweep.py > /dev/null 2>&1
  python - "$v" gpurun_out/traffic_$tag.csv <<'P'
import csv, sys, io, collections
rows = list(csv.reader(l for l in open(sys.argv[2]) if l.startswith('"')))
h = rows[0]; mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}
for r in rows[1:]:
    agg[r[mi]].append(float(r[vi].replace(",", "")) * mult.get(r[ui], 1))
m = {k: sum(v) / len(v) for k, v in agg.items()}
print(sys.argv[1], "launches", len(agg["gpu__time_duration.sum"]), "us %.1f" % m["gpu__time_duration.sum"],
      "read MB %.0f write MB %.0f" % (m["dram__bytes_read.sum"] / 1e6, m["dram__bytes_write.sum"] / 1e6))
P
done
