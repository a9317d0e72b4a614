"""Turn gpurun_out/{launches.csv, prof_mpk.ncu-rep, plain.log} into the
committed profiles/ summaries (launch list by kernel, ncu summary of the MPK
launch, traffic.json read by bench.py).  Usage: python tools/summarize_profiles.py rNN"""
import collections, csv, io, json, pathlib, re, subprocess, sys
ROOT = pathlib.Path(__file__).resolve().parent.parent
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = ROOT / "profiles"
src = ROOT / "gpurun_out"
# ---- launch list
txt = (src / "launches.csv").read_text()
lines = [l for l in txt.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    if r[mi] == "gpu__time_duration.sum":
        name = re.sub(r"\(.*", "", r[ki]).strip()
        agg[name].append(float(r[vi].replace(",", "")) / 1e3)  # ns -> us
(out / f"{tag}_launches_raw.csv").write_text("\n".join(lines) + "\n")
tot = sum(sum(v) for v in agg.values())
s = io.StringIO()
s.write(f"# {tag} launch list: `python bench.py --steps 3 --warmup 3 --no-cpu-baseline` under\n")
s.write("# ncu --metrics gpu__time_duration.sum --clock-control none -s 0 -c 200 (cold-cache, serialised)\n")
s.write(f"# {sum(len(v) for v in agg.values())} launches, {tot:.1f} us total device time\n")
s.write("kernel,launches,total_us,mean_us,share\n")
for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    s.write(f"{name},{len(v)},{sum(v):.1f},{sum(v) / len(v):.1f},{sum(v) / tot:.3f}\n")
(out / f"{tag}_launches_summary.csv").write_text(s.getvalue())
# ---- full capture of the MPK launch
rep = src / "prof_mpk.ncu-rep"
summ = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
d = dict(zip(rr[0], rr[2]))
def num(k):
    return float(d[k].replace(",", ""))
unit = dict(zip(rr[0], rr[1]))
def to_bytes(k):
    u = unit[k].lower()
    return num(k) * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
dur = num("gpu__time_duration.sum") * ({"usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(unit["gpu__time_duration.sum"], 1e-3))
kname = d.get("Kernel Name", "")
(out / f"{tag}_mpk_ring_kernel_ncu.txt").write_text(
    f"# ncu --set full --clock-control none --import-source on -k regex:mpk_ring -s 4 -c 1 (bench.py cfg2)\n" + summ)
nnz, n, k = 55_760_000, 8_000_000, 8
Q = 12 * nnz + 4 * (n + 1) + 8 * n * (k + 1)
(out / "traffic.json").write_text(json.dumps({
    "round": int(tag[1:]), "kernel": kname, "source": f"ncu --set full --clock-control none, profiles/{tag}_mpk_ring_kernel_ncu.txt",
    "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "dram_bytes_per_launch": int(rd + wr),
    "algorithmic_bytes_per_launch": Q, "ncu_duration_ms": dur}, indent=2) + "\n")
print(s.getvalue()); print(summ); print("traffic", rd + wr, "dur ms", dur)
