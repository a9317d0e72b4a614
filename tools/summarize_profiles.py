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
# ---- one full capture per config: the dominant kernel of one steady-state step
CFG = {  # n, nnz, algorithmic bytes per launch of the dominant kernel
    "cfg1": (65_536, 326_656, lambda n, z: 12 * z + 4 * (n + 1) + 8 * n * 5),
    "cfg2": (8_000_000, 55_760_000, lambda n, z: 12 * z + 4 * (n + 1) + 8 * n * 9),
    "cfg3": (4_096_000, 109_215_352, lambda n, z: 12 * z + 4 * (n + 1) + 8 * n * 9),
    "cfg4": (4_194_304, 69_438_612, lambda n, z: 12 * z + 4 * (n + 1) + 16 * n),
    "cfg5": (2_097_152, 14_680_064, lambda n, z: 12 * z + 4 * (n + 1) + 16 * n * 6),
}
traffic = {"round": int(tag[1:])}
allsumm = ""
for rep in sorted(src.glob("prof_cfg*.ncu-rep")):
    cfg = rep.stem.split("_", 1)[1]
    summ = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep)],
                          capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) < 3:
        continue
    d = dict(zip(rr[0], rr[2]))
    unit = dict(zip(rr[0], rr[1]))

    def num(k):
        return float(d[k].replace(",", ""))

    def to_bytes(k):
        return num(k) * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(unit[k].lower(), 1)

    rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
    dur = num("gpu__time_duration.sum") * {"usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6}.get(
        unit["gpu__time_duration.sum"], 1e-3)
    n, z, qf = CFG[cfg]
    fn = f"{tag}_{cfg}_ncu.txt"
    (out / fn).write_text(
        f"# ncu --set full --clock-control none --import-source on --profile-from-start off -c 1:\n"
        f"# the dominant kernel of one steady-state step of `python bench.py --config {cfg} --profile-step`\n" + summ)
    traffic[cfg] = {"kernel": d.get("Kernel Name", ""), "source": f"profiles/{fn}",
                    "dram_read_bytes": int(rd), "dram_write_bytes": int(wr), "dram_bytes_per_launch": int(rd + wr),
                    "algorithmic_bytes_per_launch": qf(n, z), "ncu_duration_ms": dur}
    allsumm += f"== {cfg}\n{summ}\n"
(out / "traffic.json").write_text(json.dumps(traffic, indent=2) + "\n")
print(s.getvalue()); print(allsumm); print(json.dumps(traffic, indent=1))
