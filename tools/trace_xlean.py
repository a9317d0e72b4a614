"""Per-warp event trace of CTA 0 of one staged lean-walk launch on cfg2
(LMPK_TRACE): per piece, every consumer warp's busy time and the hand-offs."""
import ctypes, os, sys
os.environ["LMPK_PROFILE"] = "1"
os.environ["LMPK_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import kernels as K, _lib
k = 8
a = lm.gen_stencil_3d(int(os.environ.get("N", "200")), 2, device=True).device()
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
ctx = _lib.context()
t = K.Tiling(b, k)
print("tiling", t.info)
y = torch.zeros(k + 1, b.n, dtype=torch.float64, device="cuda"); y[0] = 1.0
cfg = K.mpk_power_cfg(k)
NE = 2 * 16384
buf = np.zeros((NE, 4), dtype=np.uint32)
for _ in range(3):
    ctx.lib.lmpk_ctx_trace(ctx.handle, buf.ctypes.data_as(ctypes.c_void_p), NE)
    K.mpk_run(t, y, cfg); torch.cuda.synchronize()
ctx.lib.lmpk_ctx_trace(ctx.handle, buf.ctypes.data_as(ctypes.c_void_p), NE)
ev = buf[:16384]
ev = ev[(ev[:, 0] | ev[:, 1]) != 0]
tm = ((ev[:, 1].astype(np.uint64) << np.uint64(32)) | ev[:, 0].astype(np.uint64)).astype(np.int64)
o = np.argsort(tm, kind="stable"); ev, tm = ev[o], tm[o]; tm -= tm[0]
kind = ev[:, 2] & 0xff; warp = ev[:, 2] >> 16; item = ev[:, 3]
print("events", len(ev), "span us", tm[-1] / 1e3)
pieces = {}
for i in range(len(ev)):
    d = pieces.setdefault(int(item[i]), {"s": {}, "e": {}})
    kd = int(kind[i])
    if kd == 10: d["s"][int(warp[i])] = tm[i]
    elif kd == 11: d["e"][int(warp[i])] = tm[i]
    else: d.setdefault(kd, tm[i])
rows = sorted((d[2], key, d) for key, d in pieces.items() if 2 in d and len(d["e"]) >= 20)
busy = []; spans = []; starts = []
for t2, key, d in rows:
    ws = sorted(d["e"])
    dur = np.array([d["e"][w] - d["s"][w] for w in ws if w in d["s"]])
    busy.append(dur)
    spans.append(max(d["e"].values()) - min(d["s"].values()))
    starts.append(max(d["s"].values()) - min(d["s"].values()))
allb = np.concatenate(busy)
print("pieces", len(rows), "per-warp busy us: mean %.3f p50 %.3f p90 %.3f max %.3f" % (allb.mean() / 1e3, np.percentile(allb, 50) / 1e3, np.percentile(allb, 90) / 1e3, allb.max() / 1e3))
print("piece span (first start -> last end) mean %.3f; start skew mean %.3f; max-warp busy mean %.3f" % (np.mean(spans) / 1e3, np.mean(starts) / 1e3, np.mean([b.max() for b in busy]) / 1e3))
for t2, key, d in rows[len(rows) // 2: len(rows) // 2 + 4]:
    ws = sorted(d["e"])
    print(" tile", key >> 8, "p", key & 255, "tma@0 deps", d.get(4, 0) - t2, "start", [round((d["s"][w] - t2) / 1e3, 2) for w in ws], "dur", [round((d["e"][w] - d["s"][w]) / 1e3, 2) for w in ws], "pub", round((d.get(12, 0) - t2) / 1e3, 2))
# slot turnaround: publish of piece k -> TMA issue of piece k + ring depth
NP = t.info["lean_ring"]
iss = np.array([r[0] for r in rows]); pub = np.array([r[2].get(12, 0) for r in rows])
first = np.array([1 if 4 in r[2] else 0 for r in rows])
dep = np.array([r[2].get(4, r[0]) - r[2].get(1, r[0]) for r in rows])
if len(rows) > NP + 5:
    refill = iss[NP:] - pub[:-NP]
    print("ring", NP, "refill delay (publish k -> issue k+NP) us: mean %.3f p10 %.3f p50 %.3f p90 %.3f" % (refill.mean() / 1e3, np.percentile(refill, 10) / 1e3, np.percentile(refill, 50) / 1e3, np.percentile(refill, 90) / 1e3))
    d = np.diff(iss)
    print("issue-to-issue us: mean %.3f p50 %.3f p90 %.3f; deps wait of first pieces mean %.3f" % (d.mean() / 1e3, np.percentile(d, 50) / 1e3, np.percentile(d, 90) / 1e3, dep[first == 1].mean() / 1e3))
    full = np.array([min(r[2]["s"].values()) - r[0] for r in rows])
    print("issue -> first warp start mean %.3f p10 %.3f; first start -> publish mean %.3f" % (full.mean() / 1e3, np.percentile(full, 10) / 1e3, (pub - np.array([min(r[2]['s'].values()) for r in rows])).mean() / 1e3))
    k0 = len(rows) // 2
    for k in range(k0, k0 + 9):
        r = rows[k]
        print("  piece", k, "tile", r[1] >> 8, "p", r[1] & 255, "issue %.2f" % (r[0] / 1e3), "deps@ %.2f" % (r[2].get(4, 0) / 1e3), "fetch@ %.2f" % (r[2].get(1, 0) / 1e3), "firststart %.2f laststart %.2f lastend %.2f pub %.2f" % (min(r[2]["s"].values()) / 1e3, max(r[2]["s"].values()) / 1e3, max(r[2]["e"].values()) / 1e3, r[2].get(12, 0) / 1e3))
