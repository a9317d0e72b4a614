"""Event trace of CTA 0 of one cfg2 lean-walk launch (LMPK_PROFILE +
LMPK_TRACE): where a piece's time goes (dependency wait, TMA, consumers)."""
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
t = K.Tiling(b, k, queue_slack=int(os.environ.get("SLACK", "0")))
print("tiling", {x: t.info[x] for x in ("n_tiles", "queue_slack", "max_fwd_reach", "lean_bytes")})
y = torch.zeros(k + 1, b.n, dtype=torch.float64, device="cuda"); y[0] = 1.0
cfg = K.mpk_power_cfg(k)
buf = np.zeros((2 * 16384, 4), dtype=np.uint32)
for _ in range(3):
    ctx.lib.lmpk_ctx_trace(ctx.handle, buf.ctypes.data_as(ctypes.c_void_p), 2 * 16384)
    K.mpk_run(t, y, cfg); torch.cuda.synchronize()
ctx.lib.lmpk_ctx_trace(ctx.handle, buf.ctypes.data_as(ctypes.c_void_p), 2 * 16384)
for cta in (0, 1):
    ev = buf[cta * 16384:(cta + 1) * 16384]
    ev = ev[(ev[:, 0] | ev[:, 1]) != 0]
    tm = ((ev[:, 1].astype(np.uint64) << np.uint64(32)) | ev[:, 0].astype(np.uint64)).astype(np.int64)
    o = np.argsort(tm, kind="stable"); ev, tm = ev[o], tm[o]; tm -= tm[0]
    kind = ev[:, 2] & 0xff; warp = ev[:, 2] >> 16; item = ev[:, 3]
    span = tm[-1] / 1e3
    # per piece (tile, p): tma issue, warp-0 start/end, last-warp time
    pc = {}
    for i in range(len(ev)):
        key = int(item[i]); kd = int(kind[i])
        d = pc.setdefault(key, {})
        if kd == 10 or kd == 11:
            d.setdefault((kd, int(warp[i])), tm[i])
        else:
            d.setdefault(kd, tm[i])
    rows = sorted((d.get(2, 0), key, d) for key, d in pc.items() if 2 in d)
    tma_to_start, busy, gaps, dep = [], [], [], []
    prev_last = None
    for t2, key, d in rows:
        s0 = min(v for kk, v in d.items() if isinstance(kk, tuple) and kk[0] == 10) if any(isinstance(kk, tuple) and kk[0] == 10 for kk in d) else None
        if s0 is None or 12 not in d:
            continue
        tma_to_start.append(s0 - t2)
        busy.append(d[12] - s0)
        if prev_last is not None:
            gaps.append(max(0, s0 - prev_last))
        prev_last = d[12]
    fetch_dep = [pc[key][4] - pc[key][1] for key in pc if 1 in pc[key] and 4 in pc[key]]
    f = lambda v: (round(float(np.mean(v)) / 1e3, 3), round(float(np.percentile(v, 90)) / 1e3, 3)) if len(v) else None
    print(f"CTA {cta}: span {span:.1f} us, pieces {len(busy)}; mean/p90 us: fetch->deps {f(fetch_dep)}, "
          f"tma->start {f(tma_to_start)}, start->last {f(busy)}, gap last->next start {f(gaps)}; "
          f"busy frac {sum(busy) / 1e3 / span:.2f}")
    if cta == 0:
        for t2, key, d in rows[len(rows) // 2: len(rows) // 2 + 12]:
            print("   tile", key >> 8, "p", key & 255, {str(kk): round((v - t2) / 1e3, 2) for kk, v in sorted(d.items(), key=lambda z: z[1])})
