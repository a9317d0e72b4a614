"""Event trace of CTAs 0-1 of one cfg2 MPK launch (LMPK_PROFILE + LMPK_TRACE):
prints the per-slot timeline of a steady-state window and per-item phase
statistics."""
import ctypes, os, sys
os.environ["LMPK_PROFILE"] = "1"
os.environ["LMPK_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
N = int(os.environ.get("N", "200")); k = 8
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0] - 1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
ctx = _lib.context()
t = K.Tiling(b, k, slots=int(os.environ.get("SLOTS", "2")), tile_nnz=int(os.environ.get("TILE", "0")),
             mode_flags=int(os.environ.get("MODE_FLAGS", "0")), queue_slack=int(os.environ.get("SLACK", "0")))
print("tiling", t.info)
y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
cfg = K.mpk_power_cfg(k)
flags = int(os.environ.get("FLAGS", "0"))
K.mpk_run(t, y, cfg, flags=flags); torch.cuda.synchronize()
buf = np.zeros((2 * 16384, 4), dtype=np.uint32)
ctx.lib.lmpk_ctx_trace(ctx.handle, buf.ctypes.data_as(ctypes.c_void_p), 2 * 16384)
K.mpk_run(t, y, cfg, flags=flags); torch.cuda.synchronize()
cnt = ctx.lib.lmpk_ctx_trace(ctx.handle, buf.ctypes.data_as(ctypes.c_void_p), 2 * 16384)
ev = buf[:16384]
ev = ev[ev[:, 0] | ev[:, 1] != 0]
tm = (ev[:, 1].astype(np.uint64) << np.uint64(32)) | ev[:, 0].astype(np.uint64)
order = np.argsort(tm)
ev, tm = ev[order], tm[order].astype(np.int64)
tm -= tm[0]
kind = ev[:, 2] & 0xff; slot = (ev[:, 2] >> 8) & 0xff; warp = ev[:, 2] >> 16; item = ev[:, 3]
names = {1: "fetched", 2: "tma_issue", 3: "staged", 4: "deps_ok", 5: "push", 6: "freed", 10: "c_start", 11: "c_end", 12: "c_last"}
print("events", len(ev), "span us", tm[-1] / 1e3)
# steady-state window
mid = tm[-1] // 2
sel = (tm > mid) & (tm < mid + 40000)
for i in np.nonzero(sel)[0][:int(os.environ.get('NEV', '60'))]:
    print(f"{tm[i]/1e3:9.3f} us  slot {slot[i]} warp {warp[i]:2d} {names.get(int(kind[i]), kind[i]):10s} tile {item[i] >> 8:5d} p {item[i] & 255}")
# per-item phase durations (producer view), by (slot, item)
import collections
per = collections.defaultdict(dict)
for i in range(len(ev)):
    key = (int(slot[i]), int(item[i]))
    kd = int(kind[i])
    if kd in (1, 2, 3, 4, 5, 6, 12) and kd not in per[key]:
        per[key][kd] = tm[i]
def stat(a_, b_):
    d = [v[b_] - v[a_] for v in per.values() if a_ in v and b_ in v]
    return (np.mean(d) / 1e3, np.percentile(d, 90) / 1e3, len(d)) if d else None
for a_, b_ in ((1, 2), (2, 3), (2, 4), (3, 5), (4, 5), (5, 12), (12, 6), (5, 6)):
    print(f"{names[a_]:>9s} -> {names[b_]:<9s}: mean/p90 us {stat(a_, b_)}")
