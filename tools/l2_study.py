"""cfg2 L2-retention study: tiling geometry, L2/HBM read bandwidth vs buffer
size, flag latency, and one launch per (slack, policy) stream spec (run it
under `ncu --metrics dram__bytes_read.sum,...` to get per-launch traffic)."""
import os, sys, json, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
N = int(os.environ.get("N", "200")); k = int(os.environ.get("K", "8"))
ctx = _lib.context()
if os.environ.get("PROBES", "1") == "1":
    # micro-benchmarks live outside the product library: make -C tools/ubench
    probe = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ubench", "libprobe.so"))
    for mb in (8, 16, 32, 48, 64, 96, 128, 256, 1024):
        g = ctypes.c_double()
        probe.lmpk_probe_read_bw(ctypes.c_void_p(ctx.handle.value if hasattr(ctx.handle, 'value') else ctx.handle), ctypes.c_int64(mb << 20), 20 if mb < 512 else 3, 3, ctypes.byref(g))
        print(f"read bw {mb:5d} MB: {g.value:8.0f} GB/s", flush=True)
    lat = ctypes.c_double()
    probe.lmpk_probe_flag_latency(ctypes.c_void_p(ctx.handle.value if hasattr(ctx.handle, 'value') else ctx.handle), 2000, ctypes.byref(lat))
    print(f"flag latency one-way {lat.value:.0f} ns", flush=True)
rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0] - 1
a = K.DeviceCsr.from_host(rp, c, v)
perm, inv, lp = K.bfs_levels(a, 0)
b = K.permute_symmetric(a, perm, inv)
lvl = np.diff(lp.cpu().numpy() if hasattr(lp, "cpu") else np.asarray(lp))
print("levels", len(lvl), "max rows/level", int(lvl.max()), "n", n, "nnz", int(rp[-1]))
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
specs = json.loads(os.environ.get("SPECS", "[[2,0,0],[2,10,0],[2,37,0],[2,90,0],[2,37,1],[2,37,2],[2,10,1]]"))
for slots, slack, pol in specs:
    t = K.Tiling(b, k, tile_nnz=0, slots=slots, mode_flags=_lib.FLAG_MODE_STREAM, queue_slack=slack)
    cfg = K.mpk_power_cfg(k)
    y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = x
    K.mpk_run(t, y, cfg, flags=pol << 8)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); K.mpk_run(t, y, cfg, flags=pol << 8, check_errors=False); e1.record(); e1.synchronize()
    print(json.dumps(dict(slots=slots, slack=t.info["queue_slack"], pol=pol, info=t.info,
                          ms=round(e0.elapsed_time(e1), 4))), flush=True)
