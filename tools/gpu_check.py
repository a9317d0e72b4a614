"""First GPU session: probes, bitwise parity of every kernel, cfg2 timings."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K
from paper_2205_01598_b200 import _lib
from oracle import levelmpk_oracle as O

def ev_time(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts), sum(ts)/len(ts)

out = {}
ctx = K.context()
print("device", torch.cuda.get_device_name(), "SMs", ctx.sm_count, "smem/blk", ctx.max_smem_block, "smem/sm", ctx.max_smem_sm, "L2", ctx.l2_bytes)
for mb in ([] if os.environ.get("NOPROBE") else (8, 32, 64, 96)):
    g = K.probe_read_bw(mb << 20, reps=50, trials=5); out[f"read_bw_{mb}MB"] = g; print(f"read bw {mb} MB: {g:.0f} GB/s")
g = 0 if os.environ.get("NOPROBE") else K.probe_read_bw(4 << 30, reps=1, trials=5); out["read_bw_4GB"] = g; print(f"read bw 4 GB: {g:.0f} GB/s")
lat = 0 if os.environ.get("NOPROBE") else K.probe_flag_latency(20000); out["flag_one_way_ns"] = lat; print(f"flag one-way latency {lat:.0f} ns")

def check_matrix(name, rp, c, v, p_m=8, root=0):
    n = rp.shape[0] - 1
    a = K.DeviceCsr.from_host(rp, c, v)
    perm, inv, lp = K.bfs_levels(a, root)
    o_perm, o_lp = O.bfs_levels(rp, c, root, method="keysort")
    ok_bfs = np.array_equal(perm.cpu().numpy(), o_perm) and np.array_equal(lp, o_lp)
    b = K.permute_symmetric(a, perm, inv)
    orp, oc, ov = O.permute_symmetric(rp, c, v, o_perm)
    hb = b.to_host()
    ok_perm = np.array_equal(hb[0], orp) and np.array_equal(hb[1], oc) and np.array_equal(hb[2], ov)
    x = np.random.default_rng(0).uniform(-1, 1, n)
    ref = O.mpk_powers(orp, oc, ov, x, p_m)
    y = torch.zeros(p_m + 1, n, dtype=torch.float64, device="cuda"); y[0] = torch.from_numpy(x)
    K.mpk_baseline(b, y, p_m)
    ok_base = np.array_equal(y.cpu().numpy(), ref)
    res = {"bfs": ok_bfs, "permute": ok_perm, "baseline": ok_base, "levels": len(lp) - 1}
    for mode, fl in (("resident", _lib.FLAG_MODE_RESIDENT), ("streaming", _lib.FLAG_MODE_STREAM)):
        try:
            t = K.Tiling(b, p_m, mode_flags=fl)
            y3 = torch.zeros_like(y); y3[0] = y[0]
            K.mpk_run(t, y3, K.mpk_power_cfg(p_m), flags=_lib.FLAG_SWEEP)
            res[mode + "_sweep"] = bool(np.array_equal(y3.cpu().numpy(), ref))
            y2 = torch.zeros_like(y); y2[0] = y[0]
            K.mpk_run(t, y2, K.mpk_power_cfg(p_m))
            res[mode] = bool(np.array_equal(y2.cpu().numpy(), ref))
            res[mode + "_info"] = t.info
        except Exception as e:
            res[mode] = f"ERR {e}"
    print(name, json.dumps(res))
    return res

rp, c, v = O.gen_stencil_3d(24); out["s24"] = check_matrix("3d-24", rp, c, v)
rp, c, v = O.gen_stencil_2d7pt(64, 64); out["2d64"] = check_matrix("2d7pt-64", rp, c, v, p_m=5)
rng = np.random.default_rng(3)
n = 3000; m = 5000; r = rng.integers(0, n, m); cc = rng.integers(0, n, m)
rp, c, v = O.from_triplets(n, np.concatenate([r, np.arange(n)]), np.concatenate([cc, np.arange(n)]), rng.standard_normal(m + n))
out["rand_asym"] = check_matrix("random-asym", rp, c, v, p_m=4, root=17)
rp, c, v = O.gen_stencil_3d(64); out["s64"] = check_matrix("3d-64", rp, c, v)

# ---- cfg2 timings
t0 = time.time(); rp, c, v = O.gen_stencil_3d(200); print("gen cfg2 %.1fs" % (time.time() - t0))
n = rp.shape[0] - 1; nnz = int(rp[-1]); k = 8
a = K.DeviceCsr.from_host(rp, c, v)
torch.cuda.synchronize(); t0 = time.time(); perm, inv, lp = K.bfs_levels(a, 0); torch.cuda.synchronize(); tb = time.time() - t0
t0 = time.time(); perm, inv, lp = K.bfs_levels(a, 0); torch.cuda.synchronize(); tb2 = time.time() - t0
t0 = time.time(); b = K.permute_symmetric(a, perm, inv); torch.cuda.synchronize(); tp = time.time() - t0
print(f"cfg2 bfs {tb*1e3:.1f} ms (2nd {tb2*1e3:.1f} ms) levels {len(lp)-1} permute {tp*1e3:.1f} ms")
out["cfg2_bfs_ms"] = tb2 * 1e3; out["cfg2_permute_ms"] = tp * 1e3; out["cfg2_levels"] = len(lp) - 1
x = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = x
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tmin, tmean = ev_time(lambda: K.mpk_baseline(b, y, k))
Q_ro = 12 * nnz + 4 * (n + 1) + 8 * n * (k + 1); F = 2 * nnz * k
print(f"baseline k=8: {tmin:.3f} ms min {tmean:.3f} mean; {F/tmin/1e6:.0f} GF/s")
out["cfg2_baseline_ms"] = tmin
yb = y.clone()
results = []
configs = [(_lib.FLAG_MODE_RESIDENT, 0, 0, 0, 0, 0), (_lib.FLAG_MODE_RESIDENT, 0, 0, 0, 0, 3), (_lib.FLAG_MODE_RESIDENT, 0, 0, 0, 0, 4),
           (_lib.FLAG_MODE_RESIDENT, 0, 0, 0, 0, 6), (_lib.FLAG_MODE_RESIDENT, 0, 0, 0, 0, 8),
           (_lib.FLAG_MODE_STREAM, 0, 0, 0, 0, 3), (_lib.FLAG_MODE_STREAM, 0, 0, 0, 0, 2),
           ("sweep", 0, 0, 0, 0, 2), ("sweep", 0, 0, 0, 0, 3)]
for fl, tile, cps, thr, slack, slots in configs:
    try:
        sweep = fl == "sweep"
        t = K.Tiling(b, k, tile_nnz=tile, ctas_per_sm=cps, threads=thr, queue_slack=slack, slots=slots,
                     mode_flags=_lib.FLAG_MODE_STREAM if sweep else fl)
        cfg = K.mpk_power_cfg(k)
        y2 = torch.zeros_like(y); y2[0] = x
        def run():
            K.mpk_run(t, y2, cfg, check_errors=False, flags=_lib.FLAG_SWEEP if sweep else 0)
        tmin, tmean = ev_time(run, reps=10)
        K.mpk_run(t, y2, cfg, flags=_lib.FLAG_SWEEP if sweep else 0)
        same = bool(torch.equal(y2, yb))
        r = dict(mode="sweep" if sweep else t.mode, tile=t.info["tile_nnz_cap"], ctas=t.info["grid"] // ctx.sm_count,
                 threads=t.info["block"], slack=t.info["queue_slack"], slots=slots, n_tiles=t.info["n_tiles"],
                 chain=t.info["chain_reach"], fwd=t.info["max_fwd_reach"], ms_min=tmin, ms_mean=tmean,
                 gflops=F / tmin / 1e6, ro_frac=Q_ro / (tmin * 1e-3) / 6531.6e9, bitwise=same)
    except Exception as e:
        r = dict(flags=fl, tile=tile, cps=cps, err=str(e)[:200])
    print(json.dumps(r)); results.append(r)
out["cfg2_mpk"] = results
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/gpu_check.json", "w"), indent=1, default=str)
