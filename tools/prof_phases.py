"""Phase counters of the group-walk kernel on cfg2 (LMPK_PROFILE=1).
SPECS: JSON list of [q, slots, tile_nnz, slack]; q = 0 -> sweep."""
import ctypes, json, os, sys
os.environ["LMPK_PROFILE"] = "1"
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
buf = (ctypes.c_ulonglong * 16)()
for spec in json.loads(os.environ.get("SPECS", '[[1,2,0,0],[2,2,0,0],[0,2,0,0]]')):
    q, slots, tile, slack, xf = (list(spec) + [0] * 5)[:5]
    fl = _lib.FLAG_MODE_RESIDENT if q == k else _lib.FLAG_MODE_STREAM
    t = K.Tiling(b, k, tile_nnz=tile, slots=slots, mode_flags=fl, group=max(q, 1), queue_slack=slack)
    y = torch.zeros(k + 1, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
    cfg = K.mpk_power_cfg(k); f = (_lib.FLAG_SWEEP if q == 0 else 0) | int(xf)
    K.mpk_run(t, y, cfg, flags=f); torch.cuda.synchronize()
    ctx.lib.lmpk_ctx_profile(ctx.handle, buf, 1)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); K.mpk_run(t, y, cfg, flags=f); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.lib.lmpk_ctx_profile(ctx.handle, buf, 1)
    v = list(buf)
    nw = v[2] or 1
    print(json.dumps(dict(q=q, flags=xf, cons_busy_frac=round(v[13] / max(v[12] + v[13], 1), 3), slots=slots, tiles=t.info["n_tiles"], ms=round(ms, 3),
        cons_wait_frac=round(v[0] / max(v[0] + v[1], 1), 3), cons_compute_us_per_item_warp=round(v[1] / nw / 1e3, 3),
        cons_wait_us_per_item_warp=round(v[0] / nw / 1e3, 3), polls=v[3], notready_frac=round(v[4] / max(v[3], 1), 3),
        prod_alive_ms_per_cta=round(v[5] / 148 / 1e6, 3), items_grabbed=v[6],
        us_tma_wait_per_item=round(v[7] / max(v[6], 1) / 1e3, 3), us_dep_wait_per_item=round(v[8] / max(v[6], 1) / 1e3, 3),
        us_free_wait_per_item=round(v[9] / max(v[6], 1) / 1e3, 3), us_xstage_per_item=round(v[11] / max(v[6], 1) / 1e3, 3), dep_rounds=v[3], ready_spins=v[13], q_items=v[14], p1_items=v[15], us_fetch_per_item=round(v[0] / max(v[6], 1) / 1e3, 3), us_push_per_item=round(v[1] / max(v[6], 1) / 1e3, 3), us_entrywait_per_qitem=round(v[10] / max(v[14], 1) / 1e3, 3), cas_fail=v[12], xstaged=t.info.get('x_staged_tiles'))), flush=True)
