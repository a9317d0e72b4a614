"""CRS SpMV kernel rate (lmpk_spmv_rows) for 3D 7-pt stencils of several sizes:
HBM-resident (200^3) vs L2-resident (<= 100^3) matrices, level-permuted."""
import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_01598_b200 import kernels as K, _lib
from oracle import levelmpk_oracle as O
for N in (200, 128, 100, 80, 64):
    rp, c, v = O.gen_stencil_3d(N); n = rp.shape[0] - 1; nnz = int(rp[-1])
    a = K.DeviceCsr.from_host(rp, c, v)
    perm, inv, lp = K.bfs_levels(a, 0)
    b = K.permute_symmetric(a, perm, inv)
    y = torch.zeros(9, n, dtype=torch.float64, device="cuda"); y[0] = 1.0
    for _ in range(3): K.mpk_baseline(b, y, 8)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): K.mpk_baseline(b, y, 8)
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 80 * 1e-3
    t2 = None
    try:
        til = K.Tiling(b, 8)
        cfg = K.mpk_power_cfg(8)
        for _ in range(3): K.mpk_run(til, y, cfg, check_errors=False)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): K.mpk_run(til, y, cfg, check_errors=False)
        e1.record(); e1.synchronize(); t2 = e0.elapsed_time(e1) / 10 * 1e-3
    except Exception as ex:
        print(ex)
    print(f"N={N}^3 nnz={nnz/1e6:.1f}M matrix {12*nnz/1e6:.0f} MB: CRS SpMV {t*1e6:.1f} us = "
          f"{nnz/t/148/1.9e9:.2f} nnz/clk/SM, {(12*nnz+16*n)/t/1e9:.0f} GB/s;  MPK k=8 {t2*1e6 if t2 else 0:.1f} us "
          f"(= {t2/t/8 if t2 else 0:.2f} SpMV-equivalents per power)", flush=True)
