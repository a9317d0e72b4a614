"""BASELINE config 5 on one GPU: Chebyshev time propagation of a complex128
state on the 3D Anderson Hamiltonian 128^3 (W = 16.5), polynomial degree 64
run as 8 batches of k = 8 with the fused three-term recurrence and
coefficient accumulation.  Times ChebPropagator.step (device state) for the
default plan, the round-1 group walk on plain blocks, and per-power sweeps."""
import os, sys, json, time, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200.cheb import ChebCoeffs, cheb_coeffs_schrodinger, gershgorin_bounds
n = int(os.environ.get("N", "128"))
a = lm.gen_anderson_3d(n, seed=2)
lo, hi = gershgorin_bounds(a)
c = cheb_coeffs_schrodinger(8.0, lo, hi).c
c = np.resize(c, 65) if c.size < 65 else c[:65]
coeffs = ChebCoeffs(c=c.astype(np.complex128), dt=8.0, lam_min=lo, lam_max=hi, tol=1e-12)
rng = np.random.default_rng(0)
psi = np.exp(2j * np.pi * rng.random(a.n_rows)) / np.sqrt(a.n_rows)
xd = torch.from_numpy(psi).cuda()
flops = 2.0 * a.n_nz * 64 * 2
out = {}
ref = None
warm = lm.ChebPropagator(a, 8.0, coeffs=coeffs, p_m_batch=8, cache_bytes=126e6)  # clocks / caches up
for _ in range(3):
    warm.step(xd)
torch.cuda.synchronize()
del warm
for name, kw, sched in (("ring_walk", {}, "walk"), ("ring_tiles_sweep", {}, "sweep"), ("auto", {}, "auto"),
                        ("group_plain_walk", {"tiling_params": {"mode_flags": _lib.FLAG_MODE_STREAM}}, "walk"),
                        ("baseline_variant", {"variant": "baseline"}, "auto")):
    os.environ["LMPK_SCHEDULE"] = sched
    prop = lm.ChebPropagator(a, 8.0, coeffs=coeffs, p_m_batch=8, cache_bytes=126e6, **kw)
    y = prop.step(xd); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); y = prop.step(xd); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
    if ref is None:
        ref = y
    out[name] = {"ms": round(min(ts), 3), "gflops": round(flops / (min(ts) * 1e-3) / 1e9),
                 "bitwise_vs_first": bool(torch.equal(y, ref)),
                 "rel_err_vs_first": float((y - ref).abs().max() / ref.abs().max())}
print(json.dumps({"case": f"cfg5 cheb anderson {n}^3 complex, M=64, 8 x k=8", "nnz": a.n_nz, **out}))
