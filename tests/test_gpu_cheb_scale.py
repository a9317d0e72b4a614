"""GPU: fused Chebyshev propagation (real: bitwise vs the reference's own
outputs; complex128: bitwise vs the oracle) and the BASELINE.json configs at
or near full size (BFS / permutation / MPK bitwise vs the C oracle)."""

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from matrices import sha
from oracle import cpu as C
from oracle import levelmpk_oracle as O
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pb", [1, 3, 4])
def test_cheb_heat_bitwise_vs_reference(pb, golden):
    facts, arr = golden
    a = lm.gen_stencil_3d(8, 2)
    prop = lm.ChebPropagator(a, 0.08, tol=1e-6, p_m_batch=pb, cache_bytes=40_000)
    assert prop.coeffs.n_moments == facts[f"cheb_3d8_pb{pb}_moments"]
    got = prop.step(arr["cheb/3d-8/x"])
    assert np.array_equal(got, arr[f"cheb/3d-8/pb{pb}"])


def test_cheb_matches_dense_exponential_and_batches(rng):
    a = lm.gen_stencil_3d(8, 2)
    x = rng.standard_normal(a.n_rows)
    w, v = np.linalg.eigh(a.to_dense())
    expect = v @ (np.exp(-0.05 * w) * (v.T @ x))
    outs = {pb: lm.ChebPropagator(a, 0.05, tol=1e-4, p_m_batch=pb, cache_bytes=50_000).step(x)
            for pb in (1, 2, 4, 8)}
    assert np.linalg.norm(outs[4] - expect) / np.linalg.norm(expect) <= 1e-3
    for pb in (2, 4, 8):
        assert np.array_equal(outs[pb], outs[1])
    end, rec = lm.ChebPropagator(a, 0.02, tol=1e-4, p_m_batch=2, cache_bytes=20_000).propagate(x, 3)
    assert len(rec) == 3 and all(r["seconds"] > 0 for r in rec)


def test_cheb_complex_schrodinger_vs_oracle():
    a = lm.gen_anderson_3d(10, seed=4)
    lo, hi = lm.gershgorin_bounds(a)
    co = lm.cheb_coeffs_schrodinger(0.2, lo, hi, tol=1e-12)
    psi = np.exp(1j * np.random.default_rng(2).uniform(0, 2 * np.pi, a.n_rows)) / np.sqrt(a.n_rows)
    prop = lm.ChebPropagator(a, 0.2, coeffs=co, p_m_batch=8, cache_bytes=50_000)
    got = prop.step(psi)
    b = lm.scale_for_heat(a, lo, hi)
    p = prop.pre.perm.perm
    rp, c, v = C.permute_symmetric(b.row_ptr, b.col, b.val, p)
    accp = O.cheb_batches(rp, c, v, psi[p], co.c.real, co.c.imag)
    ref = np.empty_like(accp)
    ref[p] = accp
    assert np.array_equal(got, ref)
    assert abs(np.linalg.norm(got) - 1.0) < 1e-9  # unitary evolution


def test_cfg1_full_size_vs_reference(golden):
    """BASELINE config 1 at full size: levels, permutation and A x..A^4 x
    bitwise equal to the reference's own run (hashes from make_golden.py)."""
    facts, arr = golden
    rec = facts["matrices"]["cfg1"]
    a = lm.gen_laplace_2d5pt(256, 256)
    levels, perm = lm.bfs_levels(a, 0)
    assert sha(perm.perm) == rec["bfs0_perm"] and levels.n_levels == 511
    x = np.random.default_rng(99).standard_normal(a.n_rows)
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", 4, 126e6)
    assert [sha(res.y.data[p]) for p in range(5)] == rec["baseline_y"]


def test_rmat_restart_tail_vs_oracle():
    """R-MAT scale 16: ~half the vertices are isolated singleton levels (the
    reference's restart loop, levels.py:98-100)."""
    a = lm.gen_rmat(16)
    levels, perm = lm.bfs_levels(a, 0)
    op, olp = C.bfs_levels(a.row_ptr, a.col, 0)
    assert np.array_equal(perm.perm, op) and np.array_equal(levels.level_ptr, olp)
    assert levels.n_levels > a.n_rows // 4
    x = np.random.default_rng(0).uniform(0, 1, a.n_rows)
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", 6, 126e6)
    rp, c, v = C.permute_symmetric(a.row_ptr, a.col, a.val, pre.perm.perm)
    ref = np.zeros((7, a.n_rows))
    ref[0] = x[pre.perm.perm]
    C.mpk_baseline(rp, c, v, ref, 6)
    assert np.array_equal(res.y.data, ref)


def test_cfg2_full_size_bitwise():
    """BASELINE config 2 at full size (8M rows, 55.76M nnz, k=8): GPU levels,
    permutation and level-blocked powers equal the C oracle bit for bit."""
    import torch

    a = lm.gen_stencil_3d(200, 2)
    pre = lm.prepare(a, "lb_lg_p2p", 8, 126e6)
    assert pre.levels.n_levels == 598
    op, olp = C.bfs_levels(a.row_ptr, a.col, 0)
    assert np.array_equal(pre.perm.perm, op) and np.array_equal(pre.levels.level_ptr, olp)
    rp, c, v = C.permute_symmetric(a.row_ptr, a.col, a.val, op)
    assert np.array_equal(pre.a.row_ptr, rp) and np.array_equal(pre.a.col, c)
    assert np.array_equal(pre.a.val, v)
    x = np.random.default_rng(0).uniform(-1, 1, a.n_rows)
    ref = np.zeros((9, a.n_rows))
    ref[0] = x[op]
    C.mpk_baseline(rp, c, v, ref, 8)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    for params in ({},  # the default plan: ring walk over compressed tiles
                   {"mode_flags": _lib.FLAG_MODE_STREAM, "slots": 2},
                   {"mode_flags": _lib.FLAG_MODE_STREAM | _lib.FLAG_COMPRESS, "slots": 2},
                   {"mode_flags": _lib.FLAG_MODE_RESIDENT, "slots": 2}):
        t = plan.tiling(**params)
        y = torch.zeros((9, a.n_rows), dtype=torch.float64, device="cuda")
        y[0] = torch.from_numpy(ref[0])
        K.mpk_run(t, y, plan.power_config())
        assert np.array_equal(y.cpu().numpy(), ref), params


def test_cfg3_and_cfg5_reduced_size():
    """27-point perturbed (config 3 shape) and periodic Anderson (config 5)."""
    for a, k in ((lm.gen_stencil_3d27pt(40, seed=1), 4), (lm.gen_anderson_3d(32, seed=2), 8)):
        x = np.random.default_rng(1).uniform(-1, 1, a.n_rows)
        res, pre = lm.run_mpk(a, x, "lb_lg_p2p", k, 126e6)
        rp, c, v = C.permute_symmetric(a.row_ptr, a.col, a.val, pre.perm.perm)
        ref = np.zeros((k + 1, a.n_rows))
        ref[0] = x[pre.perm.perm]
        C.mpk_baseline(rp, c, v, ref, k)
        assert np.array_equal(res.y.data, ref)


@pytest.mark.parametrize("case", ["stencil3d", "27pt", "rmat"])
def test_fast_fma_mode_within_north_star_tolerance(case):
    """Without LMPK_FLAG_EXACT the ordered row sums use DFMA; the contract
    (BASELINE.json north_star) is relative L2 error <= 1e-12 per power."""
    import torch

    from paper_2205_01598_b200 import kernels as K

    a = {"stencil3d": lambda: lm.gen_stencil_3d(40, 2),
         "27pt": lambda: lm.gen_stencil_3d27pt(24, seed=3),
         "rmat": lambda: lm.gen_rmat(14)}[case]()
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    k = 8
    x = np.random.default_rng(5).uniform(-1, 1, a.n_rows)
    ref = np.zeros((k + 1, a.n_rows))
    ref[0] = x
    C.mpk_baseline(ap.row_ptr, ap.col, ap.val, ref, k)
    t = K.Tiling(ap.device(), k)
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k), exact=False)
    got = y.cpu().numpy()
    for p in range(1, k + 1):
        rel = np.linalg.norm(got[p] - ref[p]) / max(np.linalg.norm(ref[p]), 1e-300)
        assert rel <= 1e-12, (p, rel)


def test_rmat_scale18_mpk_bitwise():
    """Config-4 shape at scale 18 (262K rows, ~4.2M nnz, a giant level next to
    113K singleton levels): the level-blocked walk equals k baseline sweeps."""
    import torch

    from paper_2205_01598_b200 import kernels as K

    a = lm.gen_rmat(18)
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    k = 6
    x = np.random.default_rng(1).uniform(0, 1, a.n_rows)
    ref = np.zeros((k + 1, a.n_rows))
    ref[0] = x
    C.mpk_baseline(ap.row_ptr, ap.col, ap.val, ref, k)
    t = K.Tiling(ap.device(), k)
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k))
    assert np.array_equal(y.cpu().numpy(), ref)


def test_cfg5_full_size_propagation_schedules_bitwise():
    """BASELINE config 5 as specified: complex128 Chebyshev propagation on the
    Anderson 128^3 Hamiltonian, degree 64 as 8 batches of k=8.  The ring walk,
    the per-power sweeps over the same tiles and the round-1 group walk on
    plain blocks give the same bits; the result is a unitary propagation
    (norm preserved to the truncation tolerance)."""
    import os
    import torch
    from paper_2205_01598_b200.cheb import ChebCoeffs, cheb_coeffs_schrodinger, gershgorin_bounds

    a = lm.gen_anderson_3d(128, seed=2)
    lo, hi = gershgorin_bounds(a)
    c = cheb_coeffs_schrodinger(2.0, lo, hi, tol=1e-14).c
    assert c.size <= 65
    coeffs = ChebCoeffs(c=c, dt=2.0, lam_min=lo, lam_max=hi, tol=1e-14)
    rng = np.random.default_rng(0)
    psi = np.exp(2j * np.pi * rng.random(a.n_rows)) / np.sqrt(a.n_rows)
    xd = torch.from_numpy(psi).cuda()
    outs = []
    old = os.environ.get("LMPK_SCHEDULE")
    try:
        for sched, kw in (("walk", {}), ("sweep", {}),
                          ("walk", {"tiling_params": {"mode_flags": _lib.FLAG_MODE_STREAM}})):
            os.environ["LMPK_SCHEDULE"] = sched
            prop = lm.ChebPropagator(a, 2.0, coeffs=coeffs, p_m_batch=8, cache_bytes=126e6, **kw)
            outs.append(prop.step(xd))
    finally:
        if old is None:
            os.environ.pop("LMPK_SCHEDULE", None)
        else:
            os.environ["LMPK_SCHEDULE"] = old
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert abs(float(torch.linalg.vector_norm(outs[0])) - 1.0) < 1e-10
