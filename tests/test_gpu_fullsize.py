"""GPU parity at the BASELINE.json sizes of configs 3, 4 and 5 (SURVEY.md
§8c): levels / permutation bit-exact against the C oracle, power vectors
bitwise against k back-to-back oracle SpMVs on the permuted matrix (the
reference's run_baseline, executor.py:261-266, to which every variant is
bitwise equal, test_acceptance.py:59-87), and the complex Chebyshev
propagation of config 5 against the oracle's restatement of cheb.py:221-246
(bitwise) and the linearity restatement of SURVEY §8c (four real
propagations, relative error <= 1e-12)."""

import os

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from oracle import cpu as C
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


def _oracle_powers(rp, c, v, x, k):
    ref = np.zeros((k + 1, rp.shape[0] - 1))
    ref[0] = x
    C.mpk_baseline(rp, c, v, ref, k)
    return ref


def _check_levels(a, pre):
    op, olp = C.bfs_levels(a.row_ptr, a.col, 0)
    assert np.array_equal(pre.perm.perm, op) and np.array_equal(pre.levels.level_ptr, olp)
    rp, c, v = C.permute_symmetric(a.row_ptr, a.col, a.val, op)
    assert np.array_equal(pre.a.row_ptr, rp) and np.array_equal(pre.a.col, c) and np.array_equal(pre.a.val, v)
    return op, rp, c, v


@pytest.fixture(scope="module")
def cfg3():
    a = lm.gen_stencil_3d27pt(160, seed=1, device=True)
    assert a.n_rows == 4_096_000 and a.n_nz == 109_215_352
    return a


@pytest.mark.parametrize("k", [2, 4, 8, 16])
def test_cfg3_full_size(cfg3, k):
    """Config 3: 27-point 160^3 perturbed, k = 2/4/8/16; the plan's chosen
    schedule and the level-blocked walk forced, both bitwise."""
    import torch

    a = cfg3
    x = np.random.default_rng(3).uniform(-1, 1, a.n_rows)
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", k, 126e6)
    op, rp, c, v = _check_levels(a, pre)
    ref = _oracle_powers(rp, c, v, x[op], k)
    assert np.array_equal(res.y.data, ref)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    t = plan.tiling()
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(ref[0])
    K.mpk_run(t, y, plan.power_config())  # the walk itself, whatever _schedule picks
    assert torch.equal(y, torch.from_numpy(ref).cuda())


def test_cfg4_full_size():
    """Config 4: R-MAT scale 22 (4.19M vertices, 69.4M nnz, 2.2M singleton
    levels) -- BFS bit-exact with the oracle's key-sort restatement (the
    reference's own BFS needs hours here), then MPK k = 6."""
    a = lm.gen_rmat(22, device=True)
    assert a.n_rows == 4_194_304 and a.n_nz == 69_438_612
    x = np.random.default_rng(1).uniform(0, 1, a.n_rows)
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", 6, 126e6)
    op, rp, c, v = _check_levels(a, pre)
    assert pre.levels.n_levels > 2_000_000
    assert np.array_equal(res.y.data, _oracle_powers(rp, c, v, x[op], 6))


def _spmv_c(rp, c, v, x):
    y = np.zeros((2, x.shape[0]))
    y[0] = x
    C.mpk_baseline(rp, c, v, y, 1)
    return y[1]


def _cheb_real(rp, c, v, x, coef):
    """Real ChebPropagator.step restated (cheb.py:221-246; C SpMVs)."""
    acc = coef[0] * x
    t_prev, t = x, _spmv_c(rp, c, v, x)
    acc = acc + coef[1] * t
    for j in range(2, coef.size):
        t_new = 2.0 * _spmv_c(rp, c, v, t) - t_prev
        acc = acc + coef[j] * t_new
        t_prev, t = t, t_new
    return acc


def _cheb_complex(rp, c, v, x, cr, ci):
    """The complex step in the kernel's arithmetic order (oracle.cheb_batches
    with C SpMVs): acc_re += c_re t_re - c_im t_im, acc_im += c_re t_im + c_im t_re."""
    xr, xi = np.ascontiguousarray(x.real), np.ascontiguousarray(x.imag)
    ar, ai = cr[0] * xr - ci[0] * xi, cr[0] * xi + ci[0] * xr
    pr, pi = xr, xi
    tr, ti = _spmv_c(rp, c, v, xr), _spmv_c(rp, c, v, xi)
    ar, ai = ar + (cr[1] * tr - ci[1] * ti), ai + (cr[1] * ti + ci[1] * tr)
    for j in range(2, cr.size):
        nr, ni = 2.0 * _spmv_c(rp, c, v, tr) - pr, 2.0 * _spmv_c(rp, c, v, ti) - pi
        ar, ai = ar + (cr[j] * nr - ci[j] * ni), ai + (cr[j] * ni + ci[j] * nr)
        pr, pi, tr, ti = tr, ti, nr, ni
    return ar + 1j * ai


def test_cfg5_full_size_complex_chebyshev():
    """Config 5 as specified: Anderson 128^3 periodic (W = 16.5), complex128
    state with random phases, degree-64 Schroedinger expansion run as 8
    batches of k = 8 with the fused recurrence and accumulation."""
    import torch
    from paper_2205_01598_b200.cheb import ChebCoeffs, cheb_coeffs_schrodinger, gershgorin_bounds

    a = lm.gen_anderson_3d(128, seed=2, device=True)
    lo, hi = gershgorin_bounds(a)
    c = cheb_coeffs_schrodinger(2.0, lo, hi, tol=1e-14).c
    c = np.concatenate([c, np.zeros(65 - c.size, dtype=c.dtype)])  # degree 64 exactly
    coeffs = ChebCoeffs(c=c, dt=2.0, lam_min=lo, lam_max=hi, tol=1e-14)
    rng = np.random.default_rng(0)
    psi = np.exp(2j * np.pi * rng.random(a.n_rows)) / np.sqrt(a.n_rows)
    prop = lm.ChebPropagator(a, 2.0, coeffs=coeffs, p_m_batch=8, cache_bytes=126e6)
    assert coeffs.n_moments == 64 and prop.p_b == 8
    got = prop.step(torch.from_numpy(psi).cuda()).cpu().numpy()
    b = lm.scale_for_heat(a, lo, hi)
    p = prop.pre.perm.perm
    rp, cc, v = C.permute_symmetric(b.row_ptr, b.col, b.val, p)
    accp = _cheb_complex(rp, cc, v, psi[p], c.real, c.imag)
    ref = np.empty_like(accp)
    ref[p] = accp
    assert np.array_equal(got, ref)
    # linearity restatement: four real propagations
    sr = _cheb_real(rp, cc, v, np.ascontiguousarray(psi[p].real), c.real)
    si = _cheb_real(rp, cc, v, np.ascontiguousarray(psi[p].imag), c.imag)
    sri = _cheb_real(rp, cc, v, np.ascontiguousarray(psi[p].imag), c.real)
    sir = _cheb_real(rp, cc, v, np.ascontiguousarray(psi[p].real), c.imag)
    lin = np.empty(a.n_rows, dtype=np.complex128)
    lin[p] = (sr - si) + 1j * (sri + sir)
    assert np.linalg.norm(got - lin) / np.linalg.norm(lin) <= 1e-12
    assert abs(np.linalg.norm(got) - 1.0) < 1e-10
