"""GPU tests of the default walk (the lean ring kernel) and of the public
run_plan host path: bitwise against the oracle, the non-finite slow path of
padded rows, the epoch-counter wrap, a 1,000-rep torture with a host
watchdog (pkg/tests/test_executor.py:134-152), and run_plan on the
reference's own PowerVectors / plan objects (the LEVELMPK_BACKEND=cuda seam
of INTEGRATION.md)."""

import os
import threading
import types

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from oracle import levelmpk_oracle as O
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200 import executor as E
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


def _permuted(a, root=0):
    perm, _ = O.bfs_levels(a.row_ptr, a.col, root)
    rp, c, v = O.permute_symmetric(a.row_ptr, a.col, a.val, perm)
    return rp, c, v, perm


def _lean_tiling(rp, c, v, k):
    d = K.DeviceCsr.from_host(rp, c, v)
    t = K.Tiling(d, k)
    assert t.info["lean_bytes"] > 0, "expected a lean (uniform W <= 8) tiling"
    return d, t


@pytest.mark.parametrize("gen,k", [(lambda: lm.gen_stencil_3d(24, 2), 8), (lambda: lm.gen_laplace_2d5pt(64, 64), 4),
                                   (lambda: lm.gen_anderson_3d(16, seed=3), 8)])
def test_lean_walk_bitwise(gen, k):
    import torch

    a = gen()
    rp, c, v, perm = _permuted(a)
    d, t = _lean_tiling(rp, c, v, k)
    x = np.random.default_rng(5).uniform(-1, 1, a.n_rows)
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k), exact=True)
    assert np.array_equal(y.cpu().numpy(), O.mpk_powers(rp, c, v, x, k))


def test_lean_padding_nonfinite_slow_path():
    """Padded rows repeat their last column with the value +0.0; an infinite
    operand there would turn an Inf row sum into NaN, so such rows are
    recomputed with their true length -- results equal the reference's IEEE
    sums element for element (Inf stays Inf, NaN stays NaN)."""
    import torch

    a = lm.gen_stencil_3d(20, 2)  # boundary rows: 4-6 entries in 7-wide slices
    rp, c, v, perm = _permuted(a)
    d, t = _lean_tiling(rp, c, v, 3)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, a.n_rows)
    # infinities at the LAST column of some short (padded) rows
    lens = np.diff(rp)
    short = np.flatnonzero((lens > 0) & (lens < 7))
    pick = rng.choice(short, 40, replace=False)
    x[c[rp[pick + 1] - 1]] = np.inf
    x[rng.choice(a.n_rows, 3, replace=False)] = -np.inf
    x[rng.choice(a.n_rows, 2, replace=False)] = np.nan
    y = torch.zeros((4, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(3), exact=True)
    got = y.cpu().numpy()
    with np.errstate(invalid="ignore", over="ignore"):
        ref = O.mpk_powers(rp, c, v, x, 3)
    assert np.isinf(ref[1]).sum() > 40
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    assert np.array_equal(got[~np.isnan(got)], ref[~np.isnan(ref)])


def test_lean_chebyshev_and_complex_vs_oracle():
    """The general epilogue of the lean walk: Chebyshev steps with the
    accumulator, real and complex128 state (real matrix)."""
    import torch

    a = lm.gen_anderson_3d(16, seed=4)
    rp, c, v, perm = _permuted(a)
    n = a.n_rows
    d, t = _lean_tiling(rp, c, v, 6)
    rng = np.random.default_rng(11)
    cr, ci = rng.standard_normal(7), rng.standard_normal(7)
    # slots: 0 = T_0 = x, p = T_p; power 1 is a plain SpMV, powers >= 2 Chebyshev
    p = np.arange(1, 7)
    kern = np.where(p == 1, 0, 1)
    for cplx in (False, True):
        x = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cplx else 0)
        cfg = K.power_cfg(6, p, p - 1, np.maximum(p - 2, 0), kern, cr[1:], ci[1:] if cplx else None)
        if cplx:
            y = torch.zeros((7, n), dtype=torch.complex128, device="cuda")
            y[0] = torch.from_numpy(x)
            acc = torch.from_numpy(cr[0] * x.real - ci[0] * x.imag + 1j * (cr[0] * x.imag + ci[0] * x.real)).cuda()
            yv = torch.view_as_real(y).reshape(7, -1)
            av = torch.view_as_real(acc).reshape(-1)
            K.mpk_run(t, yv, cfg, acc=av, use_acc=True, complex_state=True, exact=True)
            ref = O.cheb_batches(rp, c, v, x, cr, ci)
        else:
            y = torch.zeros((7, n), dtype=torch.float64, device="cuda")
            y[0] = torch.from_numpy(x)
            acc = torch.from_numpy(cr[0] * x).cuda()
            K.mpk_run(t, y, cfg, acc=acc, use_acc=True, exact=True)
            ref = O.cheb_batches(rp, c, v, x, cr)
        assert np.array_equal(acc.cpu().numpy(), ref)


def test_epoch_wrap_keeps_other_tilings_correct():
    """after the 2^24 epoch wrap every tiling's stale progress
    words are cleared before its next launch, not only the launching one's."""
    import torch

    ctx = _lib.context()
    a1, a2 = lm.gen_stencil_3d(18, 2), lm.gen_laplace_2d5pt(90, 90)
    runs = []
    for a in (a1, a2):
        rp, c, v, perm = _permuted(a)
        d, t = _lean_tiling(rp, c, v, 5)
        x = np.random.default_rng(2).uniform(-1, 1, a.n_rows)
        runs.append((t, x, O.mpk_powers(rp, c, v, x, 5)))

    def go(i):
        t, x, ref = runs[i]
        y = torch.zeros((6, x.shape[0]), dtype=torch.float64, device="cuda")
        y[0] = torch.from_numpy(x)
        K.mpk_run(t, y, K.mpk_power_cfg(5), exact=True)
        assert np.array_equal(y.cpu().numpy(), ref)

    go(0)
    go(1)
    old = ctx.lib.lmpk_ctx_set_epoch(ctx.handle, (1 << 24) - 2)
    try:
        for _ in range(3):  # crosses the wrap on tiling 1, then runs tiling 0 with old tags
            go(1)
            go(0)
    finally:
        ctx.lib.lmpk_ctx_set_epoch(ctx.handle, max(int(old), 1))


def test_torture_default_walk_1000_reps():
    """pkg/tests/test_executor.py:134-152 on the GPU: the default persistent
    walk repeated LEVELMPK_TORTURE_REPS (1,000) times, every result bitwise
    the first; a host watchdog fails the test instead of hanging (the device
    watchdog aborts a launch stuck for 8 s)."""
    import torch

    reps = int(os.environ.get("LEVELMPK_TORTURE_REPS", "1000"))
    a = lm.gen_stencil_3d(48, 2)
    rp, c, v, perm = _permuted(a)
    d, t = _lean_tiling(rp, c, v, 8)
    x = np.random.default_rng(3).uniform(-1, 1, a.n_rows)
    ref = torch.from_numpy(O.mpk_powers(rp, c, v, x, 8)).cuda()
    y = torch.zeros_like(ref)
    y[0] = ref[0]
    bad = []
    done = threading.Event()

    def body():
        try:
            for i in range(reps):
                y[1:].zero_()
                K.mpk_run(t, y, K.mpk_power_cfg(8), exact=True)
                if not torch.equal(y, ref):
                    bad.append(i)
        finally:
            done.set()

    th = threading.Thread(target=body, daemon=True)
    th.start()
    assert done.wait(timeout=300), "torture run hung (host watchdog)"
    assert not bad, f"results differ at reps {bad[:10]}"


class _RefPowerVectors:
    """Shape of the reference's PowerVectors (executor.py:33-53): n_rows,
    p_max, data; no on_device attribute."""

    def __init__(self, n_rows, p_max, n_slots=None):
        self.n_rows = n_rows
        self.p_max = p_max
        self.data = np.zeros((n_slots or p_max + 1, n_rows))


def test_run_plan_foreign_powervectors_and_host_x():
    """run_plan(adopt_plan(plan), y=<reference PowerVectors>) --
    the INTEGRATION.md patch -- updates y in place; run_plan(plan, x=numpy)
    returns host vectors in page-locked memory with y[0] == x."""
    a = lm.gen_stencil_3d(22, 2)
    pre = lm.prepare(a, "lb_lg_p2p", 6, 2e6)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    x = np.random.default_rng(9).uniform(-1, 1, a.n_rows)
    rp, c, v = pre.a.row_ptr, pre.a.col, pre.a.val
    ref = O.mpk_powers(rp, c, v, x, 6)
    res = lm.run_plan(plan, x=x)
    assert isinstance(res.y.data, np.ndarray) and np.array_equal(res.y.data, ref)
    assert res.seconds > 0 and res.e2e_seconds >= res.seconds
    pv = _RefPowerVectors(a.n_rows, 6)
    pv.data[0] = x
    plan2 = E.adopt_plan(types.SimpleNamespace(**{f: getattr(plan, f) for f in E._PLAN_FIELDS}, a=plan.a))
    res2 = lm.run_plan(plan2, y=pv)
    assert res2.y is pv and np.array_equal(pv.data, ref)


def test_run_plan_host_chebyshev_slots():
    """Host y with Chebyshev slots (the ChebPropagator driver of
    cheb.py:209-246 on host buffers): the input slot goes up, the written
    slots come down, the host accumulator is updated in place."""
    a = lm.gen_anderson_3d(14, seed=1)
    pm = 5
    pre = lm.prepare(a, "lb_lg_p2p", pm, 2e6)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    coef = np.random.default_rng(6).standard_normal(pm + 1)
    p = plan.power
    plan.in_slot[:] = p - 1
    plan.out_slot[:] = p
    plan.prev_slot[:] = np.maximum(p - 2, 0)
    plan.kernel[:] = np.where(p == 1, 0, 1)
    plan.acc_coef[:] = coef[p]
    x = np.random.default_rng(8).uniform(-1, 1, a.n_rows)
    pv = _RefPowerVectors(a.n_rows, pm, n_slots=pm + 2)
    pv.data[0] = x
    pv.data[pm + 1] = 123.0  # an untouched slot keeps its contents
    acc = coef[0] * x
    lm.run_plan(plan, y=pv, acc=acc, use_acc=True)
    rp, c, v = pre.a.row_ptr, pre.a.col, pre.a.val
    assert np.array_equal(acc, O.cheb_batches(rp, c, v, x, coef))
    assert np.all(pv.data[pm + 1] == 123.0) and np.array_equal(pv.data[0], x)


def test_schedule_choice_key_includes_plain():
    """a plan timed as plain real MPK ('crs' may win) must not hand
    that choice to a later Chebyshev / accumulating call of the same plan."""
    a = lm.gen_stencil_3d(10, 2)
    pre = lm.prepare(a, "lb_lg_p2p", 3, 1e6)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    plan.set_schedule_choice(False, "crs", True)
    assert plan.schedule_choice(False, True) == "crs"
    assert plan.schedule_choice(False, False) is None
