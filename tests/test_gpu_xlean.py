"""GPU tests of the opt-in lean-walk variants (lean_kernel.cuh):

* LMPK_XLEAN=1 -- x staging: a ring piece is [lean block | x buffer], the runs
  of y_{p-1} a tile gathers are bulk-copied behind its block (k_lean_xplan),
  gathers read shared memory; static per-CTA work lists or the ticket queue;
* XP blocks (row records, units of up to 4 uniform slices) with staged
  (LMPK_XLEAN=1) or global (LMPK_XP=1) gathers.

Every variant must reproduce the oracle's power vectors bit for bit
(executor.py:127-147 row body, csr.py:195-201 summation order), for plain
MPK, the fused Chebyshev recurrence with accumulation, complex vectors,
non-finite operands in padded rows and odd row counts (the staged kernel
then falls back to the ring kernel: bulk copies need 16-byte aligned runs).
"""

import os

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from oracle import levelmpk_oracle as O
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu

KNOBS = ("LMPK_XLEAN", "LMPK_XP", "LMPK_NO_XP", "LMPK_XLEAN_ROWS", "LMPK_NO_WORKLIST", "LMPK_XP_RUN", "LMPK_XLEAN_PUB")
VARIANTS = {
    "xs_xp": {"LMPK_XLEAN": "1"},
    "xs_xp_queue": {"LMPK_XLEAN": "1", "LMPK_NO_WORKLIST": "1", "LMPK_XLEAN_PUB": "4"},
    "xs_lean": {"LMPK_XLEAN": "1", "LMPK_NO_XP": "1"},
    "xs_small": {"LMPK_XLEAN": "1", "LMPK_XLEAN_ROWS": "416", "LMPK_XP_RUN": "2"},
    "xp_global": {"LMPK_XP": "1"},
}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


@pytest.fixture
def knobs():
    saved = {k: os.environ.pop(k, None) for k in KNOBS}

    def set_(var):
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(VARIANTS[var])

    yield set_
    for k in KNOBS:
        os.environ.pop(k, None)
    for k, v in saved.items():
        if v is not None:
            os.environ[k] = v


def _permuted(a, root=0):
    perm, _ = O.bfs_levels(a.row_ptr, a.col, root)
    return O.permute_symmetric(a.row_ptr, a.col, a.val, perm)


GENS = {
    "3d7pt": (lambda: lm.gen_stencil_3d(28, 2), 8),
    "2d5pt": (lambda: lm.gen_laplace_2d5pt(96, 80), 4),
    "anderson": (lambda: lm.gen_anderson_3d(16, seed=3), 8),
    "3d7pt_odd": (lambda: lm.gen_stencil_3d(21, 2), 5),  # n = 9261 (odd): staged kernel not runnable on real vectors
}


@pytest.mark.parametrize("var", sorted(VARIANTS))
@pytest.mark.parametrize("name", sorted(GENS))
def test_variants_plain_mpk_bitwise(knobs, var, name):
    import torch

    gen, k = GENS[name]
    a = gen()
    rp, c, v = _permuted(a)
    knobs(var)
    t = K.Tiling(K.DeviceCsr.from_host(rp, c, v), k)
    info = t.info
    assert info["lean_bytes"] > 0
    if var.startswith("xs") and name != "anderson":
        assert info["lean_xstaged"] in (1, 2), info
    x = np.random.default_rng(5).uniform(-1, 1, a.n_rows)
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    for _ in range(2):  # second call: epoch-tagged progress words, work lists reused
        y[1:] = 0
        K.mpk_run(t, y, K.mpk_power_cfg(k), exact=True)
    assert np.array_equal(y.cpu().numpy(), O.mpk_powers(rp, c, v, x, k))
    # fewer powers than the tiling was built for
    y[1:] = 0
    K.mpk_run(t, y, K.mpk_power_cfg(2), exact=True)
    assert np.array_equal(y[:3].cpu().numpy(), O.mpk_powers(rp, c, v, x, 2))
    t.close()


@pytest.mark.parametrize("var", sorted(VARIANTS))
@pytest.mark.parametrize("cplx", [False, True])
def test_variants_chebyshev_accumulate_bitwise(knobs, var, cplx):
    """Fused T_{n+1} = 2 A T_n - T_{n-1} with acc += c_n T_n (executor.py:131-135)."""
    import torch

    a = lm.gen_stencil_3d(24, 2)
    rp, c, v = _permuted(a)
    v = v / 12.5  # spectrum inside [-1, 1]
    n, k = a.n_rows, 6
    knobs(var)
    t = K.Tiling(K.DeviceCsr.from_host(rp, c, v), k, mode_flags=_lib.FLAG_COMPLEX if cplx else 0)
    rng = np.random.default_rng(11)
    dt = np.complex128 if cplx else np.float64
    t0 = rng.uniform(-1, 1, n).astype(dt)
    t1 = rng.uniform(-1, 1, n).astype(dt)
    if cplx:
        t0 = t0 + 1j * rng.uniform(-1, 1, n)
        t1 = t1 + 1j * rng.uniform(-1, 1, n)
    coef = rng.uniform(-1, 1, k) + (1j * rng.uniform(-1, 1, k) if cplx else 0)
    acc0 = rng.uniform(-1, 1, n).astype(dt)
    # oracle: slots 0 = T_{n-1}, 1 = T_n, then k recurrence steps
    ys = [t0, t1]
    acc = acc0.copy()
    for i in range(k):
        s = (O.spmv(rp, c, v, ys[-1].real) + 1j * O.spmv(rp, c, v, ys[-1].imag)) if cplx else O.spmv(rp, c, v, ys[-1])
        nxt = 2.0 * s - ys[-2]
        ys.append(nxt)
        if cplx:
            cr, ci = coef[i].real, coef[i].imag
            acc = (acc.real + (cr * nxt.real - ci * nxt.imag)) + 1j * (acc.imag + (cr * nxt.imag + ci * nxt.real))
        else:
            acc = acc + coef[i] * nxt
    tdt = torch.complex128 if cplx else torch.float64
    y = torch.zeros((k + 2, n), dtype=tdt, device="cuda")
    y[0] = torch.from_numpy(t0)
    y[1] = torch.from_numpy(t1)
    accd = torch.from_numpy(acc0.copy()).cuda()
    cfg = K.power_cfg(k, out_slot=list(range(2, k + 2)), in_slot=list(range(1, k + 1)), prev_slot=list(range(0, k)),
                      kernel=[1] * k, coef_re=list(np.real(coef)), coef_im=list(np.imag(coef)) if cplx else None)
    yv = torch.view_as_real(y).reshape(k + 2, -1) if cplx else y
    av = torch.view_as_real(accd).reshape(-1) if cplx else accd
    K.mpk_run(t, yv, cfg, acc=av, use_acc=True, complex_state=cplx, exact=True)
    got = y.cpu().numpy()
    for i in range(k + 2):
        assert np.array_equal(got[i], ys[i]), (var, cplx, i)
    assert np.array_equal(accd.cpu().numpy(), acc)
    t.close()


@pytest.mark.parametrize("var", ["xs_xp", "xs_lean", "xp_global"])
def test_variants_nonfinite_padded_rows(knobs, var):
    """Padding repeats the row's last column with value +0.0: an infinite
    operand there is recomputed with the row's true length (Inf stays Inf)."""
    import torch

    a = lm.gen_stencil_3d(20, 2)
    rp, c, v = _permuted(a)
    knobs(var)
    t = K.Tiling(K.DeviceCsr.from_host(rp, c, v), 3)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, a.n_rows)
    lens = np.diff(rp)
    short = np.flatnonzero((lens > 0) & (lens < 7))
    x[c[rp[rng.choice(short, 40, replace=False) + 1] - 1]] = np.inf
    x[rng.choice(a.n_rows, 3, replace=False)] = -np.inf
    x[rng.choice(a.n_rows, 2, replace=False)] = np.nan
    y = torch.zeros((4, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(3), exact=True)
    with np.errstate(all="ignore"):
        ref = O.mpk_powers(rp, c, v, x, 3)
    got = y.cpu().numpy()
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    m = ~np.isnan(ref)
    assert np.array_equal(got[m], ref[m])
    t.close()


def test_xplan_runs_cover_columns(knobs):
    """k_lean_xplan through the tiling: every tile reports a staged piece that
    fits the shared-memory ring at depth >= 2."""
    a = lm.gen_stencil_3d(32, 2)
    rp, c, v = _permuted(a)
    knobs("xs_xp")
    t = K.Tiling(K.DeviceCsr.from_host(rp, c, v), 4)
    assert t.info["lean_xstaged"] in (1, 2) and 2 <= t.info["lean_ring"] <= 4
    assert t.info["lean_ring"] * t.info["lean_piece"] <= 227 * 1024
    t.close()
