"""GPU parity of DP tilings (diagonal-private dictionary blocks, csrc/mpk_dp.cuh
and the "DP units" of csrc/lean_kernel.cuh): operators whose off-diagonal
values come from one small dictionary while the diagonal differs row by row
(Anderson / Schroedinger: stencil + potential).  The walk and the per-power
sweep over these blocks must give the bits of the oracle's sequential CRS sums
(pkg/src/levelmpk/executor.py:127-135, csr.py:195-201) for real MPK, and the
bits of the ring blocks (LMPK_NO_DP) for the complex Chebyshev kernel."""

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from oracle import levelmpk_oracle as O
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


def _level_ordered(a):
    _, perm = lm.bfs_levels(a, 0)
    return lm.permute_symmetric(a, perm)


def _potential_2d(nx=61, ny=47, seed=3):
    """2D 5-point stencil (boundary rows of 3..4 entries: padded slices) with a
    random diagonal; n is not a multiple of 32."""
    rng = np.random.default_rng(seed)
    idx = np.arange(nx * ny).reshape(nx, ny)
    rows, cols, vals = [idx.ravel()], [idx.ravel()], [rng.uniform(-4, 4, nx * ny)]
    for a, b in ((idx[1:], idx[:-1]), (idx[:, 1:], idx[:, :-1])):
        rows += [a.ravel(), b.ravel()]
        cols += [b.ravel(), a.ravel()]
        vals += [np.full(a.size, -1.0), np.full(a.size, -0.5)]
    return lm.CsrMatrix.from_triplets(nx * ny, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def _band_far(n=50_001, seed=5):
    """Band (+-1, +-37) with couplings at +-40000 (column offsets beyond
    int16), a random diagonal on most rows, no diagonal on every 7th row and
    empty rows at multiples of 1000."""
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    rows, cols, vals = [], [], []
    for d, v in ((1, -1.0), (37, 0.25)):
        rows += [i[:-d], i[d:]]
        cols += [i[d:], i[:-d]]
        vals += [np.full(n - d, v), np.full(n - d, v)]
    far = np.arange(0, n - 40_000, 997)
    rows += [far, far + 40_000]
    cols += [far + 40_000, far]
    vals += [np.full(far.size, 3.0), np.full(far.size, 3.0)]
    dg = i[i % 7 != 0]
    rows.append(dg)
    cols.append(dg)
    vals.append(rng.standard_normal(dg.size))
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    keep = r % 1000 != 0
    return lm.CsrMatrix.from_triplets(n, r[keep], c[keep], v[keep])


MATRICES = {
    "anderson-16": lambda: _level_ordered(lm.gen_anderson_3d(16, seed=3)),
    "anderson-24-natural": lambda: lm.gen_anderson_3d(24, seed=1),
    "potential-2d": lambda: _level_ordered(_potential_2d()),
    "band-far": _band_far,
}


def _mpk(ap, k, x, sweep=False, tiling=None):
    import torch

    t = tiling if tiling is not None else K.Tiling(ap.device(), k)
    y = torch.zeros((k + 1, ap.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k), flags=_lib.FLAG_SWEEP if sweep else 0, exact=True)
    return t, y.cpu().numpy()


@pytest.mark.parametrize("name", list(MATRICES))
@pytest.mark.parametrize("tile_kb", [None, "4"])
def test_dp_mpk_bitwise(name, tile_kb, monkeypatch):
    if tile_kb:
        monkeypatch.setenv("LMPK_DP_TILE_KB", tile_kb)
    ap = MATRICES[name]()
    k = 7
    x = np.random.default_rng(17).uniform(-1, 1, ap.n_rows)
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    t, y = _mpk(ap, k, x)
    assert t.info["dp_tiles"] == t.info["n_tiles"] > 0 and t.info["lean_bytes"] > 0
    assert np.array_equal(y, ref)
    for _ in range(3):  # repeated launches on the same tiling (epoch-tagged progress words)
        _, y = _mpk(ap, k, x, tiling=t)
        assert np.array_equal(y, ref)
    _, ys = _mpk(ap, k, x, sweep=True, tiling=t)
    assert np.array_equal(ys, ref)
    _, y3 = _mpk(ap, 3, x, tiling=t)  # fewer powers than the tiling was planned for
    assert np.array_equal(y3, ref[:4])


def test_dp_block_bytes():
    """A level-ordered Anderson operator: ~1.5 bytes per entry plus the
    8-byte private diagonal per row, against >= 10 for the ring blocks."""
    ap = MATRICES["anderson-16"]()
    t = K.Tiling(ap.device(), 8)
    assert t.info["dp_tiles"] > 0
    assert t.info["lean_bytes"] < 4.0 * ap.n_nz


def test_dp_not_taken(monkeypatch):
    """Constant stencils keep the dictionary lean blocks; random off-diagonal
    values and LMPK_NO_DP keep the ring blocks; forced (LMPK_DP=2) a constant
    stencil runs as DP with the same bits."""
    a = _level_ordered(lm.gen_stencil_3d(16, 2))
    k = 5
    x = np.random.default_rng(2).uniform(-1, 1, a.n_rows)
    ref = O.mpk_powers(a.row_ptr, a.col, a.val, x, k)
    t, y = _mpk(a, k, x)
    assert t.info["dp_tiles"] == 0 and np.array_equal(y, ref)
    monkeypatch.setenv("LMPK_DP", "2")
    t, y = _mpk(a, k, x)
    assert t.info["dp_tiles"] == t.info["n_tiles"] and np.array_equal(y, ref)
    monkeypatch.delenv("LMPK_DP")
    rng = np.random.default_rng(4)
    b = lm.CsrMatrix(a.n_rows, a.row_ptr, a.col, rng.standard_normal(a.n_nz))
    xb = rng.uniform(-1, 1, b.n_rows)
    t, y = _mpk(b, k, xb)
    assert t.info["dp_tiles"] == 0
    assert np.array_equal(y, O.mpk_powers(b.row_ptr, b.col, b.val, xb, k))
    monkeypatch.setenv("LMPK_NO_DP", "1")
    ap = MATRICES["anderson-16"]()
    xa = rng.uniform(-1, 1, ap.n_rows)
    t, y = _mpk(ap, k, xa)
    assert t.info["dp_tiles"] == 0
    assert np.array_equal(y, O.mpk_powers(ap.row_ptr, ap.col, ap.val, xa, k))


@pytest.mark.parametrize("name", ["anderson-16", "potential-2d", "band-far"])
def test_dp_complex_cheb_bitwise(name, monkeypatch):
    """Complex state, Chebyshev kernel + accumulation: DP blocks against the
    ring blocks (LMPK_NO_DP), walk and sweep."""
    import torch

    ap = MATRICES[name]()
    n, k = ap.n_rows, 6
    rng = np.random.default_rng(9)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    cre, cim = rng.standard_normal(k), rng.standard_normal(k)
    p = np.arange(1, k + 1)
    cfg = K.power_cfg(k, p + 1, p, p - 1, np.full(k, _lib.KERNEL_CHEB), cre, cim)
    outs = []
    # the third tiling is built for real vectors (paired units) and run with complex state
    for no_dp, fl, mf in ((False, 0, _lib.FLAG_COMPLEX), (False, _lib.FLAG_SWEEP, _lib.FLAG_COMPLEX), (False, 0, 0),
                          (True, 0, _lib.FLAG_COMPLEX)):
        if no_dp:
            monkeypatch.setenv("LMPK_NO_DP", "1")
        t = K.Tiling(ap.device(), k, mode_flags=mf)
        assert (t.info["dp_tiles"] == 0) == no_dp
        y = torch.zeros((k + 2, 2 * n), dtype=torch.float64, device="cuda")
        y[0] = torch.from_numpy(x.view(np.float64).copy())
        y[1] = torch.from_numpy((0.5 * x).view(np.float64).copy())
        acc = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
        K.mpk_run(t, y, cfg, acc=acc, use_acc=True, complex_state=True, exact=True, flags=fl)
        outs.append((y.cpu().numpy(), acc.cpu().numpy()))
    for o in outs[1:]:
        assert np.array_equal(outs[0][0], o[0])
        assert np.array_equal(outs[0][1], o[1])


def test_dp_real_cheb_acc_vs_oracle():
    """Real Chebyshev batches with accumulation through DP blocks against the
    oracle's cheb_batches (cheb.py:162-246 restated)."""
    a = lm.gen_anderson_3d(12, seed=6)
    lo, hi = lm.gershgorin_bounds(a)
    co = lm.cheb_coeffs_heat(0.05, lo, hi, tol=1e-10)
    x = np.random.default_rng(1).uniform(-1, 1, a.n_rows)
    prop = lm.ChebPropagator(a, 0.05, coeffs=co, p_m_batch=4, cache_bytes=50_000)
    got = prop.step(x)
    til = prop._plan_for[4].tiling(complex_state=False)
    assert til is not None and til.info["dp_tiles"] > 0
    b = lm.scale_for_heat(a, lo, hi)
    p = prop.pre.perm.perm
    rp, c, v = O.permute_symmetric(b.row_ptr, b.col, b.val, p)
    accp = O.cheb_batches(rp, c, v, x[p], co.c)
    ref = np.empty_like(accp)
    ref[p] = accp
    assert np.array_equal(got, ref)


def test_dp_nonfinite_padded_rows():
    """Padded rows with a non-finite operand take the exact-length slow path:
    Inf stays Inf where the CRS sweep gives Inf (no NaN from 0 * Inf)."""
    ap = MATRICES["potential-2d"]()
    k = 3
    x = np.random.default_rng(8).uniform(-1, 1, ap.n_rows)
    x[5] = np.inf
    x[ap.n_rows - 3] = -np.inf
    with np.errstate(invalid="ignore", over="ignore"):
        ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    t, y = _mpk(ap, k, x)
    assert t.info["dp_tiles"] > 0
    assert np.array_equal(y, ref, equal_nan=True)
    assert np.array_equal(np.isnan(y), np.isnan(ref))


def test_dp_torture_repeated_runs():
    """500 launches of the walk on one DP tiling, bitwise stable."""
    import torch

    ap = MATRICES["anderson-16"]()
    k = 8
    x = np.random.default_rng(5).uniform(-1, 1, ap.n_rows)
    ref = torch.from_numpy(O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)).cuda()
    t = K.Tiling(ap.device(), k)
    y = torch.zeros((k + 1, ap.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    cfg = K.mpk_power_cfg(k)
    for rep in range(500):
        y[1:] = 0
        K.mpk_run(t, y, cfg, exact=True, check_errors=(rep % 50 == 49))
        if rep % 10 == 9:
            assert torch.equal(y, ref), rep


def test_dp_periodic_constant_stencil():
    """A constant 7-point stencil on a periodic 112^3 grid: its values fit one
    dictionary, but the level-ordered column offsets exceed int16 (a level's
    neighbours lie up to two level widths away), which used to leave the
    tiling without lean blocks; it now takes DP blocks.  Bitwise against the
    CRS k x SpMV on the same GPU (itself pinned to the oracle elsewhere)."""
    import torch

    offs = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    a = lm.grid_operator((112, 112, 112), [(o, -1.0) for o in offs], periodic=True, diagonal=np.full(112**3, 6.0))
    ap = _level_ordered(a)
    k = 6
    t = K.Tiling(ap.device(), k)
    assert t.info["dp_tiles"] == t.info["n_tiles"] > 0  # a level holds ~19.6K rows: offsets up to +-39K
    x = torch.from_numpy(np.random.default_rng(6).uniform(-1, 1, ap.n_rows)).cuda()
    y = torch.zeros((k + 1, ap.n_rows), dtype=torch.float64, device="cuda")
    y[0] = x
    K.mpk_run(t, y, K.mpk_power_cfg(k), exact=True)
    yb = torch.zeros_like(y)
    yb[0] = x
    K.mpk_baseline(ap.device(), yb, k)
    assert torch.equal(y, yb)
    print("periodic 112^3:", {kk: t.info[kk] for kk in ("n_tiles", "dp_tiles", "lean_bytes", "block_bytes")})
