"""GPU parity of the compressed tile blocks (LMPK_FLAG_COMPRESS: int16 column
offsets, per-tile value dictionary): the MPK, the sweep and the complex
Chebyshev path must give the same bits as the oracle's sequential CRS sums
(executor.py:121-135) on matrices that exercise every block format -- all
dictionary tiles, raw-value tiles, plain tiles for slices whose column offsets
do not fit int16, and tilings that mix the three."""

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


def _band_mixed(n=50_000, seed=5):
    """Band matrix (offsets +-1, +-37) with a few long-range couplings
    (|col - row| > 32767 in some slices) and small-set values in the first
    half, distinct random values in the second half."""
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    rows, cols = [i], [i]
    for d in (1, 37):
        rows += [i[:-d], i[d:]]
        cols += [i[d:], i[:-d]]
    far = np.arange(0, n - 40_000, 997)
    rows += [far, far + 40_000]
    cols += [far + 40_000, far]
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.where(r < n // 2, rng.choice([-1.0, 0.5, 2.25, 6.0], r.size), rng.standard_normal(r.size))
    return lm.CsrMatrix.from_triplets(n, r, c, v)


def _with_empty_rows(n=3001):
    """2D stencil rows interleaved with empty rows; n not a multiple of 32."""
    a = lm.gen_stencil_2d7pt(40, 40)
    r, c, v = a.to_triplets()
    return lm.CsrMatrix.from_triplets(n, r, c, v)


MATRICES = {
    "3d-24-o2": lambda: _level_ordered(lm.gen_stencil_3d(24, 2)),
    "3d-16-o4": lambda: _level_ordered(lm.gen_stencil_3d(16, 4)),
    "27pt-perturbed-20": lambda: _level_ordered(lm.gen_stencil_3d27pt(20)),
    "anderson-12": lambda: _level_ordered(lm.gen_anderson_3d(12)),
    "rmat-s12": lambda: _level_ordered(lm.gen_rmat(12)),
    "band-mixed": _band_mixed,
    "empty-rows": _with_empty_rows,
}


def _run(ap, k, mode, slots, tile, x, sweep=False):
    import torch

    fl = (_lib.FLAG_MODE_RESIDENT if mode == "res" else _lib.FLAG_MODE_STREAM) | _lib.FLAG_COMPRESS
    t = K.Tiling(ap.device(), k, tile_nnz=tile, slots=slots, mode_flags=fl)
    y = torch.zeros((k + 1, ap.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k), flags=_lib.FLAG_SWEEP if sweep else 0, exact=True)
    return t, y.cpu().numpy()


@pytest.mark.parametrize("name", list(MATRICES))
@pytest.mark.parametrize("mode,slots,tile", [("stream", 2, 0), ("stream", 4, 600), ("res", 3, 900)])
def test_compressed_mpk_bitwise(name, mode, slots, tile):
    ap = MATRICES[name]()
    k = 6
    x = np.random.default_rng(17).uniform(-1, 1, ap.n_rows)
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    try:
        t, y = _run(ap, k, mode, slots, tile, x)
    except RuntimeError as e:  # the resident walk needs its window of tiles co-resident
        assert mode == "res" and "no feasible tiling" in str(e)
        pytest.skip("resident walk infeasible for this tiling")
    assert t.info["compressed_tiles"] > 0 or name == "rmat-s12"
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("name", ["3d-24-o2", "band-mixed"])
def test_compressed_sweep_bitwise(name):
    ap = MATRICES[name]()
    k = 4
    x = np.random.default_rng(3).uniform(-1, 1, ap.n_rows)
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    _, y = _run(ap, k, "stream", 2, 500, x, sweep=True)
    assert np.array_equal(y, ref)


def test_block_formats_present():
    """band-mixed must produce all three formats: dictionary tiles (first
    half), raw-value tiles (second half) and plain tiles (far couplings)."""
    ap = _band_mixed()
    t = K.Tiling(ap.device(), 4, tile_nnz=2000, slots=2, mode_flags=_lib.FLAG_MODE_STREAM | _lib.FLAG_COMPRESS)
    info = t.info
    assert 0 < info["dict_tiles"] < info["compressed_tiles"] < info["n_tiles"]
    plain = K.Tiling(ap.device(), 4, tile_nnz=2000, slots=2, mode_flags=_lib.FLAG_MODE_STREAM)
    assert plain.info["compressed_tiles"] == 0
    assert info["block_bytes"] < plain.info["block_bytes"]


def test_stencil_dictionary_bytes():
    """A level-ordered 7-point stencil compresses to ~3 bytes per entry."""
    ap = MATRICES["3d-24-o2"]()
    t = K.Tiling(ap.device(), 8, slots=2, mode_flags=_lib.FLAG_MODE_STREAM | _lib.FLAG_COMPRESS)
    assert t.info["dict_tiles"] == t.info["n_tiles"]
    assert t.info["block_bytes"] < 4.0 * ap.n_nz


def test_compressed_complex_cheb_bitwise():
    """Complex state through the compressed blocks, Chebyshev kernel + acc."""
    import torch

    ap = MATRICES["anderson-12"]()
    n, k = ap.n_rows, 5
    rng = np.random.default_rng(9)
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n))
    cre = rng.standard_normal(k)
    cim = rng.standard_normal(k)
    outs = []
    for fl in (_lib.FLAG_COMPRESS, 0):
        t = K.Tiling(ap.device(), k, tile_nnz=700, slots=2,
                     mode_flags=_lib.FLAG_MODE_STREAM | _lib.FLAG_COMPLEX | fl)
        y = torch.zeros((k + 2, 2 * n), dtype=torch.float64, device="cuda")
        y[0] = torch.from_numpy(x.view(np.float64).copy())
        y[1] = torch.from_numpy((0.5 * x).view(np.float64).copy())
        acc = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
        p = np.arange(1, k + 1)
        cfg = K.power_cfg(k, p + 1, p, p - 1, np.full(k, _lib.KERNEL_CHEB), cre, cim)
        K.mpk_run(t, y, cfg, acc=acc, use_acc=True, complex_state=True, exact=True)
        outs.append((y.cpu().numpy(), acc.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("name", ["3d-24-o2", "27pt-perturbed-20", "band-mixed"])
@pytest.mark.parametrize("misaligned", [False, True])
@pytest.mark.parametrize("ring", [False, True])
def test_compressed_x_staged_bitwise(name, misaligned, ring, monkeypatch):
    """Compressed blocks whose gathers come from the staged x-segments (local
    int16 columns, LMPK_XFRAC); a slot stride that is not 16-byte aligned
    takes the cooperative-copy path."""
    import torch

    monkeypatch.setenv("LMPK_XFRAC", "50")
    ap = MATRICES[name]()
    n, k = ap.n_rows, 6
    x = np.random.default_rng(23).uniform(-1, 1, n)
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    fl = (_lib.FLAG_RING if ring else _lib.FLAG_MODE_STREAM) | _lib.FLAG_COMPRESS
    t = K.Tiling(ap.device(), k, tile_nnz=1500 if not ring else 4000, slots=2 if not ring else 6, mode_flags=fl)
    assert t.info["x_staged_tiles"] > 0 and t.info["compressed_tiles"] > 0
    assert (t.info["mode"] == 3) == ring
    ld = n + (1 if misaligned and n % 2 == 0 else 0)
    buf = torch.zeros((k + 1) * ld + 1, dtype=torch.float64, device="cuda")
    y = buf[1:1 + (k + 1) * ld].view(k + 1, ld)[:, :n] if misaligned else buf[:(k + 1) * ld].view(k + 1, ld)
    y[0] = torch.from_numpy(x)
    for _ in range(2):
        K.mpk_run(t, y, K.mpk_power_cfg(k), exact=True)
        assert np.array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("name", ["3d-24-o2", "27pt-perturbed-20", "band-mixed", "rmat-s12", "empty-rows"])
@pytest.mark.parametrize("comp,pieces,run", [(1, 6, 0), (1, 4, 3000), (0, 8, 5000), (1, 16, 1)])
def test_ring_walk_bitwise(name, comp, pieces, run):
    """Ring walk (LMPK_FLAG_RING): tiles streamed through a ring of smem
    pieces, items = runs of tiles; plain and compressed tiles, tiny runs
    (run = 1 nnz: one tile per item) and deep rings."""
    import torch

    ap = MATRICES[name]()
    n, k = ap.n_rows, 7
    x = np.random.default_rng(31).uniform(-1, 1, n)
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    fl = _lib.FLAG_MODE_STREAM | _lib.FLAG_RING | (_lib.FLAG_COMPRESS if comp else 0)
    t = K.Tiling(ap.device(), k, tile_nnz=run, slots=pieces, mode_flags=fl)
    assert t.info["mode"] == 3 and t.info["super_tiles"] >= 1
    y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    for rep in range(3):
        K.mpk_run(t, y, K.mpk_power_cfg(k), exact=True)
        assert np.array_equal(y.cpu().numpy(), ref), rep
    y[1:] = 0
    K.mpk_run(t, y, K.mpk_power_cfg(k), flags=_lib.FLAG_SWEEP, exact=True)
    assert np.array_equal(y.cpu().numpy(), ref)


def test_ring_cheb_complex_bitwise():
    """Complex Chebyshev + accumulation through the ring walk equals the group walk."""
    import torch

    ap = MATRICES["anderson-12"]()
    n, k = ap.n_rows, 6
    rng = np.random.default_rng(4)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    cre, cim = rng.standard_normal(k), rng.standard_normal(k)
    outs = []
    for fl in (_lib.FLAG_RING | _lib.FLAG_COMPRESS, 0):
        t = K.Tiling(ap.device(), k, tile_nnz=2000, slots=4, mode_flags=_lib.FLAG_MODE_STREAM | _lib.FLAG_COMPLEX | fl)
        y = torch.zeros((k + 2, 2 * n), dtype=torch.float64, device="cuda")
        y[0] = torch.from_numpy(x.view(np.float64).copy())
        y[1] = torch.from_numpy((0.25 * x).view(np.float64).copy())
        acc = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
        p = np.arange(1, k + 1)
        cfg = K.power_cfg(k, p + 1, p, p - 1, np.full(k, _lib.KERNEL_CHEB), cre, cim)
        K.mpk_run(t, y, cfg, acc=acc, use_acc=True, complex_state=True, exact=True)
        outs.append((y.cpu().numpy(), acc.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_hub_rows_fall_back_to_crs_sweeps():
    """A star graph (row 0 couples to all 70,000 rows) exceeds the tile
    format's 65535-entry rows: run_mpk runs the plan as CRS sweeps, same bits."""
    n = 70_000
    i = np.arange(1, n)
    rows = np.concatenate([np.zeros(n - 1, dtype=np.int64), i, np.arange(n)])
    cols = np.concatenate([i, np.zeros(n - 1, dtype=np.int64), np.arange(n)])
    vals = np.concatenate([np.full(n - 1, -1e-3), np.full(n - 1, -1e-3), np.full(n, 2.0)])
    a = lm.CsrMatrix.from_triplets(n, rows, cols, vals)
    x = np.random.default_rng(2).uniform(-1, 1, n)
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", 4, 126e6)
    ap = pre.a
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, pre.perm.apply_to_vector(x), 4)
    assert np.array_equal(np.asarray(res.y.data), ref)


def _star(n, off=-1e-3, diag=2.0):
    i = np.arange(1, n)
    rows = np.concatenate([np.zeros(n - 1, dtype=np.int64), i, np.arange(n)])
    cols = np.concatenate([i, np.zeros(n - 1, dtype=np.int64), np.arange(n)])
    vals = np.concatenate([np.full(n - 1, off), np.full(n - 1, off), np.full(n, diag)])
    return lm.CsrMatrix.from_triplets(n, rows, cols, vals)


@pytest.mark.parametrize("cplx", [False, True])
def test_hub_rows_chebyshev_plans_run_as_crs_sweeps(cplx):
    """Chebyshev propagation (fused recurrence + accumulation, real heat and
    complex Schrodinger coefficients) on the star graph: its 70,000-entry row
    exceeds the tile format, so every batch runs as lmpk_mpk_crs_run sweeps --
    bitwise the oracle's restatement of ChebPropagator.step (cheb.py:221-246)."""
    from oracle import cpu as C

    a = _star(70_000, off=-1e-4, diag=0.5)
    lo, hi = lm.gershgorin_bounds(a)
    rng = np.random.default_rng(3)
    if cplx:
        co = lm.cheb_coeffs_schrodinger(0.3, lo, hi, tol=1e-10)
        x = np.exp(1j * rng.uniform(0, 2 * np.pi, a.n_rows)) / np.sqrt(a.n_rows)
        prop = lm.ChebPropagator(a, 0.3, coeffs=co, p_m_batch=4, cache_bytes=126e6)
    else:
        prop = lm.ChebPropagator(a, 0.3, tol=1e-8, p_m_batch=4, cache_bytes=126e6)
        co = prop.coeffs
        x = rng.uniform(-1, 1, a.n_rows)
    assert prop._plan_for[4].tiling(complex_state=cplx) is None  # the tile format refuses the hub row
    got = prop.step(x)
    b = lm.scale_for_heat(a, lo, hi)
    p = prop.pre.perm.perm
    rp, c, v = C.permute_symmetric(b.row_ptr, b.col, b.val, p)
    accp = O.cheb_batches(rp, c, v, x[p], np.real(co.c), np.imag(co.c) if cplx else None)
    ref = np.empty_like(accp)
    ref[p] = accp
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("sched", ["walk", "sweep", "crs", "auto"])
def test_schedule_choice_bitwise(sched, monkeypatch):
    """The executor's walk / sweep choice (LMPK_SCHEDULE) never changes the bits."""
    monkeypatch.setenv("LMPK_SCHEDULE", sched)
    a = lm.gen_stencil_3d27pt(72, seed=3)  # > 4M nnz: 'auto' times both
    x = np.random.default_rng(8).uniform(-1, 1, a.n_rows)
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", 4, 126e6)
    ap = pre.a
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, pre.perm.apply_to_vector(x), 4)
    assert np.array_equal(np.asarray(res.y.data), ref)


def test_ring_oversize_slices_read_from_global():
    """Rows of 40,000 entries make slices far larger than a ring piece: those
    tiles stay plain and are read from global memory by the consumers
    (the ring kernel's long-row variant); the rest are compressed."""
    import torch

    n, k = 50_000, 3
    rng = np.random.default_rng(12)
    i = np.arange(n)
    rows, cols = [i, i[:-1], i[1:]], [i, i[1:], i[:-1]]
    hubs = np.array([10, 20_000, 49_990])
    for h in hubs:
        nb = rng.choice(n, 40_000, replace=False)
        rows += [np.full(nb.size, h), nb]
        cols += [nb, np.full(nb.size, h)]
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    a = lm.CsrMatrix.from_triplets(n, r, c, rng.uniform(-1, 1, r.size) * 1e-3)
    x = rng.uniform(-1, 1, n)
    ref = O.mpk_powers(a.row_ptr, a.col, a.val, x, k)
    t = K.Tiling(a.device(), k)
    assert t.info["mode"] == 3 and 0 < t.info["compressed_tiles"] < t.info["n_tiles"]
    y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k), exact=True)
    assert np.array_equal(y.cpu().numpy(), ref)
