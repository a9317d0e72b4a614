"""GPU parity: every liblmpk kernel against the reference's own fixtures and
the oracle, bit for bit.  Mirrors the reference's test pyramid
(pkg/tests/test_levels.py, test_csr.py, test_executor.py, test_acceptance.py
criteria 1/2/7) on the B200."""

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from matrices import CORPUS, sha
from oracle import cpu as C
from oracle import levelmpk_oracle as O
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu

SMALL = [k for k in CORPUS if k != "cfg1"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


# ------------------------------------------------------------------ BFS levels
@pytest.mark.parametrize("name", list(CORPUS))
def test_bfs_levels_bitexact_vs_reference(name, golden):
    facts, arr = golden
    a = CORPUS[name]()
    rec = facts["matrices"][name]
    roots = [int(k[3:-5]) for k in rec if k.startswith("bfs") and k.endswith("_perm")]
    for root in roots:
        levels, perm = lm.bfs_levels(a, root)
        assert sha(perm.perm) == rec[f"bfs{root}_perm"]
        assert np.array_equal(levels.level_ptr, arr[f"{name}/bfs{root}/level_ptr"])
        assert np.array_equal(perm.perm[perm.inv_perm], np.arange(a.n_rows))


def test_bfs_known_answers():
    levels, perm = lm.bfs_levels(lm.gen_stencil_2d7pt(8, 8), 0)
    assert levels.n_levels == 15 and levels.level_ptr.tolist()[:4] == [0, 1, 3, 6]
    a = lm.CsrMatrix.from_triplets(1, [0], [0], [1.0])
    levels, perm = lm.bfs_levels(a, 0)
    assert levels.level_ptr.tolist() == [0, 1] and perm.perm.tolist() == [0]
    path = lm.CsrMatrix.from_triplets(4, [0, 1, 1, 2, 2, 3], [1, 0, 2, 1, 3, 2], np.ones(6))
    levels, perm = lm.bfs_levels(path, 0)
    assert levels.level_ptr.tolist() == [0, 1, 2, 3, 4] and perm.perm.tolist() == [0, 1, 2, 3]
    with pytest.raises(ValueError, match="root"):
        lm.bfs_levels(lm.gen_stencil_2d7pt(3, 3), 9)


@pytest.mark.parametrize("seed", range(12))
def test_bfs_random_graphs_vs_oracle(seed):
    """Asymmetric, disconnected, isolated vertices, arbitrary roots."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 3000))
    m = int(rng.integers(0, 3 * n))
    r, c = rng.integers(0, n, m), rng.integers(0, n, m)
    if m == 0:
        r, c = np.array([0]), np.array([0])
    a = lm.CsrMatrix.from_triplets(n, r, c, np.ones(r.size))
    root = int(rng.integers(0, n))
    levels, perm = lm.bfs_levels(a, root)
    op, olp = O.bfs_levels(a.row_ptr, a.col, root, method="frontier")
    assert np.array_equal(perm.perm, op) and np.array_equal(levels.level_ptr, olp)


def test_symmetrized_pattern_vs_oracle():
    a = CORPUS["asym-300"]()
    rp, col = lm.symmetrized_pattern(a)
    orp, ocol = O.symmetrized_pattern(a.row_ptr, a.col)
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol)


# ------------------------------------------------------------------ permutation + SpMV
@pytest.mark.parametrize("name", list(CORPUS))
def test_permute_symmetric_bitexact(name, golden):
    facts, _ = golden
    a = CORPUS[name]()
    _, perm = lm.bfs_levels(a, 0)
    b = lm.permute_symmetric(a, perm)
    assert [sha(b.row_ptr), sha(b.col), sha(b.val)] == facts["matrices"][name]["perm_csr"]


def test_permute_random_and_long_rows(rng):
    a = lm.gen_rmat(12)  # rows up to several hundred entries -> long-row sort path
    p = rng.permutation(a.n_rows)
    b = lm.permute_symmetric(a, lm.Permutation(p))
    o = O.permute_symmetric(a.row_ptr, a.col, a.val, p)
    assert all(np.array_equal(x, y) for x, y in zip((b.row_ptr, b.col, b.val), o))
    assert lm.permute_symmetric(a, lm.Permutation.identity(a.n_rows)) == a


def test_spmv_range_semantics(rng):
    a = lm.CsrMatrix.from_triplets(3, [0, 1, 1, 2], [0, 0, 1, 2], [2.0, 1.0, 3.0, 5.0])
    out = np.full(3, -7.0)
    lm.spmv_range(a, np.ones(3), out, 1, 1)
    assert out.tolist() == [-7.0, 4.0, -7.0]
    b = lm.gen_stencil_2d7pt(9, 6)
    x = rng.standard_normal(b.n_rows)
    full = np.zeros(b.n_rows)
    lm.spmv_range(b, x, full, 0, b.n_rows - 1)
    assert np.array_equal(full, O.spmv(b.row_ptr, b.col, b.val, x))
    parts = np.zeros(b.n_rows)
    for lo, hi in ((0, 11), (11, 12), (12, 30), (30, b.n_rows)):
        lm.spmv_range(b, x, parts, lo, hi - 1)
    assert np.array_equal(full, parts)
    with pytest.raises(ValueError, match="alias"):
        lm.spmv_range(b, x, x, 0, 3)
    with pytest.raises(ValueError, match="out of bounds"):
        lm.spmv_range(b, x, parts, 0, b.n_rows)


# ------------------------------------------------------------------ MPK
@pytest.mark.parametrize("name", list(CORPUS))
def test_baseline_vs_reference_hashes(name, golden):
    facts, _ = golden
    rec = facts["matrices"][name]
    a = CORPUS[name]()
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    x = np.random.default_rng(99).standard_normal(a.n_rows)
    res = lm.run_baseline(ap, perm.apply_to_vector(x), rec["baseline_p_m"])
    assert [sha(res.y.data[p]) for p in range(rec["baseline_p_m"] + 1)] == rec["baseline_y"]


@pytest.mark.parametrize("name", SMALL)
def test_all_variants_bitwise_equal_reference(name, golden):
    """Acceptance criterion 1 (test_acceptance.py:59-87) on the GPU: every
    variant and p_m equals the reference's baseline power vectors bitwise."""
    a = CORPUS[name]()
    x = np.random.default_rng(99).standard_normal(a.n_rows)
    cache = max(12 * a.n_nz // 4, 3_000)
    for p_m in (1, 2, 4, 5, 8):
        oracle = None
        for variant, s_m in (("lb", 0), ("lb_lg", 0), ("lb_lg_p2p", 0), ("lb_lg_p2p_rec", 0)):
            res, pre = lm.run_mpk(a, x, variant, p_m, cache, s_m=s_m, workers=2)
            if oracle is None:
                rp, c, v = C.permute_symmetric(a.row_ptr, a.col, a.val, pre.perm.perm)
                oracle = O.mpk_powers(rp, c, v, pre.perm.apply_to_vector(x), p_m)
            assert np.array_equal(res.y.data, oracle), (name, variant, p_m)


@pytest.mark.parametrize("name", [k for k in SMALL if not k.startswith("rmat")])
def test_plan_checks_match_reference(name, golden):
    facts, arr = golden
    a = CORPUS[name]()
    pre = lm.prepare(a, "lb_lg_p2p", 4, facts["matrices"][name]["groups_cache"])
    got = [[g.row_start, g.row_end, g.nnz, g.boundary_left_end, g.boundary_right_start,
            g.n_levels, bool(g.violates)] for g in pre.tree.groups]
    assert got == facts["matrices"][name]["groups_p4"]
    plan = lm.build_plan(pre, "lb_lg_p2p", 2)
    for key in ("check_ptr", "check_item", "check_kind"):
        assert np.array_equal(getattr(plan, key), arr[f"{name}/{key}"]), key
    assert np.array_equal(plan.chunks, arr[f"{name}/chunks_w2"])
    assert np.diff(plan.check_ptr).max() <= 2
    assert all(np.diff(plan.check_ptr)[k] == 0 for k in range(plan.n_items) if plan.power[k] == 1)


@pytest.mark.parametrize("mode,slots,tile", [
    ("res", 2, 0), ("res", 4, 0), ("res", 3, 700), ("stream", 2, 0), ("stream", 3, 400),
    ("stream", 4, 0), ("sweep", 2, 0), ("sweep", 4, 300)])
def test_kernel_modes_bitwise(mode, slots, tile):
    """Resident / streaming / sweep, several tile sizes and slot counts: all
    produce the same bits (tiny tiles stress the dependency machinery)."""
    a = lm.gen_stencil_3d(24, 2)
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    x = np.random.default_rng(3).standard_normal(a.n_rows)
    k = 8
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    import torch

    fl = _lib.FLAG_MODE_RESIDENT if mode == "res" else _lib.FLAG_MODE_STREAM
    t = K.Tiling(ap.device(), k, tile_nnz=tile, slots=slots, mode_flags=fl)
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k), flags=_lib.FLAG_SWEEP if mode == "sweep" else 0)
    assert np.array_equal(y.cpu().numpy(), ref)


def test_torture_repeated_runs_bitwise_stable():
    """Liveness / race hunt (test_executor.py:134-152, criterion 7)."""
    import torch

    a = lm.gen_stencil_3d(24, 2)
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    x = np.random.default_rng(13).standard_normal(a.n_rows)
    ref = torch.from_numpy(O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, 8)).cuda()
    for fl, slots, tile in ((_lib.FLAG_MODE_STREAM, 3, 500), (_lib.FLAG_MODE_RESIDENT, 4, 800)):
        t = K.Tiling(ap.device(), 8, tile_nnz=tile, slots=slots, mode_flags=fl)
        y = torch.zeros_like(ref)
        y[0] = ref[0]
        cfg = K.mpk_power_cfg(8)
        for rep in range(300):
            K.mpk_run(t, y, cfg, check_errors=(rep % 50 == 0))
            if rep % 50 == 0:
                assert torch.equal(y, ref), rep
        K.mpk_run(t, y, cfg)
        assert torch.equal(y, ref)


def test_x_never_mutated_and_undo(rng):
    a = lm.gen_stencil_2d7pt(8, 8)
    x = rng.standard_normal(a.n_rows)
    keep = x.copy()
    res, pre = lm.run_mpk(a, x, "lb_lg_p2p", 3, 4_000, workers=2)
    assert np.array_equal(x, keep)
    assert np.array_equal(res.y[0], pre.perm.apply_to_vector(x))
    orig = lm.undo_permutation(res, pre.perm)
    assert np.array_equal(orig[0], x)
    nat = lm.run_baseline(a, x, 3)
    for p in range(1, 4):
        assert np.max(np.abs(orig[p] - nat.y[p]) / np.maximum(np.abs(nat.y[p]), 1e-300)) < 1e-13


def test_barrier_count_and_gflops():
    a = lm.gen_stencil_2d7pt(8, 8)
    pre = lm.prepare(a, "lb_lg", 3, 3_000)
    res = lm.run_plan(lm.build_plan(pre, "lb_lg", 2), x=np.ones(a.n_rows))
    assert res.barrier_count == len(pre.tree.groups) * 3
    res2 = lm.run_plan(lm.build_plan(lm.prepare(a, "lb_lg_p2p", 3, 3_000), "lb_lg_p2p", 2),
                       x=np.ones(a.n_rows))
    assert res2.barrier_count == 0
    assert res2.gflops(a.n_nz, 3) == pytest.approx(2 * a.n_nz * 3 / res2.seconds / 1e9)


def test_error_contract():
    a = lm.gen_stencil_2d7pt(3, 3)
    with pytest.raises(ValueError, match="length"):
        lm.run_baseline(a, np.ones(5), 2)
    with pytest.raises(ValueError, match="variant"):
        lm.run_mpk(a, np.ones(9), "bogus", 2, 1000)
    with pytest.raises(ValueError, match="p_m"):
        lm.run_mpk(a, np.ones(9), "lb_lg_p2p", 0, 1000)


def test_device_resident_power_vectors():
    import torch

    a = lm.gen_stencil_3d(16, 2)
    pre = lm.prepare(a, "lb_lg_p2p", 6, 200_000)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    x = torch.rand(a.n_rows, dtype=torch.float64, device="cuda")
    res = lm.run_plan(plan, x=x)
    assert res.y.on_device
    host = lm.run_plan(plan, x=x.cpu().numpy())
    assert np.array_equal(res.y.data.cpu().numpy(), host.y.data)


@pytest.mark.parametrize("variant", ["ready_queue", "x_staged", "x_staged_misaligned"])
def test_opt_in_walks_bitwise(variant, monkeypatch):
    """Opt-in paths of the group kernel: the dependency-driven ready-queue walk
    (LMPK_FLAG_READY_QUEUE) and x-segment staging (LMPK_XFRAC; a slot stride
    that is not 16-byte aligned takes the cooperative-copy fallback)."""
    import torch

    a = lm.gen_stencil_3d(24, 2)
    _, perm = lm.bfs_levels(a, 0)
    ap = lm.permute_symmetric(a, perm)
    n, k = a.n_rows, 6
    x = np.random.default_rng(21).standard_normal(n)
    ref = O.mpk_powers(ap.row_ptr, ap.col, ap.val, x, k)
    flags = 0
    if variant.startswith("x_staged"):
        monkeypatch.setenv("LMPK_XFRAC", "30")
    else:
        flags = _lib.FLAG_READY_QUEUE
    t = K.Tiling(ap.device(), k, tile_nnz=700, slots=2, mode_flags=_lib.FLAG_MODE_STREAM)
    if variant.startswith("x_staged"):
        assert t.info["x_staged_tiles"] > 0
    ld = n + (1 if variant == "x_staged_misaligned" and n % 2 == 0 else 0)
    buf = torch.zeros((k + 1) * ld + 1, dtype=torch.float64, device="cuda")
    y = buf[1:1 + (k + 1) * ld].view(k + 1, ld)[:, :n] if variant == "x_staged_misaligned" \
        else buf[:(k + 1) * ld].view(k + 1, ld)
    y[0] = torch.from_numpy(x)
    for _ in range(3):
        K.mpk_run(t, y, K.mpk_power_cfg(k), flags=flags)
        assert np.array_equal(y.cpu().numpy(), ref)
