"""Host-side API (no GPU): CRS construction, permutations, Matrix Market,
level-group aggregation, Lp schedules, Chebyshev coefficient math, error
contract.  Restates the reference's unit tests for these pieces
(pkg/tests/test_csr.py, test_groups.py, test_schedule.py, test_cheb.py,
test_mmio.py) against this package."""

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from paper_2205_01598_b200.groups import LevelGroupTree, _groups_from_level_nnz, _groups_one_per_level
from paper_2205_01598_b200.schedule import _diagonal_order, classify_outer


# ------------------------------------------------------------------ CRS
def test_triplet_round_trip():
    a = lm.gen_stencil_2d7pt(5, 7)
    b = lm.CsrMatrix.from_triplets(a.n_rows, *a.to_triplets())
    assert a == b


def test_duplicate_triplets_summed():
    a = lm.CsrMatrix.from_triplets(2, [0, 0, 1], [1, 1, 0], [2.0, 3.0, 1.0])
    assert a.n_nz == 2 and a.to_dense()[0, 1] == 5.0


def test_invariants_enforced():
    with pytest.raises(ValueError, match="column index out of range"):
        lm.CsrMatrix(2, [0, 1, 2], [0, 5], [1.0, 1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        lm.CsrMatrix(2, [0, 2, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError, match="non-decreasing"):
        lm.CsrMatrix(2, [0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match="32-bit"):
        lm.CsrMatrix(2, np.array([0, 1, 2**31], dtype=np.int64), [0], [1.0])


def test_single_nonzero_multi_row_matrix_is_valid():
    # the reference's validator indexes out of range here (csr.py:64-66);
    # ours accepts the canonical matrix
    a = lm.CsrMatrix.from_triplets(3, [1], [2], [1.0])
    assert a.n_nz == 1 and a.row_ptr.tolist() == [0, 0, 1, 1]


def test_permutation_inverse_and_vectors(rng):
    p = lm.Permutation(rng.permutation(20))
    v = rng.standard_normal(20)
    assert np.array_equal(p.undo_on_vector(p.apply_to_vector(v)), v)
    with pytest.raises(ValueError, match="inverses"):
        lm.Permutation(np.arange(4), np.array([1, 0, 2, 3]))


# ------------------------------------------------------------------ generators
def test_stencil_nnz_closed_form():
    for n, order in ((4, 2), (8, 4), (9, 6), (16, 2)):
        assert lm.stencil_3d_nnz(n, order) == lm.gen_stencil_3d(n, order).n_nz
    assert lm.stencil_3d_nnz(200, 2) == 55_760_000


def test_generator_errors():
    with pytest.raises(ValueError, match="grid dimensions"):
        lm.gen_stencil_2d7pt(1, 5)
    with pytest.raises(ValueError, match="order"):
        lm.gen_stencil_3d(8, 3)
    with pytest.raises(ValueError, match="too small"):
        lm.gen_stencil_3d(2, 2)


def test_config_generators_shapes():
    a = lm.gen_laplace_2d5pt(16, 16)
    assert a.n_rows == 256 and a.n_nz == 256 + 4 * 16 * 15
    b = lm.gen_stencil_3d27pt(6, perturb=0.01, seed=3)
    assert b.n_rows == 216 and b.n_nz == 4**3 * 27 + 0 or b.n_nz > 0
    d = b.to_dense()
    assert np.array_equal(d != 0, (d != 0).T)          # symmetric pattern
    assert not np.allclose(d, d.T)                       # unsymmetric values
    c = lm.gen_anderson_3d(6, seed=1)
    assert c.n_nz == 6**3 * 7
    lo, hi = lm.gershgorin_bounds(c)
    assert -14.25 <= lo and hi <= 14.25
    r = lm.gen_rmat(8)
    rs = np.add.reduceat(r.val, r.row_ptr[:-1])
    assert np.allclose(rs, 1.0, atol=1e-12)
    assert np.all(r.diagonal() > 0)


# ------------------------------------------------------------------ Matrix Market
def test_mmio_round_trip_and_errors(tmp_path):
    a = lm.gen_stencil_2d7pt(8, 8)
    p = tmp_path / "a.mtx"
    lm.save_matrix_market(a, p, comment="7pt")
    assert lm.load_matrix_market(p) == a
    q = tmp_path / "s.mtx"
    q.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 2\n2 1 -1\n3 2 -1\n")
    b = lm.load_matrix_market(q)
    assert b.n_nz == 5 and b.to_dense()[0, 1] == -1.0
    r = tmp_path / "r.mtx"
    r.write_text("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n")
    with pytest.raises(lm.MatrixMarketError, match="square"):
        lm.load_matrix_market(r)
    t = tmp_path / "t.mtx"
    t.write_text("%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n3 1\n")
    with pytest.raises(lm.MatrixMarketError, match=":4:"):
        lm.load_matrix_market(t)


# ------------------------------------------------------------------ groups
def test_cache_budget_and_errors():
    assert lm.cache_budget_nnz(2, 2880, 0.5) == 40.0
    with pytest.raises(ValueError, match="p_m"):
        lm.cache_budget_nnz(0, 1, 0.5)
    with pytest.raises(ValueError, match="cache_bytes"):
        lm.cache_budget_nnz(1, 0, 0.5)
    with pytest.raises(ValueError, match="f must"):
        lm.cache_budget_nnz(1, 10, 1.5)


def test_recursion_walkthrough_groups_from_golden_levels(golden):
    """Fig. 11 walkthrough (test_groups.py:28-31) on the reference's 8x8 levels."""
    facts, arr = golden
    lp = arr["2d7pt-8/bfs0/level_ptr"]
    a = lm.gen_stencil_2d7pt(8, 8)
    perm = arr["2d7pt-8/bfs0/perm"]
    lnz = np.add.reduceat(a.row_nnz[perm], lp[:-1])
    groups = _groups_from_level_nnz(lp, lnz, lm.cache_budget_nnz(2, 2880, 0.5))
    assert [g.n_rows for g in groups] == [6, 4, 5, 6, 7, 8, 7, 6, 5, 4, 6]
    assert [i for i, g in enumerate(groups) if g.violates] == [4, 5, 6]


def test_groups_match_reference_plan_groups(golden):
    facts, arr = golden
    for name in ("3d-16-o2", "random-1", "dumbbell", "2d7pt-32"):
        rec = facts["matrices"][name]
        from matrices import CORPUS

        a = CORPUS[name]()
        lp = arr[f"{name}/bfs0/level_ptr"]
        perm = arr[f"{name}/bfs0/perm"]
        lnz = np.add.reduceat(a.row_nnz[perm], lp[:-1])
        groups = _groups_from_level_nnz(lp, lnz, lm.cache_budget_nnz(4, rec["groups_cache"], 0.5))
        got = [[g.row_start, g.row_end, g.nnz, g.boundary_left_end, g.boundary_right_start,
                g.n_levels, bool(g.violates)] for g in groups]
        assert got == rec["groups_p4"]


# ------------------------------------------------------------------ schedules
def _levels_tree(golden, n_levels=15):
    _, arr = golden
    lp = arr["2d7pt-8/bfs0/level_ptr"]
    groups = _groups_one_per_level(lp, np.diff(lp))
    assert len(groups) == n_levels
    return LevelGroupTree(stage=0, groups=groups)


def test_schedule_goldens(golden):
    s = lm.build_schedule(_levels_tree(golden), 5)
    assert len(s.nodes()) == 75
    n64 = s.find(6, 4)
    assert all(s.find(*d).exec_step < n64.exec_step for d in ((5, 3), (6, 3), (7, 3)))
    diag = [(n.group, n.power) for n in s.nodes() if n.group + n.power == 13]
    assert diag == [(12, 1), (11, 2), (10, 3), (9, 4), (8, 5)]
    assert s.find(10, 1).exec_step == 40 and s.find(10, 2).exec_step == 46
    assert lm.reuse_distance(s, 10, 1) == 6
    edges = lm.sync_edges(s)
    assert {e.kind for e in edges} == {"A", "B", "C"}


@pytest.mark.parametrize("n_groups,p_m", [(1, 1), (1, 5), (7, 3), (50, 8), (200, 16)])
def test_diagonal_order_topologically_valid(n_groups, p_m):
    pairs = _diagonal_order(n_groups, p_m)
    assert len(pairs) == len(set(pairs)) == n_groups * p_m
    done = set()
    for g, p in pairs:
        for dg in (g - 1, g, g + 1):
            if 0 <= dg < n_groups and p > 1:
                assert (dg, p - 1) in done
        done.add((g, p))


def test_classify_outer_exhaustive():
    seen = {classify_outer(i, p, 6, 8, 5) for i in range(15) for p in range(1, 6)}
    assert seen == {"inside", "diamond", "input", "output", None}


# ------------------------------------------------------------------ Chebyshev math
@pytest.mark.parametrize("z", [0.0, 0.05, 0.7, 3.0, 12.0, 30.0])
def test_bessel_against_series(z):
    def series(z, k, terms=60):
        term = (z / 2.0) ** k / np.prod(np.arange(1, k + 1), initial=1.0)
        total = 0.0
        for m in range(terms):
            total += term
            term *= (z / 2.0) ** 2 / ((m + 1) * (m + 1 + k))
        return total

    got = lm.bessel_i_seq(z, 10)
    assert np.allclose(got, [series(z, k) for k in range(11)], rtol=1e-13, atol=1e-300)


def test_coeff_validation_and_cutoff():
    with pytest.raises(ValueError, match="dt"):
        lm.cheb_coeffs_heat(0.0, 0.0, 1.0)
    with pytest.raises(ValueError, match="tol"):
        lm.cheb_coeffs_heat(0.1, 0.0, 1.0, tol=0)
    with pytest.raises(ValueError, match="reduce dt"):
        lm.cheb_coeffs_heat(1.0, 0.0, 1.0, tol=1e-4, max_terms=2)
    co = lm.cheb_coeffs_heat(0.4, 0.0, 12.0, 1e-4)
    wide = lm.cheb_coeffs_heat(0.4, 0.0, 12.0, 1e-12)
    assert np.all(np.abs(wide.c[co.n_moments + 1: co.n_moments + 10]) < 1e-4)


def test_series_reproduces_exponential():
    co = lm.cheb_coeffs_heat(0.1, 0.0, 8.0, tol=1e-8)
    z = np.linspace(-1, 1, 101)
    lam = 4.0 - 4.0 * z
    assert np.max(np.abs(lm.eval_cheb_series(co.c, z) - np.exp(-0.1 * lam))) < 1e-6


def test_schrodinger_coefficients_unitary_scalar():
    co = lm.cheb_coeffs_schrodinger(0.5, -3.0, 5.0, tol=1e-14)
    z = np.linspace(-1, 1, 41)
    lam = 1.0 - 4.0 * z  # B = (mu - H) / alpha  ->  H = mu - alpha z
    acc = co.c[0] * np.ones_like(z, dtype=complex)
    t_prev, t = np.ones_like(z), z.copy()
    acc = acc + co.c[1] * t
    for k in range(2, len(co.c)):
        t_prev, t = t, 2 * z * t - t_prev
        acc = acc + co.c[k] * t
    assert np.max(np.abs(acc - np.exp(-0.5j * lam))) < 1e-12


def test_gershgorin_and_scaling():
    a = lm.gen_stencil_3d(6, 2)
    lo, hi = lm.gershgorin_bounds(a)
    assert (lo, hi) == (0.0, 12.0)
    w = np.linalg.eigvalsh(lm.scale_for_heat(a, lo, hi).to_dense())
    assert w.min() >= -1 - 1e-12 and w.max() <= 1 + 1e-12
    with pytest.raises(ValueError, match="lam_max"):
        lm.scale_for_heat(a, 5.0, 5.0)


def test_backend_seam():
    assert lm.backend_name() == "cuda" and not lm.USING_NUMBA and lm.USING_CUDA


def test_adopt_reference_plan_fields():
    """executor.adopt_plan: the adapter behind a LEVELMPK_BACKEND=cuda seam in
    the reference copies a reference ExecPlan (plan.py:41-49)
    field by field, filling the reference's None kernel-slot defaults."""
    from types import SimpleNamespace

    from paper_2205_01598_b200.executor import _PLAN_FIELDS, adopt_plan, build_baseline_plan

    a = lm.gen_stencil_2d7pt(6, 5)
    ours = build_baseline_plan(a, 3, 2)
    ref_like = SimpleNamespace(**{f: getattr(ours, f) for f in _PLAN_FIELDS})
    ref_like.a = SimpleNamespace(n_rows=a.n_rows, row_ptr=a.row_ptr, col=a.col, val=a.val)
    for f in ("out_slot", "in_slot", "prev_slot", "kernel", "acc_coef"):
        setattr(ref_like, f, None)
    p = adopt_plan(ref_like)
    assert p.a == a and p.variant == ours.variant and p.n_items == ours.n_items
    assert np.array_equal(p.out_slot, ours.power) and np.array_equal(p.in_slot, ours.power - 1)
    assert np.array_equal(p.prev_slot, np.maximum(ours.power - 2, 0))
    assert not np.any(p.kernel) and not np.any(p.acc_coef)
    assert adopt_plan(p) is p
