"""Pin the oracle (numpy restatement + C restatement) against fixtures that the
reference itself produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from matrices import CORPUS, sha
from oracle import cpu as C
from oracle import levelmpk_oracle as O

SMALL = [k for k in CORPUS if k != "cfg1"]


def _csr(name):
    a = CORPUS[name]()
    return a.row_ptr, a.col, a.val


@pytest.mark.parametrize("name", list(CORPUS))
def test_generators_match_reference_matrices(name, golden):
    facts, _ = golden
    rp, col, val = _csr(name)
    rec = facts["matrices"][name]
    assert (sha(rp), sha(col), sha(val)) == (rec["row_ptr"], rec["col"], rec["val"])


@pytest.mark.parametrize("name", list(CORPUS))
def test_oracle_bfs_matches_reference(name, golden):
    facts, arr = golden
    rp, col, _ = _csr(name)
    rec = facts["matrices"][name]
    roots = [int(k[3:-5]) for k in rec if k.startswith("bfs") and k.endswith("_perm")]
    for root in roots:
        lp_ref = arr[f"{name}/bfs{root}/level_ptr"]
        for perm, lp in (O.bfs_levels(rp, col, root, method="keysort"), C.bfs_levels(rp, col, root)):
            assert sha(perm) == rec[f"bfs{root}_perm"]
            assert np.array_equal(lp, lp_ref)
        if rp.shape[0] <= 200_001:
            perm, lp = O.bfs_levels(rp, col, root, method="frontier")
            assert sha(perm) == rec[f"bfs{root}_perm"] and np.array_equal(lp, lp_ref)


@pytest.mark.parametrize("name", SMALL + ["cfg1"])
def test_oracle_permute_and_powers_match_reference(name, golden):
    facts, arr = golden
    rp, col, val = _csr(name)
    rec = facts["matrices"][name]
    perm, _ = C.bfs_levels(rp, col, 0)
    for prp, pcol, pval in (O.permute_symmetric(rp, col, val, perm),
                            C.permute_symmetric(rp, col, val, perm)):
        assert [sha(prp), sha(pcol), sha(pval)] == rec["perm_csr"]
    prp, pcol, pval = C.permute_symmetric(rp, col, val, perm)
    p_m = rec["baseline_p_m"]
    x = np.random.default_rng(99).standard_normal(rp.shape[0] - 1)
    y = O.mpk_powers(prp, pcol, pval, x[perm], p_m)
    assert [sha(y[p]) for p in range(p_m + 1)] == rec["baseline_y"]
    yc = np.zeros_like(y)
    yc[0] = x[perm]
    C.mpk_baseline(prp, pcol, pval, yc, p_m, 4)
    assert np.array_equal(yc, y)


@pytest.mark.parametrize("name", [k for k in SMALL if not k.startswith("rmat")])
def test_oracle_walker_and_plan_match_reference(name, golden):
    """The C restatement of the p2p walker + the geometry-derived checks
    reproduce the reference's plan checks and bitwise power vectors."""
    facts, arr = golden
    rp, col, val = _csr(name)
    rec = facts["matrices"][name]
    perm, lp = C.bfs_levels(rp, col, 0)
    prp, pcol, pval = C.permute_symmetric(rp, col, val, perm)
    plan = C.CpuPlan(prp, pcol, lp, 4, rec["groups_cache"], workers=2, variant="lb_lg_p2p")
    assert [list(g[:6]) + [bool(g[6])] for g in plan.groups] == rec["groups_p4"]
    assert np.array_equal(plan.check_ptr, arr[f"{name}/check_ptr"])
    assert np.array_equal(plan.check_item, arr[f"{name}/check_item"])
    assert np.array_equal(plan.check_kind, arr[f"{name}/check_kind"])
    assert np.array_equal(plan.chunks, arr[f"{name}/chunks_w2"])
    x = np.random.default_rng(99).standard_normal(rp.shape[0] - 1)
    ref = O.mpk_powers(prp, pcol, pval, x[perm], 4)
    for W in (1, 3):
        p = C.CpuPlan(prp, pcol, lp, 4, rec["groups_cache"], workers=W, variant="lb_lg_p2p")
        y = np.zeros_like(ref)
        y[0] = x[perm]
        C.mpk_walk(prp, pcol, pval, y, p)
        assert np.array_equal(y, ref)


def test_oracle_cheb_matches_reference(golden):
    import paper_2205_01598_b200 as lm

    facts, arr = golden
    a = lm.gen_stencil_3d(8, 2)
    b = lm.scale_for_heat(a, *lm.gershgorin_bounds(a))
    assert [sha(b.row_ptr), sha(b.col), sha(b.val)] == facts["scale_for_heat_3d8"]
    co = lm.cheb_coeffs_heat(0.08, *lm.gershgorin_bounds(a), tol=1e-6)
    assert np.array_equal(co.c, arr["cheb/3d-8/coeffs"])
    perm, _ = C.bfs_levels(b.row_ptr, b.col, 0)
    prp, pcol, pval = C.permute_symmetric(b.row_ptr, b.col, b.val, perm)
    x = arr["cheb/3d-8/x"]
    accp = O.cheb_batches(prp, pcol, pval, x[perm], co.c)
    out = np.empty_like(accp)
    out[perm] = accp
    for pb in (1, 3, 4):  # batch size never changes a bit (test_cheb.py:210-218)
        assert np.array_equal(out, arr[f"cheb/3d-8/pb{pb}"])


def test_oracle_complex_cheb_by_linearity():
    """Complex state restated by linearity on the real oracle."""
    import paper_2205_01598_b200 as lm

    a = lm.gen_stencil_3d(5, 2)
    lo, hi = lm.gershgorin_bounds(a)
    b = lm.scale_for_heat(a, lo, hi)
    co = lm.cheb_coeffs_schrodinger(0.3, lo, hi, tol=1e-12)
    rng = np.random.default_rng(3)
    psi = np.exp(1j * rng.uniform(0, 2 * np.pi, a.n_rows))
    got = O.cheb_batches(b.row_ptr, b.col, b.val, psi, co.c.real, co.c.imag)

    def S(c, v):
        return O.cheb_batches(b.row_ptr, b.col, b.val, v, c)

    lin = (S(co.c.real, psi.real) - S(co.c.imag, psi.imag)) + 1j * (
        S(co.c.real, psi.imag) + S(co.c.imag, psi.real))
    assert np.linalg.norm(got - lin) / np.linalg.norm(lin) < 1e-13
    import scipy.linalg as sl

    ref = sl.expm(-1j * 0.3 * a.to_dense()) @ psi
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-10


def test_bessel_golden(golden):
    import paper_2205_01598_b200 as lm

    _, arr = golden
    assert np.array_equal(lm.bessel_i_seq(3.0, 10), arr["bessel/z3_k10"])
