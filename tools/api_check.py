"""GPU check of the reference-facing API against the oracle (quick)."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_01598_b200 as lm
from oracle import levelmpk_oracle as O
import __graft_entry__ as G
G.smoke()
a = lm.gen_stencil_3d(24, 2)
x = np.random.default_rng(1).standard_normal(a.n_rows)
for variant in ("lb", "lb_lg", "lb_lg_p2p", "lb_lg_p2p_rec"):
    res, pre = lm.run_mpk(a, x, variant, 5, 12 * a.n_nz // 4, workers=3)
    base = lm.run_baseline(pre.a, pre.perm.apply_to_vector(x), 5)
    rp, c, v = O.permute_symmetric(a.row_ptr, a.col, a.val, pre.perm.perm)
    ref = O.mpk_powers(rp, c, v, pre.perm.apply_to_vector(x), 5)
    print(variant, np.array_equal(res.y.data, ref), np.array_equal(base.y.data, ref), res.plan.n_items, res.barrier_count)
orig = lm.undo_permutation(res, pre.perm)
print("undo", np.array_equal(orig[0], x))
# Chebyshev: GPU vs oracle (same permuted B)
prop = lm.ChebPropagator(a, 0.05, tol=1e-6, p_m_batch=4, cache_bytes=50_000)
got = prop.step(x)
b = lm.scale_for_heat(a, *lm.gershgorin_bounds(a))
p = prop.pre.perm.perm
brp, bc, bv = O.permute_symmetric(b.row_ptr, b.col, b.val, p)
accp = O.cheb_batches(brp, bc, bv, x[p], prop.coeffs.c)
ref = np.empty_like(accp); ref[p] = accp
print("cheb bitwise", np.array_equal(got, ref), np.abs(got - ref).max())
# complex Schrodinger
co = lm.cheb_coeffs_schrodinger(0.2, *lm.gershgorin_bounds(a), tol=1e-12)
prop2 = lm.ChebPropagator(a, 0.2, coeffs=co, p_m_batch=8, cache_bytes=50_000)
psi = np.exp(1j * np.random.default_rng(2).uniform(0, 2 * np.pi, a.n_rows)) / np.sqrt(a.n_rows)
got2 = prop2.step(psi)
p2 = prop2.pre.perm.perm
accp2 = O.cheb_batches(brp, bc, bv, psi[p2], co.c.real, co.c.imag)
ref2 = np.empty_like(accp2); ref2[p2] = accp2
print("cheb complex bitwise", np.array_equal(got2, ref2), "norm", np.linalg.norm(got2))
