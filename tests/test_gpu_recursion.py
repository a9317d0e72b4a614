"""Recursive level refinement (s_m >= 1) on the GPU against the reference
itself: tests/golden/golden_r2.* holds, for 83 (matrix, p_m, s_m, cache)
cases, what the reference's prepare / build_plan / run_plan produced
(tests/golden/make_golden_r2.py) -- the final permutation, the level-group
tree with refined spans and diamond halos (groups.py:192-366), the flattened
lb_lg_p2p_rec plan (plan.py:52-181, :322-370) and the power vectors.
Everything must be equal: bit-exact integers, bitwise fp64."""

import json
import pathlib

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from matrices import CORPUS, sha
from oracle import levelmpk_oracle as O

pytestmark = pytest.mark.gpu

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
FACTS = json.loads((GOLD / "golden_r2.json").read_text())["recursion"]
ARR = np.load(GOLD / "golden_r2.npz")

MATS = dict(CORPUS)
MATS["3d-12"] = lambda: lm.gen_stencil_3d(12, 2)
MATS["2d-40x33"] = lambda: lm.gen_stencil_2d7pt(40, 33)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


def tree_record(tree):
    def halo(split):
        if split is None:
            return None
        return {"side": split.side, "groups": [list(g) for g in split.groups],
                "levels": {str(gi): [{"row_start": lv.row_start, "row_end": lv.row_end,
                                      "portions": [list(p) for p in lv.portions], "keys": list(lv.keys)}
                                     for lv in lvs]
                           for gi, lvs in split.levels_by_group.items()}}
    return {
        "stage": tree.stage,
        "groups": [[g.row_start, g.row_end, g.nnz, g.boundary_left_end, g.boundary_right_start,
                    g.n_levels, bool(g.violates), g.children is not None] for g in tree.groups],
        "spans": [{"first_group": s.first_group, "last_group": s.last_group, "row_start": s.row_start,
                   "row_end": s.row_end, "level_ptr": [int(v) for v in s.levels.level_ptr],
                   "root": int(s.levels.root), "tree": tree_record(s.tree),
                   "left": halo(s.left_split), "right": halo(s.right_split)} for s in tree.spans],
    }


@pytest.mark.parametrize("key", sorted(FACTS))
def test_refinement_plan_and_powers_equal_reference(key):
    rec = FACTS[key]
    a = MATS[rec["matrix"]]()
    p_m = rec["p_m"]
    pre = lm.prepare(a, "lb_lg_p2p_rec", p_m, rec["cache"], s_m=rec["s_m"])
    assert np.array_equal(pre.perm.perm, ARR[f"{key}/perm"]), "final permutation"
    assert np.array_equal(pre.perm.perm[pre.perm.inv_perm], np.arange(a.n_rows))
    assert pre.tree.max_depth() == rec["depth"]
    assert tree_record(pre.tree) == rec["tree"], "level-group tree / halos"
    assert [sha(pre.a.row_ptr), sha(pre.a.col), sha(pre.a.val)] == rec["perm_csr"]
    assert len(pre.flagged_leaves()) == rec["flagged_leaves"]
    plan = lm.build_plan(pre, "lb_lg_p2p_rec", 2)
    items = np.array([[it.row_start, it.row_end, it.power, it.stage, 0 if it.kind == "group" else 1,
                       it.boundary_end] for it in plan.items], dtype=np.int64)
    assert np.array_equal(items, ARR[f"{key}/items"]), "flattened items (diamond merge order)"
    assert [list(it.label) for it in plan.items] == rec["labels"]
    for f in ("check_ptr", "check_item", "check_kind"):
        assert np.array_equal(getattr(plan, f), ARR[f"{key}/{f}"]), f
    assert np.array_equal(plan.chunks, ARR[f"{key}/chunks_w2"])
    x = np.random.default_rng(99).standard_normal(a.n_rows)
    res = lm.run_plan(plan, x=pre.perm.apply_to_vector(x))
    assert [sha(res.y.data[p]) for p in range(p_m + 1)] == rec["y"], "power vectors (bitwise)"


@pytest.mark.parametrize("n,k,s_m,cache", [(40, 4, 2, 2e6), (48, 8, 3, 4e6), (32, 3, 1, 6e5)])
def test_refined_27pt_walk_bitwise_vs_oracle(n, k, s_m, cache):
    """cfg3's shape (27-point, perturbed values) at desk size: the refined
    ordering through every schedule of the plan, bitwise against the oracle's
    baseline sweeps on the same permuted matrix."""
    import os

    a = lm.gen_stencil_3d27pt(n, seed=3)
    pre = lm.prepare(a, "lb_lg_p2p_rec", k, cache, s_m=s_m)
    assert pre.tree.max_depth() >= 1
    plan = lm.build_plan(pre, "lb_lg_p2p_rec", 1)
    x = np.random.default_rng(1).uniform(-1, 1, a.n_rows)
    xp = pre.perm.apply_to_vector(x)
    ref = O.mpk_powers(pre.a.row_ptr, pre.a.col, pre.a.val, xp, k)
    for sched in ("walk", "sweep", "crs"):
        os.environ["LMPK_SCHEDULE"] = sched
        try:
            res = lm.run_plan(plan, x=xp)
        finally:
            os.environ.pop("LMPK_SCHEDULE", None)
        assert np.array_equal(res.y.data, ref), sched


def test_item_deps_vs_oracle():
    """lmpk_item_deps against the definition (plan.py:103-129) on a random
    item list over a random matrix."""
    from paper_2205_01598_b200 import kernels as K

    rng = np.random.default_rng(5)
    n = 3000
    r, c = rng.integers(0, n, 20000), rng.integers(0, n, 20000)
    a = lm.CsrMatrix.from_triplets(n, np.concatenate([r, np.arange(n)]), np.concatenate([c, np.arange(n)]),
                                   np.ones(20000 + n))
    items = []
    for p in (1, 2, 3, 5):
        cuts = np.unique(np.concatenate(([0, n], rng.integers(0, n, 40))))
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            if rng.random() < 0.85:
                items.append((int(lo), int(hi), p))
    order = rng.permutation(len(items))
    items = [items[i] for i in order]
    rs, re, pw = (np.array(v, dtype=np.int64) for v in zip(*items))
    dep_ptr, dep = K.item_deps(a.device(), rs, re, pw)
    owner = {p: np.full(n, -1, dtype=np.int64) for p in set(pw.tolist())}
    for u, (lo, hi, p) in enumerate(items):
        owner[p][lo:hi] = u
    for u, (lo, hi, p) in enumerate(items):
        prev = owner.get(p - 1)
        want = np.empty(0, dtype=np.int64)
        if prev is not None:
            cols = a.col[a.row_ptr[lo]:a.row_ptr[hi]]
            d = np.unique(prev[np.unique(np.concatenate([cols.astype(np.int64), np.arange(lo, hi)]))])
            want = d[d >= 0]
        assert np.array_equal(dep[dep_ptr[u]:dep_ptr[u + 1]], want), u
