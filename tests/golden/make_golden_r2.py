"""Round-2 golden fixtures, produced by running the REFERENCE package itself
(read-only at /root/reference; it does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_r2.py

Writes tests/golden/golden_r2.npz + golden_r2.json:

* traffic/...: simulate_traffic reports (traffic.py:192-226) for baseline,
  lb_lg_p2p and recursive plans at several capacities and line sizes, with the
  plan arrays the replay consumed (so the CPU tests need no GPU to rebuild
  the plans);
* rec/...: recursive refinement (groups.py:192-366) -- the final permutation,
  the level-group tree with its refined spans and diamond halos, the
  flattened plan items, checks and chunks of lb_lg_p2p_rec plans
  (plan.py:52-181, :322-370), and the power vectors of run_plan.
"""

import hashlib
import json
import os
import pathlib
import sys

import numpy as np

REF = os.environ.get("LEVELMPK_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, str(pathlib.Path(REF).parent / "tests"))
import levelmpk as L  # noqa: E402
from conftest import corpus, dumbbell_matrix  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tree_record(tree):
    """JSON form of a LevelGroupTree (groups.py:51-138)."""
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


def traffic_cases(arrays, facts):
    cases = []
    a8 = L.gen_stencil_3d(8, 2)
    a12 = L.gen_stencil_3d(12, 2)
    a2d = L.gen_stencil_2d7pt(20, 17)
    plans = {
        "base-3d8-p3": L.build_baseline_plan(a8, 3, 1),
        "base-3d12-p4": L.build_baseline_plan(a12, 4, 1),
        "p2p-3d8-p4": L.build_plan(L.prepare(a8, "lb_lg_p2p", 4, 6_000), "lb_lg_p2p", 1),
        "p2p-2d-p5": L.build_plan(L.prepare(a2d, "lb_lg_p2p", 5, 9_000), "lb_lg_p2p", 1),
        "rec-3d12-p4": L.build_plan(L.prepare(a12, "lb_lg_p2p_rec", 4, 100_000, s_m=4), "lb_lg_p2p_rec", 1),
    }
    for name, plan in plans.items():
        a = plan.a
        for k in ("row_start", "row_end", "power", "in_slot", "out_slot"):
            arrays[f"traffic/{name}/{k}"] = np.asarray(getattr(plan, k))
        arrays[f"traffic/{name}/row_ptr"] = a.row_ptr
        arrays[f"traffic/{name}/col"] = a.col
        for cap, line in ((0, 64), (1, 64), (2_048, 64), (10_000, 64), (50_000, 64), (1 << 20, 64),
                          (1 << 26, 64), (20_000, 128), (20_000, 32), (3_000, 8)):
            rep = L.simulate_traffic(plan, L.CacheModel(cap, line))
            key = f"traffic/{name}/cap{cap}_line{line}"
            arrays[key] = rep.by_power
            cases.append({"plan": name, "cap": cap, "line": line, "key": key, "p_m": int(plan.p_m),
                          "n_nz": int(a.n_nz), "n_rows": int(a.n_rows),
                          "matrix_bytes": int(rep.matrix_bytes), "row_ptr_bytes": int(rep.row_ptr_bytes),
                          "vector_bytes": int(rep.vector_bytes), "n_accesses": int(rep.n_accesses),
                          "n_misses": int(rep.n_misses), "code_balance": float(rep.code_balance)})
    facts["traffic"] = cases


def recursion_cases(arrays, facts):
    mats = {name: build() for name, build in corpus().items()}
    mats["dumbbell"] = dumbbell_matrix()
    mats["3d-12"] = L.gen_stencil_3d(12, 2)
    mats["3d-16-o2"] = L.gen_stencil_3d(16, 2)
    mats["2d-40x33"] = L.gen_stencil_2d7pt(40, 33)
    out = {}
    for name, a in mats.items():
        if a.n_rows < 60:
            continue
        for p_m, s_m, frac in ((4, 1, 8), (3, 2, 10), (5, 3, 12), (2, 2, 10), (1, 2, 10)):
            cache = max(12 * a.n_nz // frac, 2_000)
            pre = L.prepare(a, "lb_lg_p2p_rec", p_m, cache, s_m=s_m)
            if pre.tree.max_depth() == 0:
                continue
            key = f"rec/{name}/p{p_m}_s{s_m}"
            plan = L.build_plan(pre, "lb_lg_p2p_rec", 2)
            x = np.random.default_rng(99).standard_normal(a.n_rows)
            res = L.run_plan(plan, x=pre.perm.apply_to_vector(x))
            base = L.run_baseline(pre.a, pre.perm.apply_to_vector(x), p_m)
            assert all(np.array_equal(res.y.data[p], base.y.data[p]) for p in range(p_m + 1))
            arrays[f"{key}/perm"] = pre.perm.perm.astype(np.int32)
            arrays[f"{key}/items"] = np.array(
                [[it.row_start, it.row_end, it.power, it.stage, 0 if it.kind == "group" else 1,
                  it.boundary_end] for it in plan.items], dtype=np.int64)
            arrays[f"{key}/check_ptr"] = plan.check_ptr
            arrays[f"{key}/check_item"] = plan.check_item
            arrays[f"{key}/check_kind"] = plan.check_kind
            arrays[f"{key}/chunks_w2"] = plan.chunks
            out[key] = {"matrix": name, "p_m": p_m, "s_m": s_m, "cache": cache,
                        "depth": pre.tree.max_depth(), "tree": tree_record(pre.tree),
                        "perm_csr": [sha(pre.a.row_ptr), sha(pre.a.col), sha(pre.a.val)],
                        "y": [sha(res.y.data[p]) for p in range(p_m + 1)],
                        "flagged_leaves": len(pre.flagged_leaves()),
                        "labels": [list(it.label) for it in plan.items]}
    facts["recursion"] = out


def main():
    arrays, facts = {}, {"reference": REF, "numba": L.USING_NUMBA}
    traffic_cases(arrays, facts)
    recursion_cases(arrays, facts)
    np.savez_compressed(OUT / "golden_r2.npz", **arrays)
    (OUT / "golden_r2.json").write_text(json.dumps(facts, sort_keys=True, default=int))
    print("wrote", len(arrays), "arrays;", len(facts["traffic"]), "traffic cases;",
          len(facts["recursion"]), "recursion cases")


if __name__ == "__main__":
    main()
