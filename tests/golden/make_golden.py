"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (the reference is read-only at /root/reference and
does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/golden.npz (arrays) and tests/golden/golden.json
(hashes and scalar facts).  Everything is produced through the reference's
public API (levelmpk.__init__): generators, bfs_levels, permute_symmetric,
run_baseline, prepare/build_plan, ChebPropagator.
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
from conftest import corpus, disconnected_matrix, dumbbell_matrix, random_symmetric_pattern  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rmat_ref(scale, edge_factor=8, a=0.57, b=0.19, c=0.19, seed=1):
    """Same construction as paper_2205_01598_b200.stencils.gen_rmat, built with
    the reference's from_triplets (pins the generator and the CRS build)."""
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(m)
        right = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        down = r >= a + b
        src |= down.astype(np.int64) << bit
        dst |= right.astype(np.int64) << bit
    rows = np.concatenate([src, dst, np.arange(n)])
    cols = np.concatenate([dst, src, np.arange(n)])
    pat = L.CsrMatrix.from_triplets(n, rows, cols, np.ones(rows.size))
    v = rng.uniform(0.0, 1.0, pat.n_nz)
    rs = np.add.reduceat(v, pat.row_ptr[:-1])
    v = v / np.repeat(rs, np.diff(pat.row_ptr))
    return L.CsrMatrix(n, pat.row_ptr, pat.col, v)


def laplace_2d5pt_ref(nx, ny):
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    ix, iy = ix.ravel(), iy.ravel()
    ids = ix * ny + iy
    rows, cols, vals = [ids], [ids], [np.full(ids.size, 4.0)]
    for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        jx, jy = ix + dx, iy + dy
        ok = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny)
        rows.append(ids[ok])
        cols.append(jx[ok] * ny + jy[ok])
        vals.append(np.full(int(ok.sum()), -1.0))
    return L.CsrMatrix.from_triplets(nx * ny, np.concatenate(rows), np.concatenate(cols),
                                     np.concatenate(vals))


def main():
    arrays = {}
    facts = {"reference": REF, "numba": L.USING_NUMBA, "matrices": {}}
    mats = {name: build() for name, build in corpus().items()}
    mats["dumbbell"] = dumbbell_matrix()
    mats["rmat-s10"] = rmat_ref(10)
    mats["rmat-s12"] = rmat_ref(12)
    g7 = np.random.default_rng(7)
    r7, c7 = g7.integers(0, 300, 900), g7.integers(0, 300, 900)
    mats["asym-300"] = L.CsrMatrix.from_triplets(300, r7, c7, np.ones(900))
    mats["cfg1"] = laplace_2d5pt_ref(256, 256)
    for name, a in mats.items():
        rec = {"n": a.n_rows, "nnz": a.n_nz, "row_ptr": sha(a.row_ptr), "col": sha(a.col),
               "val": sha(a.val)}
        for root in ((0, 17 % a.n_rows) if name in ("random-1", "asym-300", "rmat-s10") else (0,)):
            lv, pm = L.bfs_levels(a, root)
            key = f"{name}/bfs{root}"
            rec[f"bfs{root}_perm"] = sha(pm.perm)
            rec[f"bfs{root}_n_levels"] = int(lv.n_levels)
            arrays[f"{key}/level_ptr"] = lv.level_ptr
            if a.n_rows <= 70_000:
                arrays[f"{key}/perm"] = pm.perm
        lv, pm = L.bfs_levels(a, 0)
        ap = L.permute_symmetric(a, pm)
        rec["perm_csr"] = [sha(ap.row_ptr), sha(ap.col), sha(ap.val)]
        p_m = 4 if name == "cfg1" else 5
        x = np.random.default_rng(99).standard_normal(a.n_rows)
        base = L.run_baseline(ap, pm.apply_to_vector(x), p_m)
        rec["baseline_p_m"] = p_m
        rec["baseline_y"] = [sha(base.y.data[p]) for p in range(p_m + 1)]
        if a.n_rows <= 5000:
            arrays[f"{name}/baseline_y"] = base.y.data
        if name != "cfg1" and not name.startswith("rmat"):
            cache = max(12 * a.n_nz // 4, 3_000)
            pre = L.prepare(a, "lb_lg_p2p", 4, cache)
            rec["groups_p4"] = [[g.row_start, g.row_end, g.nnz, g.boundary_left_end,
                                 g.boundary_right_start, g.n_levels, bool(g.violates)]
                                for g in pre.tree.groups]
            rec["groups_cache"] = cache
            plan = L.build_plan(pre, "lb_lg_p2p", 2)
            arrays[f"{name}/check_ptr"] = plan.check_ptr
            arrays[f"{name}/check_item"] = plan.check_item
            arrays[f"{name}/check_kind"] = plan.check_kind
            arrays[f"{name}/chunks_w2"] = plan.chunks
            res = L.run_plan(plan, x=pre.perm.apply_to_vector(x))
            rec["p2p_equals_baseline"] = all(
                np.array_equal(res.y.data[p], L.run_baseline(pre.a, pre.perm.apply_to_vector(x), 4).y.data[p])
                for p in range(5))
        facts["matrices"][name] = rec
    # Chebyshev (heat) on the 3d-8 stencil: reference propagator output
    a = L.gen_stencil_3d(8, 2)
    x = np.random.default_rng(5).standard_normal(a.n_rows)
    for pb in (1, 3, 4):
        prop = L.ChebPropagator(a, 0.08, tol=1e-6, p_m_batch=pb, cache_bytes=40_000)
        arrays[f"cheb/3d-8/pb{pb}"] = prop.step(x)
        facts[f"cheb_3d8_pb{pb}_moments"] = int(prop.coeffs.n_moments)
    arrays["cheb/3d-8/x"] = x
    co = L.cheb_coeffs_heat(0.08, *L.gershgorin_bounds(a), tol=1e-6)
    arrays["cheb/3d-8/coeffs"] = co.c
    b = L.scale_for_heat(a, *L.gershgorin_bounds(a))
    facts["scale_for_heat_3d8"] = [sha(b.row_ptr), sha(b.col), sha(b.val)]
    # Bessel values
    arrays["bessel/z3_k10"] = L.bessel_i_seq(3.0, 10)
    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(facts, indent=1, sort_keys=True))
    print("wrote", len(arrays), "arrays;", len(facts["matrices"]), "matrices")


if __name__ == "__main__":
    main()
