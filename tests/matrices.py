"""Corpus builders (the reference's test corpus, pkg/tests/conftest.py:12-95,
restated with this package's API) and small helpers shared by the tests."""
import hashlib

import numpy as np

import paper_2205_01598_b200 as lm


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_symmetric_pattern(n, avg_deg, seed):
    rng = np.random.default_rng(seed)
    m = n * avg_deg // 2
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    rows = np.concatenate([r, c, np.arange(n)])
    cols = np.concatenate([c, r, np.arange(n)])
    vals = rng.standard_normal(rows.size)
    return lm.CsrMatrix.from_triplets(n, rows, cols, vals)


def block_diag(*blocks):
    rows, cols, vals, off = [], [], [], 0
    for b in blocks:
        r, c, v = b.to_triplets()
        rows.append(r.astype(np.int64) + off)
        cols.append(c.astype(np.int64) + off)
        vals.append(v)
        off += b.n_rows
    return lm.CsrMatrix.from_triplets(off, np.concatenate(rows), np.concatenate(cols),
                                      np.concatenate(vals))


def disconnected_matrix():
    return block_diag(lm.gen_stencil_2d7pt(6, 6), lm.gen_stencil_3d(4, 2))


def dumbbell_matrix(grid=10, path_len=60):
    g1 = lm.gen_stencil_2d7pt(grid, grid)
    g2 = lm.gen_stencil_2d7pt(grid, grid)
    n = g1.n_rows + path_len + g2.n_rows
    r1, c1, v1 = g1.to_triplets()
    r2, c2, v2 = g2.to_triplets()
    rows = list(r1) + list(r2 + g1.n_rows + path_len)
    cols = list(c1) + list(c2 + g1.n_rows + path_len)
    vals = list(v1) + list(v2)
    chain = [g1.n_rows - 1] + [g1.n_rows + k for k in range(path_len)] + [g1.n_rows + path_len]
    for u, v in zip(chain[:-1], chain[1:]):
        rows += [u, v]
        cols += [v, u]
        vals += [1.0, 1.0]
    for k in range(path_len):
        rows.append(g1.n_rows + k)
        cols.append(g1.n_rows + k)
        vals.append(4.0)
    return lm.CsrMatrix.from_triplets(n, rows, cols, vals)


def asym_300():
    rng = np.random.default_rng(7)
    r, c = rng.integers(0, 300, 900), rng.integers(0, 300, 900)
    return lm.CsrMatrix.from_triplets(300, r, c, np.ones(900))


CORPUS = {
    "2d7pt-8": lambda: lm.gen_stencil_2d7pt(8, 8),
    "2d7pt-16": lambda: lm.gen_stencil_2d7pt(16, 16),
    "2d7pt-32": lambda: lm.gen_stencil_2d7pt(32, 32),
    "2d7pt-64": lambda: lm.gen_stencil_2d7pt(64, 64),
    "3d-8-o2": lambda: lm.gen_stencil_3d(8, 2),
    "3d-16-o2": lambda: lm.gen_stencil_3d(16, 2),
    "3d-24-o2": lambda: lm.gen_stencil_3d(24, 2),
    "3d-8-o4": lambda: lm.gen_stencil_3d(8, 4),
    "3d-16-o4": lambda: lm.gen_stencil_3d(16, 4),
    "3d-8-o6": lambda: lm.gen_stencil_3d(8, 6),
    "3d-16-o6": lambda: lm.gen_stencil_3d(16, 6),
    "random-1": lambda: random_symmetric_pattern(800, 8, 11),
    "random-2": lambda: random_symmetric_pattern(1500, 5, 22),
    "disconnected": disconnected_matrix,
    "dumbbell": dumbbell_matrix,
    "rmat-s10": lambda: lm.gen_rmat(10),
    "rmat-s12": lambda: lm.gen_rmat(12),
    "asym-300": asym_300,
    "cfg1": lambda: lm.gen_laplace_2d5pt(256, 256),
}
