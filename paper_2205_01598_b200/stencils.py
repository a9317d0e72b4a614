"""Synthetic matrices: the reference's stencils plus the BASELINE.json configs.

All generators are instances of one builder, ``grid_operator``: a list of
(offset, weight) couplings applied on a lexicographically numbered grid, with
Dirichlet truncation or periodic wrap-around, assembled by
CsrMatrix.from_triplets (duplicates summed, canonical column order).

* gen_stencil_2d7pt / gen_stencil_3d / stencil_3d_nnz reproduce
  pkg/src/levelmpk/stencils.py:20-91 exactly (same couplings, weights,
  numbering; verified against the reference's own tests and goldens);
* gen_laplace_2d5pt, gen_stencil_3d27pt, gen_rmat and gen_anderson_3d are the
  seeded stand-ins for BASELINE.json configs 1, 3, 4 and 5, which the
  reference does not ship.
These are the host-side CRS-build front end; the GPU hot path starts at the
CsrMatrix they return.
"""

import itertools

import numpy as np

from .csr import CsrMatrix

#: -d2/dx2 central-difference weights per spatial order (stencils.py:20-24)
FD_WEIGHTS = {
    2: (2.0, -1.0),
    4: (5.0 / 2.0, -4.0 / 3.0, 1.0 / 12.0),
    6: (49.0 / 18.0, -3.0 / 2.0, 3.0 / 20.0, -1.0 / 90.0),
}


def grid_operator(shape, couplings, periodic=False, diagonal=None, device=False) -> CsrMatrix:
    """Operator on a lexicographic grid.

    device=True builds the CRS from the triplets in HBM (lmpk_csr_from_triplets,
    bit-exact with the host build).

    ``couplings`` is a list of (offset tuple, weight); a zero offset adds to the
    diagonal.  Off-grid neighbours are dropped (Dirichlet) or wrapped
    (``periodic``).  ``diagonal`` (array) is added to the diagonal as well.
    """
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    coords = np.indices(shape).reshape(len(shape), -1)
    strides = np.array([int(np.prod(shape[d + 1:])) for d in range(len(shape))], dtype=np.int64)
    ids = (coords.T @ strides).astype(np.int64)
    rows, cols, vals = [], [], []
    for offset, weight in couplings:
        tgt = coords + np.asarray(offset, dtype=np.int64)[:, None]
        if periodic:
            tgt = tgt % np.asarray(shape)[:, None]
            keep = np.ones(n, dtype=bool)
        else:
            keep = np.all((tgt >= 0) & (tgt < np.asarray(shape)[:, None]), axis=0)
        rows.append(ids[keep])
        cols.append((tgt[:, keep].T @ strides).astype(np.int64))
        vals.append(np.full(int(keep.sum()), float(weight)))
    if diagonal is not None:
        rows.append(ids)
        cols.append(ids)
        vals.append(np.asarray(diagonal, dtype=np.float64))
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    if device:
        import torch

        r, c, v = (torch.from_numpy(t).cuda() for t in (r, c, v))
    return CsrMatrix.from_triplets(n, r, c, v)


def gen_stencil_2d7pt(nx: int, ny: int) -> CsrMatrix:
    """2d seven-point stencil on an nx-by-ny grid: 7 on the diagonal, -1 to the
    four axis neighbours and the two antidiagonal ones (stencils.py:31-50)."""
    if nx < 2 or ny < 2:
        raise ValueError(f"grid dimensions must be >= 2, got ({nx}, {ny})")
    offs = [(-1, 0), (1, 0), (0, -1), (0, 1), (1, -1), (-1, 1)]
    return grid_operator((nx, ny), [((0, 0), 7.0)] + [(o, -1.0) for o in offs])


def gen_stencil_3d(n: int, order: int = 2, device: bool = False) -> CsrMatrix:
    """Finite-difference -Laplacian of the given spatial order on an n^3 grid,
    Dirichlet truncation (stencils.py:53-80)."""
    if order not in FD_WEIGHTS:
        raise ValueError(f"unsupported spatial order {order} (choose 2, 4, or 6)")
    if n < order + 1:
        raise ValueError(f"grid size {n} too small for order {order} (need n >= {order + 1})")
    w = FD_WEIGHTS[order]
    couplings = [((0, 0, 0), 3.0 * w[0])]
    for axis in range(3):
        for dist in range(1, len(w)):
            for sign in (-1, 1):
                off = [0, 0, 0]
                off[axis] = sign * dist
                couplings.append((tuple(off), w[dist]))
    return grid_operator((n, n, n), couplings, device=device)


def stencil_3d_nnz(n: int, order: int = 2) -> int:
    """Closed-form nonzero count of gen_stencil_3d (stencils.py:83-91)."""
    if order not in FD_WEIGHTS:
        raise ValueError(f"unsupported spatial order {order}")
    reach = order // 2
    pairs_per_line = 2 * sum(n - k for k in range(1, reach + 1))
    return n**3 + 3 * n**2 * pairs_per_line


# ----------------------------------------------------------------- BASELINE configs
def gen_laplace_2d5pt(nx: int, ny: int, device: bool = False) -> CsrMatrix:
    """Config 1: 2D 5-point Laplacian, Dirichlet, diag 4.0 / off -1.0, ids ix*ny + iy."""
    offs = [(-1, 0), (1, 0), (0, -1), (0, 1)]
    return grid_operator((nx, ny), [((0, 0), 4.0)] + [(o, -1.0) for o in offs], device=device)


def gen_stencil_3d27pt(n: int, perturb: float = 0.01, seed: int = 0, device: bool = False) -> CsrMatrix:
    """Config 3: 27-point stencil on n^3 (Dirichlet), diag 26.0, off -1.0, plus a
    seeded uniform[-perturb, perturb] perturbation added to every stored entry
    in canonical CRS order (pattern symmetric, values not)."""
    couplings = [(o, 26.0 if o == (0, 0, 0) else -1.0)
                 for o in itertools.product((-1, 0, 1), repeat=3)]
    a = grid_operator((n, n, n), couplings, device=device)
    if perturb:
        rng = np.random.default_rng(seed)
        a = CsrMatrix(a.n_rows, a.row_ptr, a.col, a.val + rng.uniform(-perturb, perturb, a.n_nz))
    return a


def gen_rmat(scale: int, edge_factor: int = 8, a: float = 0.57, b: float = 0.19,
             c: float = 0.19, seed: int = 1, device: bool = False) -> CsrMatrix:
    """Config 4: R-MAT graph (2**scale vertices, edge_factor * 2**scale edges),
    symmetrised with duplicates merged, self-loops added, values uniform[0,1]
    (seeded, canonical CRS order) then each row normalised to sum 1."""
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(m)
        right = ((r >= a) & (r < a + b)) | (r >= a + b + c)  # quadrants b and d
        down = r >= a + b                                     # quadrants c and d
        src |= down.astype(np.int64) << bit
        dst |= right.astype(np.int64) << bit
    rows = np.concatenate([src, dst, np.arange(n)])
    cols = np.concatenate([dst, src, np.arange(n)])
    ones = np.ones(rows.size)
    if device:
        import torch

        rows, cols, ones = (torch.from_numpy(t).cuda() for t in (rows, cols, ones))
    pat = CsrMatrix.from_triplets(n, rows, cols, ones)
    v = rng.uniform(0.0, 1.0, pat.n_nz)
    rs = np.add.reduceat(v, pat.row_ptr[:-1]) if pat.n_nz else np.zeros(n)
    v = v / np.repeat(rs, np.diff(pat.row_ptr))
    return CsrMatrix(n, pat.row_ptr, pat.col, v)


def gen_anderson_3d(n: int, disorder: float = 16.5, seed: int = 0, hopping: float = -1.0,
                    device: bool = False) -> CsrMatrix:
    """Config 5: 3D Anderson Hamiltonian on an n^3 periodic grid: hopping to the
    six wrapped neighbours, on-site energies uniform[-W/2, W/2] (seeded)."""
    rng = np.random.default_rng(seed)
    eps = rng.uniform(-disorder / 2, disorder / 2, n**3)
    offs = [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    return grid_operator((n, n, n), [(o, hopping) for o in offs], periodic=True, diagonal=eps, device=device)
