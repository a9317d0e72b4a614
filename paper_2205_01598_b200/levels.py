"""Breadth-first level construction and level-ordered renumbering (GPU).

Mirrors pkg/src/levelmpk/levels.py: ``LevelSet`` (levels.py:24-45),
``symmetrized_pattern`` (levels.py:48-61) and ``bfs_levels``
(levels.py:106-114), computed by liblmpk's frontier kernels
(lmpk_bfs_levels / lmpk_symmetrized_pattern).  Levels and permutation are
bit-exact with the reference: BFS distance classes of A|A^T from the root,
each level sorted ascending, exhausted components restarted at the lowest
unvisited vertex.
"""

from dataclasses import dataclass

import numpy as np

from . import kernels as K
from .csr import CsrMatrix, Permutation


@dataclass(frozen=True)
class LevelSet:
    """level_ptr[i] is the first permuted row of level i; L_m levels total."""

    level_ptr: np.ndarray
    root: int

    def __post_init__(self):
        object.__setattr__(
            self, "level_ptr", np.ascontiguousarray(self.level_ptr, dtype=np.int64)
        )

    @property
    def n_levels(self) -> int:
        return self.level_ptr.shape[0] - 1

    @property
    def n_rows(self) -> int:
        return int(self.level_ptr[-1])

    def level_sizes(self) -> np.ndarray:
        return np.diff(self.level_ptr)


def symmetrized_pattern(a: CsrMatrix):
    """Pattern of A | A^T as host (row_ptr int64, col int32) in canonical order."""
    res = K.symmetrized_pattern(a.device())
    if res is None:  # already symmetric: the pattern of A itself
        return a.row_ptr.astype(np.int64), a.col.copy()
    rp, col = res
    return rp.cpu().numpy(), col.cpu().numpy()


def bfs_levels_device(a: CsrMatrix, root: int = 0):
    """(LevelSet, perm tensor, inv_perm tensor) with the permutation kept in HBM."""
    if not (0 <= root < a.n_rows):
        raise ValueError(f"root {root} out of range for n={a.n_rows}")
    perm, inv, level_ptr = K.bfs_levels(a.device(), int(root))
    return LevelSet(level_ptr, root), perm, inv


def bfs_levels(a: CsrMatrix, root: int = 0):
    """BFS levels of the (symmetrized) matrix graph plus the level ordering.

    The permutation numbers vertices consecutively within levels, level i-1
    before level i (levels.py:106-114).
    """
    levels, perm, inv = bfs_levels_device(a, root)
    return levels, Permutation._from_device(perm, inv)
