"""ctypes front end of oracle/_build/liboracle.so (the C restatement).

TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's CPU legs).  Provides
the reference's CPU MPK pipeline restated in C: BFS levels, symmetric
permutation, k-sweep baseline and the point-to-point level-blocked walker
(executor.py:84-179), plus the host plan construction it needs (greedy level
groups groups.py:141-164, diagonal order schedule.py:91-99, nnz-balanced
chunks plan.py:221-233, checks plan.py:322-370 for whole groups).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

from . import levelmpk_oracle as O

_HERE = pathlib.Path(__file__).resolve().parent
_SO = _HERE / "_build" / "liboracle.so"
_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def lib():
    global _lib
    if _lib is None:
        if not _SO.exists():
            subprocess.run(["make", "-C", str(_HERE)], check=True, capture_output=True)
        L = ctypes.CDLL(str(_SO))
        L.oracle_spmv_rows.argtypes = [_p, _p, _p, _p, _p, _i64, _i64]
        L.oracle_mpk_baseline.argtypes = [_i64, _p, _p, _p, _p, _i64, _i32, _i32]
        L.oracle_mpk_walk.argtypes = [_p, _p, _p, _p, _i64, _p, _i32, _i64, _p, _p, _p, _p, _p,
                                      _p, _p, _i32, _p, _p, _p, _i32]
        L.oracle_bfs_levels.argtypes = [_i64, _p, _p, _i64, _p, _p]
        L.oracle_bfs_levels.restype = _i64
        L.oracle_permute_symmetric.argtypes = [_i64, _p, _p, _p, _p, _p, _p, _p, _p, _i32]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def threads():
    return int(os.environ.get("ORACLE_THREADS", lib().oracle_max_threads()))


def bfs_levels(row_ptr, col, root=0):
    """levels.py:106-114 on a pattern (symmetrized first if needed)."""
    n = row_ptr.shape[0] - 1
    sp, sc = O.symmetrized_pattern(row_ptr, col) if not _is_symmetric(row_ptr, col) else (
        np.asarray(row_ptr, dtype=np.int64), np.asarray(col, dtype=np.int32))
    sp = np.ascontiguousarray(sp, dtype=np.int64)
    sc = np.ascontiguousarray(sc, dtype=np.int32)
    perm = np.empty(n, dtype=np.int32)
    lp = np.empty(n + 1, dtype=np.int64)
    L = lib().oracle_bfs_levels(n, _ptr(sp), _ptr(sc), int(root), _ptr(perm), _ptr(lp))
    return perm, lp[: L + 1].copy()


def _is_symmetric(row_ptr, col):
    n = row_ptr.shape[0] - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(row_ptr.astype(np.int64)))
    k1 = rows * n + col
    k2 = col.astype(np.int64) * n + rows
    return np.array_equal(np.sort(k1), np.sort(k2))


def permute_symmetric(row_ptr, col, val, perm):
    n = row_ptr.shape[0] - 1
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    inv = np.empty(n, dtype=np.int32)
    inv[perm] = np.arange(n, dtype=np.int32)
    out_rp = np.empty(n + 1, dtype=np.int32)
    out_col = np.empty(col.shape[0], dtype=np.int32)
    out_val = np.empty(val.shape[0], dtype=np.float64)
    lib().oracle_permute_symmetric(n, _ptr(np.ascontiguousarray(row_ptr, dtype=np.int32)),
                                   _ptr(np.ascontiguousarray(col, dtype=np.int32)),
                                   _ptr(np.ascontiguousarray(val, dtype=np.float64)), _ptr(perm),
                                   _ptr(inv), _ptr(out_rp), _ptr(out_col), _ptr(out_val), threads())
    return out_rp, out_col, out_val


def mpk_baseline(row_ptr, col, val, y, p_m, nthreads=None):
    """y: float64 [p_m+1, n] with y[0] = x; filled in place."""
    n = row_ptr.shape[0] - 1
    lib().oracle_mpk_baseline(n, _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(y), y.shape[1], p_m,
                              nthreads or threads())
    return y


class CpuPlan:
    """Reference ExecPlan arrays for the level-blocked walker (s_m = 0)."""

    def __init__(self, row_ptr, col, level_ptr, p_m, cache_bytes, f=0.5, workers=1,
                 variant="lb_lg_p2p"):
        lnz = row_ptr[level_ptr[1:]].astype(np.int64) - row_ptr[level_ptr[:-1]]
        if variant == "lb":
            groups = [(int(level_ptr[i]), int(level_ptr[i + 1]), int(lnz[i]), int(level_ptr[i + 1]),
                       int(level_ptr[i]), 1, False) for i in range(len(lnz))]
        else:
            groups = O.level_groups(level_ptr, lnz, p_m, cache_bytes, f)
        self.groups = groups
        order = O.diagonal_order(len(groups), p_m) if variant != "baseline" else [(0, p) for p in range(1, p_m + 1)]
        if variant == "baseline":
            n = row_ptr.shape[0] - 1
            groups = [(0, n, 0, 0, 0, 1, False)]
        n_items = len(order)
        W = workers
        self.n_items = n_items
        self.workers = W
        self.barrier = 1 if variant in ("baseline", "lb", "lb_lg") else 0
        power = np.array([p for _, p in order], dtype=np.int64)
        self.out_slot = power.copy()
        self.in_slot = power - 1
        self.prev_slot = np.maximum(power - 2, 0)
        self.kernel = np.zeros(n_items, dtype=np.int64)
        self.acoef = np.zeros(n_items, dtype=np.float64)
        chunks = np.empty((n_items, W + 1), dtype=np.int64)
        bnd = np.empty((n_items, W), dtype=np.int64)
        for k, (i, p) in enumerate(order):
            rs, re = groups[i][0], groups[i][1]
            lo, hi = int(row_ptr[rs]), int(row_ptr[re])
            if re <= rs or hi == lo:
                b = np.full(W + 1, rs, dtype=np.int64)
            else:
                t = lo + (hi - lo) * np.arange(1, W, dtype=np.int64) // W
                cuts = np.searchsorted(row_ptr[rs:re + 1], t, side="left")
                b = np.empty(W + 1, dtype=np.int64)
                b[0], b[1:W], b[W] = rs, rs + cuts, re
                b = np.maximum.accumulate(b)
            chunks[k] = b
            bnd[k] = np.clip(groups[i][3] if variant != "baseline" else 0, b[:-1], b[1:])
        self.chunks = chunks
        self.bnd_point = bnd
        # checks (A) + (C) from the per-group column range, as plan.py:322-370
        ptr = np.zeros(n_items + 1, dtype=np.int64)
        items, kinds = [], []
        if not self.barrier:
            index = {ip: k for k, ip in enumerate(order)}
            mx = np.array([int(col[row_ptr[g[1]] - 1]) if g[1] > g[0] and row_ptr[g[1]] > row_ptr[g[0]] else -1
                           for g in groups])
            # exact per-group max column (rows sorted, so the last entry of each row)
            last = np.where(np.diff(row_ptr) > 0, col[np.maximum(row_ptr[1:] - 1, 0)], -1)
            mx = np.array([last[g[0]:g[1]].max() if g[1] > g[0] else -1 for g in groups])
            for k, (i, p) in enumerate(order):
                c = []
                if p > 1:
                    c.append((index[(i, p - 1)], 0))
                    if i + 1 < len(groups) and mx[i] >= groups[i + 1][0]:
                        c.append((index[(i + 1, p - 1)], 1 if mx[i] < groups[i + 1][3] else 0))
                ptr[k + 1] = ptr[k] + len(c)
                for m, kd in c:
                    items.append(m)
                    kinds.append(kd)
        self.check_ptr = ptr
        self.check_item = np.asarray(items, dtype=np.int64)
        self.check_kind = np.asarray(kinds, dtype=np.int64)


def mpk_walk(row_ptr, col, val, y, plan: CpuPlan, acc=None, use_acc=False):
    """Run the restated p2p walker with plan.workers threads (in place on y)."""
    accp = acc if acc is not None else np.zeros(1)
    lib().oracle_mpk_walk(
        _ptr(row_ptr), _ptr(col), _ptr(val), _ptr(y), y.shape[1], _ptr(accp), 1 if use_acc else 0,
        plan.n_items, _ptr(plan.out_slot), _ptr(plan.in_slot), _ptr(plan.prev_slot),
        _ptr(plan.kernel), _ptr(plan.acoef), _ptr(plan.chunks), _ptr(plan.bnd_point),
        plan.barrier, _ptr(plan.check_ptr), _ptr(plan.check_item), _ptr(plan.check_kind),
        plan.workers)
    return y
