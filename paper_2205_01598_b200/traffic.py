"""Software cache oracle: replay an execution plan through an LRU model.

Mirrors pkg/src/levelmpk/traffic.py: CacheModel (traffic.py:31-40),
TrafficReport (traffic.py:43-75), simulate_traffic (traffic.py:192-226) and
roofline_estimate (traffic.py:229-233).  The replay itself -- a single-level,
fully associative, line-granular LRU over the per-row accesses of the plan in
its sequential order (traffic.py:118-189) -- is liblmpk's host routine
lmpk_simulate_traffic (csrc/traffic.cu) instead of the reference's numba loop.

It is the desk-scale cross-check of the DRAM bytes ncu measures
(SURVEY.md section 8f-4): ``gpu_walk_plan`` turns the item order the GPU
actually walks (tiles x powers along the skewed wavefront) into the arrays the
replay takes, so the same model prices the kernel's own schedule.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .plan import ExecPlan

S_VAL, S_COL, S_ROWPTR, S_Y = 0, 1, 2, 3


@dataclass(frozen=True)
class CacheModel:
    capacity_bytes: int
    line_bytes: int = 64

    def __post_init__(self):
        if self.capacity_bytes < 0:
            raise ValueError("capacity must be >= 0")
        if self.line_bytes <= 0 or self.line_bytes % 4:
            raise ValueError("line size must be a positive multiple of 4")


@dataclass
class TrafficReport:
    matrix_bytes: int
    row_ptr_bytes: int
    vector_bytes: int
    n_nz: int
    p_m: int
    by_power: np.ndarray  # (p_m + 1, 3): matrix / row_ptr / vector bytes per power
    n_accesses: int = 0
    line_bytes: int = 64
    bypass: bool = False

    @property
    def total_bytes(self) -> int:
        return self.matrix_bytes + self.row_ptr_bytes + self.vector_bytes

    @property
    def n_misses(self) -> int:
        if self.bypass:  # no cache: every access misses
            return self.n_accesses
        return self.total_bytes // self.line_bytes

    @property
    def n_hits(self) -> int:
        return self.n_accesses - self.n_misses

    @property
    def code_balance(self) -> float:
        return self.total_bytes / (2.0 * self.n_nz * self.p_m)

    @property
    def matrix_code_balance(self) -> float:
        return self.matrix_bytes / (2.0 * self.n_nz * self.p_m)


def _replay(row_ptr, col, n_rows, row_start, row_end, power, in_slot, out_slot, n_powers,
            cap_lines, line_bytes, bypass):
    """by_power int64[n_powers, 4] (val / col / row_ptr / y bytes) from liblmpk."""
    lib = _lib.load_library()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    arrs = [np.ascontiguousarray(v, dtype=np.int64) for v in (row_start, row_end, power, in_slot, out_slot)]
    by_power = np.zeros((int(n_powers), 4), dtype=np.int64)
    vp = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _lib.check(lib.lmpk_simulate_traffic(
        int(n_rows), vp(rp), vp(cl), int(arrs[0].shape[0]), *[vp(a) for a in arrs], int(n_powers),
        int(cap_lines), int(line_bytes), 1 if bypass else 0, vp(by_power)), "simulate_traffic")
    return by_power


def simulate_traffic(plan: ExecPlan, cache: CacheModel) -> TrafficReport:
    """Replay a plan's sequential row order through the cache model."""
    a = plan.a
    n_powers = int(np.max(plan.out_slot)) + 1
    cap_lines = cache.capacity_bytes // cache.line_bytes
    bypass = cache.capacity_bytes == 0
    row_ptr = a.row_ptr
    by_power = _replay(row_ptr, a.col, a.n_rows, plan.row_start, plan.row_end, plan.power,
                       plan.in_slot, plan.out_slot, n_powers, cap_lines, cache.line_bytes, bypass)
    merged = np.stack(
        [by_power[:, S_VAL] + by_power[:, S_COL], by_power[:, S_ROWPTR], by_power[:, S_Y]], axis=1)
    rs = np.asarray(plan.row_start, dtype=np.int64)
    re = np.asarray(plan.row_end, dtype=np.int64)
    nnzs = row_ptr[re].astype(np.int64) - row_ptr[rs].astype(np.int64)
    return TrafficReport(
        matrix_bytes=int(merged[:, 0].sum()),
        row_ptr_bytes=int(merged[:, 1].sum()),
        vector_bytes=int(merged[:, 2].sum()),
        n_nz=a.n_nz,
        p_m=plan.p_m,
        by_power=merged,
        n_accesses=int((2 * (re - rs) + 3 * nnzs).sum()),
        line_bytes=cache.line_bytes,
        bypass=bypass,
    )


def roofline_estimate(code_balance: float, mem_bw: float) -> float:
    """Memory-bound performance ceiling: bandwidth / code balance [flop/s]."""
    if code_balance <= 0 or mem_bw <= 0:
        raise ValueError("code balance and bandwidth must be positive")
    return mem_bw / code_balance


def gpu_walk_plan(plan: ExecPlan, complex_state=False) -> ExecPlan:
    """The plan the GPU kernel really walks, as an ExecPlan for simulate_traffic:
    one item per (tile, power) in the order of the kernel's item queue (the
    skewed wavefront over the plan's tiling), with the plan's slots per power.
    Lets the LRU model price the device schedule next to ncu's dram__bytes."""
    from .plan import FlatItem

    til = plan.tiling(complex_state=complex_state)
    if til is None:
        raise ValueError("the plan has no tiling (rows beyond the tile format run as CRS sweeps)")
    tile_row, _, _ = til.geometry()
    order = til.item_order()  # (tile, power) pairs in queue order
    cfg = plan.power_config()
    rs = tile_row[order[:, 0]].astype(np.int64)
    re = tile_row[order[:, 0] + 1].astype(np.int64)
    pw = order[:, 1].astype(np.int64)
    items = [FlatItem(int(a_), int(b_), int(p_), 0, "group", int(a_)) for a_, b_, p_ in zip(rs, re, pw)]
    out_slot = np.array([cfg.out_slot[p - 1] for p in pw], dtype=np.int64)
    in_slot = np.array([cfg.in_slot[p - 1] for p in pw], dtype=np.int64)
    z = np.zeros(0, dtype=np.int64)
    return ExecPlan(
        variant=plan.variant, p_m=plan.p_m, workers=1, n_rows=plan.n_rows, items=items, barrier=False,
        row_start=rs, row_end=re, power=pw, chunks=np.stack([rs, re], axis=1), bnd_point=rs[:, None].copy(),
        check_ptr=np.zeros(len(items) + 1, dtype=np.int64), check_item=z, check_kind=z, a=plan.a,
        out_slot=out_slot, in_slot=in_slot, prev_slot=np.maximum(in_slot - 1, 0),
        kernel=np.zeros(len(items), dtype=np.int64), acc_coef=np.zeros(len(items)))
