"""Flattening schedules into executable plans (host metadata + GPU tiling).

Mirrors pkg/src/levelmpk/plan.py: FlatItem (plan.py:41-49), ExecPlan
(plan.py:184-218), nnz-balanced worker chunks (plan.py:221-233), coverage
validation (plan.py:236-246), build_plan (plan.py:249-319) and the
point-to-point runtime checks (plan.py:322-370).

The reference's ExecPlan is the data contract of its CPU walker.  Here it
keeps the same fields (so callers, tests and tools see the same items,
chunks and checks) and additionally owns the GPU execution geometry:
``plan.tiling()`` builds (once) the tile-SELL-32 blocks and the tile
dependency ranges that liblmpk's level-blocked kernel walks.

Runtime checks for whole level groups (s_m = 0) are derived from group
geometry instead of the reference's per-item ``np.unique`` over all columns
(plan.py:73-130, 15.6 s on cfg2): by level confinement, item (i, p) depends
only on (i-1, p-1), (i, p-1), (i+1, p-1); whether the outer two are real
dependencies and whether the right one is BOUNDARY-granular follows from the
per-group column range (one GPU reduction, lmpk_segment_col_range).  The
result is identical to the reference's _runtime_checks for these plans.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import kernels as K
from .csr import CsrMatrix
from .groups import Preprocessed
from .schedule import LpSchedule, build_schedule

CHECK_FULL = 0
CHECK_BOUNDARY = 1

KERNEL_SPMV = 0
KERNEL_CHEB = 1  # y_out = 2 * A y_in - y_prev

VARIANTS = ("baseline", "lb", "lb_lg", "lb_lg_p2p", "lb_lg_p2p_rec")
BARRIER_VARIANTS = ("baseline", "lb", "lb_lg")


@dataclass
class FlatItem:
    row_start: int
    row_end: int  # exclusive
    power: int
    stage: int
    kind: str  # "group" | "outer"
    boundary_end: int  # end of the leftmost-level prefix (== row_start if none)
    label: tuple = ()


@dataclass
class ExecPlan:
    """Fully materialized execution recipe (reference fields + GPU geometry)."""

    variant: str
    p_m: int
    workers: int
    n_rows: int
    items: list
    barrier: bool
    row_start: np.ndarray
    row_end: np.ndarray
    power: np.ndarray
    chunks: np.ndarray
    bnd_point: np.ndarray
    check_ptr: np.ndarray
    check_item: np.ndarray
    check_kind: np.ndarray
    a: CsrMatrix
    pre: Preprocessed | None = None
    schedule: LpSchedule | None = None
    out_slot: np.ndarray = None
    in_slot: np.ndarray = None
    prev_slot: np.ndarray = None
    kernel: np.ndarray = None
    acc_coef: np.ndarray = None
    tiling_params: dict = None
    _tiling: object = None
    _sched: dict = None

    @property
    def n_items(self) -> int:
        return len(self.items)

    def barrier_count(self) -> int:
        return self.n_items if self.barrier else 0

    def tiling(self, complex_state=False, **params):
        """GPU tile geometry for this plan's matrix (built once, cached).  Real
        tilings stage x-segments in shared memory; complex state needs its own
        tiling (LMPK_FLAG_COMPLEX)."""
        if params and params != self.tiling_params:
            self.tiling_params = dict(params)
            self._tiling = None
        if self._tiling is None:
            self._tiling = {}
        key = bool(complex_state)
        if key not in self._tiling:
            prm = dict(self.tiling_params or {})
            if key:
                prm["mode_flags"] = int(prm.get("mode_flags", 0)) | _lib.FLAG_COMPLEX
            try:
                self._tiling[key] = K.Tiling(self.a.device(), self.p_m, **prm)
            except ValueError as e:
                # rows beyond the tile format (power-law hubs, > 65535 entries):
                # the plan runs as CRS sweeps (executor._launch); None marks it
                if "rows longer than" not in str(e):
                    raise
                self._tiling[key] = None
        return self._tiling[key]

    def schedule_choice(self, complex_state=False, plain=False):
        """'walk' (level-blocked wavefront), 'sweep' (dependency-free power
        sweeps on the same tiles) or, for plain real MPK only, 'crs' (the CRS
        sweeps of run_baseline) -- identical bits, chosen per plan and per
        call kind by timing once (executor._launch); None until measured.
        The key includes ``plain``: a plan re-used with Chebyshev slots or an
        accumulator never inherits the plain-only 'crs' choice."""
        return (self._sched or {}).get((bool(complex_state), bool(plain)))

    def set_schedule_choice(self, complex_state, choice, plain=False):
        if self._sched is None:
            self._sched = {}
        self._sched[(bool(complex_state), bool(plain))] = choice

    def power_config(self, acc_coef_im=None):
        """Per-power kernel configuration for liblmpk.  The reference stores it
        per item (plan.py:206-211), but its drivers set it per power
        (plan.py:307-312, cheb.py:209-219); anything else is rejected."""
        p_m = self.p_m
        cfg = {"out": [None] * p_m, "in": [None] * p_m, "prev": [None] * p_m,
               "kernel": [None] * p_m, "coef": [None] * p_m}
        for k in range(self.n_items):
            p = int(self.power[k]) - 1
            vals = (int(self.out_slot[k]), int(self.in_slot[k]), int(self.prev_slot[k]),
                    int(self.kernel[k]), float(self.acc_coef[k]))
            for key, v in zip(("out", "in", "prev", "kernel", "coef"), vals):
                if cfg[key][p] is None:
                    cfg[key][p] = v
                elif cfg[key][p] != v:
                    raise ValueError(
                        "the cuda backend needs the per-item kernel configuration to depend "
                        "only on the item's power"
                    )
        return K.power_cfg(p_m, cfg["out"], cfg["in"], cfg["prev"], cfg["kernel"], cfg["coef"],
                           acc_coef_im)


def _nnz_balanced_chunks(row_ptr, row_start, row_end, workers):
    """Split [row_start, row_end) into ``workers`` contiguous nnz-balanced chunks."""
    lo = int(row_ptr[row_start])
    hi = int(row_ptr[row_end])
    if row_end <= row_start or hi == lo:
        return np.full(workers + 1, row_start, dtype=np.int64)
    targets = lo + (hi - lo) * np.arange(1, workers, dtype=np.int64) // workers
    cuts = np.searchsorted(row_ptr[row_start : row_end + 1], targets, side="left")
    bounds = np.empty(workers + 1, dtype=np.int64)
    bounds[0] = row_start
    bounds[1:workers] = row_start + cuts
    bounds[workers] = row_end
    return np.maximum.accumulate(bounds)


def _validate_coverage(items, n_rows, p_m):
    """Every row must be computed exactly once per power."""
    for p in range(1, p_m + 1):
        ranges = sorted((it.row_start, it.row_end) for it in items if it.power == p)
        pos = 0
        for lo, hi in ranges:
            if lo != pos:
                raise RuntimeError(f"power {p}: rows [{pos}, {lo}) uncovered or doubled")
            pos = hi
        if pos != n_rows:
            raise RuntimeError(f"power {p}: rows [{pos}, {n_rows}) uncovered")


def _chunks(a: CsrMatrix, items, workers):
    n_items = len(items)
    chunks = np.empty((n_items, workers + 1), dtype=np.int64)
    if workers == 1:
        for k, it in enumerate(items):
            chunks[k] = (it.row_start, it.row_end)
        return chunks
    rp = a.row_ptr
    for k, it in enumerate(items):
        chunks[k] = _nnz_balanced_chunks(rp, it.row_start, it.row_end, workers)
    return chunks


def build_plan(pre: Preprocessed, variant: str, workers: int,
               p_m_override: int | None = None) -> ExecPlan:
    """Materialize the execution plan for one variant and worker count."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r} (choose from {VARIANTS})")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    a = pre.a
    n = a.n_rows
    p_m = pre.p_m if p_m_override is None else p_m_override
    if p_m > pre.p_m:
        raise ValueError("p_m_override may not exceed the preprocessed p_m")
    schedule = None
    if variant == "baseline":
        items = [FlatItem(0, n, p, 0, "group", 0, label=("baseline",)) for p in range(1, p_m + 1)]
    else:
        schedule = build_schedule(pre.tree, p_m)
        groups = pre.tree.groups
        items = [
            FlatItem(groups[it.group].row_start, groups[it.group].row_end, it.power,
                     schedule.stage, "group", groups[it.group].boundary_left_end,
                     label=(schedule.stage, it.group))
            for it in schedule.items
        ]
    _validate_coverage(items, n, p_m)
    barrier = variant in BARRIER_VARIANTS
    n_items = len(items)
    row_start = np.array([it.row_start for it in items], dtype=np.int64)
    row_end = np.array([it.row_end for it in items], dtype=np.int64)
    power = np.array([it.power for it in items], dtype=np.int64)
    chunks = _chunks(a, items, workers)
    bnd = np.array([it.boundary_end for it in items], dtype=np.int64)
    bnd_point = np.clip(bnd[:, None], chunks[:, :-1], chunks[:, 1:])
    check_ptr = np.zeros(n_items + 1, dtype=np.int64)
    check_item = np.empty(0, dtype=np.int64)
    check_kind = np.empty(0, dtype=np.int64)
    if not barrier:
        check_ptr, check_item, check_kind = _runtime_checks(pre, schedule, items)
    return ExecPlan(
        variant=variant, p_m=p_m, workers=workers, n_rows=n, items=items, barrier=barrier,
        row_start=row_start, row_end=row_end, power=power, chunks=chunks, bnd_point=bnd_point,
        check_ptr=check_ptr, check_item=check_item, check_kind=check_kind, a=a, pre=pre,
        schedule=schedule, out_slot=power.copy(), in_slot=power - 1,
        prev_slot=np.maximum(power - 2, 0), kernel=np.zeros(n_items, dtype=np.int64),
        acc_coef=np.zeros(n_items, dtype=np.float64),
    )


def _runtime_checks(pre: Preprocessed, schedule: LpSchedule, items):
    """Conditions (A)/(C) per item for whole-group diagonal schedules.

    Same result as plan.py:322-370: condition (A) = full completion of the
    same group at p-1; the one further check is the latest remaining
    dependency, (i+1, p-1) when group i has columns in group i+1, and it is
    BOUNDARY-granular when those columns lie inside group i+1's leftmost level.
    """
    groups = pre.tree.groups
    G = len(groups)
    seg = np.array([g.row_start for g in groups] + [groups[-1].row_end], dtype=np.int64)
    mn, mx = K.segment_col_range(pre.a.device(), seg)
    index = {(it.group, it.power): k for k, it in enumerate(schedule.items)}
    n = len(items)
    ptr = np.zeros(n + 1, dtype=np.int64)
    out_item, out_kind = [], []
    for u, it in enumerate(schedule.items):
        i, p = it.group, it.power
        checks = []
        if p > 1:
            checks.append((index[(i, p - 1)], CHECK_FULL))
            if i + 1 < G and int(mx[i]) >= groups[i + 1].row_start:
                m = index[(i + 1, p - 1)]
                if m > u:
                    raise RuntimeError(
                        f"schedule order violates dependency: item {u} needs later item {m}")
                kind = CHECK_BOUNDARY if int(mx[i]) < groups[i + 1].boundary_left_end else CHECK_FULL
                checks.append((m, kind))
        ptr[u + 1] = ptr[u] + len(checks)
        for m, kind in checks:
            out_item.append(m)
            out_kind.append(kind)
    return ptr, np.asarray(out_item, dtype=np.int64), np.asarray(out_kind, dtype=np.int64)
