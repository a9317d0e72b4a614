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

Refined spans (recursion): a SubgraphCall expands into the child schedule's
items merged with the diamond pieces of the neighbouring outer groups
(plan.py:73-181).  The merge is list scheduling against the true data
dependencies; those come from the GPU (lmpk_item_deps: one bitmap row per
item over the previous power's row intervals) instead of the reference's
per-item ``np.unique`` over every read column, and the runtime checks of such
plans (plan.py:322-370) use the same dependency lists plus one
lmpk_item_col_max_in_range reduction for the boundary-granular decision.

Runtime checks for whole level groups (s_m = 0) are derived from group
geometry instead of the reference's per-item ``np.unique`` over all columns
(plan.py:73-130, 15.6 s on cfg2): by level confinement, item (i, p) depends
only on (i-1, p-1), (i, p-1), (i+1, p-1); whether the outer two are real
dependencies and whether the right one is BOUNDARY-granular follows from the
per-group column range (one GPU reduction, lmpk_segment_col_range).  The
result is identical to the reference's _runtime_checks for these plans.
"""

import heapq
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import kernels as K
from .csr import CsrMatrix
from .groups import Preprocessed
from .schedule import LpNode, LpSchedule, SubgraphCall, build_schedule

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
        items = _flatten(schedule, pre.tree, a)
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
        if pre.tree.spans:
            check_ptr, check_item, check_kind = _runtime_checks_general(items, a)
        else:
            check_ptr, check_item, check_kind = _runtime_checks(pre, schedule, items)
    return ExecPlan(
        variant=variant, p_m=p_m, workers=workers, n_rows=n, items=items, barrier=barrier,
        row_start=row_start, row_end=row_end, power=power, chunks=chunks, bnd_point=bnd_point,
        check_ptr=check_ptr, check_item=check_item, check_kind=check_kind, a=a, pre=pre,
        schedule=schedule, out_slot=power.copy(), in_slot=power - 1,
        prev_slot=np.maximum(power - 2, 0), kernel=np.zeros(n_items, dtype=np.int64),
        acc_coef=np.zeros(n_items, dtype=np.float64),
    )


def _flatten(sched: LpSchedule, tree, a_perm):
    """Flat items of a schedule; SubgraphCalls expand recursively (plan.py:52-70)."""
    out = []
    for it in sched.items:
        if isinstance(it, LpNode):
            g = tree.groups[it.group]
            out.append(FlatItem(g.row_start, g.row_end, it.power, sched.stage, "group",
                                g.boundary_left_end, label=(sched.stage, it.group)))
        else:
            inner = _flatten(it.child, it.span.tree, a_perm)
            out.extend(_merge_diamond(inner, _diamond_pieces(it), a_perm))
    return out


def _diamond_pieces(call: SubgraphCall):
    """(item, priority) of every outer diamond piece of one subgraph step: halo
    group at distance delta runs its powers delta+1 .. p_m-delta in level /
    key-portion pieces (plan.py:73-100); priority = (power, side, delta, level,
    key, portion)."""
    p_m = call.child.p_m
    out = []
    for side, split in enumerate((call.span.left_split, call.span.right_split)):
        if split is None:
            continue
        for gi, delta in split.groups:
            for p in range(delta + 1, p_m - delta + 1):
                for li, lev in enumerate(split.levels_by_group[gi]):
                    for k, ((lo, hi), key) in enumerate(zip(lev.portions, lev.keys)):
                        if hi > lo:
                            out.append((FlatItem(lo, hi, p, call.stage, "outer", lo, label=(call.stage, gi, li, k)),
                                        (p, side, delta, li, key, k)))
    return out


def _item_dep_lists(items, a_perm):
    """dep_ptr, dep of a flat item list from the GPU (plan.py:103-129)."""
    return K.item_deps(a_perm.device(), [it.row_start for it in items], [it.row_end for it in items],
                       [it.power for it in items])


def _merge_diamond(inner, pieces, a_perm):
    """List-schedule child items and outer pieces against their true
    dependencies (plan.py:132-175): a ready outer piece always goes first
    (lowest priority tuple), otherwise the ready child item that comes first
    in the child walk."""
    if not pieces:
        return inner
    items = list(inner) + [it for it, _ in pieces]
    n_in, n = len(inner), len(items)
    dep_ptr, dep = _item_dep_lists(items, a_perm)
    unmet = np.diff(dep_ptr).astype(np.int64)
    users = [[] for _ in range(n)]
    for u in range(n):
        for d in dep[dep_ptr[u]:dep_ptr[u + 1]]:
            users[int(d)].append(u)
    ready_in, ready_out = [], []

    def release(u):
        if u < n_in:
            heapq.heappush(ready_in, u)
        else:
            heapq.heappush(ready_out, (pieces[u - n_in][1], u))

    for u in np.flatnonzero(unmet == 0):
        release(int(u))
    order = []
    while ready_in or ready_out:
        u = heapq.heappop(ready_out)[1] if ready_out else heapq.heappop(ready_in)
        order.append(u)
        for v in users[u]:
            unmet[v] -= 1
            if unmet[v] == 0:
                release(v)
    if len(order) != n:
        raise RuntimeError("cyclic dependencies in diamond merge (bug)")
    return [items[u] for u in order]


def _runtime_checks_general(items, a_perm):
    """Spin checks of an arbitrary flat plan (plan.py:322-370): condition (A) =
    the latest dependency overlapping the item's own rows (else the latest
    dependency), FULL; one more check on the latest dependency after it,
    BOUNDARY-granular when the item's columns inside that target stay left
    of its boundary_end.  Also validates the topological order."""
    n = len(items)
    dep_ptr, dep = _item_dep_lists(items, a_perm)
    rs = np.array([it.row_start for it in items], dtype=np.int64)
    re = np.array([it.row_end for it in items], dtype=np.int64)
    first = np.full(n, -1, dtype=np.int64)
    second = np.full(n, -1, dtype=np.int64)
    for u in range(n):
        d = dep[dep_ptr[u]:dep_ptr[u + 1]]
        if not d.size:
            continue
        if d[-1] >= u:
            bad = items[int(d[-1])]
            raise RuntimeError(
                f"schedule order violates dependency: item {u} {items[u].label} "
                f"p={items[u].power} needs later item {bad.label} p={bad.power}")
        own = d[(rs[d] < re[u]) & (re[d] > rs[u])]
        first[u] = own[-1] if own.size else d[-1]
        if d[-1] > first[u]:
            second[u] = d[-1]
    has2 = second >= 0
    tgt = np.where(has2, second, 0)
    col_lo = np.where(has2, rs[tgt], 0)
    col_hi = np.where(has2, re[tgt], 0)
    cmax = K.item_col_max_in_range(a_perm.device(), rs, re, col_lo, col_hi) if has2.any() else None
    bnd = np.array([it.boundary_end for it in items], dtype=np.int64)
    ptr = np.zeros(n + 1, dtype=np.int64)
    out_item, out_kind = [], []
    for u in range(n):
        if first[u] >= 0:
            out_item.append(int(first[u]))
            out_kind.append(CHECK_FULL)
            if has2[u]:
                m = int(second[u])
                out_item.append(m)
                out_kind.append(CHECK_BOUNDARY if 0 <= cmax[u] < bnd[m] else CHECK_FULL)
        ptr[u + 1] = len(out_item)
    return ptr, np.asarray(out_item, dtype=np.int64), np.asarray(out_kind, dtype=np.int64)


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
