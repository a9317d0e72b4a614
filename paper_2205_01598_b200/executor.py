"""MPK execution on the B200 (run_plan / run_baseline / run_mpk).

Mirrors pkg/src/levelmpk/executor.py: PowerVectors (executor.py:33-53),
MpkResult (executor.py:56-66), undo_permutation (executor.py:69-76),
run_plan (executor.py:213-230), build_baseline_plan / run_baseline
(executor.py:233-266), prepare / run_mpk (executor.py:269-298), warmup
(executor.py:301-306).

Execution goes through liblmpk only:

* level-blocked variants (lb, lb_lg, lb_lg_p2p, lb_lg_p2p_rec) run the
  persistent level-blocked kernel (lmpk_mpk_run) over the plan's tiling;
* ``baseline`` plans run p_m back-to-back CRS SpMV launches
  (lmpk_mpk_baseline), the blocking-free comparator.

Every variant computes each row with the reference's per-row summation, so
power vectors are bitwise identical across variants AND bitwise identical
to the reference's numba backend.  ``PowerVectors`` may hold host (numpy)
or device (torch CUDA) storage; host storage is staged through HBM.
``MpkResult.seconds`` is the device time of the kernel launches (CUDA
events); ``e2e_seconds`` adds the host<->device copies of a host call.
"""

from __future__ import annotations

import time

import os

import numpy as np

from . import _lib
from . import kernels as K
from .csr import CsrMatrix, Permutation
from .groups import Preprocessed, preprocess
from .plan import VARIANTS, ExecPlan, FlatItem, _validate_coverage, build_plan


def _torch():
    import torch

    return torch


class PowerVectors:
    """The p_max + 1 dense vectors y_0..y_{p_max}, each contiguous.

    y_0 is the caller-supplied input and is never written by kernels.
    ``data`` is a numpy array (host) or, with ``device=True``, a CUDA tensor.
    """

    def __init__(self, n_rows, p_max, n_slots=None, data=None, device=False, dtype=np.float64):
        self.n_rows = n_rows
        self.p_max = p_max
        slots = n_slots if n_slots is not None else p_max + 1
        if data is not None:
            assert tuple(data.shape) == (slots, n_rows)
            self.data = data
        elif device:
            torch = _torch()
            tdt = torch.complex128 if np.dtype(dtype) == np.complex128 else torch.float64
            self.data = torch.zeros((slots, n_rows), dtype=tdt, device="cuda")
        else:
            self.data = np.zeros((slots, n_rows), dtype=dtype)

    @property
    def on_device(self) -> bool:
        return not isinstance(self.data, np.ndarray)

    def vec(self, p):
        return self.data[p]

    def __getitem__(self, p):
        return self.data[p]

    def to_host(self) -> "PowerVectors":
        if not self.on_device:
            return self
        return PowerVectors(self.n_rows, self.p_max, n_slots=self.data.shape[0],
                            data=self.data.cpu().numpy())


class MpkResult:
    def __init__(self, y, seconds, variant, workers, plan=None, e2e_seconds=None):
        self.y = y
        self.seconds = seconds
        self.e2e_seconds = seconds if e2e_seconds is None else e2e_seconds
        self.variant = variant
        self.workers = workers
        self.plan = plan
        self.barrier_count = plan.barrier_count() if plan is not None else 0

    def gflops(self, n_nz, p_m) -> float:
        return 2.0 * n_nz * p_m / self.seconds / 1e9


def undo_permutation(result, perm: Permutation) -> PowerVectors:
    """Bring power vectors computed in permuted order back to the original."""
    y = result.y if isinstance(result, MpkResult) else result
    if perm.n != y.n_rows:
        raise ValueError(f"permutation length {perm.n} != vector length {y.n_rows}")
    if y.on_device:
        out = PowerVectors(y.n_rows, y.p_max, n_slots=y.data.shape[0], device=True,
                           dtype=np.complex128 if y.data.is_complex() else np.float64)
        K.permute_vectors(perm.device()[0], y.data, out.data, scatter=True)
        return out
    out = PowerVectors(y.n_rows, y.p_max, n_slots=y.data.shape[0], dtype=y.data.dtype)
    out.data[:, perm.perm] = y.data
    return out


def _to_device_f64(arr):
    torch = _torch()
    if isinstance(arr, torch.Tensor):
        return arr
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


def _schedule(plan: ExecPlan, til, yv, cfg, av, use_acc, cplx, flags):
    """Wavefront walk, per-power sweeps on the tiles, or (plain real MPK) the
    CRS sweeps of run_baseline for this plan -- same bits.  The walk
    pays when the level window fits the L2 (cfg2, cfg5 shapes); for very wide
    levels (cfg3 27-point 160^3: 20 MB per level) the blocks are re-read from
    HBM at every power anyway and the dependency-free sweep is faster.  Chosen
    once per (plan, complex, plain) by timing each candidate on scratch copies
    (min of 3 calls); LMPK_SCHEDULE=walk|sweep|crs forces it."""
    forced = os.environ.get("LMPK_SCHEDULE", "auto")
    plain = not cplx and not use_acc and not np.any(plan.kernel != 0) and K.EXACT_DEFAULT
    if forced in ("walk", "sweep") or (forced == "crs" and plain):
        return forced
    got = plan.schedule_choice(cplx, plain)
    if got is not None:
        return got
    torch = _torch()
    ys = yv.clone()
    as_ = av.clone() if av is not None else None
    times = {}
    cands = [("walk", 0), ("sweep", _lib.FLAG_SWEEP)]
    if plain:  # plain real MPK: the CRS sweeps of run_baseline are a candidate too (same bits, EXACT)
        cands.append(("crs", None))
    for name, f in cands:
        def once():
            if f is None:
                K.mpk_baseline(plan.a.device(), ys, plan.p_m)
            else:
                K.mpk_run(til, ys, cfg, acc=as_, use_acc=use_acc, complex_state=cplx, flags=flags | f,
                          check_errors=False)
        once()
        best = None
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            once()
            e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        times[name] = best
    del ys, as_
    choice = min(times, key=times.get)
    plan.set_schedule_choice(cplx, choice, plain)
    return choice


def _launch(plan: ExecPlan, yd, accd, use_acc, flags=0, sync=True):
    """Run one plan on device buffers; returns device seconds (with
    ``sync=False``: a callable that waits for the launches and returns them,
    so the caller can queue copies behind the kernel first)."""
    torch = _torch()
    cplx = yd.is_complex()
    yv = torch.view_as_real(yd).reshape(yd.shape[0], -1) if cplx else yd
    av = None
    if use_acc:
        av = torch.view_as_real(accd).reshape(-1) if accd.is_complex() else accd
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if plan.variant == "baseline":
        if cplx or use_acc or np.any(plan.kernel != 0):
            # baseline plans with Chebyshev slots: tiled dependency-free sweeps
            cfg = plan.power_config()
            K.mpk_run(plan.tiling(complex_state=cplx), yv, cfg, acc=av, use_acc=use_acc, complex_state=cplx,
                      flags=flags | _lib.FLAG_SWEEP)
        else:
            K.mpk_baseline(plan.a.device(), yv, plan.p_m)
    else:
        cfg = plan.power_config()
        til = plan.tiling(complex_state=cplx)
        if til is None:
            # rows too long for the tile format (power-law hubs): sweeps over the
            # CRS arrays, the plan's Chebyshev steps / accumulation fused in
            if cplx or use_acc or np.any(plan.kernel != 0):
                K.mpk_crs_run(plan.a.device(), yv, cfg, acc=av, use_acc=use_acc, complex_state=cplx)
            else:
                K.mpk_baseline(plan.a.device(), yv, plan.p_m)
        else:
            sched = _schedule(plan, til, yv, cfg, av, use_acc, cplx, flags)
            if sched == "crs":
                K.mpk_baseline(plan.a.device(), yv, plan.p_m)
            else:
                f = flags | (_lib.FLAG_SWEEP if sched == "sweep" else 0)
                K.mpk_run(til, yv, cfg, acc=av, use_acc=use_acc, complex_state=cplx, flags=f)
    e1.record()

    def finish():
        e1.synchronize()
        ctx = _lib.context()
        _lib.check(ctx.lib.lmpk_ctx_check(ctx.handle, _lib.stream_handle()), "run_plan")
        return e0.elapsed_time(e1) * 1e-3

    return finish() if sync else finish


def plan_launcher(plan: ExecPlan, yd, accd=None, use_acc=False, flags=0):
    """(launch, schedule): a callable that queues exactly what run_plan
    launches for this plan on device buffers -- the chosen walk / sweep / CRS
    schedule -- without synchronizing or checking errors (timed loops; call
    lmpk_ctx_check afterwards), and the schedule's name."""
    torch = _torch()
    cplx = yd.is_complex()
    yv = torch.view_as_real(yd).reshape(yd.shape[0], -1) if cplx else yd
    av = None
    if use_acc:
        av = torch.view_as_real(accd).reshape(-1) if accd.is_complex() else accd
    cfg = plan.power_config()
    if plan.variant == "baseline":
        return (lambda: K.mpk_baseline(plan.a.device(), yv, plan.p_m)), "crs"
    til = plan.tiling(complex_state=cplx)
    if til is None:
        if cplx or use_acc or np.any(plan.kernel != 0):
            return (lambda: K.mpk_crs_run(plan.a.device(), yv, cfg, acc=av, use_acc=use_acc, complex_state=cplx)), "crs"
        return (lambda: K.mpk_baseline(plan.a.device(), yv, plan.p_m)), "crs"
    sched = _schedule(plan, til, yv, cfg, av, use_acc, cplx, flags)
    if sched == "crs":
        return (lambda: K.mpk_baseline(plan.a.device(), yv, plan.p_m)), sched
    f = flags | (_lib.FLAG_SWEEP if sched == "sweep" else 0)
    return (lambda: K.mpk_run(til, yv, cfg, acc=av, use_acc=use_acc, complex_state=cplx, flags=f,
                              check_errors=False)), sched


_PLAN_FIELDS = ("variant", "p_m", "workers", "n_rows", "items", "barrier", "row_start", "row_end",
                "power", "chunks", "bnd_point", "check_ptr", "check_item", "check_kind",
                "out_slot", "in_slot", "prev_slot", "kernel", "acc_coef")


def adopt_plan(ref_plan) -> ExecPlan:
    """An ExecPlan of this package from a reference ``levelmpk.plan.ExecPlan``
    (plan.py:41-49 fields) -- the adapter behind a ``LEVELMPK_BACKEND=cuda``
    seam in the reference.  The permuted matrix is re-wrapped
    (validated) and uploaded on first use; preprocessing objects are dropped."""
    if isinstance(ref_plan, ExecPlan):
        return ref_plan
    kw = {f: getattr(ref_plan, f) for f in _PLAN_FIELDS}
    a = ref_plan.a
    kw["a"] = CsrMatrix(a.n_rows, a.row_ptr, a.col, a.val)
    for f in ("out_slot", "in_slot", "prev_slot", "kernel", "acc_coef"):
        if kw[f] is not None:
            kw[f] = np.asarray(kw[f])
    n_items = len(kw["items"])
    defaults = {"out_slot": np.asarray(kw["power"]), "in_slot": np.asarray(kw["power"]) - 1,
                "prev_slot": np.maximum(np.asarray(kw["power"]) - 2, 0),
                "kernel": np.zeros(n_items, dtype=np.int64), "acc_coef": np.zeros(n_items)}
    for f, v in defaults.items():
        if kw[f] is None:
            kw[f] = v
    return ExecPlan(**kw)


def _slot_roles(plan: ExecPlan, n_slots):
    """(input slots, output slots) of a plan's per-power configuration: a
    slot is an input when some power reads it (in_slot / prev_slot) before
    any earlier power wrote it; outputs are the out_slots."""
    cfg = plan.power_config()
    written, inputs = set(), set()
    for i in range(cfg.n_powers):
        for sl in (cfg.in_slot[i], cfg.prev_slot[i] if cfg.kernel[i] == 1 else None):
            if sl is not None and sl not in written:
                inputs.add(int(sl))
        written.add(int(cfg.out_slot[i]))
    inputs.add(0)
    return sorted(s_ for s_ in inputs if s_ < n_slots), sorted(s_ for s_ in written if s_ < n_slots)


def _index_runs(idx):
    """Sorted indices as half-open runs of consecutive values: [1, 2, 3, 7] -> [(1, 4), (7, 8)]."""
    runs = []
    for i in idx:
        if runs and runs[-1][1] == i:
            runs[-1][1] = i + 1
        else:
            runs.append([i, i + 1])
    return [(a, b) for a, b in runs]


def _host_pinned(shape, dtype):
    """A numpy array in page-locked host memory (torch's caching host
    allocator), so device<->host copies of it run at full PCIe rate."""
    torch = _torch()
    tdt = torch.complex128 if np.dtype(dtype) == np.complex128 else torch.float64
    t = torch.empty(shape, dtype=tdt, pin_memory=True)
    return t, t.numpy()


def run_plan(plan: ExecPlan, x=None, y=None, acc=None, use_acc=False, timeout=None):
    """Execute a plan on the GPU; returns an MpkResult with the power vectors.

    Semantics of executor.py:213-230: with ``y=None`` a PowerVectors is
    allocated and y[0] = x; otherwise ``y`` (any object with a ``data``
    array of shape (slots, n): this package's PowerVectors, the reference's,
    a numpy array or a CUDA tensor) is updated in place.  ``acc`` (with
    use_acc) is accumulated in place.  The device watchdog (8 s without
    progress) replaces the reference's join timeout.

    Host data moves only where the plan needs it: the input slots go up
    (slot 0 = x, plus Chebyshev state slots), the output slots come down,
    asynchronously on the launch stream; a host PowerVectors that run_plan
    allocates lives in page-locked memory, and its copy of x is written on
    the CPU while the device works.
    """
    del timeout  # device-side watchdog
    torch = _torch()
    t_start = time.perf_counter()
    n = plan.n_rows
    if y is None:
        if x is None:
            raise ValueError("either x or y must be given")
        on_dev = isinstance(x, torch.Tensor) and x.is_cuda
        if on_dev:
            dt = np.complex128 if x.is_complex() else np.float64
            pv = PowerVectors(n, plan.p_m, device=True, dtype=dt)
            pv.data[0] = x
            host_x = None
        else:
            xa = x.numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
            dt = np.complex128 if np.iscomplexobj(xa) else np.float64
            xa = np.ascontiguousarray(xa, dtype=dt)
            if xa.shape != (n,):
                raise ValueError(f"x length {xa.shape} must equal n_rows {n}")
            pin_t, arr = _host_pinned((plan.p_m + 1, n), dt)
            pv = PowerVectors(n, plan.p_m, data=arr)
            pv._pinned = pin_t
            host_x = xa
    else:
        pv = y
        host_x = None
    data = pv if isinstance(pv, (np.ndarray, torch.Tensor)) else pv.data
    on_dev = isinstance(data, torch.Tensor) and data.is_cuda
    accd = None
    if use_acc:
        if acc is None:
            raise ValueError("use_acc requires acc")
        accd = acc if isinstance(acc, torch.Tensor) and acc.is_cuda else _to_device_f64(np.asarray(acc))
    if on_dev:
        seconds = _launch(plan, data, accd, use_acc)
    else:
        host = data if isinstance(data, np.ndarray) else np.asarray(data)
        slots = host.shape[0]
        ins, outs = _slot_roles(plan, slots)
        yd = torch.empty(host.shape, dtype=torch.complex128 if np.iscomplexobj(host) else torch.float64,
                         device="cuda")
        rest = [s_ for s_ in range(slots) if s_ not in ins and s_ not in outs]
        for s_ in ins:  # slot 0 straight from the caller's x when run_plan allocated y
            src = host_x if (s_ == 0 and host_x is not None) else host[s_]
            yd[s_].copy_(torch.from_numpy(np.ascontiguousarray(src)), non_blocking=True)
        if rest:
            yd[rest] = torch.from_numpy(host[rest]).cuda(non_blocking=True)
        seconds = _launch(plan, yd, accd, use_acc, sync=False)
        pinned = getattr(pv, "_pinned", None)
        if pinned is not None:
            for a_, b_ in _index_runs(outs):  # consecutive output slots: one copy per run
                pinned[a_:b_].copy_(yd[a_:b_], non_blocking=True)
            if host_x is not None:
                host[0] = host_x  # the reference's y[0] = x, on the CPU while the copies run
            seconds = seconds()
            torch.cuda.current_stream().synchronize()
        else:
            seconds = seconds()
            out_h = yd[outs].cpu().numpy()
            for i, s_ in enumerate(outs):
                host[s_] = out_h[i]
    if use_acc and not (isinstance(acc, torch.Tensor) and acc.is_cuda):
        acc[...] = accd.cpu().numpy()
    e2e = time.perf_counter() - t_start
    return MpkResult(pv, seconds, plan.variant, plan.workers, plan, e2e_seconds=e2e)


def build_baseline_plan(a: CsrMatrix, p_m: int, workers: int) -> ExecPlan:
    """p_m full-range SpMV sweeps with a barrier between sweeps (executor.py:233-258)."""
    from .plan import _nnz_balanced_chunks

    n = a.n_rows
    items = [FlatItem(0, n, p, 0, "group", 0, label=("baseline",)) for p in range(1, p_m + 1)]
    _validate_coverage(items, n, p_m)
    row_start = np.zeros(p_m, dtype=np.int64)
    row_end = np.full(p_m, n, dtype=np.int64)
    power = np.arange(1, p_m + 1, dtype=np.int64)
    chunks = np.empty((p_m, workers + 1), dtype=np.int64)
    if workers == 1:
        chunks[:] = (0, n)
    else:
        chunks[:] = _nnz_balanced_chunks(a.row_ptr, 0, n, workers)
    return ExecPlan(
        variant="baseline", p_m=p_m, workers=workers, n_rows=n, items=items,
        barrier=True, row_start=row_start, row_end=row_end, power=power,
        chunks=chunks, bnd_point=chunks[:, :-1].copy(),
        check_ptr=np.zeros(p_m + 1, dtype=np.int64),
        check_item=np.empty(0, dtype=np.int64),
        check_kind=np.empty(0, dtype=np.int64),
        a=a, pre=None, schedule=None,
        out_slot=power.copy(), in_slot=power - 1,
        prev_slot=np.maximum(power - 2, 0),
        kernel=np.zeros(p_m, dtype=np.int64),
        acc_coef=np.zeros(p_m, dtype=np.float64),
    )


def run_baseline(a: CsrMatrix, x, p_m: int, workers: int = 1, timeout=None) -> MpkResult:
    """Baseline MPK: y_p = A y_{p-1} as p_m full sweeps (k back-to-back SpMVs)."""
    if tuple(np.shape(x)) != (a.n_rows,):
        raise ValueError("x length must equal n_rows")
    plan = build_baseline_plan(a, p_m, workers)
    return run_plan(plan, x=x, timeout=timeout)


def prepare(a: CsrMatrix, variant: str, p_m: int, cache_bytes: float,
            f: float = 0.5, s_m: int = 0, root: int = 0) -> Preprocessed:
    """Preprocess with the grouping implied by the variant (executor.py:269-282)."""
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if variant == "lb":
        return preprocess(a, p_m, max(cache_bytes, 1.0), f, s_m=0, root=root, grouping="levels")
    eff_sm = s_m if variant == "lb_lg_p2p_rec" else 0
    return preprocess(a, p_m, cache_bytes, f, s_m=eff_sm, root=root)


def run_mpk(a: CsrMatrix, x, variant: str, p_m: int, cache_bytes: float,
            f: float = 0.5, s_m: int = 0, workers: int = 1, root: int = 0,
            timeout=None):
    """Preprocess, execute; returns (result in permuted order, pre) (executor.py:285-298)."""
    if variant == "baseline":
        return run_baseline(a, x, p_m, workers, timeout=timeout), None
    pre = prepare(a, variant, p_m, cache_bytes, f, s_m, root)
    plan = build_plan(pre, variant, workers)
    x_perm = pre.perm.apply_to_vector(np.asarray(x, dtype=np.float64))
    return run_plan(plan, x=x_perm, timeout=timeout), pre


def warmup():
    """Load the library, create the context and touch every kernel once."""
    from .stencils import gen_stencil_2d7pt

    a = gen_stencil_2d7pt(4, 4)
    run_baseline(a, np.ones(a.n_rows), p_m=1, workers=1)
    run_mpk(a, np.ones(a.n_rows), "lb_lg_p2p", 2, 10_000)
