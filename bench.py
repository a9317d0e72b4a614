"""Benchmark of the level-blocked MPK on the BASELINE.json configs.

    python bench.py [--config cfg2] [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workloads (BASELINE.json configs; cfg2 = configs[1], the default and the
shape the metric is quoted on):
  cfg1  2D 5-point Laplacian 256^2, MPK k = 4
  cfg2  3D 7-point Laplacian 200^3 (gen_stencil_3d(200, 2)), MPK k = 8
  cfg3  3D 27-point 160^3 perturbed, MPK k = 8 (cfg3-k2 / -k4 / -k8 / -k16)
  cfg4  R-MAT scale 22 (edge factor 8, symmetrised, row-normalised), MPK k = 6
  cfg5  Anderson 128^3 periodic, complex128 Chebyshev step of degree 64 as
        8 batches of k = 8 (fused recurrence + accumulation)
Matrices are the seeded synthetic stand-ins of SURVEY.md 8d, built in HBM;
x is uniform[-1, 1] (cfg4: [0, 1]; cfg5: random phases) from seed 0.

A step is one MPK call (y_1..y_k from y_0; cfg5: one propagation step) on
HBM-resident inputs, through the product path (executor.plan_launcher: the
walk / sweep / CRS schedule run_plan picks for the plan).  Metric: effective
GFLOP/s = 2 nnz k / t (cfg5: 4 nnz 64 / t, complex state).  Every working set
exceeds the 126 MB L2 except cfg1's (6.8 MB; `l2_resident` in config).

The line carries: the read-once roofline of the dominant kernel (algorithmic
bytes per launch / CUDA-event launch time, vs MEASURED_PEAKS), the ncu DRAM
bytes of that kernel for this build (profiles/traffic.json, written by
tools/profile_round.sh), the k x SpMV comparators and their roofline
fraction, e2e through the public API with host buffers (lm.run_plan /
ChebPropagator.step), preprocessing in SpMV equivalents (cli.py:157-159),
clocks sampled under load, and the CPU baseline: the reference's lb_lg_p2p
walker restated in C (oracle/) on the host cores, its power vectors compared
with the GPU's.

--impl reference times that C restatement of the reference on the host
cores for the same config and metric.  --gpus N > 1 without torchrun
re-launches itself under torch.distributed.run (one rank per GPU, NCCL).
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PEAK_FALLBACK_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    return PEAK_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# --------------------------------------------------------------------------- configs
def _gen(name):
    import paper_2205_01598_b200 as lm

    return {
        "cfg1": lambda: lm.gen_laplace_2d5pt(256, 256, device=True),
        "cfg2": lambda: lm.gen_stencil_3d(200, 2, device=True),
        "cfg2-small": lambda: lm.gen_stencil_3d(64, 2, device=True),
        "cfg3": lambda: lm.gen_stencil_3d27pt(160, seed=1, device=True),
        "cfg4": lambda: lm.gen_rmat(22, device=True),
        "cfg5": lambda: lm.gen_anderson_3d(128, seed=2, device=True),
    }[name]


def workload(cfg):
    base = cfg.split("-k")[0] if cfg.startswith("cfg3-k") else cfg
    table = {
        "cfg1": dict(name="cfg1: 2D 5-pt Laplacian 256^2, MPK k=4", k=4, kind="mpk", xlo=-1.0),
        "cfg2": dict(name="cfg2: 3D 7-pt Laplacian 200^3 (gen_stencil_3d(200,2)), MPK k=8", k=8, kind="mpk", xlo=-1.0),
        "cfg2-small": dict(name="cfg2-small: 3D 7-pt Laplacian 64^3, MPK k=8", k=8, kind="mpk", xlo=-1.0),
        "cfg3": dict(name="cfg3: 3D 27-pt 160^3 +-0.01 perturbed, MPK k={k}", k=8, kind="mpk", xlo=-1.0),
        "cfg4": dict(name="cfg4: R-MAT scale 22 (a=.57,b=c=.19, ef 8, seed 1) sym + self-loops, row-normalised, MPK k=6",
                     k=6, kind="mpk", xlo=0.0),
        "cfg5": dict(name="cfg5: Anderson 128^3 periodic W=16.5, complex128 Chebyshev step, degree 64 = 8 x k=8",
                     k=8, kind="cheb", xlo=None, degree=64),
    }
    if base not in table:
        raise SystemExit(f"unknown config {cfg} (cfg1, cfg2, cfg2-small, cfg3[-k2|-k4|-k8|-k16], cfg4, cfg5)")
    d = dict(table[base])
    if cfg.startswith("cfg3-k"):
        d["k"] = int(cfg.split("-k")[1])
    d["name"] = d["name"].format(k=d["k"])
    d["key"] = base
    return d


def q_ro(n, nnz, k):
    """Read-once bytes of one MPK call: matrix once, x in, k powers out."""
    return 12 * nnz + 4 * (n + 1) + 8 * n * (k + 1)


def q_spmv(n, nnz):
    return 12 * nnz + 4 * (n + 1) + 16 * n


def q_cheb_batch(n, nnz):
    """Fused complex Chebyshev batch, minimal I/O: matrix, 2 states in, 2 out, acc r/w."""
    return 12 * nnz + 4 * (n + 1) + 16 * n * 6


def traffic_for(key):
    """ncu DRAM bytes (read + write) per launch of the dominant kernel of this
    config, from the round's `ncu --set full` capture (profiles/traffic.json,
    written by tools/summarize_profiles.py from tools/profile_round.sh)."""
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            ent = json.loads(tf.read_text()).get(key)
            return int(ent["dram_bytes_per_launch"]) if ent else None
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed loop runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0, enabled=True):
        self.device = device
        self.enabled = enabled
        self.proc = None
        self.lines = []

    def __enter__(self):
        if not self.enabled:  # --no-clocks (profiling runs)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def under_load(self, step, min_samples=5, max_s=5.0, all_done=None):
        """Untimed steps until nvidia-smi reported `min_samples` samples with
        the GPU busy (the timed loop alone is shorter than nvidia-smi's
        start-up); the sampled window is this load phase plus the timed loop."""
        import torch

        if self.proc is None and all_done is None:
            return
        t0 = time.perf_counter()
        n0 = None
        while True:
            for _ in range(20):
                step()
            torch.cuda.synchronize()
            if n0 is None and self.lines:
                n0 = len(self.lines)
            done = (self.proc is None or time.perf_counter() - t0 > max_s
                    or (n0 is not None and len(self.lines) - n0 >= min_samples))
            if all_done is not None:
                done = all_done(done)
            if done:
                break

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cheb_coeffs_cfg5(a):
    """Degree-64 Schroedinger expansion for cfg5 (dt = 2, tol 1e-14, padded
    with zeros to 65 moments so the step is exactly 8 batches of k = 8)."""
    from paper_2205_01598_b200.cheb import ChebCoeffs, cheb_coeffs_schrodinger, gershgorin_bounds

    lo, hi = gershgorin_bounds(a)
    c = cheb_coeffs_schrodinger(2.0, lo, hi, tol=1e-14).c
    c = np.concatenate([c, np.zeros(max(0, 65 - c.size), dtype=c.dtype)])[:65]
    return ChebCoeffs(c=c, dt=2.0, lam_min=lo, lam_max=hi, tol=1e-14)


def make_x(cfgd, n):
    rng = np.random.default_rng(0)
    if cfgd["kind"] == "cheb":
        return np.exp(2j * np.pi * rng.random(n)) / np.sqrt(n)
    return rng.uniform(cfgd["xlo"], 1.0, n)


# --------------------------------------------------------------------------- CPU reference
def _cpu_walk_timed(rp, col, val, lp, x_perm, k, budget_s, min_reps, max_reps):
    """The reference's lb_lg_p2p walker restated in C (oracle/mpk_oracle.c),
    all host threads, C = 32 MiB (cli.py:380-384): one warm call, then timed
    calls until the budget or max_reps; returns (times, y)."""
    from oracle import cpu as C

    threads = C.threads()
    plan = C.CpuPlan(rp, col, lp, k, 32 * 2**20, workers=threads, variant="lb_lg_p2p")
    y = np.zeros((k + 1, rp.shape[0] - 1))
    y[0] = x_perm
    C.mpk_walk(rp, col, val, y, plan)  # warm: thread pool, pages
    ts = []
    t_begin = time.perf_counter()
    while len(ts) < max_reps and (len(ts) < min_reps or time.perf_counter() - t_begin < budget_s):
        t0 = time.perf_counter()
        C.mpk_walk(rp, col, val, y, plan)
        ts.append(time.perf_counter() - t0)
    return ts, y, threads


def _cpu_cheb_real_step(rp, col, val, lp, xr, coef, p_b, threads):
    """One real ChebPropagator.step restated on the C walker (cheb.py:209-246:
    slot ring of p_b + 2 states, CHEB kernel, fused accumulation)."""
    from oracle import cpu as C

    m = coef.size - 1
    plan = C.CpuPlan(rp, col, lp, p_b, 32 * 2**20, workers=threads, variant="lb_lg_p2p")
    S = p_b + 2
    y = np.zeros((S, xr.shape[0]))
    y[0] = xr
    acc = coef[0] * xr
    p = plan.out_slot.copy()  # item powers
    k_done, first = 0, True
    while k_done < m:
        plan.in_slot[:] = (k_done + p - 1) % S
        plan.out_slot[:] = (k_done + p) % S
        plan.prev_slot[:] = (k_done + p - 2) % S
        plan.kernel[:] = 1
        if first:
            plan.kernel[p == 1] = 0
        plan.acoef[:] = coef[k_done + p]
        C.mpk_walk(rp, col, val, y, plan, acc=acc, use_acc=True)
        k_done += p_b
        first = False
    return acc


def cpu_reference_run(cfgd, rp, col, val, lp, x_perm, coef=None, budget_s=20.0, min_reps=2, max_reps=50):
    """The CPU baseline / reference arm: seconds per step (mean of the timed
    calls), the statistic both report, and the result for the cross-check."""
    from oracle import cpu as C

    k = cfgd["k"]
    nnz = int(rp[-1])
    if cfgd["kind"] == "cheb":
        threads = C.threads()
        ts = []
        t_begin = time.perf_counter()
        out = None
        xr = np.ascontiguousarray(x_perm.real)
        xi = np.ascontiguousarray(x_perm.imag)
        while len(ts) < max_reps and (len(ts) < min_reps or time.perf_counter() - t_begin < budget_s):
            t0 = time.perf_counter()
            # linearity restatement: one complex step = 4 real propagations
            sr = _cpu_cheb_real_step(rp, col, val, lp, xr, coef.real.copy(), k, threads)
            si = _cpu_cheb_real_step(rp, col, val, lp, xi, coef.imag.copy(), k, threads)
            sri = _cpu_cheb_real_step(rp, col, val, lp, xi, coef.real.copy(), k, threads)
            sir = _cpu_cheb_real_step(rp, col, val, lp, xr, coef.imag.copy(), k, threads)
            out = (sr - si) + 1j * (sri + sir)
            ts.append(time.perf_counter() - t0)
        flops = 4.0 * nnz * (coef.size - 1)
        sample = (f"{len(ts)} complex steps, each 4 real Chebyshev propagations of degree {coef.size - 1} "
                  f"(8 batches of the lb_lg_p2p walker, k={k}, C=32 MiB; linearity restatement SURVEY 8c)")
        return ts, out, threads, flops, sample
    ts, y, threads = _cpu_walk_timed(rp, col, val, lp, x_perm, k, budget_s, min_reps, max_reps)
    sample = f"{len(ts)} timed lb_lg_p2p calls of the full workload (mean), C=32 MiB"
    return ts, y, threads, 2.0 * nnz * k, sample


def run_reference(args, cfgd):
    """--impl reference: the reference's CPU path on the host cores (rank 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import cpu as C

    import paper_2205_01598_b200 as lm  # generators only (host arrays); no kernels on this arm

    k = cfgd["k"]
    t0 = time.perf_counter()
    a = _host_matrix(cfgd)
    rp, col, val = a
    perm, lp = C.bfs_levels(rp, col, 0)
    coef = None
    if cfgd["kind"] == "cheb":
        mat = lm.CsrMatrix(rp.shape[0] - 1, rp, col, val)
        co = cheb_coeffs_cfg5(mat)
        coef = co.c
        b = lm.scale_for_heat(mat, co.lam_min, co.lam_max)
        rp, col, val = b.row_ptr, b.col, b.val
    arp, acol, aval = C.permute_symmetric(rp, col, val, perm)
    n = arp.shape[0] - 1
    x = make_x(cfgd, n)
    prep = time.perf_counter() - t0
    # K steps, each the full workload, bounded to ~a minute of host time
    ts, _, threads, flops, sample = cpu_reference_run(cfgd, arp, acol, aval, lp, x[perm], coef,
                                                      budget_s=60.0, min_reps=2, max_reps=max(args.steps, 2))
    t = sum(ts) / len(ts)
    value = flops / t / 1e9
    line = {
        "metric": metric_name(cfgd), "value": value, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": len(ts), "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if cfgd["kind"] == "cheb" else "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": cfgd["name"], "n_rows": n, "nnz": int(arp[-1]), "k": k,
                   "variant": "lb_lg_p2p", "cache_bytes": 32 * 2**20, "workers": threads},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "preprocess_seconds": prep,
    }
    print(json.dumps(line), flush=True)


def _host_matrix(cfgd):
    """Host CRS arrays of the config (the same generators as the GPU arm)."""
    import paper_2205_01598_b200 as lm

    key = cfgd["key"]
    a = {"cfg1": lambda: lm.gen_laplace_2d5pt(256, 256), "cfg2": lambda: lm.gen_stencil_3d(200, 2),
         "cfg2-small": lambda: lm.gen_stencil_3d(64, 2), "cfg3": lambda: lm.gen_stencil_3d27pt(160, seed=1),
         "cfg4": lambda: lm.gen_rmat(22), "cfg5": lambda: lm.gen_anderson_3d(128, seed=2)}[key]()
    return a.row_ptr, a.col, a.val


def metric_name(cfgd):
    if cfgd["kind"] == "cheb":
        return "Chebyshev propagation effective GFLOP/s (4*nnz*degree per step, complex128)"
    return "MPK effective GFLOP/s (2*nnz*k per call)"


# --------------------------------------------------------------------------- GPU arm
def _event_time(fn, reps=5):
    import torch

    fn()
    torch.cuda.synchronize()
    b0 = torch.cuda.Event(enable_timing=True)
    b1 = torch.cuda.Event(enable_timing=True)
    b0.record()
    for _ in range(reps):
        fn()
    b1.record()
    b1.synchronize()
    return b0.elapsed_time(b1) * 1e-3 / reps


def run_ours(args, cfgd):
    import torch

    import paper_2205_01598_b200 as lm
    from paper_2205_01598_b200 import _lib
    from paper_2205_01598_b200 import executor as E
    from paper_2205_01598_b200 import kernels as K

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    k = cfgd["k"]
    t0 = time.perf_counter()
    a = _gen(cfgd["key"])()  # CRS built in HBM (bitwise = host build)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    n, nnz = a.n_rows, a.n_nz
    x = make_x(cfgd, n)
    lm.warmup()
    torch.cuda.synchronize()
    if world > 1 and cfgd["key"] in ("cfg1", "cfg4"):
        # cfg4: the giant component spans fewer than 2k+1 levels, so
        # level-range shards degenerate; cfg1 fits one GPU's L2: N replicas
        return run_replicas(args, cfgd, a, x, rank, world, local, t_gen)
    if world > 1:
        return run_dist(args, cfgd, a, x, rank, world, local, t_gen)
    peak, peak_kind = measured_hbm_peak()
    ctx = _lib.context()
    t0 = time.perf_counter()
    if cfgd["kind"] == "cheb":
        coeffs = cheb_coeffs_cfg5(a)
        prop = lm.ChebPropagator(a, coeffs.dt, coeffs=coeffs, p_m_batch=k, cache_bytes=126e6)
        prop.check_errors = False  # one error check after the timed loop
        xd = torch.from_numpy(x).cuda()
        prop.step(xd)  # builds the tilings and picks the schedules
        torch.cuda.synchronize()
        t_pre = time.perf_counter() - t0
        step = lambda: prop.step(xd)  # noqa: E731
        sched = prop._plan_for[k].schedule_choice(True, False)
        n_batches = (coeffs.n_moments + k - 1) // k
        flops = 4.0 * nnz * coeffs.n_moments
        pre = prop.pre
        plan = prop._plan_for[k]
    else:
        # preprocessing (cli.py:157-159 counts it in SpMV equivalents): levels +
        # groups + permutation, plan, tiling.  The first pass also pays CUDA
        # module loads and allocator growth; the second, timed pass is the one
        # the bench runs on
        pre = lm.prepare(a, "lb_lg_p2p", k, 126e6)
        plan = lm.build_plan(pre, "lb_lg_p2p", 1)
        til_ = plan.tiling()
        torch.cuda.synchronize()
        t_first = time.perf_counter() - t0
        del pre, plan, til_
        t0 = time.perf_counter()
        pre = lm.prepare(a, "lb_lg_p2p", k, 126e6)
        torch.cuda.synchronize()
        t_prep = time.perf_counter() - t0
        plan = lm.build_plan(pre, "lb_lg_p2p", 1)
        t_plan = time.perf_counter() - t0 - t_prep
        plan.tiling()
        torch.cuda.synchronize()
        t_pre = time.perf_counter() - t0
        perm_d = pre.perm.device()[0]
        y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
        K.permute_vectors(perm_d, torch.from_numpy(x).cuda().unsqueeze(0), y[0:1])
        t0 = time.perf_counter()
        launch, sched = E.plan_launcher(plan, y)  # times walk / sweep / CRS once per plan
        launch()
        torch.cuda.synchronize()
        pre_parts = {"prepare_seconds": t_prep, "build_plan_seconds": t_plan,
                     "tiling_seconds": t_pre - t_prep - t_plan, "first_pass_seconds": t_first,
                     "schedule_timing_seconds": time.perf_counter() - t0}
        step = launch
        flops = 2.0 * nnz * k
        n_batches = 1
    # ---------------- device-resident timed loop
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _lib.check(ctx.lib.lmpk_ctx_check(ctx.handle, _lib.stream_handle()), "bench warm-up")
    if args.profile_step:  # one steady-state step between cudaProfilerStart/Stop (ncu --profile-from-start off)
        torch.cuda.cudart().cudaProfilerStart()
        step()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    with ClockSampler(local, enabled=not args.no_clocks) as clocks:
        clocks.under_load(step)
        torch.cuda.synchronize()
        launches0 = ctx.launches()
        e0.record()
        for s in range(args.steps):
            step_ev[s][0].record()
            step()
            step_ev[s][1].record()
        e1.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    _lib.check(ctx.lib.lmpk_ctx_check(ctx.handle, _lib.stream_handle()), "bench")
    t_step = e0.elapsed_time(e1) * 1e-3 / args.steps
    per_step = [a_.elapsed_time(b_) * 1e-3 for a_, b_ in step_ev]
    t_kernel = sum(per_step) / len(per_step)
    value = flops / t_step / 1e9
    # ---------------- roofline of the dominant kernel
    if cfgd["kind"] == "cheb":
        Q = q_cheb_batch(n, nnz)
        t_launch = t_kernel / n_batches  # the step is n_batches walk launches (+ two permutations)
        roof_note = "fused complex Chebyshev batch (k=8 powers): 12 nnz + 4(N+1) + 16N*6 bytes per launch"
    elif sched == "crs":
        Q = q_spmv(n, nnz)
        t_launch = t_kernel / k
        roof_note = "CRS SpMV sweep (the plan's fastest schedule): 12 nnz + 4(N+1) + 16N bytes per launch"
    else:
        Q = q_ro(n, nnz, k)
        t_launch = t_kernel
        roof_note = "level-blocked walk, one launch per call: read-once bytes 12 nnz + 4(N+1) + 8N(k+1)"
    achieved = Q / t_launch / 1e9
    traffic = traffic_for(args.config)
    line = {
        "metric": metric_name(cfgd), "value": value, "unit": "GFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128" if cfgd["kind"] == "cheb" else "f64", "data": "synthetic",
        "config": {"workload": cfgd["name"], "n_rows": n, "nnz": nnz, "k": k, "schedule": sched,
                   "l2_resident": bool(q_ro(n, nnz, k) < 100e6), "inputs_exceed_l2": bool(q_ro(n, nnz, k) > 126e6),
                   "l2_flush": "none: working set > L2" if q_ro(n, nnz, k) > 126e6 else
                   "none: the config fits L2 by definition (its shape)",
                   "parallelism": "single"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_kind": peak_kind, "algorithmic_bytes_per_launch": Q,
                     "launch_seconds": t_launch, "note": roof_note},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if traffic:
        line["dram_gbs"] = traffic / t_launch / 1e9
    til = plan.tiling(complex_state=cfgd["kind"] == "cheb")
    if til is not None:
        line["config"].update({"tiles": til.info["n_tiles"], "lean_bytes": til.info["lean_bytes"],
                               "block_bytes": til.info["block_bytes"], "super_tiles": til.info["super_tiles"]})
    # ---------------- k x SpMV comparators and parity of the timed result
    if cfgd["kind"] == "cheb":
        # the same step as degree x SpMV: (a) sweeps over the CRS arrays of the
        # natural-order operator with the recurrence fused into the row store
        # (lmpk_mpk_crs_run: the "k back-to-back SpMVs" of the paper), (b)
        # per-power sweeps over the tiles of the natural-order operator
        y_walk = prop.step(xd)
        base = lm.ChebPropagator(a, coeffs.dt, coeffs=coeffs, p_m_batch=k, variant="baseline")
        base.check_errors = False
        t_tiled = _event_time(lambda: base.step(xd))
        base.force_crs = True
        y_crs = base.step(xd)
        t_crs = _event_time(lambda: base.step(xd))
        rel = float((y_crs - y_walk).abs().max() / y_walk.abs().max())
        line["kspmv_baseline"] = {
            "crs_ms": t_crs * 1e3, "tiled_sweep_ms": t_tiled * 1e3,
            "crs_roofline_frac": coeffs.n_moments * (12 * nnz + 4 * (n + 1) + 16 * n * 5) / t_crs / 1e9 / peak,
            "speedup_vs_crs": t_crs / t_kernel, "speedup_vs_best": min(t_crs, t_tiled) / t_kernel,
            "rel_diff_vs_walk": rel,
            "note": "natural order; per power 12 nnz + 4(N+1) + 16N*5 bytes (in, prev, out, acc read+write)"}
        del base
    if cfgd["kind"] == "mpk":
        yb = torch.zeros_like(y)
        yb[0] = y[0]
        K.mpk_baseline(pre.a.device(), yb, k)
        line["bitwise_vs_baseline"] = bool(torch.equal(yb, y))
        t_crs = _event_time(lambda: K.mpk_baseline(pre.a.device(), yb, k))
        cfg = plan.power_config()
        t_sweep = _event_time(lambda: K.mpk_run(til, yb, cfg, flags=_lib.FLAG_SWEEP, check_errors=False)) \
            if til is not None else None
        kq = k * q_spmv(n, nnz)
        line["kspmv_baseline"] = {
            "crs_ms": t_crs * 1e3, "crs_roofline_frac": kq / t_crs / 1e9 / peak,
            "tiled_sweep_ms": t_sweep * 1e3 if t_sweep else None,
            "speedup_vs_crs": t_crs / t_kernel,
            "speedup_vs_best": min(t_crs, t_sweep or t_crs) / t_kernel}
        line["preprocess"] = {"seconds": t_pre, "spmv_equivalents": t_pre / (t_crs / k), "generate_seconds": t_gen,
                              "note": "second pass of prepare + build_plan + tiling; the first pass also pays CUDA "
                                      "module loads and allocator growth; the walk/sweep/CRS choice is timed once "
                                      "per plan (schedule_timing_seconds)"}
        line["preprocess"].update(pre_parts)
    else:
        line["preprocess"] = {"seconds": t_pre, "generate_seconds": t_gen}
    # ---------------- end to end through the public API with host buffers
    if cfgd["kind"] == "mpk":
        # run_plan(plan, x=host): x (permuted order) from pinned host memory;
        # run_plan uploads y_0, runs the plan, and returns y_0..y_k in pinned
        # host memory (y_1..y_k copied back, y_0 = x written on the CPU meanwhile)
        hx_t = torch.from_numpy(np.ascontiguousarray(x[pre.perm.perm])).pin_memory()
        hx = hx_t.numpy()
        res = lm.run_plan(plan, x=hx)
        e2e_ok = bool(np.array_equal(res.y.data[1:], y[1:].cpu().numpy()))
        del res
        ts = []
        for _ in range(max(3, min(args.steps, 20))):
            t0 = time.perf_counter()
            res = lm.run_plan(plan, x=hx)
            ts.append(time.perf_counter() - t0)
            del res
        t_e2e = statistics.median(ts)
        line["e2e"] = {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 8 * n,
                       "d2h_bytes_per_step": 8 * n * k, "api": "paper_2205_01598_b200.run_plan(plan, x=<pinned host>)",
                       "seconds_median": t_e2e, "result_matches": e2e_ok}
    else:
        prop.check_errors = True
        hx_t = torch.from_numpy(x).pin_memory()
        hx = hx_t.numpy()
        got = prop.step(hx)
        e2e_ok = bool(np.array_equal(got, step().cpu().numpy()))
        ts = []
        for _ in range(max(3, min(args.steps, 10))):
            t0 = time.perf_counter()
            got = prop.step(hx)
            ts.append(time.perf_counter() - t0)
        t_e2e = statistics.median(ts)
        line["e2e"] = {"value": flops / t_e2e / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": 16 * n,
                       "d2h_bytes_per_step": 16 * n, "api": "ChebPropagator.step(<pinned host psi>)",
                       "seconds_median": t_e2e, "result_matches": e2e_ok}
    # ---------------- CPU baseline: the reference's walker restated in C, same run
    if not args.no_cpu_baseline:
        try:
            coef = prop.coeffs.c if cfgd["kind"] == "cheb" else None
            ts, ycpu, threads, cflops, sample = cpu_reference_run(
                cfgd, pre.a.row_ptr, pre.a.col, pre.a.val, pre.levels.level_ptr, x[pre.perm.perm], coef,
                budget_s=args.cpu_budget, min_reps=2, max_reps=20)
            tc = sum(ts) / len(ts)
            if cfgd["kind"] == "cheb":
                gpu_acc = prop.step(torch.from_numpy(x).cuda()).cpu().numpy()[pre.perm.perm]
                rel = float(np.linalg.norm(gpu_acc - ycpu) / np.linalg.norm(ycpu))
                match = {"gpu_vs_cpu_rel_l2": rel, "within_1e-12": rel <= 1e-12}
            else:
                match = {"bitwise_gpu_vs_cpu": bool(np.array_equal(ycpu, y.cpu().numpy()))}
            line["cpu_baseline"] = {"value": cflops / tc / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                                    "cpu_model": cpu_model(), "sample": sample, "seconds_mean": tc,
                                    "seconds_min": min(ts), **match}
        except Exception as e:  # keep the GPU line even if the host leg fails
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def run_replicas(args, cfgd, a, x, rank, world, local, t_gen):
    """N replicas of the single-GPU MPK (weak scaling: every rank runs the
    whole config; value = N x flops / the slowest rank's time)."""
    import torch
    import torch.distributed as dist

    import paper_2205_01598_b200 as lm
    from paper_2205_01598_b200 import _lib
    from paper_2205_01598_b200 import executor as E
    from paper_2205_01598_b200 import kernels as K

    k = cfgd["k"]
    n, nnz = a.n_rows, a.n_nz
    ctx = _lib.context()
    t0 = time.perf_counter()
    pre = lm.prepare(a, "lb_lg_p2p", k, 126e6)
    plan = lm.build_plan(pre, "lb_lg_p2p", 1)
    y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
    K.permute_vectors(pre.perm.device()[0], torch.from_numpy(x).cuda().unsqueeze(0), y[0:1])
    launch, sched = E.plan_launcher(plan, y)
    launch()
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t0
    for _ in range(args.warmup):
        launch()
    dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, enabled=not args.no_clocks) as clocks:
        def all_done(done):
            f = torch.tensor([1 if done else 0], device="cuda", dtype=torch.int32)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            return bool(f.item())

        clocks.under_load(launch, all_done=all_done)
        dist.barrier()
        torch.cuda.synchronize()
        launches0 = ctx.launches()
        e0.record()
        for _ in range(args.steps):
            launch()
        e1.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    _lib.check(ctx.lib.lmpk_ctx_check(ctx.handle, _lib.stream_handle()), "bench")
    tt = torch.tensor([e0.elapsed_time(e1) * 1e-3], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_step = float(tt.item()) / args.steps
    yb = torch.zeros_like(y)
    yb[0] = y[0]
    K.mpk_baseline(pre.a.device(), yb, k)
    ok = torch.tensor([1 if torch.equal(yb, y) else 0], device="cuda")
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    hx = torch.from_numpy(np.ascontiguousarray(x[pre.perm.perm])).pin_memory().numpy()
    dist.barrier()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        res = lm.run_plan(plan, x=hx)
        ts.append(time.perf_counter() - t0)
        del res
    te = torch.tensor([statistics.median(ts)], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    flops = 2.0 * nnz * k
    peak, peak_kind = measured_hbm_peak()
    Q = q_ro(n, nnz, k) if sched != "crs" else k * q_spmv(n, nnz)
    line = {
        "metric": metric_name(cfgd), "value": world * flops / t_step / 1e9, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfgd["name"], "n_rows": n, "nnz": nnz, "k": k, "schedule": sched,
                   "parallelism": f"replicas x{world} (no data-path collective: "
                                  + ("the giant component spans < 2k+1 levels, SURVEY 8e)" if cfgd["key"] == "cfg4"
                                     else "the whole config fits one GPU's L2)")},
        "roofline": {"bound": "hbm", "achieved": Q / t_step / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": Q / t_step / 1e9 / peak, "traffic": traffic_for(args.config), "peak_kind": peak_kind},
        "e2e": {"value": world * flops / float(te.item()) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": world * 8 * n, "d2h_bytes_per_step": world * 8 * n * k},
        "gpu_launches": launches,
        "bitwise_vs_baseline": bool(ok.item() == 1),
        "preprocess": {"seconds": t_pre, "generate_seconds": t_gen},
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_dist(args, cfgd, a, x, rank, world, local, t_gen):
    """N > 1: contiguous level-range shards with a depth-k halo (dist.py),
    each rank's window cut from the level-permuted matrix in HBM.  Strong
    scaling: one matrix split over the ranks; a step is one halo exchange of
    y_0 (cfg5: of the two newest states per batch) by one batched NCCL
    send/recv group + the local level-blocked kernel."""
    import torch
    import torch.distributed as dist

    import paper_2205_01598_b200 as lm
    from paper_2205_01598_b200 import _lib
    from paper_2205_01598_b200 import kernels as K
    from paper_2205_01598_b200.dist import DistCheb, DistMpk

    k = cfgd["k"]
    n, nnz = a.n_rows, a.n_nz
    ctx = _lib.context()
    t0 = time.perf_counter()
    if cfgd["kind"] == "cheb":
        coeffs = cheb_coeffs_cfg5(a)
        b = lm.scale_for_heat(a, coeffs.lam_min, coeffs.lam_max)
        levels, perm = lm.bfs_levels(b, 0)
        pb = lm.permute_symmetric(b, perm)
    else:
        levels, perm = lm.bfs_levels(a, 0)
        pb = lm.permute_symmetric(a, perm)
    dev = pb.device()
    lp = np.asarray(levels.level_ptr, dtype=np.int64)
    lnnz = K.level_nnz(dev, lp)
    x_perm = x[perm.perm]
    if cfgd["kind"] == "cheb":
        dm = DistCheb(dev, None, None, lp, lnnz, coeffs.c, k, rank, world, device=f"cuda:{local}")
        s = dm.shard
        x_own = torch.from_numpy(x_perm[s.own_lo:s.own_hi].copy()).cuda()
        run = lambda: dm.step(x_own)  # noqa: E731
        flops = 4.0 * nnz * coeffs.n_moments
        red = dm.shards.redundant_flops() // k * coeffs.n_moments * 2
    else:
        dm = DistMpk(dev, None, None, lp, lnnz, k, rank, world, device=f"cuda:{local}")
        s = dm.shard
        x_own = torch.from_numpy(x_perm[s.own_lo:s.own_hi].copy()).cuda()
        run = lambda: dm.run(x_own, check_errors=False)  # noqa: E731
        flops = 2.0 * nnz * k
        red = dm.shards.redundant_flops()
    run()
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t0
    for _ in range(args.warmup):
        run()
    dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, enabled=not args.no_clocks) as clocks:
        def all_done(done):
            f = torch.tensor([1 if done else 0], device="cuda", dtype=torch.int32)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            return bool(f.item())

        clocks.under_load(run, all_done=all_done)
        dist.barrier()
        torch.cuda.synchronize()
        launches0 = ctx.launches()
        e0.record()
        for _ in range(args.steps):
            run()
        e1.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    _lib.check(ctx.lib.lmpk_ctx_check(ctx.handle, _lib.stream_handle()), "bench")
    t_local = torch.tensor([e0.elapsed_time(e1) * 1e-3], device="cuda")
    dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    t_step = float(t_local.item()) / args.steps
    # parity of the owned rows against the single-GPU computation
    if cfgd["kind"] == "cheb":
        prop = lm.ChebPropagator(a, coeffs.dt, coeffs=coeffs, p_m_batch=k, cache_bytes=126e6)
        ref = prop.step(torch.from_numpy(x).cuda())[torch.from_numpy(perm.perm).cuda().long()]
        ok = torch.tensor([1 if torch.equal(ref[s.own_lo:s.own_hi], dm.step(x_own)) else 0], device="cuda")
        hb, db = 16 * s.n_own, 16 * s.n_own
    else:
        yb = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
        yb[0] = torch.from_numpy(x_perm)
        K.mpk_baseline(dev, yb, k)
        ok = torch.tensor([1 if torch.equal(yb[:, s.own_lo:s.own_hi], dm.run(x_own)) else 0], device="cuda")
        hb, db = 8 * s.n_own, 8 * s.n_own * k
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    # end to end: the rank's owned x from pinned host memory, results back to pinned host memory
    hx = x_own.cpu().pin_memory()
    dist.barrier()
    c0 = time.perf_counter()
    for _ in range(max(3, min(args.steps, 20))):
        x_own.copy_(hx, non_blocking=True)
        out = run()
        host = out[1:].cpu() if cfgd["kind"] == "mpk" else out.cpu()
    torch.cuda.synchronize()
    te = torch.tensor([(time.perf_counter() - c0) / max(3, min(args.steps, 20))], device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    del host
    peak, peak_kind = measured_hbm_peak()
    Qc = q_ro(n, nnz, k) if cfgd["kind"] == "mpk" else q_cheb_batch(n, nnz) * (coeffs.n_moments // k)
    line = {
        "metric": metric_name(cfgd), "value": flops / t_step / 1e9, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c128" if cfgd["kind"] == "cheb" else "f64", "data": "synthetic",
        "config": {"workload": cfgd["name"], "n_rows": n, "nnz": nnz, "k": k,
                   "parallelism": f"level-range shards x{world}, depth-{k} halo (one NCCL send/recv group per "
                                  + ("call)" if cfgd["kind"] == "mpk" else "batch)"),
                   "windows": "cut in HBM (lmpk_csr_window)"},
        "redundant_flop_frac": red / flops,
        "halo_bytes_per_call": int(sum(dm.shards.halo_bytes(g) for g in range(world))),
        "roofline": {"bound": "hbm", "achieved": Qc / world / t_step / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": Qc / world / t_step / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                     "note": "per-GPU share of the algorithmic bytes / step time (includes the halo exchange)"},
        "e2e": {"value": flops / float(te.item()) / 1e9, "unit": "GFLOP/s",
                "h2d_bytes_per_step": int(hb) * world, "d2h_bytes_per_step": int(db) * world},
        "gpu_launches": launches,
        "bitwise_vs_single_gpu": bool(ok.item() == 1),
        "preprocess": {"seconds": t_pre, "generate_seconds": t_gen},
        "clocks": clocks.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU-baseline timing")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-step", action="store_true",
                    help="wrap one steady-state step in cudaProfilerStart/Stop (for ncu --profile-from-start off)")
    ap.add_argument("--no-clocks", action="store_true",
                    help="skip the nvidia-smi sampler and its load phase (ncu runs)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfgd = workload(args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # self-launch: one rank per GPU under torch.distributed.run (NCCL)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py")] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd, env=env))
    if args.impl == "reference":
        run_reference(args, cfgd)
    else:
        run_ours(args, cfgd)


if __name__ == "__main__":
    main()
