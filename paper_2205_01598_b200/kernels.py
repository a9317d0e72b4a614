"""Torch-facing wrappers of the C-ABI (include/lmpk.h).

torch is used only for device memory and streams: every tensor here is a
buffer handed to liblmpk by pointer.  All functions fail loudly when the
library or a CUDA device is missing.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, context, ptr, stream_handle


def _torch():
    import torch

    return torch


@dataclass
class DeviceCsr:
    """CRS arrays resident in HBM (row_ptr int32[n+1], col int32[nnz], val f64[nnz])."""

    n: int
    row_ptr: "object"
    col: "object"
    val: "object"

    @property
    def nnz(self) -> int:
        return int(self.col.shape[0])

    def hub_flag(self) -> int:
        """FLAG_NO_HUB_ROWS when no row holds more than 128 entries (one device
        reduction, cached): the CRS sweeps then skip their per-call hub-row scan
        and its host synchronisation."""
        f = getattr(self, "_hub_flag", None)
        if f is None:
            mx = int((self.row_ptr[1:] - self.row_ptr[:-1]).max().item()) if self.n > 0 else 0
            f = _lib.FLAG_NO_HUB_ROWS if mx <= 128 else 0
            self._hub_flag = f
        return f

    @classmethod
    def from_host(cls, row_ptr, col, val, device=None):
        torch = _torch()
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        rp = torch.from_numpy(np.ascontiguousarray(row_ptr, dtype=np.int32)).to(dev, non_blocking=False)
        c = torch.from_numpy(np.ascontiguousarray(col, dtype=np.int32)).to(dev)
        v = torch.from_numpy(np.ascontiguousarray(val, dtype=np.float64)).to(dev)
        return cls(int(rp.shape[0] - 1), rp, c, v)

    def to_host(self):
        return (self.row_ptr.cpu().numpy(), self.col.cpu().numpy(), self.val.cpu().numpy())


def spmv_rows(a: DeviceCsr, x, out, r0, r1, flags=0, stream=None):
    """out[r] = sum val*x[col] for r in [r0, r1) (csr.py:195-201 bitwise)."""
    ctx = context()
    check(ctx.lib.lmpk_spmv_rows(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), ptr(a.val),
                                 ptr(x), ptr(out), int(r0), int(r1), int(flags) | a.hub_flag(),
                                 stream_handle(stream)), "spmv_rows")


def mpk_baseline(a: DeviceCsr, y, p_m, flags=0, stream=None):
    """p_m back-to-back SpMV sweeps on the slots of y (shape [>=p_m+1, n])."""
    ctx = context()
    check(ctx.lib.lmpk_mpk_baseline(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), ptr(a.val),
                                    ptr(y), int(y.stride(0)), int(p_m), int(flags) | a.hub_flag(),
                                    stream_handle(stream)), "mpk_baseline")


class Tiling:
    """Tile geometry of one device matrix for the level-blocked kernel."""

    def __init__(self, a: DeviceCsr, p_m, tile_nnz=0, ctas_per_sm=0, mode_flags=0, threads=0,
                 queue_slack=0, slots=0, group=0, stream=None):
        self.ctx = context()
        self.a = a
        self.p_m = int(p_m)
        h = ctypes.c_void_p()
        info = _lib.TilingInfo()
        prm = _lib.TilingParams(int(tile_nnz), int(ctas_per_sm), int(threads), int(queue_slack),
                                int(mode_flags), int(slots), int(group))
        check(self.ctx.lib.lmpk_tiling_create(
            self.ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), ptr(a.val), int(p_m),
            ctypes.byref(prm), ctypes.byref(h), ctypes.byref(info), stream_handle(stream)),
            "tiling_create")
        self.handle = h
        self.info = info.as_dict()

    @property
    def mode(self) -> str:
        return {1: "resident", 2: "streaming", 3: "ring"}[self.info["mode"]]

    @property
    def group(self) -> int:
        """Powers computed per staged tile block (q)."""
        return self.info["powers_per_item"]

    def geometry(self):
        nt = self.info["n_tiles"]
        tr = np.empty(nt + 1, dtype=np.int32)
        lo = np.empty(nt, dtype=np.int32)
        hi = np.empty(nt, dtype=np.int32)
        check(self.ctx.lib.lmpk_tiling_geometry(
            self.handle, tr.ctypes.data_as(ctypes.c_void_p), lo.ctypes.data_as(ctypes.c_void_p),
            hi.ctypes.data_as(ctypes.c_void_p)))
        return tr, lo, hi

    def item_order(self):
        """int32 [n, 2] (tile, power) pairs in the order the kernel's item queue
        hands them out (an item of q powers expands to q rows)."""
        n = ctypes.c_int64()
        check(self.ctx.lib.lmpk_tiling_items(self.handle, None, 0, ctypes.byref(n)))
        raw = np.empty((int(n.value), 3), dtype=np.int32)
        check(self.ctx.lib.lmpk_tiling_items(self.handle, raw.ctypes.data_as(ctypes.c_void_p),
                                             int(n.value), ctypes.byref(n)))
        reps = raw[:, 2]
        tiles = np.repeat(raw[:, 0], reps)
        first = np.repeat(raw[:, 1], reps)
        offs = np.arange(int(reps.sum())) - np.repeat(np.cumsum(reps) - reps, reps)
        return np.stack([tiles, first + offs], axis=1).astype(np.int64)

    def close(self):
        if getattr(self, "handle", None):
            self.ctx.lib.lmpk_tiling_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def power_cfg(n_powers, out_slot, in_slot, prev_slot, kernel, coef_re=None, coef_im=None):
    cfg = _lib.PowerCfg()
    if not 1 <= n_powers <= _lib.MAX_POWERS:
        raise ValueError(f"p_m must be in [1, {_lib.MAX_POWERS}] for the cuda backend")
    cfg.n_powers = int(n_powers)
    for i in range(n_powers):
        cfg.out_slot[i] = int(out_slot[i])
        cfg.in_slot[i] = int(in_slot[i])
        cfg.prev_slot[i] = int(prev_slot[i])
        cfg.kernel[i] = int(kernel[i])
        cfg.acc_coef_re[i] = float(coef_re[i]) if coef_re is not None else 0.0
        cfg.acc_coef_im[i] = float(coef_im[i]) if coef_im is not None else 0.0
    return cfg


def mpk_power_cfg(p_m):
    """Plain MPK: out = p, in = p-1, prev = max(p-2, 0) (plan.py:307-312)."""
    p = np.arange(1, p_m + 1)
    return power_cfg(p_m, p, p - 1, np.maximum(p - 2, 0), np.zeros(p_m, dtype=int))


# Row sums of the level-blocked kernel: True = separately rounded multiply and
# add (bitwise identical to the reference), False = fused multiply-add chain
# (same order; relative error far inside the 1e-12 contract).  LMPK_EXACT=0/1
# overrides the default.
EXACT_DEFAULT = os.environ.get("LMPK_EXACT", "1") != "0"


def mpk_run(tiling: Tiling, y, cfg, acc=None, use_acc=False, complex_state=False, flags=0,
            stream=None, check_errors=True, exact=None):
    """Level-blocked MPK over the slots of y (torch float64, [n_slots, n] or
    [n_slots, 2n] for complex state viewed as float64)."""
    ctx = tiling.ctx
    if exact is None:
        exact = EXACT_DEFAULT
    f = int(flags) | (_lib.FLAG_COMPLEX if complex_state else 0) | (_lib.FLAG_EXACT if exact else 0)
    check(ctx.lib.lmpk_mpk_run(ctx.handle, tiling.handle, ptr(y), int(y.stride(0)), int(y.shape[0]),
                               ctypes.byref(cfg), ptr(acc), 1 if use_acc else 0, f,
                               stream_handle(stream)), "mpk_run")
    if check_errors:
        check(ctx.lib.lmpk_ctx_check(ctx.handle, stream_handle(stream)), "mpk_run")


def mpk_crs_run(a: DeviceCsr, y, cfg, acc=None, use_acc=False, complex_state=False, stream=None):
    """A plan's powers as sweeps over the CRS arrays with the per-power kernel
    (SpMV / Chebyshev) and accumulation fused (lmpk_mpk_crs_run): the path of
    level-blocked plans on matrices whose rows exceed the tile format."""
    ctx = context()
    f = (_lib.FLAG_COMPLEX if complex_state else 0) | _lib.FLAG_EXACT | a.hub_flag()
    check(ctx.lib.lmpk_mpk_crs_run(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), ptr(a.val), ptr(y),
                                   int(y.stride(0)), int(y.shape[0]), ctypes.byref(cfg), ptr(acc),
                                   1 if use_acc else 0, f, stream_handle(stream)), "mpk_crs_run")


def bfs_levels(a: DeviceCsr, root=0, stream=None):
    """Returns (perm int32 tensor, inv_perm int32 tensor, level_ptr int64 numpy)."""
    torch = _torch()
    ctx = context()
    dev = a.row_ptr.device
    perm = torch.empty(a.n, dtype=torch.int32, device=dev)
    inv = torch.empty(a.n, dtype=torch.int32, device=dev)
    lp = torch.empty(a.n + 1, dtype=torch.int64, device=dev)
    nl = ctypes.c_int64()
    check(ctx.lib.lmpk_bfs_levels(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), int(root),
                                  ptr(perm), ptr(inv), ptr(lp), ctypes.byref(nl),
                                  stream_handle(stream)), "bfs_levels")
    L = int(nl.value)
    return perm, inv, lp[: L + 1].cpu().numpy()


def symmetrized_pattern(a: DeviceCsr, stream=None):
    """(row_ptr int64, col int32) tensors of A|A^T, or None if A is symmetric."""
    torch = _torch()
    ctx = context()
    sym = ctypes.c_int()
    nnz = ctypes.c_int64()
    check(ctx.lib.lmpk_symmetrized_pattern(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col),
                                           ctypes.byref(sym), ctypes.byref(nnz), None, None, 0,
                                           stream_handle(stream)), "symmetrized_pattern")
    if sym.value:
        return None
    dev = a.row_ptr.device
    rp = torch.empty(a.n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(int(nnz.value), 1), dtype=torch.int32, device=dev)
    check(ctx.lib.lmpk_symmetrized_pattern(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col),
                                           ctypes.byref(sym), ctypes.byref(nnz), ptr(rp), ptr(col),
                                           int(col.shape[0]), stream_handle(stream)),
          "symmetrized_pattern")
    return rp, col[: int(nnz.value)]


def csr_from_triplets(n, rows, cols, vals, sum_duplicates=True, stream=None) -> DeviceCsr:
    """Device CRS build from COO triplets (csr.py:72-94, bit-exact): rows/cols
    int64 and vals float64 CUDA tensors of one length.  Raises ValueError
    ("row index out of range" / "column index out of range") like the reference."""
    torch = _torch()
    ctx = context()
    rows = rows.to(torch.int64).contiguous()
    cols = cols.to(torch.int64).contiguous()
    vals = vals.to(torch.float64).contiguous()
    m = int(rows.shape[0])
    if int(cols.shape[0]) != m or int(vals.shape[0]) != m:
        raise ValueError("rows, cols and vals must have the same length")
    dev = rows.device
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    col = torch.empty(m, dtype=torch.int32, device=dev)
    val = torch.empty(m, dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64(0)
    rc = ctx.lib.lmpk_csr_from_triplets(ctx.handle, int(n), m, ptr(rows), ptr(cols), ptr(vals),
                                        1 if sum_duplicates else 0, ptr(rp), ptr(col), ptr(val),
                                        ctypes.byref(nnz), stream_handle(stream))
    check(rc, "csr_from_triplets")  # LMPK_ERR_ARG -> ValueError with the reference's message
    k = int(nnz.value)
    return DeviceCsr(int(n), rp, col[:k], val[:k])


def permute_symmetric(a: DeviceCsr, perm, inv, stream=None) -> DeviceCsr:
    torch = _torch()
    ctx = context()
    dev = a.row_ptr.device
    rp = torch.empty(a.n + 1, dtype=torch.int32, device=dev)
    col = torch.empty(a.nnz, dtype=torch.int32, device=dev)
    val = torch.empty(a.nnz, dtype=torch.float64, device=dev)
    check(ctx.lib.lmpk_permute_symmetric(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), ptr(a.val),
                                         ptr(perm), ptr(inv), ptr(rp), ptr(col), ptr(val),
                                         stream_handle(stream)), "permute_symmetric")
    return DeviceCsr(a.n, rp, col, val)


def permute_vectors(perm, src, dst, scatter=False, stream=None):
    """gather: dst[v][i] = src[v][perm[i]]; scatter: dst[v][perm[i]] = src[v][i].
    src/dst: float64 tensors [n_vec, n] or complex128 [n_vec, n]."""
    torch = _torch()
    ctx = context()
    width = 1
    if src.dtype == torch.complex128:
        width = 2
        src = torch.view_as_real(src)
        dst = torch.view_as_real(dst)
    if src.dim() == 1 or (width == 2 and src.dim() == 2):
        src = src.unsqueeze(0)
        dst = dst.unsqueeze(0)
    n = int(perm.shape[0])
    check(ctx.lib.lmpk_permute_vectors(ctx.handle, n, ptr(perm), ptr(src), int(src.stride(0)),
                                       ptr(dst), int(dst.stride(0)), int(src.shape[0]), width,
                                       1 if scatter else 0, stream_handle(stream)),
          "permute_vectors")


def level_nnz(a: DeviceCsr, level_ptr, stream=None):
    torch = _torch()
    ctx = context()
    lp = torch.as_tensor(np.ascontiguousarray(level_ptr, dtype=np.int64), device=a.row_ptr.device)
    L = int(lp.shape[0] - 1)
    out = torch.empty(max(L, 1), dtype=torch.int64, device=a.row_ptr.device)
    check(ctx.lib.lmpk_level_nnz(ctx.handle, ptr(a.row_ptr), ptr(lp), L, ptr(out),
                                 stream_handle(stream)), "level_nnz")
    return out[:L].cpu().numpy()


def segment_col_range(a: DeviceCsr, seg_ptr, stream=None):
    """(min col, max col) per row segment [seg_ptr[g], seg_ptr[g+1]) as numpy arrays."""
    torch = _torch()
    ctx = context()
    dev = a.row_ptr.device
    sp = torch.as_tensor(np.ascontiguousarray(seg_ptr, dtype=np.int64), device=dev)
    G = int(sp.shape[0] - 1)
    mn = torch.empty(max(G, 1), dtype=torch.int32, device=dev)
    mx = torch.empty(max(G, 1), dtype=torch.int32, device=dev)
    check(ctx.lib.lmpk_segment_col_range(ctx.handle, ptr(a.row_ptr), ptr(a.col), G, ptr(sp),
                                         ptr(mn), ptr(mx), stream_handle(stream)),
          "segment_col_range")
    return mn[:G].cpu().numpy(), mx[:G].cpu().numpy()


def csr_window(a: DeviceCsr, lo, hi, stream=None) -> DeviceCsr:
    """Rows [lo, hi) of a device matrix, columns outside the range dropped and
    shifted by -lo (one rank's level-range window, cut in HBM)."""
    torch = _torch()
    ctx = context()
    w = int(hi) - int(lo)
    dev = a.row_ptr.device
    rp = torch.empty(w + 1, dtype=torch.int32, device=dev)
    cap = int(a.row_ptr[int(hi)].item()) - int(a.row_ptr[int(lo)].item()) if w > 0 else 0
    col = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    val = torch.empty(max(cap, 1), dtype=torch.float64, device=dev)
    nnz = ctypes.c_int64()
    check(ctx.lib.lmpk_csr_window(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), ptr(a.val), int(lo), int(hi),
                                  ptr(rp), ptr(col), ptr(val), ctypes.byref(nnz), stream_handle(stream)),
          "csr_window")
    k = int(nnz.value)
    return DeviceCsr(w, rp, col[:k].clone() if k < col.shape[0] else col, val[:k].clone() if k < val.shape[0] else val)


def vec_scale(x, c, out, stream=None):
    """out = c * x (float64 or complex128 tensors of equal shape) in the
    reference's arithmetic (the ChebPropagator accumulator start c_0 T_0)."""
    torch = _torch()
    ctx = context()
    cplx = x.is_complex()
    xv = torch.view_as_real(x).reshape(-1) if cplx else x.reshape(-1)
    ov = torch.view_as_real(out).reshape(-1) if cplx else out.reshape(-1)
    n = xv.shape[0] // 2 if cplx else xv.shape[0]
    check(ctx.lib.lmpk_vec_scale(ctx.handle, int(n), ptr(xv), float(np.real(c)), float(np.imag(c)),
                                 1 if cplx else 0, ptr(ov), stream_handle(stream)), "vec_scale")
    return out


# ---------------------------------------------------------------- planning (include/lmpk_plan.h)
def _np_ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def sym_pattern_device(a: DeviceCsr):
    """(ptr tensor, col tensor, ptr64) of A|A^T in HBM; A's own arrays when the
    pattern is already symmetric (levels.py:48-61)."""
    res = symmetrized_pattern(a)
    if res is None:
        return a.row_ptr, a.col, 0
    return res[0], res[1], 1


def level_nnz_perm(a: DeviceCsr, perm, level_ptr, stream=None):
    """nnz per level of rows perm[level_ptr[i]:level_ptr[i+1]] of the original matrix."""
    torch = _torch()
    ctx = context()
    lp = torch.as_tensor(np.ascontiguousarray(level_ptr, dtype=np.int64), device=a.row_ptr.device)
    L = int(lp.shape[0] - 1)
    out = torch.empty(max(L, 1), dtype=torch.int64, device=a.row_ptr.device)
    check(ctx.lib.lmpk_level_nnz_perm(ctx.handle, ptr(a.row_ptr), ptr(perm), ptr(lp), L, ptr(out),
                                      stream_handle(stream)), "level_nnz_perm")
    return out[:L].cpu().numpy()


def refine_span(n, sym, perm, r0, r1, stream=None):
    """Induced-subgraph BFS of permuted rows [r0, r1); reorders perm[r0:r1] in
    place and returns the child level_ptr (numpy int64, relative to r0)."""
    torch = _torch()
    ctx = context()
    sp, sc, ptr64 = sym
    lp = torch.empty(int(r1) - int(r0) + 1, dtype=torch.int64, device=perm.device)
    nl = ctypes.c_int64()
    check(ctx.lib.lmpk_refine_span(ctx.handle, int(n), ptr(sp), int(ptr64), ptr(sc), ptr(perm), int(r0), int(r1),
                                   ptr(lp), ctypes.byref(nl), stream_handle(stream)), "refine_span")
    return lp[: int(nl.value) + 1].cpu().numpy()


def halo_seed(n, perm, group_ptr, key_orig, stream=None):
    torch = _torch()
    ctx = context()
    gp = torch.as_tensor(np.ascontiguousarray(group_ptr, dtype=np.int64), device=perm.device)
    check(ctx.lib.lmpk_halo_seed(ctx.handle, int(n), ptr(perm), int(gp.shape[0] - 1), ptr(gp), ptr(key_orig),
                                 stream_handle(stream)), "halo_seed")


def halo_level_sort(n, sym, perm, key_orig, lo, hi, stream=None):
    """Stable key sort of the halo level [lo, hi) of perm; returns the sorted keys (numpy)."""
    torch = _torch()
    ctx = context()
    sp, sc, ptr64 = sym
    keys = torch.empty(max(int(hi) - int(lo), 1), dtype=torch.int32, device=perm.device)
    check(ctx.lib.lmpk_halo_level_sort(ctx.handle, int(n), ptr(sp), int(ptr64), ptr(sc), ptr(perm), ptr(key_orig),
                                       int(lo), int(hi), ptr(keys), stream_handle(stream)), "halo_level_sort")
    return keys[: int(hi) - int(lo)].cpu().numpy()


def invert_perm(perm, stream=None):
    torch = _torch()
    ctx = context()
    inv = torch.empty_like(perm)
    check(ctx.lib.lmpk_invert_perm(ctx.handle, int(perm.shape[0]), ptr(perm), ptr(inv), stream_handle(stream)),
          "invert_perm")
    return inv


def item_deps(a: DeviceCsr, row_start, row_end, power, stream=None):
    """True dependencies of a flat item list (plan.py:103-129) as (dep_ptr, dep)
    numpy int64 arrays: item u depends on dep[dep_ptr[u]:dep_ptr[u+1]] (ascending)."""
    ctx = context()
    rs = np.ascontiguousarray(row_start, dtype=np.int64)
    re = np.ascontiguousarray(row_end, dtype=np.int64)
    pw = np.ascontiguousarray(power, dtype=np.int64)
    n_items = int(rs.shape[0])
    dep_ptr = np.zeros(n_items + 1, dtype=np.int64)
    out = ctypes.c_void_p()
    check(ctx.lib.lmpk_item_deps(ctx.handle, a.n, ptr(a.row_ptr), ptr(a.col), n_items, _np_ptr(rs), _np_ptr(re),
                                 _np_ptr(pw), _np_ptr(dep_ptr), ctypes.byref(out), stream_handle(stream)),
          "item_deps")
    try:
        total = int(dep_ptr[-1])
        dep = np.ctypeslib.as_array(ctypes.cast(out, ctypes.POINTER(ctypes.c_int64)), shape=(max(total, 1),))[:total].copy()
    finally:
        ctx.lib.lmpk_host_free(out)
    return dep_ptr, dep


def item_col_max_in_range(a: DeviceCsr, row_start, row_end, col_lo, col_hi, stream=None):
    """Largest column of each item's rows inside [col_lo, col_hi) (-1: none)."""
    ctx = context()
    arrs = [np.ascontiguousarray(v, dtype=np.int64) for v in (row_start, row_end, col_lo, col_hi)]
    out = np.full(arrs[0].shape[0], -1, dtype=np.int32)
    check(ctx.lib.lmpk_item_col_max_in_range(ctx.handle, ptr(a.row_ptr), ptr(a.col), int(arrs[0].shape[0]),
                                             *[_np_ptr(v) for v in arrs], _np_ptr(out), stream_handle(stream)),
          "item_col_max_in_range")
    return out
