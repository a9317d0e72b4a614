"""Multi-GPU MPK: contiguous level-range shards with a depth-k halo.

The reference has no multi-process code; this module
is the greenfield multi-GPU layer north_star asks for.  It rests on level
confinement (Eq. 4 of the paper; pkg/src/levelmpk/levels.py, test_levels.py:
58-88): in the level-permuted matrix a row of level l only couples to levels
l-1..l+1.  Hence:

  * rank g owns a contiguous LEVEL range [a_g, b_g), balanced by nnz, i.e. a
    contiguous row range of the permuted matrix;
  * its WINDOW is levels [a_g - k, b_g + k) (clamped): to produce y_1..y_k on
    the owned rows it needs y_0 on the window only, and the window matrix is
    the contiguous row block of the permuted matrix with the columns outside
    the window dropped.  Rows whose entries were dropped sit in the outermost
    window levels; their error moves inward one level per power, so after p
    powers levels [a_g - k + p, b_g + k - p) are exact -- the owned rows at
    every power p <= k (bitwise identical to the single-GPU result: same
    rows, same entries in the same order);
  * y_0 halos are exchanged ONCE per MPK call: the left halo [win_lo, own_lo)
    comes from rank g-1, the right halo [own_hi, win_hi) from rank g+1, as one
    batched NCCL send/recv group over NVLink (torch.distributed P2P ops);
  * the redundant work is the halo rows computed at every power:
    2 * k * (nnz(window) - nnz(owned)) flops per call, reported by
    ``LevelShards.redundant_flops``.

Each rank needs at least k levels so the halo comes from direct neighbours
only; ``LevelShards`` raises ValueError otherwise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    level_lo: int  # owned levels [level_lo, level_hi)
    level_hi: int
    own_lo: int    # owned rows (permuted order)
    own_hi: int
    win_lo: int    # window rows: levels [level_lo - k, level_hi + k) clamped
    win_hi: int

    @property
    def n_own(self) -> int:
        return self.own_hi - self.own_lo

    @property
    def n_win(self) -> int:
        return self.win_hi - self.win_lo

    @property
    def own_offset(self) -> int:
        """First owned row inside the window."""
        return self.own_lo - self.win_lo

    @property
    def left_halo(self) -> int:
        return self.own_lo - self.win_lo

    @property
    def right_halo(self) -> int:
        return self.win_hi - self.own_hi


class LevelShards:
    """Partition of a level-permuted matrix into `world` level ranges."""

    def __init__(self, level_ptr, level_nnz, world: int, k: int):
        level_ptr = np.asarray(level_ptr, dtype=np.int64)
        level_nnz = np.asarray(level_nnz, dtype=np.int64)
        L = int(level_ptr.shape[0] - 1)
        if world < 1:
            raise ValueError("world must be >= 1")
        if k < 1:
            raise ValueError("p_m must be >= 1")
        if level_nnz.shape[0] != L:
            raise ValueError("level_nnz length must equal the number of levels")
        if world > 1 and L < world * k:
            raise ValueError(f"{L} levels cannot give {world} shards of >= k={k} levels "
                             "(depth-k halos must come from direct neighbours)")
        self.world, self.k, self.n_levels = world, k, L
        self.level_ptr = level_ptr
        self.level_nnz = level_nnz
        bounds = self._balanced_bounds(level_nnz, world, k)
        self.level_bounds = bounds
        self.shards = []
        for g in range(world):
            a, b = int(bounds[g]), int(bounds[g + 1])
            wa, wb = max(0, a - k), min(L, b + k)
            self.shards.append(Shard(g, a, b, int(level_ptr[a]), int(level_ptr[b]),
                                     int(level_ptr[wa]), int(level_ptr[wb])))

    @staticmethod
    def _balanced_bounds(level_nnz, world, k):
        """Level boundaries with ~equal owned nnz and >= k levels per shard."""
        L = level_nnz.shape[0]
        if world == 1:
            return np.array([0, L], dtype=np.int64)
        csum = np.concatenate([[0], np.cumsum(level_nnz)])
        total = csum[-1]
        bounds = [0]
        for g in range(1, world):
            target = total * g / world
            b = int(np.searchsorted(csum, target, side="left"))
            lo = bounds[-1] + k                # >= k levels for shard g-1
            hi = L - (world - g) * k           # leave >= k levels for the rest
            bounds.append(int(min(max(b, lo), hi)))
        bounds.append(L)
        return np.array(bounds, dtype=np.int64)

    def __getitem__(self, g) -> Shard:
        return self.shards[g]

    def nnz_range(self, lo_level, hi_level) -> int:
        return int(self.level_nnz[lo_level:hi_level].sum())

    def window_nnz(self, g) -> int:
        s = self.shards[g]
        return self.nnz_range(max(0, s.level_lo - self.k), min(self.n_levels, s.level_hi + self.k))

    def owned_nnz(self, g) -> int:
        s = self.shards[g]
        return self.nnz_range(s.level_lo, s.level_hi)

    def redundant_flops(self, g=None) -> int:
        """2*k*(window nnz - owned nnz): halo rows recomputed at every power
        (an upper bound: dropped out-of-window entries are not computed)."""
        gs = range(self.world) if g is None else [g]
        return int(sum(2 * self.k * (self.window_nnz(i) - self.owned_nnz(i)) for i in gs))

    def halo_bytes(self, g, width=1) -> int:
        s = self.shards[g]
        return 8 * width * (s.left_halo + s.right_halo)


def window_csr(row_ptr, col, val, lo: int, hi: int):
    """Rows [lo, hi) of a CRS matrix with columns shifted by -lo and the
    entries whose column falls outside [lo, hi) dropped (entry order kept)."""
    row_ptr = np.asarray(row_ptr)
    col = np.asarray(col)
    val = np.asarray(val)
    e0, e1 = int(row_ptr[lo]), int(row_ptr[hi])
    c = col[e0:e1].astype(np.int64)
    keep = (c >= lo) & (c < hi)
    lens = np.diff(row_ptr[lo:hi + 1].astype(np.int64))
    row_id = np.repeat(np.arange(hi - lo), lens)
    kept_per_row = np.bincount(row_id[keep], minlength=hi - lo)
    rp = np.zeros(hi - lo + 1, dtype=np.int32)
    np.cumsum(kept_per_row, out=rp[1:])
    return rp, (c[keep] - lo).astype(np.int32), np.ascontiguousarray(val[e0:e1][keep])


def _real_view(v):
    import torch

    return torch.view_as_real(v) if v.is_complex() else v


def halo_exchange(shards: "LevelShards", rank: int, group, vecs):
    """One batched P2P group: for every window-local vector, send my first /
    last owned rows to the left / right neighbour (their halos) and receive
    my left / right halo from them (NCCL over NVLink on GPUs, gloo on CPU)."""
    if shards.world == 1:
        return
    import torch.distributed as dist

    s = shards[rank]
    o0, o1 = s.own_offset, s.own_offset + s.n_own
    ops = []
    for v in vecs:
        v = _real_view(v)
        if rank > 0:
            left = shards[rank - 1]
            ops.append(dist.P2POp(dist.isend, v[o0:o0 + left.right_halo], rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, v[0:s.left_halo], rank - 1, group))
        if rank < shards.world - 1:
            right = shards[rank + 1]
            ops.append(dist.P2POp(dist.isend, v[o1 - right.left_halo:o1], rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, v[o1:o1 + s.right_halo], rank + 1, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def _is_device_csr(a) -> bool:
    from .kernels import DeviceCsr

    return isinstance(a, DeviceCsr)


def _window(row_ptr, col, val, lo, hi):
    """The window matrix: cut in HBM (lmpk_csr_window) when the permuted
    matrix is a DeviceCsr, else on the host (window_csr)."""
    if _is_device_csr(row_ptr):
        from . import kernels as K

        return K.csr_window(row_ptr, lo, hi)
    return window_csr(row_ptr, col, val, lo, hi)


class CudaWindowMpk:
    """Local MPK on one rank's window: the single-GPU level-blocked kernel."""

    def __init__(self, rp, col, val, k, **tiling_kw):
        from . import kernels as K

        self.K = K
        self.k = k
        self.a = rp if _is_device_csr(rp) else K.DeviceCsr.from_host(rp, col, val)
        self.tiling = K.Tiling(self.a, k, **tiling_kw)
        self.cfg = K.mpk_power_cfg(k)

    def __call__(self, y, check_errors=True):
        self.K.mpk_run(self.tiling, y, self.cfg, check_errors=check_errors)
        return y


class DistMpk:
    """Level-range sharded MPK on one rank of a torch.distributed group.

    ``run(x_own)`` takes y_0 on the owned rows (permuted order) and returns
    the [k+1, n_own] block of y_0..y_k for those rows.  ``local`` computes the
    window MPK in place on a [k+1, n_win] tensor; the default is the CUDA
    kernel (CudaWindowMpk); tests inject a CPU computation with gloo.
    """

    def __init__(self, row_ptr, col, val, level_ptr, level_nnz, k, rank, world, group=None,
                 device=None, local=None, **tiling_kw):
        import torch

        self.torch = torch
        self.rank, self.world, self.k, self.group = rank, world, k, group
        self.shards = LevelShards(level_ptr, level_nnz, world, k)
        self.shard = self.shards[rank]
        s = self.shard
        win = _window(row_ptr, col, val, s.win_lo, s.win_hi)
        self.window = win
        self.device = torch.device("cpu") if device is None else torch.device(device)
        if local is None:
            local = CudaWindowMpk(win, None, None, k, **tiling_kw) if _is_device_csr(win) \
                else CudaWindowMpk(*win, k, **tiling_kw)
        self.local = local
        self.y = torch.zeros((k + 1, s.n_win), dtype=torch.float64, device=self.device)

    def exchange(self, *vecs):
        """Fill the halo rows of window-local vectors from the neighbour ranks."""
        halo_exchange(self.shards, self.rank, self.group, vecs)

    def run(self, x_own, check_errors=True):
        s = self.shard
        y = self.y
        y[0, s.own_offset:s.own_offset + s.n_own].copy_(self.torch.as_tensor(x_own, device=self.device))
        self.exchange(y[0])
        self.local(y, check_errors=check_errors)
        return y[:, s.own_offset:s.own_offset + s.n_own]

    @property
    def redundant_flops(self) -> int:
        return self.shards.redundant_flops(self.rank)


def cheb_batch_config(coeffs_c, k_base, pb, n_slots, first_batch):
    """Per-power slots/kernels/coefficients of one Chebyshev batch over a ring
    of n_slots state vectors (cheb.py:209-219, ChebPropagator._configure)."""
    from .plan import KERNEL_CHEB, KERNEL_SPMV

    p = np.arange(1, pb + 1)
    out_slot = (k_base + p) % n_slots
    in_slot = (k_base + p - 1) % n_slots
    prev_slot = (k_base + p - 2) % n_slots
    kernel = np.full(pb, KERNEL_CHEB)
    if first_batch:
        kernel[0] = KERNEL_SPMV
    c = np.asarray(coeffs_c)[k_base + 1:k_base + pb + 1]
    return out_slot, in_slot, prev_slot, kernel, np.real(c), (np.imag(c) if np.iscomplexobj(c) else None)


class CudaWindowCheb:
    """Chebyshev batches on one rank's window through the level-blocked kernel."""

    def __init__(self, rp, col, val, p_b, complex_state, **tiling_kw):
        from . import _lib
        from . import kernels as K

        self.K, self._lib = K, _lib
        self.a = rp if _is_device_csr(rp) else K.DeviceCsr.from_host(rp, col, val)
        flags = int(tiling_kw.pop("mode_flags", 0)) | (_lib.FLAG_COMPLEX if complex_state else 0)
        self.tiling = K.Tiling(self.a, p_b, mode_flags=flags, **tiling_kw)
        self.complex = complex_state

    def __call__(self, ring, acc, coeffs_c, k_base, pb, first_batch):
        import torch

        o, i, pv, kern, cre, cim = cheb_batch_config(coeffs_c, k_base, pb, ring.shape[0], first_batch)
        cfg = self.K.power_cfg(pb, o, i, pv, kern, cre, cim)
        yv = torch.view_as_real(ring).reshape(ring.shape[0], -1) if self.complex else ring
        av = torch.view_as_real(acc).reshape(-1) if self.complex else acc
        self.K.mpk_run(self.tiling, yv, cfg, acc=av, use_acc=True, complex_state=self.complex)


class DistCheb:
    """Level-range sharded Chebyshev propagation (BASELINE config 5 shape).

    Every rank holds a ring of p_b + 2 Chebyshev states T_k over its window
    (depth-p_b halo).  Before each batch of <= p_b powers the halos of the two
    newest states (T_k and T_{k-1}) are exchanged in one P2P group; the
    accumulator needs no exchange (only owned rows are returned).  Owned rows
    are bitwise identical to the single-GPU propagator: the same rows, entries
    and summation order.  ``local(ring, acc, coeffs_c, k_base, pb, first)``
    runs one batch on the window (CUDA by default)."""

    def __init__(self, row_ptr, col, val, level_ptr, level_nnz, coeffs_c, p_b, rank, world, group=None,
                 device=None, local=None, complex_state=None, **tiling_kw):
        import torch

        self.torch = torch
        self.c = np.asarray(coeffs_c)
        self.complex = bool(np.iscomplexobj(self.c)) if complex_state is None else bool(complex_state)
        self.m = self.c.shape[0] - 1
        self.p_b = max(1, min(int(p_b), self.m)) if self.m >= 1 else 1
        self.rank, self.world, self.group = rank, world, group
        self.shards = LevelShards(level_ptr, level_nnz, world, self.p_b)
        s = self.shard = self.shards[rank]
        win = _window(row_ptr, col, val, s.win_lo, s.win_hi)
        self.device = torch.device("cpu") if device is None else torch.device(device)
        if local is None:
            local = CudaWindowCheb(win, None, None, self.p_b, self.complex, **tiling_kw) if _is_device_csr(win) \
                else CudaWindowCheb(*win, self.p_b, self.complex, **tiling_kw)
        self.local = local
        dt = torch.complex128 if self.complex else torch.float64
        self.ring = torch.zeros((self.p_b + 2, s.n_win), dtype=dt, device=self.device)

    def step(self, x_own):
        """One propagation step; x_own = T_0 on the owned rows (level-permuted
        order).  Returns acc = sum_k c_k T_k on the owned rows."""
        torch = self.torch
        s, S = self.shard, self.ring.shape[0]
        ring = self.ring
        o0, o1 = s.own_offset, s.own_offset + s.n_own
        ring[0, o0:o1].copy_(torch.as_tensor(x_own, device=self.device).to(ring.dtype))
        halo_exchange(self.shards, self.rank, self.group, [ring[0]])
        c0 = complex(self.c[0]) if self.complex else float(np.real(self.c[0]))
        acc = torch.empty_like(ring[0])
        if ring.is_cuda:  # acc = c_0 T_0 by liblmpk (oracle order)
            from . import kernels as K

            K.vec_scale(ring[0], c0, acc)
        elif self.complex:  # CPU ranks of the gloo tests: the same products spelled out
            acc.real.copy_(ring[0].real * c0.real - ring[0].imag * c0.imag)
            acc.imag.copy_(ring[0].imag * c0.real + ring[0].real * c0.imag)
        else:
            acc.copy_(ring[0] * c0)
        k = 0
        while k < self.m:
            pb = min(self.p_b, self.m - k)
            if k > 0:
                halo_exchange(self.shards, self.rank, self.group, [ring[k % S], ring[(k - 1) % S]])
            self.local(ring, acc, self.c, k, pb, k == 0)
            k += pb
        return acc[o0:o1]

    @property
    def redundant_flops_per_step(self) -> int:
        return self.shards.redundant_flops(self.rank) // self.p_b * max(self.m, 1)
