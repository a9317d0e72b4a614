"""ctypes binding of liblmpk.so, the C-ABI declared in include/lmpk.h.

The reference binds libc with ctypes for its spin-loop barriers
(pkg/src/levelmpk/backend.py:48-59); this package binds its CUDA library the
same way.  There is no CPU fallback: if the shared library or a CUDA device
is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = pathlib.Path(os.environ.get("LMPK_LIB", _HERE / "_lib" / "liblmpk.so"))

LMPK_OK = 0
LMPK_ERR_ARG = -1
LMPK_ERR_CUDA = -2
LMPK_ERR_WATCHDOG = -3
LMPK_ERR_NOMEM = -4
LMPK_ERR_UNSUPPORTED = -5

KERNEL_SPMV = 0
KERNEL_CHEB = 1

FLAG_COMPLEX = 0x1
FLAG_MODE_STREAM = 0x10
FLAG_MODE_RESIDENT = 0x20
FLAG_NO_TMA = 0x40
FLAG_SWEEP = 0x80
FLAG_EXACT = 0x400
FLAG_READY_QUEUE = 0x1000
FLAG_COMPRESS = 0x2000
FLAG_NO_HUB_ROWS = 0x10000
FLAG_RING = 0x4000
FLAG_PLAIN = 0x8000

MAX_POWERS = 64

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_int = ctypes.c_int


class TilingInfo(ctypes.Structure):
    _fields_ = [
        ("n_tiles", _i32), ("p_m", _i32), ("mode", _i32), ("grid", _i32),
        ("block", _i32), ("smem_bytes", _i32), ("tile_nnz_cap", _i32),
        ("max_fwd_reach", _i32), ("chain_reach", _i32), ("max_row_nnz", _i32),
        ("queue_slack", _i32), ("nnz", _i64), ("block_bytes", _i64),
        ("powers_per_item", _i32), ("slots", _i32), ("x_staged_tiles", _i32),
        ("compressed_tiles", _i32), ("dict_tiles", _i32), ("super_tiles", _i32),
        ("lean_bytes", _i64), ("lean_pattern_tiles", _i32),
        ("lean_xstaged", _i32), ("lean_ring", _i32), ("lean_piece", _i32),
        ("dp_tiles", _i32),
    ]

    def as_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


class TilingParams(ctypes.Structure):
    _fields_ = [("tile_nnz_hint", _i32), ("ctas_per_sm", _i32), ("threads", _i32),
                ("queue_slack", _i32), ("mode_flags", _i32), ("slots", _i32),
                ("powers_per_item", _i32)]


class PowerCfg(ctypes.Structure):
    _fields_ = [
        ("n_powers", _i32),
        ("out_slot", _i32 * MAX_POWERS),
        ("in_slot", _i32 * MAX_POWERS),
        ("prev_slot", _i32 * MAX_POWERS),
        ("kernel", _i32 * MAX_POWERS),
        ("acc_coef_re", ctypes.c_double * MAX_POWERS),
        ("acc_coef_im", ctypes.c_double * MAX_POWERS),
    ]


# name -> (restype, argtypes); every symbol include/lmpk.h declares
SIGNATURES = {
    "lmpk_abi_version": (_int, []),
    "lmpk_last_error": (ctypes.c_char_p, []),
    "lmpk_device_info": (_int, [_int] + [ctypes.POINTER(_int)] * 6),
    "lmpk_ctx_create": (_int, [ctypes.POINTER(_vp), _int]),
    "lmpk_ctx_destroy": (_int, [_vp]),
    "lmpk_ctx_launch_count": (_i64, [_vp]),
    "lmpk_ctx_check": (_int, [_vp, _vp]),
    "lmpk_ctx_set_epoch": (_i64, [_vp, _i64]),
    "lmpk_csr_window": (_int, [_vp, _i32, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp, ctypes.POINTER(_i64), _vp]),
    "lmpk_vec_scale": (_int, [_vp, _i64, _vp, ctypes.c_double, ctypes.c_double, _int, _vp, _vp]),
    "lmpk_ctx_profile": (_int, [_vp, _vp, _int]),
    "lmpk_ctx_trace": (_int, [_vp, _vp, _i64]),
    "lmpk_spmv_rows": (_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _i32, _i32, _int, _vp]),
    "lmpk_mpk_baseline": (_int, [_vp, _i32, _vp, _vp, _vp, _vp, _i64, _i32, _int, _vp]),
    "lmpk_tiling_create": (_int, [_vp, _i32, _vp, _vp, _vp, _i32, ctypes.POINTER(TilingParams),
                                  ctypes.POINTER(_vp), ctypes.POINTER(TilingInfo), _vp]),
    "lmpk_tiling_destroy": (_int, [_vp]),
    "lmpk_tiling_geometry": (_int, [_vp, _vp, _vp, _vp]),
    "lmpk_mpk_run": (_int, [_vp, _vp, _vp, _i64, _i32, ctypes.POINTER(PowerCfg), _vp, _int,
                            _int, _vp]),
    "lmpk_mpk_crs_run": (_int, [_vp, _i32, _vp, _vp, _vp, _vp, _i64, _i32, ctypes.POINTER(PowerCfg), _vp,
                                _int, _int, _vp]),
    "lmpk_bfs_levels": (_int, [_vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp, _i64p, _vp]),
    "lmpk_symmetrized_pattern": (_int, [_vp, _i32, _vp, _vp, ctypes.POINTER(_int), _i64p,
                                        _vp, _vp, _i64, _vp]),
    "lmpk_csr_from_triplets": (_int, [_vp, _i32, _i64, _vp, _vp, _vp, _int, _vp, _vp, _vp, _vp, _vp]),
    "lmpk_permute_symmetric": (_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lmpk_permute_vectors": (_int, [_vp, _i32, _vp, _vp, _i64, _vp, _i64, _i32, _i32, _int, _vp]),
    "lmpk_level_nnz": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "lmpk_segment_col_range": (_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "lmpk_tiling_items": (_int, [_vp, _vp, _i64, _i64p]),
    # include/lmpk_plan.h
    "lmpk_level_nnz_perm": (_int, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "lmpk_refine_span": (_int, [_vp, _i32, _vp, _int, _vp, _vp, _i32, _i32, _vp, _i64p, _vp]),
    "lmpk_halo_seed": (_int, [_vp, _i32, _vp, _i64, _vp, _vp, _vp]),
    "lmpk_halo_level_sort": (_int, [_vp, _i32, _vp, _int, _vp, _vp, _vp, _i32, _i32, _vp, _vp]),
    "lmpk_invert_perm": (_int, [_vp, _i32, _vp, _vp, _vp]),
    "lmpk_item_deps": (_int, [_vp, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp, ctypes.POINTER(_vp), _vp]),
    "lmpk_host_free": (None, [_vp]),
    "lmpk_item_col_max_in_range": (_int, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "lmpk_simulate_traffic": (_int, [_i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                     _int, _vp]),
}

_lib = None
_lock = threading.Lock()


def load_library(path=None):
    """Load liblmpk.so and attach the signatures; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = pathlib.Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"liblmpk.so not found at {p}: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.lmpk_abi_version() != 1:
            raise RuntimeError("liblmpk ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def check(rc, what=""):
    """Map a status code to the reference's exception types."""
    if rc == LMPK_OK:
        return
    msg = load_library().lmpk_last_error()
    msg = msg.decode() if msg else ""
    text = f"{what}: {msg}" if what else msg
    if rc == LMPK_ERR_ARG:
        raise ValueError(text)
    raise RuntimeError(text)


def _require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the cuda backend needs a CUDA device (no CPU fallback)")
    return torch


class Context:
    """Owns one lmpk_ctx (per-device scratch, epoch counters, queue word)."""

    def __init__(self, device=None):
        torch = _require_cuda()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.lib = load_library()
        h = _vp()
        with torch.cuda.device(self.device):
            check(self.lib.lmpk_ctx_create(ctypes.byref(h), self.device), "lmpk_ctx_create")
        self.handle = h
        vals = [_int() for _ in range(6)]
        check(self.lib.lmpk_device_info(self.device, *[ctypes.byref(v) for v in vals]))
        (self.sm_count, self.max_smem_block, self.max_smem_sm, self.l2_bytes,
         self.cc_major, self.cc_minor) = (v.value for v in vals)

    def launches(self) -> int:
        return int(self.lib.lmpk_ctx_launch_count(self.handle))

    def close(self):
        if self.handle:
            self.lib.lmpk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass


_ctxs: dict = {}


def context(device=None) -> Context:
    torch = _require_cuda()
    dev = torch.cuda.current_device() if device is None else int(device)
    c = _ctxs.get(dev)
    if c is None:
        c = Context(dev)
        _ctxs[dev] = c
    return c


def stream_handle(stream=None):
    """cudaStream_t of `stream` (default: torch's current stream of the current
    device).  The raw-stream query costs ~0.3 us against ~7 us for building a
    torch.cuda.Stream object -- five of these were 15% of a cfg1 run_plan call."""
    import torch

    if stream is None:
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        if raw is not None:
            return _vp(raw(torch.cuda.current_device()))
        stream = torch.cuda.current_stream()
    return _vp(stream.cuda_stream)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    return _vp(0) if t is None else _vp(t.data_ptr())
