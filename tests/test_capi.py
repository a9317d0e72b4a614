"""The C-ABI boundary (include/lmpk.h) without a GPU: the shared library
loads, exports every declared entry point with the declared layout, and
fails loudly (no CPU fallback) when no device is present."""

import ctypes
import pathlib
import re
import subprocess

import pytest

from paper_2205_01598_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADERS = sorted((ROOT / "include").glob("*.h"))  # lmpk.h, lmpk_plan.h


def declared_functions():
    names = set()
    for header in HEADERS:
        text = re.sub(r"/\*.*?\*/", "", header.read_text(), flags=re.S)
        names |= set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(lmpk_\w+)\s*\(", text, re.M))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    names = declared_functions()
    assert len(names) >= 34
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.lmpk_abi_version() == 1


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "lmpk.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(lmpk_tiling_info), offsetof(lmpk_tiling_info, nnz),
         sizeof(lmpk_tiling_params), sizeof(lmpk_power_cfg), offsetof(lmpk_power_cfg, acc_coef_re),
         offsetof(lmpk_tiling_info, block_bytes));
  return 0;
}''')
    exe = tmp_path / "layout"
    subprocess.run(["/usr/bin/gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.TilingInfo), _lib.TilingInfo.nnz.offset,
            ctypes.sizeof(_lib.TilingParams), ctypes.sizeof(_lib.PowerCfg),
            _lib.PowerCfg.acc_coef_re.offset, _lib.TilingInfo.block_bytes.offset]
    assert got == want


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    lib = _lib.load_library()
    h = ctypes.c_void_p()
    rc = lib.lmpk_ctx_create(ctypes.byref(h), 0)
    assert rc != 0 and not h.value
    assert lib.lmpk_last_error()
    with pytest.raises(RuntimeError):
        _lib.context()


def test_kernels_compiled_for_sm100a():
    so = ROOT / "paper_2205_01598_b200" / "_lib" / "liblmpk.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
