"""GPU parity of the hub-row paths of the CRS kernels (csrc/spmv.cu): rows of
more than 128 entries take a warp each, rows of more than 4096 entries a whole
CTA (producer warps + one adding thread over a shared-memory ring).  Both must
give the bits of the sequential storage-order sum of the reference row kernel
(pkg/src/levelmpk/csr.py:195-201, executor.py:127-135) at every row length
around the stage boundaries (128 / 896 entries per stage)."""

import numpy as np
import pytest

import paper_2205_01598_b200 as lm
from oracle import levelmpk_oracle as O
from paper_2205_01598_b200 import _lib
from paper_2205_01598_b200 import kernels as K

pytestmark = pytest.mark.gpu

LENGTHS = [129, 255, 256, 4096, 4097, 4100, 4096 + 895, 4096 + 896, 4096 + 897, 5 * 896 - 1, 5 * 896, 5 * 896 + 1,
           8 * 896 + 3, 20_001, 70_003]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    lm.warmup()


def _hub_matrix():
    """n = 80,000 rows: a tridiagonal background plus one hub row per length in
    LENGTHS (random columns, random values of mixed magnitude)."""
    n = 80_000
    rng = np.random.default_rng(21)
    i = np.arange(n)
    rows, cols = [i, i[:-1], i[1:]], [i, i[1:], i[:-1]]
    hubs = 1000 + 4000 * np.arange(len(LENGTHS))
    for h, ln in zip(hubs, LENGTHS):
        nb = rng.choice(n, ln, replace=False)
        rows.append(np.full(ln, h))
        cols.append(nb)
    r, c = np.concatenate(rows), np.concatenate(cols)
    v = rng.standard_normal(r.size) * 10.0 ** rng.integers(-6, 3, r.size)
    a = lm.CsrMatrix.from_triplets(n, r, c, v)
    lens = np.diff(a.row_ptr)
    assert lens.max() >= 70_003 and (lens > 4096).sum() >= 10
    return a


@pytest.fixture(scope="module")
def hub_matrix():
    return _hub_matrix()


def test_hub_spmv_rows_bitwise(hub_matrix):
    import torch

    a = hub_matrix
    x = np.random.default_rng(1).uniform(-1, 1, a.n_rows)
    ref = O.spmv(a.row_ptr, a.col, a.val, x)
    d = a.device()
    xd = torch.from_numpy(x).cuda()
    out = torch.zeros(a.n_rows, dtype=torch.float64, device="cuda")
    K.spmv_rows(d, xd, out, 0, a.n_rows)
    assert np.array_equal(out.cpu().numpy(), ref)
    # a row range that cuts the hub list
    out.zero_()
    K.spmv_rows(d, xd, out, 4_000, 42_000)
    got = out.cpu().numpy()
    assert np.array_equal(got[4_000:42_000], ref[4_000:42_000]) and not got[:4_000].any() and not got[42_000:].any()


def test_hub_baseline_powers_bitwise(hub_matrix):
    import torch

    a = hub_matrix
    k = 3
    x = np.random.default_rng(2).uniform(-1, 1, a.n_rows) * 1e-3
    ref = O.mpk_powers(a.row_ptr, a.col, a.val, x, k)
    y = torch.zeros((k + 1, a.n_rows), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_baseline(a.device(), y, k)
    assert np.array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("cplx", [False, True])
def test_hub_crs_run_cheb_bitwise(hub_matrix, cplx):
    """lmpk_mpk_crs_run (Chebyshev kernel + accumulation, real and complex)
    against the oracle's cheb_batches on the same matrix."""
    import torch

    a = hub_matrix
    n, k = a.n_rows, 4
    rng = np.random.default_rng(5)
    s = 1.0 / np.abs(a.val).sum() * a.n_rows  # keep the recurrence bounded
    b = lm.CsrMatrix(n, a.row_ptr, a.col, a.val * s)
    cr, ci = rng.standard_normal(k + 1), rng.standard_normal(k + 1)
    x = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cplx else 0)
    p = np.arange(1, k + 1)
    kern = np.where(p == 1, _lib.KERNEL_SPMV, _lib.KERNEL_CHEB)
    cfg = K.power_cfg(k, p, p - 1, np.maximum(p - 2, 0), kern, cr[1:], ci[1:] if cplx else None)
    if cplx:
        y = torch.zeros((k + 1, n), dtype=torch.complex128, device="cuda")
        y[0] = torch.from_numpy(x)
        acc = torch.from_numpy(cr[0] * x.real - ci[0] * x.imag + 1j * (cr[0] * x.imag + ci[0] * x.real)).cuda()
        K.mpk_crs_run(b.device(), torch.view_as_real(y).reshape(k + 1, -1), cfg,
                      acc=torch.view_as_real(acc).reshape(-1), use_acc=True, complex_state=True)
        ref = O.cheb_batches(b.row_ptr, b.col, b.val, x, cr, ci)
    else:
        y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
        y[0] = torch.from_numpy(x)
        acc = torch.from_numpy(cr[0] * x).cuda()
        K.mpk_crs_run(b.device(), y, cfg, acc=acc, use_acc=True)
        ref = O.cheb_batches(b.row_ptr, b.col, b.val, x, cr)
    assert np.array_equal(acc.cpu().numpy(), ref)


@pytest.mark.parametrize("lo,hi", [(20, 31), (10, 128), (90, 128)])
def test_stream_rows_bitwise(lo, hi):
    """Medium rows without hubs (10..128 entries, empty rows in between): the
    row-per-thread kernel on full and partial row ranges and as k x SpMV."""
    import torch

    n = 20_011
    rng = np.random.default_rng(lo * 1000 + hi)
    lens = rng.integers(lo, hi + 1, n)
    lens[::97] = 0  # empty rows
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rp[1:])
    col = np.concatenate([np.sort(rng.choice(n, int(k), replace=False)) for k in lens if k]).astype(np.int32)
    val = rng.standard_normal(col.size) * 10.0 ** rng.integers(-5, 3, col.size)
    a = lm.CsrMatrix(n, rp.astype(np.int32), col, val)
    x = rng.uniform(-1, 1, n)
    ref = O.spmv(a.row_ptr, a.col, a.val, x)
    d = a.device()
    xd = torch.from_numpy(x).cuda()
    out = torch.zeros(n, dtype=torch.float64, device="cuda")
    K.spmv_rows(d, xd, out, 0, n)
    assert np.array_equal(out.cpu().numpy(), ref)
    out.zero_()
    K.spmv_rows(d, xd, out, 77, 19_001)
    got = out.cpu().numpy()
    assert np.array_equal(got[77:19_001], ref[77:19_001]) and not got[:77].any() and not got[19_001:].any()
    k = 3
    s = 1.0 / np.abs(val).max() / hi
    b = lm.CsrMatrix(n, a.row_ptr, a.col, a.val * s)
    refp = O.mpk_powers(b.row_ptr, b.col, b.val, x, k)
    y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
    y[0] = xd
    K.mpk_baseline(b.device(), y, k)
    assert np.array_equal(y.cpu().numpy(), refp)
