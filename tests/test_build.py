"""Device CRS build from COO triplets (lmpk_csr_from_triplets) against the
reference's canonicalisation (pkg/src/levelmpk/csr.py:72-94), bit for bit.
Mirrors pkg/tests/test_csr.py's from_triplets cases (duplicates summed,
range errors) and adds segments long enough to reach numpy's pairwise
summation branches."""

import numpy as np
import pytest

from oracle import levelmpk_oracle as O


# ---------------------------------------------------------------- CPU: the model the kernel mirrors
@pytest.mark.parametrize("seed", range(6))
def test_segment_sum_model_matches_numpy_reduceat(seed):
    rng = np.random.default_rng(seed)
    for length in list(range(1, 20)) + [31, 64, 127, 128, 129, 130, 200, 257, 300, 1000, 2049]:
        seg = rng.standard_normal(length) * 10.0 ** rng.integers(-8, 9, size=length)
        got = O.segment_sum_model(seg)
        want = float(np.add.reduceat(seg, [0])[0])
        assert np.float64(got).tobytes() == np.float64(want).tobytes(), length


def test_segment_sum_model_signed_zero():
    for seg in ([-0.0], [-0.0, -0.0], [0.0, -0.0], [-0.0] * 9, [-0.0] * 130):
        got = O.segment_sum_model(np.array(seg))
        want = float(np.add.reduceat(np.array(seg), [0])[0])
        assert np.float64(got).tobytes() == np.float64(want).tobytes()


# ---------------------------------------------------------------- GPU parity
def _triplets(seed, n, m, dup_rate):
    rng = np.random.default_rng(seed)
    rows = rng.integers(0, n, size=m)
    cols = rng.integers(0, n, size=m)
    nd = int(m * dup_rate)
    if nd:
        src = rng.integers(0, m, size=nd)
        dst = rng.integers(0, m, size=nd)
        rows[dst] = rows[src]
        cols[dst] = cols[src]
    vals = rng.standard_normal(m) * 10.0 ** rng.integers(-6, 7, size=m)
    return rows, cols, vals


def _device_build(n, rows, cols, vals, sum_duplicates=True):
    import torch

    from paper_2205_01598_b200 import kernels as K

    d = K.csr_from_triplets(n, torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda(),
                            torch.from_numpy(vals).cuda(), sum_duplicates=sum_duplicates)
    return d.to_host()


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n,m,dup", [(0, 1, 1, 0.0), (1, 5, 40, 0.5), (2, 1000, 20000, 0.3),
                                          (3, 70000, 300000, 0.1), (4, 3, 5000, 0.0),
                                          (5, 200000, 2000000, 0.05)])
def test_from_triplets_bitwise(seed, n, m, dup):
    rows, cols, vals = _triplets(seed, n, m, dup)
    rp, col, val = _device_build(n, rows, cols, vals)
    erp, ecol, ev = O.from_triplets(n, rows, cols, vals)
    assert np.array_equal(rp.astype(np.int64), erp)
    assert np.array_equal(col.astype(np.int64), ecol)
    assert val.tobytes() == ev.tobytes()


@pytest.mark.gpu
def test_from_triplets_long_duplicate_runs():
    # one (row, col) repeated 1000x (pairwise recursion), one 130x, one 9x
    rng = np.random.default_rng(7)
    rows = np.concatenate([np.full(1000, 2), np.full(130, 0), np.full(9, 1), rng.integers(0, 4, 50)])
    cols = np.concatenate([np.full(1000, 3), np.full(130, 1), np.full(9, 0), rng.integers(0, 4, 50)])
    perm = rng.permutation(rows.size)
    rows, cols = rows[perm], cols[perm]
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.integers(-8, 9, size=rows.size)
    rp, col, val = _device_build(4, rows, cols, vals)
    erp, ecol, ev = O.from_triplets(4, rows, cols, vals)
    assert np.array_equal(rp.astype(np.int64), erp) and np.array_equal(col.astype(np.int64), ecol)
    assert val.tobytes() == ev.tobytes()


@pytest.mark.gpu
def test_from_triplets_stencil_matches_host_build():
    import paper_2205_01598_b200 as lm

    a = lm.gen_stencil_3d(24, 2)
    r, c, v = a.to_triplets()
    rng = np.random.default_rng(3)
    p = rng.permutation(r.size)
    rp, col, val = _device_build(a.n_rows, r[p].astype(np.int64), c[p].astype(np.int64), v[p])
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(col, a.col)
    assert val.tobytes() == a.val.tobytes()


@pytest.mark.gpu
def test_from_triplets_no_sum_and_empty():
    rows = np.array([1, 0, 1, 1], dtype=np.int64)
    cols = np.array([0, 1, 0, 2], dtype=np.int64)
    vals = np.array([1.0, 2.0, 3.0, 4.0])
    rp, col, val = _device_build(3, rows, cols, vals, sum_duplicates=False)
    erp, ecol, ev = O.from_triplets(3, rows, cols, vals, sum_duplicates=False)
    assert np.array_equal(rp.astype(np.int64), erp) and np.array_equal(col.astype(np.int64), ecol)
    assert val.tobytes() == ev.tobytes()
    e = np.zeros(0, dtype=np.int64)
    rp, col, val = _device_build(3, e, e, np.zeros(0))
    assert rp.tolist() == [0, 0, 0, 0] and col.size == 0 and val.size == 0


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols,msg", [([0, 3], [0, 0], "row index out of range"),
                                           ([0, -1], [0, 0], "row index out of range"),
                                           ([0, 1], [0, 5], "column index out of range")])
def test_from_triplets_range_errors(rows, cols, msg):
    with pytest.raises(ValueError, match=msg):
        _device_build(3, np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), np.ones(2))


@pytest.mark.gpu
def test_csrmatrix_from_triplets_device_tensors():
    import torch

    import paper_2205_01598_b200 as lm

    rows, cols, vals = _triplets(11, 500, 5000, 0.2)
    host = lm.CsrMatrix.from_triplets(500, rows, cols, vals)
    dev = lm.CsrMatrix.from_triplets(500, torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda(),
                                     torch.from_numpy(vals).cuda())
    assert np.array_equal(dev.row_ptr, host.row_ptr) and np.array_equal(dev.col, host.col)
    assert dev.val.tobytes() == host.val.tobytes()
    with pytest.raises(ValueError, match="strictly increasing"):
        lm.CsrMatrix.from_triplets(3, torch.tensor([0, 0]).cuda(), torch.tensor([1, 1]).cuda(),
                                   torch.tensor([1.0, 2.0], dtype=torch.float64).cuda(), sum_duplicates=False)


@pytest.mark.gpu
# 32: one thread sorts each row; 33 and 4096: one CTA per row (bitonic);
# 4097 and 5000: the two full radix passes
@pytest.mark.parametrize("row_len", [32, 33, 4096, 4097, 5000])
def test_from_triplets_short_row_boundary(row_len):
    rng = np.random.default_rng(row_len)
    n = 64
    rows = np.repeat(np.arange(n), row_len)
    cols = rng.integers(0, min(n, max(8, row_len // 4)), size=rows.size)  # many duplicates per row
    p = rng.permutation(rows.size)
    rows, cols = rows[p].astype(np.int64), cols[p].astype(np.int64)
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.integers(-8, 9, size=rows.size)
    rows[:3] = 5  # an uneven row next to the full ones
    rp, col, val = _device_build(n, rows, cols, vals)
    erp, ecol, ev = O.from_triplets(n, rows, cols, vals)
    assert np.array_equal(rp.astype(np.int64), erp) and np.array_equal(col.astype(np.int64), ecol)
    assert val.tobytes() == ev.tobytes()


@pytest.mark.gpu
def test_load_matrix_market_device_build(tmp_path):
    import paper_2205_01598_b200 as lm

    p = tmp_path / "s.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real symmetric\n4 4 6\n"
                 "1 1 2.5\n2 1 -1e-17\n2 1 1.0\n3 3 4\n4 2 0.125\n4 4 1e16\n")
    host = lm.load_matrix_market(p)
    dev = lm.load_matrix_market(p, device=True)
    assert np.array_equal(dev.row_ptr, host.row_ptr) and np.array_equal(dev.col, host.col)
    assert dev.val.tobytes() == host.val.tobytes()


@pytest.mark.gpu
def test_gen_stencil_3d_device_build():
    import paper_2205_01598_b200 as lm

    host = lm.gen_stencil_3d(20, 4)
    dev = lm.gen_stencil_3d(20, 4, device=True)
    assert dev.n_nz == host.n_nz == lm.stencil_3d_nnz(20, 4)
    assert np.array_equal(dev.row_ptr, host.row_ptr) and np.array_equal(dev.col, host.col)
    assert dev.val.tobytes() == host.val.tobytes()
