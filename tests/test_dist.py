"""Multi-GPU level-range sharding: partition, window
extraction, halo exchange and the bitwise single-rank equivalence.

CPU tests run the sharded logic with the oracle as the local window MPK
(test-only) -- sequentially, and across a real world_size=2 gloo group.  The
gpu test runs every shard's window through the CUDA kernel in one process
(the shards never wait on each other, so this is not a multi-rank stand-in)."""

import os
import pathlib
import socket

import numpy as np
import pytest

from oracle import levelmpk_oracle as O
from paper_2205_01598_b200.dist import DistMpk, LevelShards, window_csr


def _level_permuted(n=12, order=2):
    rp, col, val = O.gen_stencil_3d(n, order)
    perm, level_ptr = O.bfs_levels(rp, col, 0)
    prp, pcol, pval = O.permute_symmetric(rp, col, val, perm)
    level_ptr = np.asarray(level_ptr, dtype=np.int64)
    level_nnz = prp[level_ptr[1:]].astype(np.int64) - prp[level_ptr[:-1]]
    return prp, pcol, pval, level_ptr, level_nnz


def _oracle_local(k):
    """Window MPK by the oracle (in place on a torch [k+1, n_win] tensor)."""

    def run(y, rp, col, val, check_errors=True):
        out = O.mpk_powers(rp, col, val, y[0].cpu().numpy(), k)
        y.copy_(__import__("torch").from_numpy(out))
        return y

    return run


@pytest.mark.parametrize("world,k", [(1, 4), (2, 4), (3, 3), (4, 4), (5, 2)])
def test_partition_properties(world, k):
    prp, pcol, pval, lp, lnnz = _level_permuted(12)
    sh = LevelShards(lp, lnnz, world, k)
    n = prp.shape[0] - 1
    assert sh.shards[0].own_lo == 0 and sh.shards[-1].own_hi == n
    for g, s in enumerate(sh.shards):
        assert s.level_hi - s.level_lo >= (k if world > 1 else 1)
        assert s.win_lo <= s.own_lo < s.own_hi <= s.win_hi
        if g > 0:
            assert s.own_lo == sh.shards[g - 1].own_hi
            # my left halo lies inside my left neighbour's owned rows
            assert s.win_lo >= sh.shards[g - 1].own_lo
        if g < world - 1:
            assert s.win_hi <= sh.shards[g + 1].own_hi
    total = int(lnnz.sum())
    owned = [sh.owned_nnz(g) for g in range(world)]
    assert sum(owned) == total
    if world > 1:
        # nnz balance within one (widest) level plus the >= k constraint slack
        assert max(owned) - min(owned) <= int(lnnz.max()) * (k + 1)
    assert sh.redundant_flops() >= 0


def test_too_few_levels_rejected():
    prp, pcol, pval, lp, lnnz = _level_permuted(6)
    with pytest.raises(ValueError, match="levels"):
        LevelShards(lp, lnnz, 8, 4)


def test_window_csr_matches_dense_slice():
    prp, pcol, pval, lp, lnnz = _level_permuted(8)
    n = prp.shape[0] - 1
    dense = np.zeros((n, n))
    for r in range(n):
        dense[r, pcol[prp[r]:prp[r + 1]]] = pval[prp[r]:prp[r + 1]]
    lo, hi = int(lp[5]), int(lp[14])
    rp, c, v = window_csr(prp, pcol, pval, lo, hi)
    w = np.zeros((hi - lo, hi - lo))
    for r in range(hi - lo):
        w[r, c[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    assert np.array_equal(w, dense[lo:hi, lo:hi])
    assert np.all(np.diff(rp) >= 0)
    for r in range(hi - lo):  # per-row order kept
        assert np.all(np.diff(c[rp[r]:rp[r + 1]]) > 0)


@pytest.mark.parametrize("world,k", [(2, 4), (3, 4), (4, 3)])
def test_sharded_windows_bitwise_equal_global(world, k):
    """Every shard's window MPK reproduces the global powers on its owned rows."""
    prp, pcol, pval, lp, lnnz = _level_permuted(12)
    n = prp.shape[0] - 1
    x = np.random.default_rng(7).uniform(-1, 1, n)
    ref = O.mpk_powers(prp, pcol, pval, x, k)
    sh = LevelShards(lp, lnnz, world, k)
    got = np.empty_like(ref)
    for s in sh.shards:
        rp, c, v = window_csr(prp, pcol, pval, s.win_lo, s.win_hi)
        yw = O.mpk_powers(rp, c, v, x[s.win_lo:s.win_hi], k)
        got[:, s.own_lo:s.own_hi] = yw[:, s.own_offset:s.own_offset + s.n_own]
    assert np.array_equal(got, ref)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, k, out_dir):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prp, pcol, pval, lp, lnnz = _level_permuted(12)
        n = prp.shape[0] - 1
        x = np.random.default_rng(11).uniform(-1, 1, n)
        sh = LevelShards(lp, lnnz, world, k)
        s = sh[rank]
        rp, c, v = window_csr(prp, pcol, pval, s.win_lo, s.win_hi)
        oracle = _oracle_local(k)
        dm = DistMpk(prp, pcol, pval, lp, lnnz, k, rank, world,
                     local=lambda y, check_errors=True: oracle(y, rp, c, v))
        # halo rows must come from the neighbours, not from a local copy of x
        y_own = dm.run(torch.from_numpy(x[s.own_lo:s.own_hi].copy()))
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), y_own.numpy())
        np.save(os.path.join(out_dir, f"halo{rank}.npy"), dm.y[0].numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange_and_mpk(tmp_path, world):
    import torch.multiprocessing as mp

    k = 4
    port = _free_port()
    mp.start_processes(_gloo_worker, args=(world, port, k, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    prp, pcol, pval, lp, lnnz = _level_permuted(12)
    n = prp.shape[0] - 1
    x = np.random.default_rng(11).uniform(-1, 1, n)
    ref = O.mpk_powers(prp, pcol, pval, x, k)
    sh = LevelShards(lp, lnnz, world, k)
    for g, s in enumerate(sh.shards):
        got = np.load(tmp_path / f"rank{g}.npy")
        assert np.array_equal(got, ref[:, s.own_lo:s.own_hi]), g
        halo = np.load(tmp_path / f"halo{g}.npy")
        assert np.array_equal(halo, x[s.win_lo:s.win_hi]), g


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_gpu_shard_windows_bitwise_equal_single_gpu(world):
    """Each shard's window through the CUDA kernel == the single-GPU MPK."""
    import torch

    from paper_2205_01598_b200 import kernels as K
    from paper_2205_01598_b200.dist import CudaWindowMpk

    k = 4
    prp, pcol, pval, lp, lnnz = _level_permuted(24)
    n = prp.shape[0] - 1
    x = np.random.default_rng(5).uniform(-1, 1, n)
    a = K.DeviceCsr.from_host(prp, pcol, pval)
    t = K.Tiling(a, k, tile_nnz=2000)
    y = torch.zeros((k + 1, n), dtype=torch.float64, device="cuda")
    y[0] = torch.from_numpy(x)
    K.mpk_run(t, y, K.mpk_power_cfg(k))
    ref = y.cpu().numpy()
    assert np.array_equal(ref, O.mpk_powers(prp, pcol, pval, x, k))
    sh = LevelShards(lp, lnnz, world, k)
    for s in sh.shards:
        rp, c, v = window_csr(prp, pcol, pval, s.win_lo, s.win_hi)
        loc = CudaWindowMpk(rp, c, v, k, tile_nnz=1500)
        yw = torch.zeros((k + 1, s.n_win), dtype=torch.float64, device="cuda")
        yw[0] = torch.from_numpy(x[s.win_lo:s.win_hi].copy())
        loc(yw)
        got = yw[:, s.own_offset:s.own_offset + s.n_own].cpu().numpy()
        assert np.array_equal(got, ref[:, s.own_lo:s.own_hi])


def _cheb_window_batch(rp, c, v):
    """Test-only CPU restatement of one Chebyshev batch on a window (the GPU
    kernel's per-power semantics, oracle spmv), in place on the torch ring."""
    import torch

    def run(ring, acc, coeffs_c, k_base, pb, first):
        S = ring.shape[0]
        cplx = ring.is_complex()
        R = ring.numpy()
        A = acc.numpy()
        for p in range(1, pb + 1):
            k = k_base + p
            tin, tprev = R[(k - 1) % S], R[(k - 2) % S]
            if cplx:
                tr = O.spmv(rp, c, v, np.ascontiguousarray(tin.real))
                ti = O.spmv(rp, c, v, np.ascontiguousarray(tin.imag))
                if not (first and p == 1):
                    tr = 2.0 * tr - tprev.real
                    ti = 2.0 * ti - tprev.imag
                cr, ci = float(np.real(coeffs_c[k])), float(np.imag(coeffs_c[k]))
                ar = A.real + (cr * tr - ci * ti)
                ai = A.imag + (cr * ti + ci * tr)
                R[k % S] = tr + 1j * ti
                A[...] = ar + 1j * ai
            else:
                t = O.spmv(rp, c, v, np.ascontiguousarray(tin))
                if not (first and p == 1):
                    t = 2.0 * t - tprev
                R[k % S] = t
                A[...] = A + float(np.real(coeffs_c[k])) * t
        return ring

    return run


def _gloo_cheb_worker(rank, world, port, p_b, cplx, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2205_01598_b200.dist import DistCheb, window_csr

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        prp, pcol, pval, lp, lnnz = _level_permuted(12)
        n = prp.shape[0] - 1
        rng = np.random.default_rng(17)
        coeffs = rng.uniform(-1, 1, 11) + (1j * rng.uniform(-1, 1, 11) if cplx else 0)
        x = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cplx else 0)
        sh = LevelShards(lp, lnnz, world, p_b)
        s = sh[rank]
        rp, c, v = window_csr(prp, pcol, pval, s.win_lo, s.win_hi)
        dc = DistCheb(prp, pcol, pval, lp, lnnz, coeffs, p_b, rank, world, local=_cheb_window_batch(rp, c, v))
        out = dc.step(torch.from_numpy(np.asarray(x[s.own_lo:s.own_hi])))
        np.save(os.path.join(out_dir, f"cheb{rank}.npy"), out.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p_b,cplx", [(2, 4, True), (3, 3, False), (2, 3, True)])
def test_gloo_sharded_chebyshev_bitwise(tmp_path, world, p_b, cplx):
    """Config-5 shape on CPU ranks: sharded Chebyshev propagation (halo of the
    two newest states exchanged per batch) equals the single-rank oracle."""
    import torch.multiprocessing as mp

    port = _free_port()
    mp.start_processes(_gloo_cheb_worker, args=(world, port, p_b, cplx, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    prp, pcol, pval, lp, lnnz = _level_permuted(12)
    n = prp.shape[0] - 1
    rng = np.random.default_rng(17)
    coeffs = rng.uniform(-1, 1, 11) + (1j * rng.uniform(-1, 1, 11) if cplx else 0)
    x = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cplx else 0)
    ref = O.cheb_batches(prp, pcol, pval, x, np.real(coeffs), np.imag(coeffs) if cplx else None)
    sh = LevelShards(lp, lnnz, world, p_b)
    for g, s in enumerate(sh.shards):
        got = np.load(tmp_path / f"cheb{g}.npy")
        assert np.array_equal(got, ref[s.own_lo:s.own_hi]), g


@pytest.mark.gpu
@pytest.mark.parametrize("cplx,p_b", [(True, 4), (False, 3)])
def test_gpu_dist_cheb_window_runner_vs_oracle(cplx, p_b):
    """DistCheb's CUDA batch runner (world 1: the window is the whole matrix)
    against the oracle propagation, bitwise."""
    import torch

    from paper_2205_01598_b200.dist import DistCheb

    prp, pcol, pval, lp, lnnz = _level_permuted(20)
    n = prp.shape[0] - 1
    rng = np.random.default_rng(23)
    coeffs = rng.uniform(-1, 1, 13) + (1j * rng.uniform(-1, 1, 13) if cplx else 0)
    x = rng.uniform(-1, 1, n) + (1j * rng.uniform(-1, 1, n) if cplx else 0)
    dc = DistCheb(prp, pcol, pval, lp, lnnz, coeffs, p_b, 0, 1, device="cuda")
    got = dc.step(torch.from_numpy(np.asarray(x)).cuda()).cpu().numpy()
    ref = O.cheb_batches(prp, pcol, pval, x, np.real(coeffs), np.imag(coeffs) if cplx else None)
    assert np.array_equal(got, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_device_windows_match_host_windows(world):
    """lmpk_csr_window (the window cut in HBM that bench.py's ranks use) is
    bitwise the host window_csr; DistMpk built from the device matrix
    computes the owned rows bitwise like the single-GPU MPK."""
    import torch

    from paper_2205_01598_b200 import kernels as K
    from paper_2205_01598_b200.dist import CudaWindowMpk, _window

    k = 3
    prp, pcol, pval, lp, lnnz = _level_permuted(20)
    n = prp.shape[0] - 1
    a = K.DeviceCsr.from_host(prp, pcol, pval)
    x = np.random.default_rng(8).uniform(-1, 1, n)
    ref = O.mpk_powers(prp, pcol, pval, x, k)
    sh = LevelShards(lp, lnnz, world, k)
    for s in sh.shards:
        rp, c, v = window_csr(prp, pcol, pval, s.win_lo, s.win_hi)
        d = _window(a, None, None, s.win_lo, s.win_hi)
        assert d.n == s.n_win
        assert np.array_equal(d.row_ptr.cpu().numpy(), rp) and np.array_equal(d.col.cpu().numpy(), c)
        assert np.array_equal(d.val.cpu().numpy(), v)
        loc = CudaWindowMpk(d, None, None, k)
        yw = torch.zeros((k + 1, s.n_win), dtype=torch.float64, device="cuda")
        yw[0] = torch.from_numpy(x[s.win_lo:s.win_hi].copy())  # the exchanged halo
        loc(yw)
        got = yw[:, s.own_offset:s.own_offset + s.n_own].cpu().numpy()
        assert np.array_equal(got, ref[:, s.own_lo:s.own_hi])


def test_bench_self_launch_command(monkeypatch):
    """bench.py --gpus N without WORLD_SIZE re-launches itself with one rank
    per GPU under torch.distributed.run on 127.0.0.1 (NCCL init logging on)."""
    import importlib
    import subprocess
    import sys

    sys.path.insert(0, str(pathlib.Path(__file__).resolve().parent.parent))
    bench = importlib.import_module("bench")
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3", "--config", "cfg2"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "3", "--config", "cfg2"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
