"""Multi-GPU level-range sharding: partition, window
extraction, halo exchange and the bitwise single-rank equivalence.

CPU tests run the sharded logic with the oracle as the local window MPK
(test-only) -- sequentially, and across a real world_size=2 gloo group.  The
gpu test runs every shard's window through the CUDA kernel in one process
(the shards never wait on each other, so this is not a multi-rank stand-in)."""

import os
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
