// spmv.cu -- bit-exact row-range SpMV and the baseline k x SpMV MPK.
//
// Replaces the reference's numba row kernel (pkg/src/levelmpk/csr.py:195-201)
// and the barrier-separated baseline sweeps (executor.py:233-266).
//
// Design (sm_100a): a persistent grid walks nnz-balanced row tiles.  Each
// tile's col/val slice is staged into shared memory by a 1-D TMA bulk copy
// (cp.async.bulk, mbarrier completion), double-buffered so the next tile's
// copy overlaps the current tile's gathers.  One thread owns one row and sums
// it in storage order with unfused multiply/add -> bitwise equal to numba.
#include <algorithm>

#include "lmpk_internal.cuh"

namespace lmpk {

struct SpmvArgs {
  const int32_t* row_ptr;
  const int32_t* col;
  const double* val;
  const double* x;
  double* out;
  int32_t r0, r1;  // row range [r0, r1)
  int64_t nz_base; // row_ptr[r0]
  int64_t nnz;     // row_ptr[r1] - row_ptr[r0]
  int32_t tile_nnz;
  int32_t cap;     // smem capacity (elements) per buffer
  int32_t n_tiles;
  int32_t use_tma;
};

__device__ __forceinline__ int32_t lower_bound_rows(const int32_t* row_ptr, int32_t lo, int32_t hi,
                                                    int64_t target) {
  // first r in [lo, hi] with row_ptr[r] >= target (hi if none)
  while (lo < hi) {
    int32_t mid = lo + ((hi - lo) >> 1);
    if (static_cast<int64_t>(__ldg(row_ptr + mid)) < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void tile_rows(const SpmvArgs& a, int32_t t, int32_t& rs, int32_t& re) {
  rs = (t == 0) ? a.r0
                : lower_bound_rows(a.row_ptr, a.r0, a.r1, a.nz_base + int64_t(t) * a.tile_nnz);
  re = (t == a.n_tiles - 1)
           ? a.r1
           : lower_bound_rows(a.row_ptr, a.r0, a.r1, a.nz_base + int64_t(t + 1) * a.tile_nnz);
}

struct TileBuf {
  int32_t* col;
  double* val;
  uint64_t* bar;
};

// Stage elements [nz0, nz1) of col/val into buffer b.  TMA moves the 16-byte
// aligned interior, threads fill the ragged edges.  Returns false (nothing
// staged) when the tile exceeds the buffer capacity.
__device__ __forceinline__ bool stage_tile(const SpmvArgs& a, const TileBuf& b, int64_t nz0,
                                           int64_t nz1, uint64_t policy) {
  if (nz1 - nz0 > a.cap) {  // oversized tile: computed from global memory
    if (threadIdx.x == 0) mbar_arrive_expect_tx(b.bar, 0);  // keep one phase per use
    return false;
  }
  const int64_t ca0 = nz0 & ~int64_t(3), ci0 = (nz0 + 3) & ~int64_t(3), ci1 = nz1 & ~int64_t(3);
  const int64_t va0 = nz0 & ~int64_t(1), vi0 = (nz0 + 1) & ~int64_t(1), vi1 = nz1 & ~int64_t(1);
  const bool col_int = a.use_tma && ci1 > ci0;
  const bool val_int = a.use_tma && vi1 > vi0;
  if (threadIdx.x == 0) {
    uint32_t bytes = (col_int ? uint32_t(ci1 - ci0) * 4u : 0u) + (val_int ? uint32_t(vi1 - vi0) * 8u : 0u);
    mbar_arrive_expect_tx(b.bar, bytes);
    if (col_int) bulk_g2s(b.col + (ci0 - ca0), a.col + ci0, uint32_t(ci1 - ci0) * 4u, b.bar, policy);
    if (val_int) bulk_g2s(b.val + (vi0 - va0), a.val + vi0, uint32_t(vi1 - vi0) * 8u, b.bar, policy);
  }
  // ragged edges (or everything when TMA is off)
  if (col_int) {
    for (int64_t e = nz0 + threadIdx.x; e < ci0; e += blockDim.x) b.col[e - ca0] = __ldg(a.col + e);
    for (int64_t e = ci1 + threadIdx.x; e < nz1; e += blockDim.x) b.col[e - ca0] = __ldg(a.col + e);
  } else {
    for (int64_t e = nz0 + threadIdx.x; e < nz1; e += blockDim.x) b.col[e - ca0] = __ldg(a.col + e);
  }
  if (val_int) {
    for (int64_t e = nz0 + threadIdx.x; e < vi0; e += blockDim.x) b.val[e - va0] = __ldg(a.val + e);
    for (int64_t e = vi1 + threadIdx.x; e < nz1; e += blockDim.x) b.val[e - va0] = __ldg(a.val + e);
  } else {
    for (int64_t e = nz0 + threadIdx.x; e < nz1; e += blockDim.x) b.val[e - va0] = __ldg(a.val + e);
  }
  return true;
}

__global__ void __launch_bounds__(512, 2) spmv_tiles_kernel(SpmvArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bars[2];
  TileBuf buf[2];
  {
    const size_t col_bytes = ((size_t(a.cap) + 8) * 4 + 15) & ~size_t(15);
    const size_t val_bytes = ((size_t(a.cap) + 4) * 8 + 15) & ~size_t(15);
    const size_t per = ((col_bytes + val_bytes) + 127) & ~size_t(127);
    for (int i = 0; i < 2; ++i) {
      unsigned char* base = smem_raw + i * per;
      buf[i].val = reinterpret_cast<double*>(base);
      buf[i].col = reinterpret_cast<int32_t*>(base + val_bytes);
      buf[i].bar = &bars[i];
    }
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();

  int32_t t = blockIdx.x;
  if (t >= a.n_tiles) return;
  int32_t rs, re;
  tile_rows(a, t, rs, re);
  int64_t nz0 = __ldg(a.row_ptr + rs), nz1 = __ldg(a.row_ptr + re);
  bool staged = stage_tile(a, buf[0], nz0, nz1, pol);
  for (int it = 0;; ++it) {
    const int b = it & 1;
    const int32_t tn = t + gridDim.x;
    int32_t rsn = 0, ren = 0;
    int64_t nz0n = 0, nz1n = 0;
    bool staged_n = false;
    if (tn < a.n_tiles) {  // prefetch next tile into the other buffer
      tile_rows(a, tn, rsn, ren);
      nz0n = __ldg(a.row_ptr + rsn);
      nz1n = __ldg(a.row_ptr + ren);
      staged_n = stage_tile(a, buf[b ^ 1], nz0n, nz1n, pol);
    }
    mbar_wait(buf[b].bar, (it >> 1) & 1);
    __syncthreads();
    const int32_t* scol = buf[b].col - (nz0 & ~int64_t(3));
    const double* sval = buf[b].val - (nz0 & ~int64_t(1));
    for (int32_t r = rs + threadIdx.x; r < re; r += blockDim.x) {
      const int32_t k0 = __ldg(a.row_ptr + r), k1 = __ldg(a.row_ptr + r + 1);
      const double* x = a.x;
      double s;
      if (staged)
        s = row_sum_exact(scol + k0, sval + k0, k1 - k0, [x](int c) { return __ldg(x + c); });
      else
        s = row_sum_exact(a.col + k0, a.val + k0, k1 - k0, [x](int c) { return __ldg(x + c); });
      a.out[r] = s;
    }
    __syncthreads();
    if (tn >= a.n_tiles) break;
    t = tn;
    rs = rsn;
    re = ren;
    nz0 = nz0n;
    nz1 = nz1n;
    staged = staged_n;
  }
}

static int spmv_launch(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                       const double* val, const double* x, double* out, int32_t r0, int32_t r1,
                       int64_t nz_base, int64_t nnz, int flags, cudaStream_t st) {
  if (r1 <= r0) return LMPK_OK;
  const int threads = 512;
  const int64_t rows = r1 - r0;
  const double avg = rows > 0 ? double(nnz) / double(rows) : 1.0;
  // ~1 row per thread per tile; rows longer than the slack run from global
  int32_t tile = static_cast<int32_t>(std::min<double>(std::max<double>(avg * threads, 512.0), 4096.0));
  tile &= ~3;
  int32_t cap = tile + 256;
  const size_t col_bytes = ((size_t(cap) + 8) * 4 + 15) & ~size_t(15);
  const size_t val_bytes = ((size_t(cap) + 4) * 8 + 15) & ~size_t(15);
  const size_t per = ((col_bytes + val_bytes) + 127) & ~size_t(127);
  const size_t smem = 2 * per;
  static bool attr_set = false;
  if (!attr_set) {
    LMPK_CHECK_CUDA(cudaFuncSetAttribute(spmv_tiles_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr_set = true;
  }
  SpmvArgs a;
  a.row_ptr = row_ptr;
  a.col = col;
  a.val = val;
  a.x = x;
  a.out = out;
  a.r0 = r0;
  a.r1 = r1;
  a.nz_base = nz_base;
  a.nnz = nnz;
  a.tile_nnz = tile;
  a.cap = cap;
  a.n_tiles = static_cast<int32_t>(std::max<int64_t>(1, (nnz + tile - 1) / tile));
  a.use_tma = (flags & LMPK_FLAG_NO_TMA) ? 0 : 1;
  if ((reinterpret_cast<uintptr_t>(col) & 15) || (reinterpret_cast<uintptr_t>(val) & 15)) a.use_tma = 0;
  int occ = 0;
  LMPK_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmv_tiles_kernel, threads, smem));
  if (occ < 1) occ = 1;
  const int grid = static_cast<int>(std::min<int64_t>(a.n_tiles, int64_t(ctx->sm_count) * occ));
  spmv_tiles_kernel<<<grid, threads, smem, st>>>(a);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

}  // namespace lmpk

using namespace lmpk;

// row_ptr[r0] / row_ptr[r1] are needed on the host to size the tile grid.
static int read_rowptr_pair(const int32_t* row_ptr, int32_t r0, int32_t r1, int64_t* a, int64_t* b,
                            cudaStream_t st) {
  int32_t h[2];
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&h[0], row_ptr + r0, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&h[1], row_ptr + r1, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  *a = h[0];
  *b = h[1];
  return LMPK_OK;
}

extern "C" int lmpk_spmv_rows(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                              const double* val, const double* x, double* out, int32_t r0,
                              int32_t r1, int flags, void* stream) {
  LMPK_ARG_CHECK(ctx != nullptr, "lmpk_spmv_rows: ctx is NULL");
  LMPK_ARG_CHECK(n >= 0 && 0 <= r0 && r0 <= r1 && r1 <= n,
                 "row range [%d, %d) out of bounds for n=%d", r0, r1, n);
  LMPK_ARG_CHECK(x != out, "in_vec and out_vec must not alias");
  if (r1 == r0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  int64_t nz0, nz1;
  LMPK_TRY(read_rowptr_pair(row_ptr, r0, r1, &nz0, &nz1, st));
  return spmv_launch(ctx, n, row_ptr, col, val, x, out, r0, r1, nz0, nz1 - nz0, flags, st);
}

extern "C" int lmpk_mpk_baseline(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr,
                                 const int32_t* col, const double* val, double* y, int64_t ldy,
                                 int32_t p_m, int flags, void* stream) {
  LMPK_ARG_CHECK(ctx != nullptr, "lmpk_mpk_baseline: ctx is NULL");
  LMPK_ARG_CHECK(p_m >= 1, "p_m must be >= 1");
  LMPK_ARG_CHECK(ldy >= n, "ldy (%lld) must be >= n (%d)", (long long)ldy, n);
  if (n == 0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  int64_t nz0, nz1;
  LMPK_TRY(read_rowptr_pair(row_ptr, 0, n, &nz0, &nz1, st));
  for (int32_t p = 1; p <= p_m; ++p) {
    LMPK_TRY(spmv_launch(ctx, n, row_ptr, col, val, y + int64_t(p - 1) * ldy, y + int64_t(p) * ldy,
                         0, n, nz0, nz1 - nz0, flags, st));
  }
  return LMPK_OK;
}
