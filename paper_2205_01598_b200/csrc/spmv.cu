// spmv.cu -- bit-exact row-range SpMV and the baseline k x SpMV MPK.
//
// Replaces the reference's numba row kernel (pkg/src/levelmpk/csr.py:195-201)
// and the barrier-separated baseline sweeps (executor.py:233-266): one thread
// per row sums it in storage order with unfused multiply/add -> bitwise equal
// to numba.  Each call is one asynchronous launch per sweep.
#include <algorithm>

#include "lmpk_internal.cuh"

namespace lmpk {

// One thread per row, grid-stride over [r0, r1).  No shared memory: the
// whole unified L1 caches the row's col/val lines (a warp's 32 consecutive
// rows share them across the 7-ish entry loads) and the gathered x lines.
// The matrix and x are immutable during a launch, so the .nc path is safe.
__global__ void __launch_bounds__(256) spmv_rows_kernel(const int32_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x, double* __restrict__ out,
                                                        int32_t r0, int32_t r1) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t r = r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < r1; r += stride) {
    const int32_t k0 = __ldg(row_ptr + r), k1 = __ldg(row_ptr + r + 1);
    out[r] = row_sum_exact(col + k0, val + k0, k1 - k0, [x](int c) { return __ldg(x + c); });
  }
}

static int spmv_launch(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col, const double* val,
                       const double* x, double* out, int32_t r0, int32_t r1, cudaStream_t st) {
  if (r1 <= r0) return LMPK_OK;
  const int threads = 256;
  const int64_t blocks = (int64_t(r1) - r0 + threads - 1) / threads;
  // enough CTAs for full occupancy (8 x 256 threads per SM), grid-stride beyond
  const int grid = static_cast<int>(std::min<int64_t>(blocks, int64_t(ctx->sm_count) * 8));
  spmv_rows_kernel<<<grid, threads, 0, st>>>(row_ptr, col, val, x, out, r0, r1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

}  // namespace lmpk

using namespace lmpk;

extern "C" int lmpk_spmv_rows(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                              const double* val, const double* x, double* out, int32_t r0,
                              int32_t r1, int flags, void* stream) {
  LMPK_ARG_CHECK(ctx != nullptr, "lmpk_spmv_rows: ctx is NULL");
  LMPK_ARG_CHECK(n >= 0 && 0 <= r0 && r0 <= r1 && r1 <= n,
                 "row range [%d, %d) out of bounds for n=%d", r0, r1, n);
  LMPK_ARG_CHECK(x != out, "in_vec and out_vec must not alias");
  (void)flags;
  if (r1 == r0) return LMPK_OK;
  return spmv_launch(ctx, row_ptr, col, val, x, out, r0, r1, as_stream(stream));
}

extern "C" int lmpk_mpk_baseline(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr,
                                 const int32_t* col, const double* val, double* y, int64_t ldy,
                                 int32_t p_m, int flags, void* stream) {
  LMPK_ARG_CHECK(ctx != nullptr, "lmpk_mpk_baseline: ctx is NULL");
  LMPK_ARG_CHECK(p_m >= 1, "p_m must be >= 1");
  LMPK_ARG_CHECK(ldy >= n, "ldy (%lld) must be >= n (%d)", (long long)ldy, n);
  if (n == 0) return LMPK_OK;
  (void)flags;
  cudaStream_t st = as_stream(stream);
  for (int32_t p = 1; p <= p_m; ++p)
    LMPK_TRY(spmv_launch(ctx, row_ptr, col, val, y + int64_t(p - 1) * ldy, y + int64_t(p) * ldy, 0, n, st));
  return LMPK_OK;
}
