// spmv.cu -- bit-exact row-range SpMV and the baseline k x SpMV MPK.
//
// Replaces the reference's numba row kernel (pkg/src/levelmpk/csr.py:195-201)
// and the barrier-separated baseline sweeps (executor.py:233-266): one thread
// per row sums it in storage order with unfused multiply/add -> bitwise equal
// to numba.  Each call is one asynchronous launch per sweep.
#include <algorithm>

#include "lmpk_internal.cuh"

namespace lmpk {

// One thread per light row (<= kHeavy entries), grid-stride over [r0, r1),
// summed in storage order with unfused multiply/add (bitwise the numba
// kernel).  No shared memory: the unified L1 caches the rows' col/val lines
// and the gathered x lines.  The matrix and x are immutable during a launch,
// so the .nc path is safe.  Heavy rows are skipped here and summed by
// spmv_heavy_kernel.
constexpr int kHeavy = 128;
__global__ void __launch_bounds__(256) spmv_rows_kernel(const int32_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col,
                                                        const double* __restrict__ val,
                                                        const double* __restrict__ x, double* __restrict__ out,
                                                        int32_t r0, int32_t r1) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t r = r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < r1; r += stride) {
    const int32_t k0 = __ldg(row_ptr + r), k1 = __ldg(row_ptr + r + 1);
    if (k1 - k0 <= kHeavy)
      out[r] = row_sum_exact(col + k0, val + k0, k1 - k0, [x](int c) { return __ldg(x + c); });
  }
}

// Rows longer than kHeavy (power-law hubs: cfg4's largest has 97,280
// entries) in [r0, r1), compacted once per call: list[0] = count.
__global__ void k_heavy_rows(const int32_t* __restrict__ row_ptr, int32_t r0, int32_t r1, int32_t* list) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t r = r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < r1; r += stride)
    if (__ldg(row_ptr + r + 1) - __ldg(row_ptr + r) > kHeavy) list[1 + atomicAdd(list, 1)] = int32_t(r);
}

// One warp per heavy row: the warp loads 32 entries at a time (coalesced)
// and forms the 32 products in parallel -- each the same rounded double as
// the sequential kernel's -- then every lane adds them in storage order from
// shuffles: bitwise the sequential sum, with the row's loads no longer one
// entry at a time and the hubs spread over all warps of the grid.
__global__ void __launch_bounds__(256) spmv_heavy_kernel(const int32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x, double* __restrict__ out,
                                                         const int32_t* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  const int32_t nh = __ldg(list);
  const int32_t nw = int32_t((int64_t(gridDim.x) * blockDim.x) >> 5);
  for (int32_t i = int32_t((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); i < nh; i += nw) {
    const int32_t r = __ldg(list + 1 + i);
    const int32_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);
    double t = 0.0;
    for (int32_t e = a; e < b; e += 32) {
      const int n = min(32, b - e);
      double m = 0.0;
      if (lane < n) m = __dmul_rn(__ldg(val + e + lane), __ldg(x + __ldg(col + e + lane)));
      if (n == 32) {
        double ms[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) ms[j] = __shfl_sync(0xffffffffu, m, j);  // shuffles off the add chain
#pragma unroll
        for (int j = 0; j < 32; ++j) t = __dadd_rn(t, ms[j]);
      } else {
        for (int j = 0; j < n; ++j) t = __dadd_rn(t, __shfl_sync(0xffffffffu, m, j));
      }
    }
    if (lane == 0) out[r] = t;
  }
}

static int spmv_launch(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col, const double* val,
                       const double* x, double* out, int32_t r0, int32_t r1, const int32_t* heavy,
                       int32_t n_heavy, cudaStream_t st) {
  if (r1 <= r0) return LMPK_OK;
  const int threads = 256;
  const int64_t blocks = (int64_t(r1) - r0 + threads - 1) / threads;
  // enough CTAs for full occupancy (8 x 256 threads per SM), grid-stride beyond
  const int grid = static_cast<int>(std::min<int64_t>(blocks, int64_t(ctx->sm_count) * 8));
  spmv_rows_kernel<<<grid, threads, 0, st>>>(row_ptr, col, val, x, out, r0, r1);
  launch_count_add(ctx, 1);
  if (n_heavy > 0) {  // no second launch for matrices without hub rows
    const int hgrid = static_cast<int>(std::min<int64_t>((int64_t(n_heavy) * 32 + threads - 1) / threads,
                                                         int64_t(ctx->sm_count) * 8));
    spmv_heavy_kernel<<<hgrid, threads, 0, st>>>(row_ptr, col, val, x, out, heavy);
    launch_count_add(ctx, 1);
  }
  LMPK_CHECK_CUDA(cudaGetLastError());
  return LMPK_OK;
}

// heavy-row list of [r0, r1) in the ctx scratch (count, then row indices)
static int heavy_list(lmpk_ctx* ctx, const int32_t* row_ptr, int32_t r0, int32_t r1, int32_t** out,
                      int32_t* n_heavy, cudaStream_t st) {
  // the list is shared ctx scratch: a call on another stream may still be
  // reading it -- order this call (and any reallocation) after that reader
  if (!ctx->heavy_ev) LMPK_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->heavy_ev, cudaEventDisableTiming));
  if (ctx->s_heavy.bytes < (size_t(r1 - r0) + 1) * 4) LMPK_CHECK_CUDA(cudaEventSynchronize(ctx->heavy_ev));
  LMPK_CHECK_CUDA(cudaStreamWaitEvent(st, ctx->heavy_ev, 0));
  LMPK_TRY(ctx->s_heavy.ensure((size_t(r1 - r0) + 1) * 4));
  int32_t* list = reinterpret_cast<int32_t*>(ctx->s_heavy.ptr);
  LMPK_CHECK_CUDA(cudaMemsetAsync(list, 0, 4, st));
  const int64_t blocks = (int64_t(r1) - r0 + 255) / 256;
  k_heavy_rows<<<static_cast<int>(std::min<int64_t>(blocks, int64_t(ctx->sm_count) * 8)), 256, 0, st>>>(row_ptr, r0,
                                                                                                          r1, list);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(n_heavy, list, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));  // once per call: decides the heavy-row launches
  *out = list;
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
  cudaStream_t st = as_stream(stream);
  int32_t* heavy = nullptr;
  int32_t n_heavy = 0;
  LMPK_TRY(heavy_list(ctx, row_ptr, r0, r1, &heavy, &n_heavy, st));
  LMPK_TRY(spmv_launch(ctx, row_ptr, col, val, x, out, r0, r1, heavy, n_heavy, st));
  LMPK_CHECK_CUDA(cudaEventRecord(ctx->heavy_ev, st));
  return LMPK_OK;
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
  int32_t* heavy = nullptr;
  int32_t n_heavy = 0;
  LMPK_TRY(heavy_list(ctx, row_ptr, 0, n, &heavy, &n_heavy, st));
  for (int32_t p = 1; p <= p_m; ++p)
    LMPK_TRY(spmv_launch(ctx, row_ptr, col, val, y + int64_t(p - 1) * ldy, y + int64_t(p) * ldy, 0, n, heavy,
                         n_heavy, st));
  LMPK_CHECK_CUDA(cudaEventRecord(ctx->heavy_ev, st));
  return LMPK_OK;
}
