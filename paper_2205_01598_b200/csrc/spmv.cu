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
// entries) in [r0, r1), compacted once per call: list[0] = rows longer than
// kHuge (filled from the front: they start first), list[1] = the other heavy
// rows (filled from the back of the cap = r1 - r0 slots behind the header).
constexpr int kHuge = 4096;
__global__ void k_heavy_rows(const int32_t* __restrict__ row_ptr, int32_t r0, int32_t r1, int32_t* list) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int32_t cap = r1 - r0;
  for (int64_t r = r0 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < r1; r += stride) {
    const int32_t len = __ldg(row_ptr + r + 1) - __ldg(row_ptr + r);
    if (len > kHuge)
      list[2 + atomicAdd(list, 1)] = int32_t(r);
    else if (len > kHeavy)
      list[2 + cap - 1 - atomicAdd(list + 1, 1)] = int32_t(r);
  }
}

// One sweep over [r0, r1).  CTAs [0, hb): one WARP per heavy row, software
// pipelined in stages of 128 entries -- the lanes load col/val (coalesced) two
// stages ahead and gather x one stage ahead, form the stage's products (each
// the same rounded double as the sequential kernel's) into shared memory, and
// lane 0 adds them in storage order from +0.0 while the next stages' loads are
// in flight: bitwise the sequential sum at the rate of its dependent add chain
// (the longest row's chain is the floor of a bit-exact sweep).  The other CTAs
// sum the light rows, one thread per row.
constexpr int kHStage = 128;
__global__ void __launch_bounds__(256) spmv_rows_heavy_kernel(const int32_t* __restrict__ row_ptr,
                                                              const int32_t* __restrict__ col,
                                                              const double* __restrict__ val,
                                                              const double* __restrict__ x,
                                                              double* __restrict__ out, int32_t r0, int32_t r1,
                                                              const int32_t* __restrict__ list, int32_t hb) {
  if (int32_t(blockIdx.x) < hb) {
    __shared__ __align__(16) double buf[8][2][kHStage];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t i = int32_t(blockIdx.x) * 8 + warp;
    const int32_t na = __ldg(list), nb = __ldg(list + 1);
    if (i >= na + nb) return;
    const int32_t r = i < na ? __ldg(list + 2 + i) : __ldg(list + 2 + (r1 - r0) - 1 - (i - na));
    const int32_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);
    const int32_t nst = (b - a + kHStage - 1) / kHStage;
    int32_t c2[4];
    double v2[4], x1[4], v1[4];
    auto load_cv = [&](int32_t s) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int32_t e = a + s * kHStage + q * 32 + lane;
        c2[q] = e < b ? __ldg(col + e) : -1;
        v2[q] = e < b ? __ldg(val + e) : 0.0;
      }
    };
    auto gather = [&]() {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x1[q] = c2[q] >= 0 ? __ldg(x + c2[q]) : 0.0;
        v1[q] = v2[q];
      }
    };
    load_cv(0);
    gather();
    if (nst > 1) load_cv(1);
    double t = 0.0;
    for (int32_t s = 0; s < nst; ++s) {
      double m[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) m[q] = __dmul_rn(v1[q], x1[q]);
      if (s + 1 < nst) gather();      // stage s + 1 (its columns arrived)
      if (s + 2 < nst) load_cv(s + 2);
      double* bw = buf[warp][s & 1];
#pragma unroll
      for (int q = 0; q < 4; ++q) bw[q * 32 + lane] = m[q];
      __syncwarp();
      if (lane == 0) {
        const int32_t cnt = min(kHStage, b - a - s * kHStage);
        const double2* b2 = reinterpret_cast<const double2*>(bw);
        int32_t k = 0;
        for (; k + 8 <= cnt; k += 8) {
          const double2 p0 = b2[k / 2], p1 = b2[k / 2 + 1], p2 = b2[k / 2 + 2], p3 = b2[k / 2 + 3];
          t = __dadd_rn(t, p0.x);
          t = __dadd_rn(t, p0.y);
          t = __dadd_rn(t, p1.x);
          t = __dadd_rn(t, p1.y);
          t = __dadd_rn(t, p2.x);
          t = __dadd_rn(t, p2.y);
          t = __dadd_rn(t, p3.x);
          t = __dadd_rn(t, p3.y);
        }
        for (; k < cnt; ++k) t = __dadd_rn(t, bw[k]);
      }
      __syncwarp();
    }
    if (lane == 0) out[r] = t;
    return;
  }
  const int64_t stride = int64_t(gridDim.x - hb) * blockDim.x;
  for (int64_t r = r0 + int64_t(blockIdx.x - hb) * blockDim.x + threadIdx.x; r < r1; r += stride) {
    const int32_t k0 = __ldg(row_ptr + r), k1 = __ldg(row_ptr + r + 1);
    if (k1 - k0 <= kHeavy)
      out[r] = row_sum_exact(col + k0, val + k0, k1 - k0, [x](int c) { return __ldg(x + c); });
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
  if (n_heavy == 0) {  // no hub rows
    spmv_rows_kernel<<<grid, threads, 0, st>>>(row_ptr, col, val, x, out, r0, r1);
  } else {
    const int hb = (n_heavy + 7) / 8;
    spmv_rows_heavy_kernel<<<hb + grid, threads, 0, st>>>(row_ptr, col, val, x, out, r0, r1, heavy, hb);
  }
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  return LMPK_OK;
}

// heavy-row list of [r0, r1) in the ctx scratch (two counts, then cap slots)
static int heavy_list(lmpk_ctx* ctx, const int32_t* row_ptr, int32_t r0, int32_t r1, int32_t** out,
                      int32_t* n_heavy, cudaStream_t st) {
  // the list is shared ctx scratch: a call on another stream may still be
  // reading it -- order this call (and any reallocation) after that reader
  if (!ctx->heavy_ev) LMPK_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->heavy_ev, cudaEventDisableTiming));
  const size_t list_bytes = (size_t(r1 - r0) + 2) * 4;
  if (ctx->s_heavy.bytes < list_bytes) LMPK_CHECK_CUDA(cudaEventSynchronize(ctx->heavy_ev));
  LMPK_CHECK_CUDA(cudaStreamWaitEvent(st, ctx->heavy_ev, 0));
  LMPK_TRY(ctx->s_heavy.ensure(list_bytes));
  int32_t* list = reinterpret_cast<int32_t*>(ctx->s_heavy.ptr);
  LMPK_CHECK_CUDA(cudaMemsetAsync(list, 0, 8, st));
  const int64_t blocks = (int64_t(r1) - r0 + 255) / 256;
  k_heavy_rows<<<static_cast<int>(std::min<int64_t>(blocks, int64_t(ctx->sm_count) * 8)), 256, 0, st>>>(row_ptr, r0,
                                                                                                          r1, list);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  int32_t head[2] = {0, 0};
  LMPK_CHECK_CUDA(cudaMemcpyAsync(head, list, 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));  // once per call: decides the heavy-row launch
  *n_heavy = head[0] + head[1];
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
