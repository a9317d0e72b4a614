// probe.cu -- micro-benchmarks that size the MPK design on the actual B200:
// HBM vs L2-resident read bandwidth and the cross-CTA release/acquire round
// trip that every wavefront dependency pays.
#include "lmpk_internal.cuh"

namespace lmpk {

__global__ void k_read_bw(const double4* __restrict__ p, size_t n4, int reps, double* sink) {
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
         i += size_t(gridDim.x) * blockDim.x) {
      double4 v;
      asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                   : "l"(p + i));
      acc += v.x + v.y + v.z + v.w;
    }
  }
  if (acc == 1234.5) sink[0] = acc;
}

__global__ void k_pingpong(uint32_t* flags, int iters, unsigned long long* out_ns) {
  // CTA 0 and CTA 1 alternate: CTA b waits for flags[b] == i then sets flags[1-b]
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (b == 0) {
      st_release_u32(flags + 1, i);
      while (ld_relaxed_u32(flags + 0) < uint32_t(i)) {
      }
      fence_acq_rel_gpu();
    } else {
      while (ld_relaxed_u32(flags + 1) < uint32_t(i)) {
      }
      fence_acq_rel_gpu();
      st_release_u32(flags + 0, i);
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (b == 0) out_ns[0] = t1 - t0;
}

}  // namespace lmpk

using namespace lmpk;

// GB/s of a streaming read over `bytes` repeated `reps` times (L2-resident
// when bytes << 126 MB), timed with CUDA events; best of `trials`.
extern "C" int lmpk_probe_read_bw(lmpk_ctx* ctx, int64_t bytes, int reps, int trials,
                                  double* gbps) {
  LMPK_ARG_CHECK(ctx && gbps && bytes >= 1024, "bad probe args");
  double4* buf = nullptr;
  double* sink = nullptr;
  LMPK_CHECK_CUDA(cudaMalloc(&buf, bytes));
  LMPK_CHECK_CUDA(cudaMalloc(&sink, 64));
  LMPK_CHECK_CUDA(cudaMemset(buf, 0, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t n4 = size_t(bytes) / sizeof(double4);
  const int grid = ctx->sm_count * 8;
  k_read_bw<<<grid, 256>>>(buf, n4, 1, sink);  // warm
  float best = 1e30f;
  for (int t = 0; t < trials; ++t) {
    cudaEventRecord(a);
    k_read_bw<<<grid, 256>>>(buf, n4, reps, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  if (e != cudaSuccess) {
    set_error("probe: %s", cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  }
  *gbps = double(bytes) * reps / (best * 1e-3) / 1e9;
  return LMPK_OK;
}

// Mean one-way latency (ns) of a release-store / relaxed-poll + acquire-fence
// hand-off between two CTAs (cooperative launch guarantees co-residency).
extern "C" int lmpk_probe_flag_latency(lmpk_ctx* ctx, int iters, double* ns_one_way) {
  LMPK_ARG_CHECK(ctx && ns_one_way && iters > 0, "bad probe args");
  uint32_t* flags = nullptr;
  unsigned long long* out = nullptr;
  LMPK_CHECK_CUDA(cudaMalloc(&flags, 256));
  LMPK_CHECK_CUDA(cudaMalloc(&out, 64));
  LMPK_CHECK_CUDA(cudaMemset(flags, 0, 256));
  void* args[] = {&flags, &iters, &out};
  LMPK_CHECK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_pingpong), dim3(2),
                                              dim3(32), args, 0, nullptr));
  unsigned long long ns = 0;
  LMPK_CHECK_CUDA(cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost));
  cudaFree(flags);
  cudaFree(out);
  *ns_one_way = double(ns) / (2.0 * iters);
  return LMPK_OK;
}
