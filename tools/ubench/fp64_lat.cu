// Micro-benchmarks: fp64 dependent-chain latency and per-SM throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, long long* cyc, int n, int kind) {
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  if (kind == 0) for (int i = 0; i < n; ++i) a = __fma_rn(a, b, c);
  else if (kind == 1) for (int i = 0; i < n; ++i) a = __dadd_rn(a, c);
  else for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// 8 independent chains per thread, many warps: throughput
__global__ void thru(double* out, int n) {
  double a0 = out[threadIdx.x], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 1.0000001, c = 1e-9;
  for (int i = 0; i < n; ++i) {
    a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c);
    a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
// pointer chase within a small (L1-resident) array: L1 hit latency
__global__ void chase(const int* nxt, long long* cyc, int n, int* sink) {
  int p = 0;
  for (int i = 0; i < 64; ++i) p = nxt[p];  // warm
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = nxt[p];
  long long t1 = clock64();
  *sink = p;
  *cyc = t1 - t0;
}
int main() {
  double* d; long long* c; int* nx; int* sink;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 8); cudaMalloc(&nx, 4096 * 4); cudaMalloc(&sink, 4);
  cudaMemset(d, 0, 1 << 26);
  const int n = 4096;
  const char* nm[3] = {"DFMA", "DADD", "DMUL"};
  for (int k = 0; k < 3; ++k) {
    chain<<<1, 32>>>(d, c, n, k); cudaDeviceSynchronize();
    chain<<<1, 32>>>(d, c, n, k);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%s dependent latency: %.2f cycles\n", nm[k], double(h) / n);
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int warps : {4, 8, 16, 32}) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    thru<<<sms, 32 * warps>>>(d, 1000);
    cudaEventRecord(a); thru<<<sms, 32 * warps>>>(d, 20000); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fma = double(sms) * 32 * warps * 8 * 20000;
    printf("DFMA throughput, %2d warps/SM: %.1f TFMA/s = %.1f lane-FMA/clk/SM (at %d MHz nominal)\n", warps,
           fma / ms / 1e9, fma / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  int h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (i * 97 + 33) % 4096;  // single cycle over 4096 entries
  cudaMemcpy(nx, h, sizeof(h), cudaMemcpyHostToDevice);
  chase<<<1, 1>>>(nx, c, 2000, sink); cudaDeviceSynchronize();
  chase<<<1, 1>>>(nx, c, 2000, sink);
  long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
  printf("LDG L1-hit chase latency: %.1f cycles\n", double(hc) / 2000);
  return 0;
}
