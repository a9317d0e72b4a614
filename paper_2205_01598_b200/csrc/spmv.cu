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

// Longest huge rows first (their CTAs are scheduled in list order and the
// longest row's add chain is the critical path of the sweep): rank sort of the
// na huge rows by (length descending, row ascending) by one CTA, through the
// free slots between the two ends of the list.
// n_cta receives the number of rows longer than kCtaRow: only those take the
// CTA path (its one adding thread per CTA is the fastest chain, but an SM
// holds three such CTAs against 24 warp-per-row chains); the other huge rows
// stay at the front of the list, so their warps start first.
constexpr int kCtaRow = 16384;
__global__ void __launch_bounds__(1024) k_sort_huge(const int32_t* __restrict__ row_ptr, int32_t* list, int32_t na,
                                                    int32_t* n_cta) {
  int32_t* rows = list + 2;
  int32_t* tmp = rows + na;
  for (int32_t i = threadIdx.x; i < na; i += blockDim.x) {
    const int32_t r = rows[i];
    const int32_t len = __ldg(row_ptr + r + 1) - __ldg(row_ptr + r);
    if (len > kCtaRow) atomicAdd(n_cta, 1);
    int32_t rank = 0;
    for (int32_t j = 0; j < na; ++j) {
      const int32_t q = rows[j];
      const int32_t lq = __ldg(row_ptr + q + 1) - __ldg(row_ptr + q);
      rank += (lq > len) || (lq == len && q < r);
    }
    tmp[rank] = r;
  }
  __syncthreads();
  for (int32_t i = threadIdx.x; i < na; i += blockDim.x) rows[i] = tmp[i];
}

// A HUGE row (> kHuge entries) takes a whole CTA: warps 1..7 load col/val,
// gather x and write the products (each the same rounded double as the
// sequential kernel's) into a shared-memory ring of stages of 896 entries;
// lane 0 of warp 0 only adds them, in storage order from +0.0, next group's
// products already in registers -- the dependent DADD chain never waits for
// anything else, so the row costs its entries x the DADD latency (cfg4's
// 97,280-entry hub: ~0.45 ms, the floor of a bit-exact sum; one warp doing
// both jobs in turns took 0.8 ms and set the time of the whole sweep).
constexpr int kHugeWarps = 7;
constexpr int kHugeStage = kHugeWarps * 128;
template <bool CPLX>
struct HugeRing {
  static constexpr int kStages = CPLX ? 2 : 4;
  static constexpr int kDoubles = kStages * kHugeStage * (CPLX ? 2 : 1);
};
template <bool CPLX>
__device__ __forceinline__ void huge_row_sum(const int32_t* __restrict__ col, const double* __restrict__ val,
                                             const double* __restrict__ x, int32_t a, int32_t b, double* ring,
                                             uint64_t* full, uint64_t* empty, double& tr, double& ti) {
  constexpr int NS = HugeRing<CPLX>::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 32 * kHugeWarps);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int32_t nst = (b - a + kHugeStage - 1) / kHugeStage;
  tr = 0.0, ti = 0.0;
  if (warp > 0) {
    const int32_t wofs = (warp - 1) * 128 + lane;
    for (int32_t s = 0; s < nst; ++s) {
      int32_t c[4];
      double v[4], mr[4], mi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int32_t e = a + s * kHugeStage + wofs + q * 32;
        c[q] = e < b ? __ldg(col + e) : -1;
        v[q] = e < b ? __ldg(val + e) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if constexpr (CPLX) {
          const double2 xx = c[q] >= 0 ? __ldg(reinterpret_cast<const double2*>(x) + c[q]) : make_double2(0.0, 0.0);
          mr[q] = __dmul_rn(v[q], xx.x);
          mi[q] = __dmul_rn(v[q], xx.y);
        } else {
          mr[q] = __dmul_rn(v[q], c[q] >= 0 ? __ldg(x + c[q]) : 0.0);
          mi[q] = 0.0;
        }
      }
      const int slot = s % NS;
      if (s >= NS) mbar_wait(&empty[slot], uint32_t(s / NS - 1) & 1u);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if constexpr (CPLX)
          reinterpret_cast<double2*>(ring)[slot * kHugeStage + wofs + q * 32] = make_double2(mr[q], mi[q]);
        else
          ring[slot * kHugeStage + wofs + q * 32] = mr[q];
      }
      mbar_arrive(&full[slot]);
    }
  } else if (lane == 0) {
    for (int32_t s = 0; s < nst; ++s) {
      const int slot = s % NS;
      mbar_wait(&full[slot], uint32_t(s / NS) & 1u);
      const int32_t cnt = min(kHugeStage, b - a - s * kHugeStage);
      // Blocks of 32 products (complex: 16), written out as four groups over
      // two register buffers: each group's shared-memory loads are issued one
      // group ahead of its adds, the first group of the next block (index
      // clamped to the stage) during the last group.  The block loop is not
      // unrolled by the compiler and has no conditional loads: an earlier
      // form with a conditional prefetch inside an unrollable loop was
      // miscompiled (one group of an unrolled remainder was dropped).
      constexpr int kPer = CPLX ? 16 : 32;  // entries per block = 16 double2 loads
      const double2* b2 = CPLX ? reinterpret_cast<const double2*>(ring) + slot * kHugeStage
                               : reinterpret_cast<const double2*>(ring + slot * kHugeStage);
      auto ld4 = [&](double2(&P)[4], int32_t i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) P[j] = b2[i + j];
      };
      auto add4 = [&](const double2(&P)[4]) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if constexpr (CPLX) {
            tr = __dadd_rn(tr, P[j].x);
            ti = __dadd_rn(ti, P[j].y);
          } else {
            tr = __dadd_rn(tr, P[j].x);
            tr = __dadd_rn(tr, P[j].y);
          }
        }
      };
      const int32_t nblk = cnt / kPer;
      double2 A[4], B[4];
      ld4(A, 0);
#pragma unroll 1
      for (int32_t blk = 0; blk < nblk; ++blk) {
        const int32_t i0 = 16 * blk;
        const int32_t inext = 16 * min(blk + 1, kHugeStage / kPer - 1);
        ld4(B, i0 + 4);
        add4(A);
        ld4(A, i0 + 8);
        add4(B);
        ld4(B, i0 + 12);
        add4(A);
        ld4(A, inext);
        add4(B);
      }
      if constexpr (CPLX) {
        for (int32_t k = kPer * nblk; k < cnt; ++k) tr = __dadd_rn(tr, b2[k].x), ti = __dadd_rn(ti, b2[k].y);
      } else {
        for (int32_t k = kPer * nblk; k < cnt; ++k) tr = __dadd_rn(tr, ring[slot * kHugeStage + k]);
      }
      mbar_arrive(&empty[slot]);
    }
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
                                                              const int32_t* __restrict__ list, int32_t ha,
                                                              int32_t hb) {
  // CTAs [0, ha): one huge row each; [ha, ha + hb): 8 heavy rows each; the rest: light rows
  __shared__ __align__(16) double smem_d[HugeRing<false>::kDoubles];
  __shared__ uint64_t bars[2 * HugeRing<false>::kStages];
  static_assert(HugeRing<false>::kDoubles >= 8 * 2 * kHStage, "heavy-row buffers share the ring's memory");
  if (int32_t(blockIdx.x) < ha) {
    const int32_t r = __ldg(list + 2 + int32_t(blockIdx.x));
    double tr, ti;
    huge_row_sum<false>(col, val, x, __ldg(row_ptr + r), __ldg(row_ptr + r + 1), smem_d, bars,
                        bars + HugeRing<false>::kStages, tr, ti);
    if (threadIdx.x == 0) out[r] = tr;
    return;
  }
  if (int32_t(blockIdx.x) < ha + hb) {
    double(*buf)[2][kHStage] = reinterpret_cast<double(*)[2][kHStage]>(smem_d);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t na = __ldg(list), nb = __ldg(list + 1);
    const int32_t i = ha + (int32_t(blockIdx.x) - ha) * 8 + warp;  // ha <= na: the longest rows took CTAs
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
  const int64_t stride = int64_t(gridDim.x - ha - hb) * blockDim.x;
  for (int64_t r = r0 + int64_t(blockIdx.x - ha - hb) * blockDim.x + threadIdx.x; r < r1; r += stride) {
    const int32_t k0 = __ldg(row_ptr + r), k1 = __ldg(row_ptr + r + 1);
    if (k1 - k0 <= kHeavy)
      out[r] = row_sum_exact(col + k0, val + k0, k1 - k0, [x](int c) { return __ldg(x + c); });
  }
}

static int spmv_launch(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col, const double* val,
                       const double* x, double* out, int32_t r0, int32_t r1, const int32_t* heavy,
                       int32_t n_huge, int32_t n_heavy, cudaStream_t st) {
  if (r1 <= r0) return LMPK_OK;
  const int threads = 256;
  const int64_t blocks = (int64_t(r1) - r0 + threads - 1) / threads;
  // enough CTAs for full occupancy (8 x 256 threads per SM), grid-stride beyond
  const int grid = static_cast<int>(std::min<int64_t>(blocks, int64_t(ctx->sm_count) * 8));
  if (n_heavy == 0) {  // no hub rows
    spmv_rows_kernel<<<grid, threads, 0, st>>>(row_ptr, col, val, x, out, r0, r1);
  } else {
    const int hb = (n_heavy - n_huge + 7) / 8;
    spmv_rows_heavy_kernel<<<n_huge + hb + grid, threads, 0, st>>>(row_ptr, col, val, x, out, r0, r1, heavy, n_huge,
                                                                   hb);
  }
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  return LMPK_OK;
}

// ---------------------------------------------------------------- CRS plan sweeps
// One power of a plan on the CRS arrays with the plan's per-power epilogue
// fused in: t = row sum (storage order, unfused, as above); Chebyshev
// t = 2 t - y_prev[r]; y_out[r] = t; acc[r] += c t (executor.py:127-147).
// Real or complex128 vectors (a real matrix: two independent sums).  This is
// the level-blocked plans' fallback for matrices the tile format cannot hold
// (rows longer than 65,535 entries), so that Chebyshev and accumulating plans
// run there too; bitwise equal to the walk's row body.
struct SweepEpi {
  const double* prev;  // y_{p-2} slot (Chebyshev), or null
  double* acc;         // accumulator, or null
  double cre, cim;
};
template <bool CPLX>
__device__ __forceinline__ void sweep_store(double* __restrict__ out, const SweepEpi& E, int64_t r, double tr,
                                            double ti) {
  if constexpr (!CPLX) {
    if (E.prev) tr = __dsub_rn(__dmul_rn(2.0, tr), E.prev[r]);
    out[r] = tr;
    if (E.acc) E.acc[r] = __dadd_rn(E.acc[r], __dmul_rn(E.cre, tr));
  } else {
    if (E.prev) {
      tr = __dsub_rn(__dmul_rn(2.0, tr), E.prev[2 * r]);
      ti = __dsub_rn(__dmul_rn(2.0, ti), E.prev[2 * r + 1]);
    }
    out[2 * r] = tr;
    out[2 * r + 1] = ti;
    if (E.acc) {
      const double pr = __dsub_rn(__dmul_rn(E.cre, tr), __dmul_rn(E.cim, ti));
      const double pi = __dadd_rn(__dmul_rn(E.cre, ti), __dmul_rn(E.cim, tr));
      E.acc[2 * r] = __dadd_rn(E.acc[2 * r], pr);
      E.acc[2 * r + 1] = __dadd_rn(E.acc[2 * r + 1], pi);
    }
  }
}

struct LdgX {
  const double* x;
  __device__ __forceinline__ double operator()(int c) const { return __ldg(x + c); }
};
struct LdgX2 {
  const double2* x;
  __device__ __forceinline__ double2 operator()(int c) const { return __ldg(x + c); }
};

template <bool CPLX>
__device__ __forceinline__ void sweep_gather(const double* __restrict__ x, int32_t c, double& xr, double& xi) {
  if constexpr (CPLX) {
    const double2 xx = c >= 0 ? __ldg(reinterpret_cast<const double2*>(x) + c) : make_double2(0.0, 0.0);
    xr = xx.x;
    xi = xx.y;
  } else {
    xr = c >= 0 ? __ldg(x + c) : 0.0;
    xi = 0.0;
  }
}

template <bool CPLX>
__global__ void __launch_bounds__(256) sweep_rows_kernel(const int32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col,
                                                         const double* __restrict__ val,
                                                         const double* __restrict__ x, double* __restrict__ out,
                                                         SweepEpi E, int32_t n, const int32_t* __restrict__ list,
                                                         int32_t ha, int32_t hb) {
  constexpr int kHW = kHStage * (CPLX ? 2 : 1);
  constexpr int kSm = HugeRing<CPLX>::kDoubles > 8 * 2 * kHW ? HugeRing<CPLX>::kDoubles : 8 * 2 * kHW;
  __shared__ __align__(16) double smem_d[kSm];
  __shared__ uint64_t bars[2 * HugeRing<CPLX>::kStages];
  if (int32_t(blockIdx.x) < ha) {
    // one CTA per huge row (huge_row_sum above)
    const int32_t r = __ldg(list + 2 + int32_t(blockIdx.x));
    double tr, ti;
    huge_row_sum<CPLX>(col, val, x, __ldg(row_ptr + r), __ldg(row_ptr + r + 1), smem_d, bars,
                       bars + HugeRing<CPLX>::kStages, tr, ti);
    if (threadIdx.x == 0) sweep_store<CPLX>(out, E, r, tr, ti);
    return;
  }
  if (int32_t(blockIdx.x) < ha + hb) {
    // one warp per heavy row, pipelined as in spmv_rows_heavy_kernel
    double(*buf)[2][kHW] = reinterpret_cast<double(*)[2][kHW]>(smem_d);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int32_t na = __ldg(list), nb = __ldg(list + 1);
    const int32_t i = ha + (int32_t(blockIdx.x) - ha) * 8 + warp;  // ha <= na: the longest rows took CTAs
    if (i >= na + nb) return;
    const int32_t r = i < na ? __ldg(list + 2 + i) : __ldg(list + 2 + n - 1 - (i - na));
    const int32_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);
    const int32_t nst = (b - a + kHStage - 1) / kHStage;
    int32_t c2[4];
    double v2[4], v1[4], x1r[4], x1i[4];
#define LMPK_SWEEP_LOAD_CV(S)                                      \
  _Pragma("unroll") for (int q = 0; q < 4; ++q) {                  \
    const int32_t e = a + (S) * kHStage + q * 32 + lane;           \
    c2[q] = e < b ? __ldg(col + e) : -1;                           \
    v2[q] = e < b ? __ldg(val + e) : 0.0;                          \
  }
#define LMPK_SWEEP_GATHER()                                        \
  _Pragma("unroll") for (int q = 0; q < 4; ++q) {                  \
    sweep_gather<CPLX>(x, c2[q], x1r[q], x1i[q]);                  \
    v1[q] = v2[q];                                                 \
  }
    LMPK_SWEEP_LOAD_CV(0)
    LMPK_SWEEP_GATHER()
    if (nst > 1) {
      LMPK_SWEEP_LOAD_CV(1)
    }
    double tr = 0.0, ti = 0.0;
    for (int32_t s = 0; s < nst; ++s) {
      double mr[4], mi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        mr[q] = __dmul_rn(v1[q], x1r[q]);
        mi[q] = CPLX ? __dmul_rn(v1[q], x1i[q]) : 0.0;
      }
      if (s + 1 < nst) {
        LMPK_SWEEP_GATHER()
      }
      if (s + 2 < nst) {
        LMPK_SWEEP_LOAD_CV(s + 2)
      }
      double* bw = buf[warp][s & 1];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if constexpr (CPLX) {
          bw[2 * (q * 32 + lane)] = mr[q];
          bw[2 * (q * 32 + lane) + 1] = mi[q];
        } else {
          bw[q * 32 + lane] = mr[q];
        }
      }
      __syncwarp();
      if (lane == 0) {
        const int32_t cnt = min(kHStage, b - a - s * kHStage);
        const double2* b2 = reinterpret_cast<const double2*>(bw);
        if constexpr (CPLX) {
          for (int32_t k = 0; k < cnt; ++k) {
            const double2 p = b2[k];
            tr = __dadd_rn(tr, p.x);
            ti = __dadd_rn(ti, p.y);
          }
        } else {
          int32_t k = 0;
          for (; k + 2 <= cnt; k += 2) {
            const double2 p = b2[k / 2];
            tr = __dadd_rn(tr, p.x);
            tr = __dadd_rn(tr, p.y);
          }
          if (k < cnt) tr = __dadd_rn(tr, bw[k]);
        }
      }
      __syncwarp();
    }
    if (lane == 0) sweep_store<CPLX>(out, E, r, tr, ti);
#undef LMPK_SWEEP_LOAD_CV
#undef LMPK_SWEEP_GATHER
    return;
  }
  const int64_t stride = int64_t(gridDim.x - ha - hb) * blockDim.x;
  for (int64_t r = int64_t(blockIdx.x - ha - hb) * blockDim.x + threadIdx.x; r < n; r += stride) {
    const int32_t k0 = __ldg(row_ptr + r), k1 = __ldg(row_ptr + r + 1);
    if (k1 - k0 > kHeavy) continue;
    if constexpr (CPLX) {
      const double2 t = row_sum_exact_c(col + k0, val + k0, k1 - k0, LdgX2{reinterpret_cast<const double2*>(x)});
      sweep_store<true>(out, E, r, t.x, t.y);
    } else {
      const double t = row_sum_exact(col + k0, val + k0, k1 - k0, LdgX{x});
      sweep_store<false>(out, E, r, t, 0.0);
    }
  }
}

// heavy-row list of [r0, r1) in the ctx scratch (two counts, then cap slots)
static int heavy_list(lmpk_ctx* ctx, const int32_t* row_ptr, int32_t r0, int32_t r1, int32_t** out,
                      int32_t* n_huge, int32_t* n_heavy, cudaStream_t st) {
  // the list is shared ctx scratch: a call on another stream may still be
  // reading it -- order this call (and any reallocation) after that reader
  if (!ctx->heavy_ev) LMPK_CHECK_CUDA(cudaEventCreateWithFlags(&ctx->heavy_ev, cudaEventDisableTiming));
  const size_t list_bytes = (size_t(r1 - r0) + 3) * 4;  // two counts, cap slots, the CTA-path count
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
  *n_huge = head[0];  // rows on the CTA path: every huge row unless the sort below narrows it
  *n_heavy = head[0] + head[1];
  if (head[0] > 0 && int64_t(r1 - r0) - head[0] - head[1] >= head[0]) {
    int32_t* d_cta = list + 2 + (r1 - r0);  // one slot behind the cap
    LMPK_CHECK_CUDA(cudaMemsetAsync(d_cta, 0, 4, st));
    k_sort_huge<<<1, 1024, 0, st>>>(row_ptr, list, head[0], d_cta);
    LMPK_CHECK_CUDA(cudaGetLastError());
    launch_count_add(ctx, 1);
    int32_t h_cta = 0;
    LMPK_CHECK_CUDA(cudaMemcpyAsync(&h_cta, d_cta, 4, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    *n_huge = h_cta;
  }
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
  if (r1 == r0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  int32_t* heavy = nullptr;
  int32_t n_heavy = 0, n_huge = 0;
  if (flags & LMPK_FLAG_NO_HUB_ROWS) {  // no scan, no sync, no shared scratch
    return spmv_launch(ctx, row_ptr, col, val, x, out, r0, r1, nullptr, 0, 0, st);
  }
  LMPK_TRY(heavy_list(ctx, row_ptr, r0, r1, &heavy, &n_huge, &n_heavy, st));
  LMPK_TRY(spmv_launch(ctx, row_ptr, col, val, x, out, r0, r1, heavy, n_huge, n_heavy, st));
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
  cudaStream_t st = as_stream(stream);
  int32_t* heavy = nullptr;
  int32_t n_heavy = 0, n_huge = 0;
  if (flags & LMPK_FLAG_NO_HUB_ROWS) {
    for (int32_t p = 1; p <= p_m; ++p)
      LMPK_TRY(spmv_launch(ctx, row_ptr, col, val, y + int64_t(p - 1) * ldy, y + int64_t(p) * ldy, 0, n, nullptr, 0,
                           0, st));
    return LMPK_OK;
  }
  LMPK_TRY(heavy_list(ctx, row_ptr, 0, n, &heavy, &n_huge, &n_heavy, st));
  for (int32_t p = 1; p <= p_m; ++p)
    LMPK_TRY(spmv_launch(ctx, row_ptr, col, val, y + int64_t(p - 1) * ldy, y + int64_t(p) * ldy, 0, n, heavy,
                         n_huge, n_heavy, st));
  LMPK_CHECK_CUDA(cudaEventRecord(ctx->heavy_ev, st));
  return LMPK_OK;
}

// Replaces run_plan's walker (executor.py:84-230) for plans on matrices whose
// rows do not fit the tile format: cfg->n_powers sweeps over the CRS arrays
// with the per-power slots, kernel (SpMV / Chebyshev) and accumulation.
extern "C" int lmpk_mpk_crs_run(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                                const double* val, double* y, int64_t ldy, int32_t n_slots,
                                const lmpk_power_cfg* cfg, double* acc, int use_acc, int flags, void* stream) {
  LMPK_ARG_CHECK(ctx && cfg && y, "lmpk_mpk_crs_run: NULL ctx/cfg/y");
  const bool cplx = (flags & LMPK_FLAG_COMPLEX) != 0;
  LMPK_ARG_CHECK(cfg->n_powers >= 1 && cfg->n_powers <= LMPK_MAX_POWERS, "n_powers out of range");
  LMPK_ARG_CHECK(ldy >= int64_t(n) * (cplx ? 2 : 1), "ldy too small");
  LMPK_ARG_CHECK(!use_acc || acc != nullptr, "use_acc requires acc");
  LMPK_ARG_CHECK(!cplx || (reinterpret_cast<uintptr_t>(y) & 15) == 0, "complex y must be 16-byte aligned");
  if (n == 0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  int32_t* heavy = nullptr;
  int32_t n_heavy = 0, n_huge = 0;
  const bool no_hubs = (flags & LMPK_FLAG_NO_HUB_ROWS) != 0;
  if (!no_hubs) LMPK_TRY(heavy_list(ctx, row_ptr, 0, n, &heavy, &n_huge, &n_heavy, st));
  const int threads = 256;
  const int64_t blocks = (int64_t(n) + threads - 1) / threads;
  const int grid = static_cast<int>(std::min<int64_t>(blocks, int64_t(ctx->sm_count) * 8));
  const int ha = n_huge, hb = (n_heavy - n_huge + 7) / 8;
  for (int32_t i = 0; i < cfg->n_powers; ++i) {
    const int32_t so = cfg->out_slot[i], si = cfg->in_slot[i], sp = cfg->prev_slot[i];
    LMPK_ARG_CHECK(so >= 0 && so < n_slots && si >= 0 && si < n_slots && so != si, "bad slots at power %d", i + 1);
    const bool cheb = cfg->kernel[i] == LMPK_KERNEL_CHEB;
    LMPK_ARG_CHECK(!cheb || (sp >= 0 && sp < n_slots), "bad prev_slot at power %d", i + 1);
    SweepEpi E{cheb ? y + int64_t(sp) * ldy : nullptr, use_acc ? acc : nullptr, cfg->acc_coef_re[i],
               cplx ? cfg->acc_coef_im[i] : 0.0};
    const double* x = y + int64_t(si) * ldy;
    double* out = y + int64_t(so) * ldy;
    if (cplx)
      sweep_rows_kernel<true><<<ha + hb + grid, threads, 0, st>>>(row_ptr, col, val, x, out, E, n, heavy, ha, hb);
    else
      sweep_rows_kernel<false><<<ha + hb + grid, threads, 0, st>>>(row_ptr, col, val, x, out, E, n, heavy, ha, hb);
    launch_count_add(ctx, 1);
  }
  LMPK_CHECK_CUDA(cudaGetLastError());
  if (!no_hubs) LMPK_CHECK_CUDA(cudaEventRecord(ctx->heavy_ev, st));
  return LMPK_OK;
}
