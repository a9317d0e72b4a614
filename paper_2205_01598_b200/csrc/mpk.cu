// mpk.cu -- level-blocked matrix power kernel for sm_100a.
//
// Reference: the diagonal Lp-diagram walk of pkg/src/levelmpk/schedule.py:91-99
// executed by the p2p walker _walk/_wait_all (executor.py:84-150) over the
// flat ExecPlan (plan.py:184-370).  The GPU form:
//
//   * the level-permuted matrix is cut into contiguous row TILES sized to the
//     shared-memory budget; tile t's dependency range [dep_lo(t), dep_hi(t)]
//     is the set of tiles owning its column indices (level confinement,
//     Eq. 4 of the paper, keeps it narrow: a tile couples only to tiles of
//     its own and the adjacent levels);
//   * a persistent grid of CTAs replaces the reference's W threads.  Each
//     (tile, power) node publishes an epoch-tagged counter with a gpu-scope
//     release after its rows are stored; a consumer polls its dependency
//     range with relaxed loads and then issues an acquire fence (which also
//     invalidates the SM's L1 so later gathers see fresh vector data).  This
//     is the device form of condition (A)/(B)/(C): "tile t at power p only
//     after tiles dep_lo..dep_hi finished p-1".
//   * RESIDENT mode (cooperative launch): a CTA grabs the next tile in order,
//     stages its CRS slice into shared memory ONCE with a TMA bulk copy and
//     computes all p_m powers on it -> the matrix is read from HBM once.
//     Deadlock freedom: the chain reach of the p_m-1 dependency steps must be
//     smaller than the number of co-resident CTAs (checked at planning time).
//   * STREAMING mode: CTAs grab (tile, power) items from a queue ordered by
//     the skewed diagonal key (t + p*D, p) -- topologically valid for any
//     D >= max forward reach -- and re-stage the slice per power (served from
//     L2 inside the diagonal window).  Deadlock-free without co-residency.
//
// Every row is summed exactly like the reference (bit-exact mode), so all
// modes and tilings produce bitwise identical power vectors.
#include <string.h>

#include <algorithm>
#include <numeric>

#include "lmpk_internal.cuh"

namespace lmpk {

constexpr int kMpkThreads = 256;
constexpr uint32_t kEpochStride = 128;  // > LMPK_MAX_POWERS
constexpr unsigned long long kWatchdogNs = 8ull * 1000 * 1000 * 1000;

struct PowerCfgDev {
  int32_t out_slot[LMPK_MAX_POWERS];
  int32_t in_slot[LMPK_MAX_POWERS];
  int32_t prev_slot[LMPK_MAX_POWERS];
  int32_t kernel[LMPK_MAX_POWERS];
  double coef_re[LMPK_MAX_POWERS];
  double coef_im[LMPK_MAX_POWERS];
};

struct MpkParams {
  const int32_t* row_ptr;
  const int32_t* col;
  const double* val;
  double* y;
  int64_t ldy;
  double* acc;
  int32_t use_acc;
  const int32_t* tile_row;
  const int32_t* dep_lo;
  const int32_t* dep_hi;
  const int32_t* items;
  uint32_t* progress;
  unsigned long long* queue;  // [0] work counter, [1] abort flag
  unsigned long long queue_base;
  uint32_t epoch_base;
  int32_t n_tiles;
  int32_t n_items;
  int32_t n_powers;
  int32_t mode;
  int32_t cap;
  int32_t rows_cap;
  int32_t use_tma;
  int* err;  // host-mapped
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct MpkSmem {
  double* val;
  int32_t* col;
  int32_t* rp;
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

// 16-byte aligned sections (TMA bulk copies need 16-byte aligned smem).
__device__ __forceinline__ MpkSmem carve(unsigned char* base, int32_t cap, int32_t rows_cap) {
  MpkSmem s;
  const size_t val_bytes = align16((size_t(cap) + 4) * 8);
  const size_t col_bytes = align16((size_t(cap) + 8) * 4);
  s.val = reinterpret_cast<double*>(base);
  s.col = reinterpret_cast<int32_t*>(base + val_bytes);
  s.rp = reinterpret_cast<int32_t*>(base + val_bytes + col_bytes);
  (void)rows_cap;
  return s;
}

__host__ __device__ inline size_t mpk_buf_bytes(int32_t cap, int32_t rows_cap) {
  size_t b = align16((size_t(cap) + 4) * 8) + align16((size_t(cap) + 8) * 4) +
             align16((size_t(rows_cap) + 8) * 4);
  return (b + 127) & ~size_t(127);
}

// Stage rows [r0, r1] pointers and elements [nz0, nz1) of tile into smem.
// Thread 0 arms the mbarrier (exactly one phase per call).  Returns false if
// the tile does not fit (then it is computed straight from global memory).
__device__ __forceinline__ bool mpk_stage(const MpkParams& P, const MpkSmem& s, uint64_t* bar,
                                          int32_t r0, int32_t r1, int64_t nz0, int64_t nz1,
                                          uint64_t policy) {
  const bool fits = (nz1 - nz0 <= P.cap) && (r1 - r0 <= P.rows_cap);
  if (!fits) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, 0);
    return false;
  }
  const int64_t ca0 = nz0 & ~int64_t(3), ci0 = (nz0 + 3) & ~int64_t(3), ci1 = nz1 & ~int64_t(3);
  const int64_t va0 = nz0 & ~int64_t(1), vi0 = (nz0 + 1) & ~int64_t(1), vi1 = nz1 & ~int64_t(1);
  const int32_t ra0 = r0 & ~3, ri0 = (r0 + 3) & ~3, ri1 = (r1 + 1) & ~3;  // rp[r0..r1] inclusive
  const bool c_tma = P.use_tma && ci1 > ci0;
  const bool v_tma = P.use_tma && vi1 > vi0;
  const bool r_tma = P.use_tma && ri1 > ri0;
  if (threadIdx.x == 0) {
    fence_proxy_async_smem();
    uint32_t bytes = (c_tma ? uint32_t(ci1 - ci0) * 4u : 0u) + (v_tma ? uint32_t(vi1 - vi0) * 8u : 0u) +
                     (r_tma ? uint32_t(ri1 - ri0) * 4u : 0u);
    mbar_arrive_expect_tx(bar, bytes);
    if (v_tma) bulk_g2s(s.val + (vi0 - va0), P.val + vi0, uint32_t(vi1 - vi0) * 8u, bar, policy);
    if (c_tma) bulk_g2s(s.col + (ci0 - ca0), P.col + ci0, uint32_t(ci1 - ci0) * 4u, bar, policy);
    if (r_tma) bulk_g2s(s.rp + (ri0 - ra0), P.row_ptr + ri0, uint32_t(ri1 - ri0) * 4u, bar, policy);
  }
  const int tid = threadIdx.x, nt = blockDim.x;
  if (c_tma) {
    for (int64_t e = nz0 + tid; e < ci0; e += nt) s.col[e - ca0] = __ldg(P.col + e);
    for (int64_t e = ci1 + tid; e < nz1; e += nt) s.col[e - ca0] = __ldg(P.col + e);
  } else {
    for (int64_t e = nz0 + tid; e < nz1; e += nt) s.col[e - ca0] = __ldg(P.col + e);
  }
  if (v_tma) {
    for (int64_t e = nz0 + tid; e < vi0; e += nt) s.val[e - va0] = __ldg(P.val + e);
    for (int64_t e = vi1 + tid; e < nz1; e += nt) s.val[e - va0] = __ldg(P.val + e);
  } else {
    for (int64_t e = nz0 + tid; e < nz1; e += nt) s.val[e - va0] = __ldg(P.val + e);
  }
  if (r_tma) {
    for (int32_t e = r0 + tid; e < ri0 && e <= r1; e += nt) s.rp[e - ra0] = __ldg(P.row_ptr + e);
    for (int32_t e = max(ri1, ri0) + tid; e <= r1; e += nt) s.rp[e - ra0] = __ldg(P.row_ptr + e);
  } else {
    for (int32_t e = r0 + tid; e <= r1; e += nt) s.rp[e - ra0] = __ldg(P.row_ptr + e);
  }
  return true;
}

// Warp 0 waits until every tile in [lo, hi] published >= target.  Returns
// false (and raises the abort flag) when the watchdog expires.
__device__ __forceinline__ bool mpk_wait(const MpkParams& P, int32_t lo, int32_t hi,
                                         uint32_t target) {
  bool ok = true;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    unsigned long long t0 = 0;
    for (int32_t i = lo + lane; i <= hi; i += 32) {
      int spins = 0;
      while (ld_relaxed_u32(P.progress + i) < target) {
        if (++spins > 8) __nanosleep(64);
        if ((spins & 255) == 0) {
          if (t0 == 0) t0 = globaltimer();
          const volatile unsigned long long* ab = P.queue + 1;
          if (*ab != 0ull) {
            ok = false;
            break;
          }
          if (globaltimer() - t0 > kWatchdogNs) {
            atomicExch(P.queue + 1, 1ull);
            *P.err = 1;
            ok = false;
            break;
          }
        }
      }
      if (!ok) break;
    }
    ok = __all_sync(0xffffffffu, ok);
    fence_acq_rel_gpu();  // acquire: order + invalidate L1 before the gathers
  }
  return ok;
}

template <bool CPLX>
__device__ __forceinline__ void mpk_compute(const MpkParams& P, const PowerCfgDev& C,
                                            const MpkSmem& s, bool staged, int32_t r0, int32_t r1,
                                            int64_t nz0, int p) {
  const int pi = p - 1;
  const int kern = C.kernel[pi];
  const double cre = C.coef_re[pi], cim = C.coef_im[pi];
  const int32_t* scol = s.col - (nz0 & ~int64_t(3));
  const double* sval = s.val - (nz0 & ~int64_t(1));
  const int32_t* srp = s.rp - (r0 & ~3);
  const int64_t w = CPLX ? 2 : 1;
  const double* yin = P.y + int64_t(C.in_slot[pi]) * P.ldy;
  const double* ypv = P.y + int64_t(C.prev_slot[pi]) * P.ldy;
  double* yout = P.y + int64_t(C.out_slot[pi]) * P.ldy;
  for (int32_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    int32_t k0, k1;
    if (staged) {
      k0 = srp[r];
      k1 = srp[r + 1];
    } else {
      k0 = __ldg(P.row_ptr + r);
      k1 = __ldg(P.row_ptr + r + 1);
    }
    const int32_t* cp = staged ? scol + k0 : P.col + k0;
    const double* vp = staged ? sval + k0 : P.val + k0;
    if constexpr (!CPLX) {
      double t = row_sum_exact(cp, vp, k1 - k0, [yin](int c) { return ld_weak(yin + c); });
      if (kern == LMPK_KERNEL_CHEB) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(ypv + r));
      yout[r] = t;
      if (P.use_acc) P.acc[r] = __dadd_rn(ld_cg(P.acc + r), __dmul_rn(cre, t));
    } else {
      const double2* yin2 = reinterpret_cast<const double2*>(yin);
      double2 t = row_sum_exact_c(cp, vp, k1 - k0, [yin2](int c) { return ld_weak2(yin2 + c); });
      if (kern == LMPK_KERNEL_CHEB) {
        t.x = __dsub_rn(__dmul_rn(2.0, t.x), ld_cg(ypv + w * r));
        t.y = __dsub_rn(__dmul_rn(2.0, t.y), ld_cg(ypv + w * r + 1));
      }
      reinterpret_cast<double2*>(yout)[r] = t;
      if (P.use_acc) {
        // acc += (cre + i cim) * t, real and imaginary parts spelled out
        const double ar = ld_cg(P.acc + w * r), ai = ld_cg(P.acc + w * r + 1);
        const double pr = __dsub_rn(__dmul_rn(cre, t.x), __dmul_rn(cim, t.y));
        const double pim = __dadd_rn(__dmul_rn(cre, t.y), __dmul_rn(cim, t.x));
        P.acc[w * r] = __dadd_rn(ar, pr);
        P.acc[w * r + 1] = __dadd_rn(ai, pim);
      }
    }
  }
}

__device__ __forceinline__ void mpk_publish(const MpkParams& P, int32_t t, int p) {
  __syncthreads();  // all rows of (t, p) stored
  if (threadIdx.x == 0) st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
}

template <bool CPLX>
__global__ void __launch_bounds__(kMpkThreads) mpk_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bars[2];
  __shared__ int32_t s_work[2];
  __shared__ int32_t s_abort;
  const size_t per = mpk_buf_bytes(P.cap, P.rows_cap);
  MpkSmem sb[2] = {carve(smem_raw, P.cap, P.rows_cap), carve(smem_raw + per, P.cap, P.rows_cap)};
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    s_abort = 0;
  }
  __syncthreads();

  if (P.mode == 1) {
    // ---------------- RESIDENT: one tile in smem across all powers
    const uint64_t pol = policy_evict_first();
    for (int it = 0;; ++it) {
      if (threadIdx.x == 0)
        s_work[0] = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
      __syncthreads();
      const int32_t t = s_work[0];
      if (t >= P.n_tiles || s_abort) break;
      const int32_t r0 = __ldg(P.tile_row + t), r1 = __ldg(P.tile_row + t + 1);
      const int64_t nz0 = __ldg(P.row_ptr + r0), nz1 = __ldg(P.row_ptr + r1);
      const bool staged = mpk_stage(P, sb[0], &bars[0], r0, r1, nz0, nz1, pol);
      const int32_t lo = __ldg(P.dep_lo + t), hi = __ldg(P.dep_hi + t);
      mbar_wait(&bars[0], it & 1);
      __syncthreads();
      for (int p = 1; p <= P.n_powers; ++p) {
        if (p > 1) {
          bool ok = mpk_wait(P, lo, hi, P.epoch_base + uint32_t(p - 1));
          if (threadIdx.x == 0 && !ok) s_abort = 1;
          __syncthreads();
          if (s_abort) break;
        }
        mpk_compute<CPLX>(P, C, sb[0], staged, r0, r1, nz0, p);
        mpk_publish(P, t, p);
      }
      __syncthreads();
      if (s_abort) break;
    }
  } else {
    // ---------------- STREAMING: (tile, power) items in skewed-diagonal order
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_drop = policy_evict_first();
    if (threadIdx.x == 0) s_work[0] = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
    __syncthreads();
    int32_t i = s_work[0];
    if (i >= P.n_items) return;
    int32_t code = __ldg(P.items + i);
    int32_t t = code >> 7, p = code & 127;
    int32_t r0 = __ldg(P.tile_row + t), r1 = __ldg(P.tile_row + t + 1);
    int64_t nz0 = __ldg(P.row_ptr + r0), nz1 = __ldg(P.row_ptr + r1);
    bool staged = mpk_stage(P, sb[0], &bars[0], r0, r1, nz0, nz1, p < P.n_powers ? pol_keep : pol_drop);
    for (int it = 0;; ++it) {
      const int b = it & 1;
      if (threadIdx.x == 0) s_work[1] = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
      __syncthreads();
      const int32_t in = s_work[1];
      int32_t tn = 0, pn = 0, r0n = 0, r1n = 0;
      int64_t nz0n = 0, nz1n = 0;
      bool staged_n = false;
      if (in < P.n_items) {  // prefetch the next item's slice into the other buffer
        const int32_t cn = __ldg(P.items + in);
        tn = cn >> 7;
        pn = cn & 127;
        r0n = __ldg(P.tile_row + tn);
        r1n = __ldg(P.tile_row + tn + 1);
        nz0n = __ldg(P.row_ptr + r0n);
        nz1n = __ldg(P.row_ptr + r1n);
        staged_n = mpk_stage(P, sb[b ^ 1], &bars[b ^ 1], r0n, r1n, nz0n, nz1n,
                             pn < P.n_powers ? pol_keep : pol_drop);
      }
      if (p > 1) {
        bool ok = mpk_wait(P, __ldg(P.dep_lo + t), __ldg(P.dep_hi + t), P.epoch_base + uint32_t(p - 1));
        if (threadIdx.x == 0 && !ok) s_abort = 1;
      }
      mbar_wait(&bars[b], (it >> 1) & 1);
      __syncthreads();
      if (s_abort) {
        // never leave the CTA with a bulk copy still landing in its smem
        if (in < P.n_items) mbar_wait(&bars[b ^ 1], ((it + 1) >> 1) & 1);
        break;
      }
      mpk_compute<CPLX>(P, C, sb[b], staged, r0, r1, nz0, p);
      mpk_publish(P, t, p);
      if (in >= P.n_items) break;
      t = tn;
      p = pn;
      r0 = r0n;
      r1 = r1n;
      nz0 = nz0n;
      nz1 = nz1n;
      staged = staged_n;
      __syncthreads();
    }
    // drain a possibly armed prefetch barrier is unnecessary: the kernel ends.
  }
}

// ---------------------------------------------------------------- tiling kernels
__global__ void k_max_row(const int32_t* row_ptr, int32_t n, int* out) {
  int m = 0;
  for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    m = max(m, __ldg(row_ptr + r + 1) - __ldg(row_ptr + r));
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_tile_bounds(const int32_t* row_ptr, int32_t n, int64_t tile_nnz, int32_t nb,
                              int32_t* out) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int64_t target = int64_t(i) * tile_nnz;
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    int32_t mid = lo + ((hi - lo) >> 1);
    if (int64_t(__ldg(row_ptr + mid)) < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[i] = lo;
}

__device__ __forceinline__ int32_t tile_of(const int32_t* tile_row, int32_t n_tiles, int32_t r) {
  // last t with tile_row[t] <= r
  int32_t lo = 0, hi = n_tiles - 1;
  while (lo < hi) {
    int32_t mid = (lo + hi + 1) >> 1;
    if (__ldg(tile_row + mid) <= r)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void k_tile_deps(const int32_t* row_ptr, const int32_t* col, const int32_t* tile_row,
                            int32_t n_tiles, int32_t* dep_lo, int32_t* dep_hi) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_tiles) return;
  const int32_t r0 = __ldg(tile_row + warp), r1 = __ldg(tile_row + warp + 1);
  int32_t mn = INT32_MAX, mx = -1;
  for (int32_t r = r0 + lane; r < r1; r += 32) {
    const int32_t a = __ldg(row_ptr + r), b = __ldg(row_ptr + r + 1);
    if (b > a) {
      mn = min(mn, __ldg(col + a));
      mx = max(mx, __ldg(col + b - 1));
    }
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    int32_t lo = warp, hi = warp;  // always depend on the own tile (Cheb prev/acc)
    if (mx >= 0) {
      lo = min(lo, tile_of(tile_row, n_tiles, mn));
      hi = max(hi, tile_of(tile_row, n_tiles, mx));
    }
    dep_lo[warp] = lo;
    dep_hi[warp] = hi;
  }
}

template <typename T>
static int dmalloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    set_error("cudaMalloc(%zu) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    return LMPK_ERR_NOMEM;
  }
  return LMPK_OK;
}

template <bool CPLX>
static cudaError_t occupancy_t(lmpk_ctx* ctx, int smem, int* occ) {
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, mpk_kernel<CPLX>);
  if (e != cudaSuccess) return e;
  const int max_dyn = ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes);
  if (smem > max_dyn) {
    *occ = 0;
    return cudaSuccess;
  }
  // the attribute is only an upper bound: set it to the device maximum
  e = cudaFuncSetAttribute(mpk_kernel<CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, mpk_kernel<CPLX>, kMpkThreads, smem);
}

static int occupancy(lmpk_ctx* ctx, int cplx, int smem, int* occ) {
  cudaError_t e = cplx ? occupancy_t<true>(ctx, smem, occ) : occupancy_t<false>(ctx, smem, occ);
  if (e != cudaSuccess) {
    cudaGetLastError();  // do not leave a sticky status for later checks
    set_error("occupancy query failed: %s", cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  }
  return LMPK_OK;
}

}  // namespace lmpk

using namespace lmpk;

extern "C" int lmpk_tiling_destroy(lmpk_tiling* t) {
  if (!t) return LMPK_OK;
  cudaFree(t->d_tile_row);
  cudaFree(t->d_dep_lo);
  cudaFree(t->d_dep_hi);
  cudaFree(t->d_items);
  cudaFree(t->d_progress);
  delete t;
  return LMPK_OK;
}

// Build tiles with at most tile_nnz nonzeros / rows_cap rows and their deps.
static int build_tiles(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr,
                       const int32_t* col, int64_t nnz, int32_t tile_nnz, int32_t max_row,
                       int32_t rows_cap, cudaStream_t st) {
  // boundaries at nnz multiples of (tile_nnz - max_row + 1) keep every tile <= tile_nnz
  int64_t step = std::max<int64_t>(1, int64_t(tile_nnz) - std::max(max_row - 1, 0));
  if (max_row > tile_nnz / 2) step = tile_nnz;  // long rows -> oversize tiles run from global
  const int32_t nb = static_cast<int32_t>(std::max<int64_t>(1, (nnz + step - 1) / step));
  int32_t* d_b = nullptr;
  LMPK_TRY(dmalloc(&d_b, nb));
  k_tile_bounds<<<div_up(nb, 256), 256, 0, st>>>(row_ptr, n, step, nb, d_b);
  std::vector<int32_t> hb(nb);
  cudaError_t e = cudaMemcpyAsync(hb.data(), d_b, nb * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_b);
  if (e != cudaSuccess) {
    set_error("tile bounds: %s", cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  }
  launch_count_add(ctx, 1);
  std::vector<int32_t> tr;
  tr.reserve(nb + 2);
  tr.push_back(0);
  for (int32_t i = 1; i < nb; ++i)
    if (hb[i] > tr.back() && hb[i] < n) tr.push_back(hb[i]);
  if (n > tr.back() || tr.size() == 1) tr.push_back(n);
  // split by row capacity
  std::vector<int32_t> out;
  out.reserve(tr.size() * 2);
  out.push_back(tr[0]);
  for (size_t i = 1; i < tr.size(); ++i) {
    int32_t a = out.back(), b = tr[i];
    while (b - a > rows_cap) {
      a += rows_cap;
      out.push_back(a);
    }
    if (b > out.back()) out.push_back(b);
  }
  if (out.size() == 1) out.push_back(n);  // n == 0
  const int32_t n_tiles = static_cast<int32_t>(out.size() - 1);
  T->h_tile_row = out;
  LMPK_TRY(dmalloc(&T->d_tile_row, n_tiles + 1));
  LMPK_TRY(dmalloc(&T->d_dep_lo, n_tiles));
  LMPK_TRY(dmalloc(&T->d_dep_hi, n_tiles));
  LMPK_TRY(dmalloc(&T->d_progress, n_tiles));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_row, out.data(), (n_tiles + 1) * 4,
                                  cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(T->d_progress, 0, n_tiles * 4, st));
  k_tile_deps<<<div_up(int64_t(n_tiles) * 32, 256), 256, 0, st>>>(row_ptr, col, T->d_tile_row,
                                                                   n_tiles, T->d_dep_lo, T->d_dep_hi);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  T->h_dep_lo.resize(n_tiles);
  T->h_dep_hi.resize(n_tiles);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->h_dep_lo.data(), T->d_dep_lo, n_tiles * 4,
                                  cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->h_dep_hi.data(), T->d_dep_hi, n_tiles * 4,
                                  cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  T->info.n_tiles = n_tiles;
  return LMPK_OK;
}

// max over t of (the p_m-1 step forward dependency chain) - t, using the
// prefix max of dep_hi (monotone, conservative).
static int32_t chain_reach(const std::vector<int32_t>& dep_hi, int32_t p_m, int32_t* max_fwd) {
  const int32_t nt = static_cast<int32_t>(dep_hi.size());
  std::vector<int32_t> H(nt);
  int32_t run = 0, mf = 0;
  for (int32_t t = 0; t < nt; ++t) {
    run = std::max(run, dep_hi[t]);
    H[t] = run;
    mf = std::max(mf, dep_hi[t] - t);
  }
  *max_fwd = mf;
  int32_t worst = 0;
  for (int32_t t = 0; t < nt; ++t) {
    int32_t c = t;
    for (int32_t j = 1; j < p_m; ++j) {
      int32_t nc = H[c];
      if (nc == c) break;
      c = nc;
    }
    worst = std::max(worst, c - t);
  }
  return worst;
}

extern "C" int lmpk_tiling_create(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr,
                                  const int32_t* col, int32_t p_m, int32_t tile_nnz_hint,
                                  int32_t ctas_per_sm_hint, int mode_flags, lmpk_tiling** out,
                                  lmpk_tiling_info* info, void* stream) {
  LMPK_ARG_CHECK(ctx && out, "lmpk_tiling_create: NULL ctx/out");
  LMPK_ARG_CHECK(p_m >= 1 && p_m <= LMPK_MAX_POWERS, "p_m must be in [1, %d]", LMPK_MAX_POWERS);
  LMPK_ARG_CHECK(n >= 0, "n must be >= 0");
  *out = nullptr;
  cudaStream_t st = as_stream(stream);
  int32_t h_nnz = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&h_nnz, row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
  int* d_max = nullptr;
  LMPK_TRY(dmalloc(&d_max, 1));
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_max, 0, 4, st));
  if (n > 0) k_max_row<<<std::min(div_up(n, 256), ctx->sm_count * 8), 256, 0, st>>>(row_ptr, n, d_max);
  int32_t max_row = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&max_row, d_max, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_max);
  launch_count_add(ctx, 1);
  const int64_t nnz = h_nnz;
  const double avg = n > 0 ? double(nnz) / double(n) : 1.0;

  bool want_stream = (mode_flags & LMPK_FLAG_MODE_STREAM) != 0;
  bool want_res = (mode_flags & LMPK_FLAG_MODE_RESIDENT) != 0;
  const bool cplx = (mode_flags & LMPK_FLAG_COMPLEX) != 0;
  const int usable_sm = ctx->max_smem_sm - 2048;  // static smem + driver reserve per CTA

  lmpk_tiling* T = nullptr;
  int mode = 0;
  int c = 0;
  int32_t tile = 0, rows_cap = 0;
  int smem = 0;
  int32_t mfwd = 0, creach = 0;
  // candidate list: resident first (unless streaming is forced)
  struct Cand {
    int mode, c;
    int32_t tile;
  };
  std::vector<Cand> cands;
  auto res_tile = [&](int cc) {
    int per = std::min(usable_sm / cc - 1024, ctx->max_smem_block - 1024);
    // per = 12*T + 4*(T/avg*1.25+40) + ~200  ->  T
    double bytes_per_nnz = 12.0 + 4.0 * 1.25 / std::max(avg, 0.25);
    return static_cast<int32_t>((per - 512) / bytes_per_nnz);
  };
  if (!want_stream) {
    if (tile_nnz_hint > 0 && ctas_per_sm_hint > 0) {
      cands.push_back({1, ctas_per_sm_hint, tile_nnz_hint});
    } else {
      int c_list[3] = {ctas_per_sm_hint > 0 ? ctas_per_sm_hint : 2, 1, 3};
      for (int cc : c_list) cands.push_back({1, cc, tile_nnz_hint > 0 ? tile_nnz_hint : res_tile(cc)});
    }
  }
  if (!want_res) {
    int cc = ctas_per_sm_hint > 0 ? ctas_per_sm_hint : 4;
    int32_t tt = tile_nnz_hint > 0 ? tile_nnz_hint
                                   : static_cast<int32_t>(std::max(512.0, std::min(avg * 4 * kMpkThreads, 12288.0)));
    cands.push_back({2, cc, tt});
  }
  for (Cand cd : cands) {
    cd.tile &= ~3;  // multiple of 4 elements
    if (cd.tile < 16) continue;
    const int32_t rc = static_cast<int32_t>(std::min<double>(cd.tile / std::max(avg, 0.25) * 1.25 + 40, cd.tile + 64.0));
    // resident mode uses one buffer; streaming double-buffers
    const int smem_need = cd.mode == 1 ? static_cast<int>(mpk_buf_bytes(cd.tile, rc))
                                       : static_cast<int>(2 * mpk_buf_bytes(cd.tile, rc));
    if (smem_need > ctx->max_smem_block) continue;
    int occ = 0;
    LMPK_TRY(occupancy(ctx, cplx, smem_need, &occ));
    if (occ < 1) continue;
    lmpk_tiling* cand = new lmpk_tiling();
    cand->ctx = ctx;
    cand->n = n;
    int rc2 = build_tiles(ctx, cand, n, row_ptr, col, nnz, cd.tile, max_row, rc, st);
    if (rc2 != LMPK_OK) {
      lmpk_tiling_destroy(cand);
      return rc2;
    }
    int32_t mf = 0;
    int32_t cr = chain_reach(cand->h_dep_hi, p_m, &mf);
    const int grid = std::min(occ, cd.c) * ctx->sm_count;
    bool ok = true;
    if (cd.mode == 1) {
      ok = (occ >= cd.c) && (cr < grid - 1) && max_row <= cd.tile / 2;
    }
    if (ok) {
      T = cand;
      mode = cd.mode;
      c = std::min(occ, cd.c);
      tile = cd.tile;
      rows_cap = rc;
      smem = smem_need;
      mfwd = mf;
      creach = cr;
      break;
    }
    lmpk_tiling_destroy(cand);
  }
  if (!T) {
    set_error("lmpk_tiling_create: no feasible tiling (mode flags 0x%x)", mode_flags);
    return want_res ? LMPK_ERR_UNSUPPORTED : LMPK_ERR_ARG;
  }
  T->rows_cap = rows_cap;
  T->info.p_m = p_m;
  T->info.mode = mode;
  T->info.block = kMpkThreads;
  T->info.smem_bytes = smem;
  T->info.tile_nnz_cap = tile;
  T->info.max_fwd_reach = mfwd;
  T->info.chain_reach = creach;
  T->info.max_row_nnz = max_row;
  T->info.nnz = nnz;
  const int32_t nt = T->info.n_tiles;
  if (mode == 1) {
    T->info.grid = c * ctx->sm_count;
  } else {
    // skewed diagonal order key (t + p*D, p), D = max forward reach
    std::vector<int64_t> keys;
    keys.reserve(int64_t(nt) * p_m);
    const int64_t D = std::max(mfwd, 0);
    for (int32_t t = 0; t < nt; ++t)
      for (int32_t p = 1; p <= p_m; ++p) keys.push_back(((t + p * D) << 8) | p);
    std::vector<int32_t> order(keys.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return keys[a] < keys[b]; });
    std::vector<int32_t> items(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
      const int32_t t = order[i] / p_m, p = order[i] % p_m + 1;
      items[i] = (t << 7) | p;
    }
    LMPK_TRY(dmalloc(&T->d_items, items.size()));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_items, items.data(), items.size() * 4,
                                    cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    T->info.grid = static_cast<int32_t>(std::min<int64_t>(int64_t(c) * ctx->sm_count, int64_t(nt) * p_m));
  }
  if (nt >= (1 << 24)) {
    lmpk_tiling_destroy(T);
    set_error("too many tiles (%d)", nt);
    return LMPK_ERR_UNSUPPORTED;
  }
  if (info) *info = T->info;
  *out = T;
  return LMPK_OK;
}

extern "C" int lmpk_tiling_geometry(const lmpk_tiling* t, int32_t* tile_row, int32_t* dep_lo,
                                    int32_t* dep_hi) {
  LMPK_ARG_CHECK(t != nullptr, "tiling is NULL");
  const size_t nt = t->info.n_tiles;
  if (tile_row) memcpy(tile_row, t->h_tile_row.data(), (nt + 1) * 4);
  if (dep_lo) memcpy(dep_lo, t->h_dep_lo.data(), nt * 4);
  if (dep_hi) memcpy(dep_hi, t->h_dep_hi.data(), nt * 4);
  return LMPK_OK;
}

extern "C" int lmpk_mpk_run(lmpk_ctx* ctx, const lmpk_tiling* T, const int32_t* row_ptr,
                            const int32_t* col, const double* val, double* y, int64_t ldy,
                            int32_t n_slots, const lmpk_power_cfg* cfg, double* acc, int use_acc,
                            int flags, void* stream) {
  LMPK_ARG_CHECK(ctx && T && cfg, "lmpk_mpk_run: NULL ctx/tiling/cfg");
  LMPK_ARG_CHECK(T->ctx == ctx, "tiling belongs to another ctx");
  const int32_t P = cfg->n_powers;
  LMPK_ARG_CHECK(P >= 1 && P <= T->info.p_m, "n_powers %d exceeds the tiling's p_m %d", P, T->info.p_m);
  const bool cplx = (flags & LMPK_FLAG_COMPLEX) != 0;
  LMPK_ARG_CHECK(ldy >= int64_t(T->n) * (cplx ? 2 : 1), "ldy too small");
  LMPK_ARG_CHECK(!use_acc || acc != nullptr, "use_acc requires acc");
  PowerCfgDev C;
  memset(&C, 0, sizeof(C));
  for (int i = 0; i < P; ++i) {
    const int32_t o = cfg->out_slot[i], a = cfg->in_slot[i], b = cfg->prev_slot[i];
    LMPK_ARG_CHECK(o >= 0 && o < n_slots && a >= 0 && a < n_slots && b >= 0 && b < n_slots,
                   "slot index out of range at power %d", i + 1);
    LMPK_ARG_CHECK(o != a, "in_vec and out_vec must not alias (power %d)", i + 1);
    LMPK_ARG_CHECK(cfg->kernel[i] == LMPK_KERNEL_SPMV || cfg->kernel[i] == LMPK_KERNEL_CHEB,
                   "unknown kernel id %d", cfg->kernel[i]);
    C.out_slot[i] = o;
    C.in_slot[i] = a;
    C.prev_slot[i] = b;
    C.kernel[i] = cfg->kernel[i];
    C.coef_re[i] = cfg->acc_coef_re[i];
    C.coef_im[i] = cplx ? cfg->acc_coef_im[i] : 0.0;
  }
  if (T->n == 0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  lmpk_tiling* Tm = const_cast<lmpk_tiling*>(T);
  ctx->epoch += 1;
  if (ctx->epoch >= (1u << 24)) {  // counter wrap: reset progress words
    LMPK_CHECK_CUDA(cudaMemsetAsync(Tm->d_progress, 0, size_t(T->info.n_tiles) * 4, st));
    ctx->epoch = 1;
  }
  MpkParams Pm;
  Pm.row_ptr = row_ptr;
  Pm.col = col;
  Pm.val = val;
  Pm.y = y;
  Pm.ldy = ldy;
  Pm.acc = acc;
  Pm.use_acc = use_acc ? 1 : 0;
  Pm.tile_row = T->d_tile_row;
  Pm.dep_lo = T->d_dep_lo;
  Pm.dep_hi = T->d_dep_hi;
  Pm.items = T->d_items;
  Pm.progress = Tm->d_progress;
  Pm.queue = reinterpret_cast<unsigned long long*>(ctx->queue_ctr);
  Pm.queue_base = ctx->queue_base;
  Pm.epoch_base = ctx->epoch * kEpochStride;
  Pm.n_tiles = T->info.n_tiles;
  Pm.n_items = T->info.n_tiles * P;
  Pm.n_powers = P;
  Pm.mode = T->info.mode;
  Pm.cap = T->info.tile_nnz_cap;
  Pm.rows_cap = T->rows_cap;
  Pm.use_tma = (flags & LMPK_FLAG_NO_TMA) ? 0 : 1;
  if ((reinterpret_cast<uintptr_t>(col) & 15) || (reinterpret_cast<uintptr_t>(val) & 15) ||
      (reinterpret_cast<uintptr_t>(row_ptr) & 15))
    Pm.use_tma = 0;
  Pm.err = ctx->err.dev;
  if (Pm.mode == 2 && P < T->info.p_m) {
    // item list was built for p_m powers: the queue order restricted to
    // p <= P is still topologically valid, but it contains P' > P items;
    // rebuild lazily is avoided by requiring n_powers == p_m in streaming.
    LMPK_ARG_CHECK(false, "streaming tiling built for p_m=%d cannot run %d powers", T->info.p_m, P);
  }
  const int grid = T->info.grid;
  const int smem = T->info.smem_bytes;
  void* args[] = {&Pm, &C};
  cudaError_t e;
  if (Pm.mode == 1) {
    e = cplx ? cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mpk_kernel<true>), dim3(grid),
                                           dim3(kMpkThreads), args, smem, st)
             : cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mpk_kernel<false>), dim3(grid),
                                           dim3(kMpkThreads), args, smem, st);
  } else {
    e = cplx ? cudaLaunchKernel(reinterpret_cast<void*>(mpk_kernel<true>), dim3(grid),
                                dim3(kMpkThreads), args, smem, st)
             : cudaLaunchKernel(reinterpret_cast<void*>(mpk_kernel<false>), dim3(grid),
                                dim3(kMpkThreads), args, smem, st);
  }
  if (e != cudaSuccess) {
    set_error("mpk launch failed: %s (grid %d, smem %d)", cudaGetErrorString(e), grid, smem);
    return LMPK_ERR_CUDA;
  }
  launch_count_add(ctx, 1);
  const int64_t work = (Pm.mode == 1) ? T->info.n_tiles : int64_t(T->info.n_tiles) * P;
  ctx->queue_base += uint64_t(work + grid);
  return LMPK_OK;
}

// Host-side check after the caller synchronized the stream.
extern "C" int lmpk_ctx_check(lmpk_ctx* ctx, void* stream) {
  LMPK_ARG_CHECK(ctx != nullptr, "ctx is NULL");
  LMPK_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  int rc = ctx_check_device_error(ctx, "mpk");
  if (rc != LMPK_OK) {
    // the aborted launch left the queue counter inconsistent: reset it
    cudaMemset(ctx->queue_ctr, 0, 64);
    cudaDeviceSynchronize();
    ctx->queue_base = 0;
  }
  return rc;
}
