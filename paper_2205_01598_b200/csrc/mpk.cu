// mpk.cu -- level-blocked matrix power kernel for sm_100a.
//
// Reference: the diagonal Lp-diagram walk of pkg/src/levelmpk/schedule.py:91-99
// executed by the p2p walker _walk/_wait_all (executor.py:84-150) over the
// flat ExecPlan (plan.py:184-370).  The GPU form:
//
//   * the level-permuted matrix is cut into contiguous row TILES (multiples
//     of 32 rows) sized to the shared-memory budget and re-laid out once as
//     "tile-SELL-32" blocks: per 32-row slice the entries are stored
//     column-major (entry j of row i at slice_base + 32*j + i), padded to the
//     slice's longest row.  One contiguous block per tile -> ONE TMA bulk
//     copy stages it; warps read it conflict-free; each row is still summed
//     in its CRS storage order (padding is predicated away), so results stay
//     bitwise identical to the reference;
//   * tile t's dependency range [dep_lo(t), dep_hi(t)] is the set of tiles
//     owning its column indices (level confinement, Eq. 4 of the paper,
//     keeps it narrow: a tile couples only to its own and adjacent levels);
//   * a persistent grid of CTAs replaces the reference's W threads.  Each
//     (tile, power) node publishes an epoch-tagged counter with a gpu-scope
//     release after its rows are stored; a consumer polls its dependency
//     range with relaxed loads and then issues an acquire fence (which also
//     invalidates the SM's L1 so later gathers see fresh vector data).  This
//     is the device form of conditions (A)/(B)/(C): "tile t at power p only
//     after tiles dep_lo..dep_hi finished p-1" (schedule.py:195-240);
//   * RESIDENT mode (cooperative launch): a CTA grabs the next tile in order,
//     stages its block into shared memory ONCE and computes all p_m powers on
//     it -> the matrix is read from HBM once.  Deadlock freedom: the chain
//     reach of the p_m-1 dependency steps must be smaller than the number of
//     co-resident CTAs (checked at planning time);
//   * STREAMING mode: CTAs grab (tile, power) items from a queue ordered by
//     the skewed diagonal key (t + p*M, p), M = D + slack, D = max forward
//     reach -- topologically valid for any M >= D; the slack keeps dependent
//     items ~2 grids apart so the queue is never a serial chain.  The block
//     is re-staged per power (served from L2 inside the diagonal window: the
//     reference's cache blocking with the 126 MB L2 as the cache).
//     Deadlock-free without co-residency;
//   * SWEEP (LMPK_FLAG_SWEEP): n_powers dependency-free passes, one launch per
//     power -- the blocking-free "k back-to-back SpMVs" baseline on the same
//     tiles and the same row kernel.
#include <string.h>

#include <algorithm>
#include <numeric>

#include "lmpk_internal.cuh"

namespace lmpk {

constexpr uint32_t kEpochStride = 128;  // > LMPK_MAX_POWERS
constexpr unsigned long long kWatchdogNs = 8ull * 1000 * 1000 * 1000;
constexpr int kMaxThreads = 512;
constexpr bool kPairSlices = false;  // measured slower on cfg2 (load imbalance per item)

struct PowerCfgDev {
  int32_t out_slot[LMPK_MAX_POWERS];
  int32_t in_slot[LMPK_MAX_POWERS];
  int32_t prev_slot[LMPK_MAX_POWERS];
  int32_t kernel[LMPK_MAX_POWERS];
  double coef_re[LMPK_MAX_POWERS];
  double coef_im[LMPK_MAX_POWERS];
};

struct MpkParams {
  const unsigned char* blocks;
  const int64_t* tile_ofs;
  const int32_t* tile_E;
  const int32_t* tile_row;
  const int32_t* dep_lo;
  const int32_t* dep_hi;
  const int32_t* items;
  double* y;
  int64_t ldy;
  double* acc;
  int32_t use_acc;
  uint32_t* progress;
  unsigned long long* queue;  // [0] work counter, [1] abort flag
  unsigned long long queue_base;
  uint32_t epoch_base;
  int32_t n_tiles;
  int32_t n_items;
  int32_t n_powers;
  int32_t mode;      // 1 resident, 2 streaming, 3 sweep (one power, no deps)
  int32_t smem_cap;  // bytes of one staging buffer
  int32_t n_slots;   // pipelined kernel: ring slots
  int32_t use_tma;
  int* err;          // host-mapped
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__host__ __device__ inline int64_t align16(int64_t b) { return (b + 15) & ~int64_t(15); }

// Block layout of a tile with ns slices and E padded entries:
//   [slice_off int32 x ns4][lens uint16 x 32*ns] | align16 | [col int32 x E][val f64 x E]
__host__ __device__ inline int64_t blk_col_off(int32_t ns) {
  const int32_t ns4 = (ns + 3) & ~3;
  return align16(int64_t(ns4) * 4 + int64_t(ns) * 64);
}
__host__ __device__ inline int64_t blk_bytes(int32_t ns, int64_t E) {
  return (blk_col_off(ns) + E * 12 + 127) & ~int64_t(127);
}

// Stage tile block [ofs, ofs+bytes) into smem with one bulk copy.  Thread 0
// arms the mbarrier (exactly one phase per call).  Returns false if the block
// does not fit -- the tile is then computed straight from global memory.
__device__ __forceinline__ bool stage_block(const MpkParams& P, unsigned char* buf, uint64_t* bar,
                                            int64_t ofs, int64_t bytes, uint64_t policy) {
  if (bytes > P.smem_cap) {
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, 0);
    return false;
  }
  if (P.use_tma) {
    if (threadIdx.x == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(bar, uint32_t(bytes));
      bulk_g2s(buf, P.blocks + ofs, uint32_t(bytes), bar, policy);
    }
  } else {
    const int4* src = reinterpret_cast<const int4*>(P.blocks + ofs);
    int4* dst = reinterpret_cast<int4*>(buf);
    for (int64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) dst[i] = __ldg(src + i);
    if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, 0);
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
        if (++spins > 4) __nanosleep(32);
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

// One power step over a staged (or global) tile block: warps stride over the
// 32-row slices, lane = row.  Entries j of the slice's rows are consecutive
// in the block, so col/val reads are conflict-free 128/256-byte rows.
template <bool CPLX>
__device__ __forceinline__ void tile_power(const MpkParams& P, const PowerCfgDev& C,
                                           const unsigned char* blk, int32_t r0, int32_t r1,
                                           int32_t E, int p, int wid, int nwarps) {
  const int pi = p - 1;
  const int kern = C.kernel[pi];
  const double cre = C.coef_re[pi], cim = C.coef_im[pi];
  const int32_t ns = (r1 - r0 + 31) >> 5;
  const int32_t* soff = reinterpret_cast<const int32_t*>(blk);
  const uint16_t* lens = reinterpret_cast<const uint16_t*>(blk + ((ns + 3) & ~3) * 4);
  const int64_t co = blk_col_off(ns);
  const int32_t* cols = reinterpret_cast<const int32_t*>(blk + co);
  const double* vals = reinterpret_cast<const double*>(blk + co + int64_t(E) * 4);
  const double* yin = P.y + int64_t(C.in_slot[pi]) * P.ldy;
  const double* ypv = P.y + int64_t(C.prev_slot[pi]) * P.ldy;
  double* yout = P.y + int64_t(C.out_slot[pi]) * P.ldy;
  const int lane = threadIdx.x & 31;
  if constexpr (!CPLX && kPairSlices) {
    // Real vectors: a warp advances TWO slices (s, s + nwarps) at a time so
    // twice as many independent gathers are in flight per lane; each row's
    // sum is still the sequential storage-order chain.
    auto finish = [&](int32_t row, double t) {
      if (row < r1) {
        if (kern == LMPK_KERNEL_CHEB) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(ypv + row));
        yout[row] = t;
        if (P.use_acc) P.acc[row] = __dadd_rn(ld_cg(P.acc + row), __dmul_rn(cre, t));
      }
    };
    for (int32_t s = wid; s < ns; s += 2 * nwarps) {
      const int32_t s2 = s + nwarps;
      const bool has2 = s2 < ns;
      const int la = lens[s * 32 + lane];
      const int lb = has2 ? lens[s2 * 32 + lane] : 0;
      const int w = __reduce_max_sync(0xffffffffu, max(la, lb));
      const int32_t* ca = cols + soff[s] + lane;
      const double* va = vals + soff[s] + lane;
      const int32_t* cb = cols + (has2 ? soff[s2] : 0) + lane;
      const double* vb = vals + (has2 ? soff[s2] : 0) + lane;
      double ta = 0.0, tb = 0.0;
      for (int j0 = 0; j0 < w; j0 += 8) {
        double xa[8], xb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < la) xa[j] = ld_weak(yin + ca[(j0 + j) * 32]);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < lb) xb[j] = ld_weak(yin + cb[(j0 + j) * 32]);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < la) ta = __dadd_rn(ta, __dmul_rn(va[(j0 + j) * 32], xa[j]));
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < lb) tb = __dadd_rn(tb, __dmul_rn(vb[(j0 + j) * 32], xb[j]));
      }
      finish(r0 + s * 32 + lane, ta);
      if (has2) finish(r0 + s2 * 32 + lane, tb);
    }
    return;
  }
  for (int32_t s = wid; s < ns; s += nwarps) {
    const int32_t row = r0 + s * 32 + lane;
    const int len = lens[s * 32 + lane];
    const int w = __reduce_max_sync(0xffffffffu, len);
    const int32_t* cs = cols + soff[s] + lane;
    const double* vs = vals + soff[s] + lane;
    if constexpr (!CPLX) {
      double t = 0.0;
      // columns first, all gathers in flight, values read only when the
      // gathered operands return (keeps the register footprint small)
      for (int j0 = 0; j0 < w; j0 += 8) {
        int cc[8];
        double xx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < w) cc[j] = cs[(j0 + j) * 32];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < len) xx[j] = ld_weak(yin + cc[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (j0 + j < len) t = __dadd_rn(t, __dmul_rn(vs[(j0 + j) * 32], xx[j]));
      }
      if (row < r1) {
        if (kern == LMPK_KERNEL_CHEB) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(ypv + row));
        yout[row] = t;
        if (P.use_acc) P.acc[row] = __dadd_rn(ld_cg(P.acc + row), __dmul_rn(cre, t));
      }
    } else {
      const double2* yin2 = reinterpret_cast<const double2*>(yin);
      double tr = 0.0, ti = 0.0;
      for (int j0 = 0; j0 < w; j0 += 4) {
        int cc[4];
        double vv[4];
        double2 xx[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j0 + j < w) {
            cc[j] = cs[(j0 + j) * 32];
            vv[j] = vs[(j0 + j) * 32];
          }
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j0 + j < len) xx[j] = ld_weak2(yin2 + cc[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j0 + j < len) {
            tr = __dadd_rn(tr, __dmul_rn(vv[j], xx[j].x));
            ti = __dadd_rn(ti, __dmul_rn(vv[j], xx[j].y));
          }
      }
      if (row < r1) {
        const int64_t r2 = 2 * int64_t(row);
        if (kern == LMPK_KERNEL_CHEB) {
          tr = __dsub_rn(__dmul_rn(2.0, tr), ld_cg(ypv + r2));
          ti = __dsub_rn(__dmul_rn(2.0, ti), ld_cg(ypv + r2 + 1));
        }
        reinterpret_cast<double2*>(yout)[row] = make_double2(tr, ti);
        if (P.use_acc) {
          // acc += (cre + i cim) * t with the products spelled out
          const double ar = ld_cg(P.acc + r2), ai = ld_cg(P.acc + r2 + 1);
          const double pr = __dsub_rn(__dmul_rn(cre, tr), __dmul_rn(cim, ti));
          const double pim = __dadd_rn(__dmul_rn(cre, ti), __dmul_rn(cim, tr));
          P.acc[r2] = __dadd_rn(ar, pr);
          P.acc[r2 + 1] = __dadd_rn(ai, pim);
        }
      }
    }
  }
}

__device__ __forceinline__ void mpk_publish(const MpkParams& P, int32_t t, int p) {
  __syncthreads();  // all rows of (t, p) stored
  if (threadIdx.x == 0) st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
}

template <bool CPLX>
__global__ void __launch_bounds__(kMaxThreads, 2) mpk_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bars[2];
  __shared__ int32_t s_work[2];
  __shared__ int32_t s_abort;
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    s_abort = 0;
  }
  __syncthreads();
  unsigned char* buf0 = smem_raw;
  unsigned char* buf1 = smem_raw + P.smem_cap;

  if (P.mode == 1) {
    // ---------------- RESIDENT: one tile in smem across all powers
    const uint64_t pol = policy_evict_first();
    for (int it = 0;; ++it) {
      if (threadIdx.x == 0) s_work[0] = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
      __syncthreads();
      const int32_t t = s_work[0];
      if (t >= P.n_tiles || s_abort) break;
      const int32_t r0 = __ldg(P.tile_row + t), r1 = __ldg(P.tile_row + t + 1);
      const int64_t ofs = __ldg(P.tile_ofs + t), bytes = __ldg(P.tile_ofs + t + 1) - ofs;
      const int32_t E = __ldg(P.tile_E + t);
      const bool staged = stage_block(P, buf0, &bars[0], ofs, bytes, pol);
      const int32_t lo = __ldg(P.dep_lo + t), hi = __ldg(P.dep_hi + t);
      mbar_wait(&bars[0], it & 1);
      __syncthreads();
      const unsigned char* blk = staged ? buf0 : P.blocks + ofs;
      for (int p = 1; p <= P.n_powers; ++p) {
        if (p > 1) {
          const bool ok = mpk_wait(P, lo, hi, P.epoch_base + uint32_t(p - 1));
          if (threadIdx.x == 0 && !ok) s_abort = 1;
          __syncthreads();
          if (s_abort) break;
        }
        tile_power<CPLX>(P, C, blk, r0, r1, E, p, threadIdx.x >> 5, blockDim.x >> 5);
        mpk_publish(P, t, p);
      }
      __syncthreads();
      if (s_abort) break;
    }
    return;
  }
  // ---------------- STREAMING / SWEEP: items in queue order, double-buffered
  // Sweep items are assigned statically (blockIdx + it*grid).  Streaming
  // grabs are issued two items ahead so the queue atomic's round trip
  // overlaps the current item's work; a CTA always computes its oldest held
  // item, which keeps the in-order deadlock argument intact.
  const uint64_t pol_keep = policy_evict_last();
  const uint64_t pol_drop = policy_evict_first();
  const bool sweep = P.mode == 3;
  auto decode = [&](int32_t i, int32_t& t, int32_t& p) {
    if (sweep) {
      t = i;
      p = 1;
    } else {
      const int32_t code = __ldg(P.items + i);
      t = code >> 7;
      p = code & 127;
    }
  };
  auto grab = [&]() -> int32_t { return int32_t(atomicAdd(P.queue, 1ull) - P.queue_base); };
  int32_t i_cur, i_next;
  if (sweep) {
    i_cur = blockIdx.x;
    i_next = blockIdx.x + gridDim.x;
  } else {
    if (threadIdx.x == 0) {
      const int32_t a = grab();
      s_work[0] = a;
      s_work[1] = a < P.n_items ? grab() : P.n_items;
    }
    __syncthreads();
    i_cur = s_work[0];
    i_next = s_work[1];
  }
  if (i_cur >= P.n_items) return;
  int32_t t, p;
  decode(i_cur, t, p);
  int64_t ofs = __ldg(P.tile_ofs + t);
  bool staged = stage_block(P, buf0, &bars[0], ofs, __ldg(P.tile_ofs + t + 1) - ofs,
                            (sweep || p == P.n_powers) ? pol_drop : pol_keep);
  for (int it = 0;; ++it) {
    const int b = it & 1;
    unsigned char* cur = b ? buf1 : buf0;
    unsigned char* nxt = b ? buf0 : buf1;
    const bool has_next = i_next < P.n_items;
    unsigned long long ticket = 0;
    if (!sweep && threadIdx.x == 0 && has_next) ticket = atomicAdd(P.queue, 1ull);  // item it+2
    int32_t tn = 0, pn = 0;
    int64_t ofsn = 0;
    bool staged_n = false;
    if (has_next) {  // prefetch the next item's block into the other buffer
      decode(i_next, tn, pn);
      ofsn = __ldg(P.tile_ofs + tn);
      staged_n = stage_block(P, nxt, &bars[b ^ 1], ofsn, __ldg(P.tile_ofs + tn + 1) - ofsn,
                             (sweep || pn == P.n_powers) ? pol_drop : pol_keep);
    }
    if (p > 1) {
      const bool ok = mpk_wait(P, __ldg(P.dep_lo + t), __ldg(P.dep_hi + t), P.epoch_base + uint32_t(p - 1));
      if (threadIdx.x == 0 && !ok) s_abort = 1;
    }
    mbar_wait(&bars[b], (it >> 1) & 1);
    __syncthreads();
    if (s_abort) {
      // never leave the CTA with a bulk copy still landing in its smem
      if (has_next) mbar_wait(&bars[b ^ 1], ((it + 1) >> 1) & 1);
      break;
    }
    const int32_t r0 = __ldg(P.tile_row + t), r1 = __ldg(P.tile_row + t + 1);
    tile_power<CPLX>(P, C, staged ? cur : P.blocks + ofs, r0, r1, __ldg(P.tile_E + t), p, threadIdx.x >> 5,
                     blockDim.x >> 5);
    int32_t i_after;
    if (sweep) {
      i_after = i_next + gridDim.x;
      __syncthreads();
    } else {
      if (threadIdx.x == 0) s_work[it & 1] = has_next ? int32_t(ticket - P.queue_base) : P.n_items;
      mpk_publish(P, t, p);  // includes the __syncthreads that publishes s_work
      i_after = s_work[it & 1];
    }
    if (!has_next) break;
    i_cur = i_next;
    i_next = i_after;
    t = tn;
    p = pn;
    ofs = ofsn;
    staged = staged_n;
  }
}

// ---------------------------------------------------------------- pipelined streaming / sweep
// One producer warp + NC consumer warps per CTA (one CTA per SM).  The
// producer grabs items in queue order, stages each tile block into a ring
// slot with one TMA bulk copy, waits for the item's dependencies (relaxed
// polls + acquire fence, which also invalidates L1) and then arrives on the
// slot's FULL mbarrier.  Consumer warps flow through the ring without any
// CTA-wide barrier: each computes its share of the slices, and the last warp
// to finish an item (acq_rel counter in smem) publishes the item's progress
// word with a gpu-scope release; every warp arrives on the slot's EMPTY
// mbarrier so the producer can refill it.  Deadlock freedom: a CTA's
// consumers never wait on other CTAs, and the producer only waits for the
// dependencies of the oldest item it has not yet released, whose
// dependencies precede it in the global queue order.
constexpr int kPipeMaxSlots = 8;
#ifndef LMPK_NC
#define LMPK_NC 24
#endif
constexpr int kPipeConsumers = LMPK_NC;

__device__ __forceinline__ bool warp_wait_deps(const MpkParams& P, int32_t lo, int32_t hi,
                                               uint32_t target) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  unsigned long long t0 = 0;
  for (int32_t i = lo + lane; i <= hi; i += 32) {
    int spins = 0;
    while (ld_relaxed_u32(P.progress + i) < target) {
      if (++spins > 4) __nanosleep(32);
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
  fence_acq_rel_gpu();  // acquire (and L1 invalidation) before the slot is released
  return ok;
}

template <bool CPLX, int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1) mpk_pipe_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kPipeMaxSlots], empty_bar[kPipeMaxSlots];
  __shared__ int64_t s_ofs[kPipeMaxSlots];
  __shared__ int32_t s_t[kPipeMaxSlots], s_p[kPipeMaxSlots], s_staged[kPipeMaxSlots];
  __shared__ uint32_t s_done[kPipeMaxSlots];
  const int S = P.n_slots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], NC);
      s_done[i] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  const bool sweep = P.mode == 3;
  if (warp == NC) {
    // ------------------------------------------------ producer warp
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_drop = policy_evict_first();
    bool abort = false;
    for (int k = 0;; ++k) {
      const int slot = k % S;
      const uint32_t use = uint32_t(k / S);
      int32_t item;
      if (sweep) {
        item = blockIdx.x + k * gridDim.x;
      } else {
        int32_t g = 0;
        if (lane == 0) g = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
        item = __shfl_sync(0xffffffffu, g, 0);
      }
      if (abort) item = P.n_items;
      if (lane == 0 && use > 0) mbar_wait(&empty_bar[slot], (use - 1) & 1);
      __syncwarp();
      if (item >= P.n_items) {
        if (lane == 0) {
          s_t[slot] = -1;
          mbar_arrive(&full_bar[slot]);
        }
        break;
      }
      int32_t t, p;
      if (sweep) {
        t = item;
        p = 1;
      } else {
        const int32_t code = __ldg(P.items + item);
        t = code >> 7;
        p = code & 127;
      }
      const int64_t ofs = __ldg(P.tile_ofs + t);
      const int64_t bytes = __ldg(P.tile_ofs + t + 1) - ofs;
      const bool staged = bytes <= P.smem_cap;
      if (lane == 0) {
        s_t[slot] = t;
        s_p[slot] = p;
        s_ofs[slot] = ofs;
        s_staged[slot] = staged ? 1 : 0;
        if (staged) {
          fence_proxy_async_smem();
          mbar_expect_tx(&full_bar[slot], uint32_t(bytes));
          bulk_g2s(smem_raw + int64_t(slot) * P.smem_cap, P.blocks + ofs, uint32_t(bytes),
                   &full_bar[slot], (sweep || p == P.n_powers) ? pol_drop : pol_keep);
        }
      }
      if (p > 1) {
        if (!warp_wait_deps(P, __ldg(P.dep_lo + t), __ldg(P.dep_hi + t), P.epoch_base + uint32_t(p - 1)))
          abort = true;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_bar[slot]);
    }
  } else {
    // ------------------------------------------------ consumer warps
    for (int k = 0;; ++k) {
      const int slot = k % S;
      mbar_wait(&full_bar[slot], uint32_t(k / S) & 1);
      const int32_t t = s_t[slot];
      if (t < 0) break;
      const int p = s_p[slot];
      const int32_t r0 = __ldg(P.tile_row + t), r1 = __ldg(P.tile_row + t + 1);
      const unsigned char* blk =
          s_staged[slot] ? smem_raw + int64_t(slot) * P.smem_cap : P.blocks + s_ofs[slot];
      tile_power<CPLX>(P, C, blk, r0, r1, __ldg(P.tile_E + t), p, warp, NC);
      __syncwarp();
      if (lane == 0) {
        if (!sweep) {
          const uint32_t old = atom_add_acqrel_cta_smem(&s_done[slot], 1u);
          if (old == NC - 1) {
            s_done[slot] = 0;
            st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
          }
        }
        mbar_arrive(&empty_bar[slot]);
      }
    }
  }
}

// ---------------------------------------------------------------- pipelined resident mode
// One producer warp + NC consumer warps per CTA (one CTA per SM).  The CTA
// holds R tiles resident in shared memory (one TMA bulk copy each, so the
// matrix is read from HBM once).  The producer polls the held tiles round
// robin WITHOUT blocking on any single one: a tile whose next power p has
// its dependencies satisfied (tiles dep_lo..dep_hi published p-1) is queued
// as a work item (slot, p) in a small smem ring; consumer warps drain the
// ring like the streaming pipeline (no CTA-wide barriers; the last warp of
// an item publishes the tile's progress word).  A tile whose last power
// completed frees its slot, which the producer refills with the next tile
// of the global in-order queue.  Deadlock freedom: tiles are grabbed in
// order, so the unfinished tiles [t0, t0 + 148*R) are always held; if the
// (p_m-1)-step dependency chain reach is below 148*R (checked when the
// tiling is built) the oldest held tile can always advance.
constexpr int kResMaxSlots = 8;
constexpr int kWorkRing = 8;

__device__ __forceinline__ bool warp_deps_ready(const MpkParams& P, int32_t lo, int32_t hi,
                                                uint32_t target) {
  bool ok = true;
  for (int32_t i = lo + int32_t(threadIdx.x & 31); i <= hi; i += 32)
    ok = ok && (ld_relaxed_u32(P.progress + i) >= target);
  return __all_sync(0xffffffffu, ok);
}

template <bool CPLX, int NC>
__global__ void __launch_bounds__(32 * (NC + 1), 1) mpk_res_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t tile_bar[kResMaxSlots];
  __shared__ uint64_t full_bar[kWorkRing], empty_bar[kWorkRing];
  __shared__ int32_t w_slot[kWorkRing], w_p[kWorkRing];
  __shared__ uint32_t w_done[kWorkRing];
  __shared__ int32_t h_t[kResMaxSlots];
  __shared__ volatile int32_t slot_free[kResMaxSlots];
  const int R = P.n_slots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < R; ++i) {
      mbar_init(&tile_bar[i], 1);
      slot_free[i] = 0;
    }
    for (int i = 0; i < kWorkRing; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], NC);
      w_done[i] = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == NC) {
    // ------------------------------------------------ producer warp
    const uint64_t pol = policy_evict_first();
    int32_t np[kResMaxSlots];      // next power to issue per held slot (lane-uniform)
    uint32_t refills[kResMaxSlots];
    int32_t lo[kResMaxSlots], hi[kResMaxSlots];
    int live = 0;
    auto refill = [&](int r) {
      int32_t g = 0;
      if (lane == 0) g = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
      const int32_t t = __shfl_sync(0xffffffffu, g, 0);
      if (t >= P.n_tiles || t < 0) {
        if (lane == 0) h_t[r] = -1;
        np[r] = 0;
        return false;
      }
      const int64_t ofs = __ldg(P.tile_ofs + t);
      const int64_t bytes = __ldg(P.tile_ofs + t + 1) - ofs;
      if (lane == 0) {
        h_t[r] = t;
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&tile_bar[r], uint32_t(bytes));
        bulk_g2s(smem_raw + int64_t(r) * P.smem_cap, P.blocks + ofs, uint32_t(bytes), &tile_bar[r], pol);
      }
      lo[r] = __ldg(P.dep_lo + t);
      hi[r] = __ldg(P.dep_hi + t);
      np[r] = 1;
      return true;
    };
    for (int r = 0; r < R; ++r) {
      refills[r] = 0;
      if (refill(r)) ++live;
    }
    int k = 0;  // work items pushed
    unsigned long long idle_since = 0;
    bool abort = false;
    while (live > 0 && !abort) {
      bool progressed = false;
      for (int r = 0; r < R; ++r) {
        if (np[r] == 0) continue;  // retired slot
        if (np[r] > P.n_powers) {
          // all powers issued: refill once the last one completed
          if (slot_free[r]) {
            __syncwarp();
            if (lane == 0) slot_free[r] = 0;
            __threadfence_block();
            ++refills[r];
            if (!refill(r)) --live;
            progressed = true;
          }
          continue;
        }
        const int p = np[r];
        bool ready;
        if (p == 1)
          ready = mbar_test(&tile_bar[r], refills[r] & 1);
        else
          ready = warp_deps_ready(P, lo[r], hi[r], P.epoch_base + uint32_t(p - 1));
        if (!ready) continue;
        if (p > 1) fence_acq_rel_gpu();  // acquire + L1 invalidation before the gathers
        const int ws = k % kWorkRing;
        if (lane == 0) {
          if (k >= kWorkRing) mbar_wait(&empty_bar[ws], uint32_t(k / kWorkRing - 1) & 1);
          w_slot[ws] = r;
          w_p[ws] = p;
          mbar_arrive(&full_bar[ws]);
        }
        __syncwarp();
        ++k;
        np[r] = p + 1;
        progressed = true;
      }
      if (progressed) {
        idle_since = 0;
      } else {
        __nanosleep(64);
        const unsigned long long now = globaltimer();
        if (idle_since == 0) idle_since = now;
        const volatile unsigned long long* ab = P.queue + 1;
        if (*ab != 0ull) abort = true;
        if (now - idle_since > kWatchdogNs) {
          if (lane == 0) {
            atomicExch(P.queue + 1, 1ull);
            *P.err = 1;
          }
          abort = true;
        }
      }
    }
    // terminator
    const int ws = k % kWorkRing;
    if (lane == 0) {
      if (k >= kWorkRing) mbar_wait(&empty_bar[ws], uint32_t(k / kWorkRing - 1) & 1);
      w_slot[ws] = -1;
      mbar_arrive(&full_bar[ws]);
    }
    // no TMA may still be landing when the CTA exits: held slots were either
    // consumed (power >= 1 issued) or are waited for here
    if (abort && lane == 0)
      for (int r = 0; r < R; ++r)
        if (np[r] == 1) mbar_wait(&tile_bar[r], refills[r] & 1);
  } else {
    // ------------------------------------------------ consumer warps
    for (int k = 0;; ++k) {
      const int ws = k % kWorkRing;
      mbar_wait(&full_bar[ws], uint32_t(k / kWorkRing) & 1);
      const int r = w_slot[ws];
      if (r < 0) break;
      const int p = w_p[ws];
      const int32_t t = h_t[r];
      const int32_t r0 = __ldg(P.tile_row + t), r1 = __ldg(P.tile_row + t + 1);
      tile_power<CPLX>(P, C, smem_raw + int64_t(r) * P.smem_cap, r0, r1, __ldg(P.tile_E + t), p, warp, NC);
      __syncwarp();
      if (lane == 0) {
        const uint32_t old = atom_add_acqrel_cta_smem(&w_done[ws], 1u);
        if (old == NC - 1) {
          w_done[ws] = 0;
          st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
          if (p == P.n_powers) {
            __threadfence_block();
            slot_free[r] = 1;
          }
        }
        mbar_arrive(&empty_bar[ws]);
      }
    }
  }
}

// ---------------------------------------------------------------- tiling kernels
__global__ void k_slice_width(const int32_t* row_ptr, int32_t n, int32_t n_slices, int32_t* width) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int32_t r = s * 32 + lane;
  const int len = r < n ? __ldg(row_ptr + r + 1) - __ldg(row_ptr + r) : 0;
  const int w = __reduce_max_sync(0xffffffffu, len);
  if (lane == 0) width[s] = w;
}

// one warp per slice: write slice offset, row lengths and column-major entries
__global__ void k_fill_blocks(const int32_t* row_ptr, const int32_t* col, const double* val,
                              int32_t n_slices, const int32_t* slice_tile, const int32_t* slice_off,
                              const int32_t* width, const int32_t* tile_row, const int64_t* tile_ofs,
                              const int32_t* tile_E, unsigned char* blocks) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int32_t t = slice_tile[s];
  const int32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const int32_t ns = (r1 - r0 + 31) >> 5;
  const int32_t ls = s - (r0 >> 5);
  unsigned char* blk = blocks + tile_ofs[t];
  int32_t* soff = reinterpret_cast<int32_t*>(blk);
  uint16_t* lens = reinterpret_cast<uint16_t*>(blk + ((ns + 3) & ~3) * 4);
  const int64_t co = blk_col_off(ns);
  const int32_t E = tile_E[t];
  int32_t* cols = reinterpret_cast<int32_t*>(blk + co);
  double* vals = reinterpret_cast<double*>(blk + co + int64_t(E) * 4);
  const int32_t base = slice_off[s];
  const int32_t r = s * 32 + lane;
  const bool valid = r < r1;
  const int32_t a = valid ? row_ptr[r] : 0;
  const int len = valid ? row_ptr[r + 1] - a : 0;
  if (lane == 0) soff[ls] = base;
  lens[ls * 32 + lane] = uint16_t(len);
  const int w = width[s];
  for (int j = 0; j < w; ++j) {
    const int64_t e = int64_t(base) + int64_t(j) * 32 + lane;
    if (j < len) {
      cols[e] = col[a + j];
      vals[e] = val[a + j];
    } else {
      cols[e] = valid ? r : r0;  // harmless in-range index, never accumulated
      vals[e] = 0.0;
    }
  }
}

__device__ __forceinline__ int32_t tile_of(const int32_t* tile_row, int32_t n_tiles, int32_t r) {
  int32_t lo = 0, hi = n_tiles - 1;  // last t with tile_row[t] <= r
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
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
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
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
    cudaGetLastError();
    set_error("cudaMalloc(%zu) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    return LMPK_ERR_NOMEM;
  }
  return LMPK_OK;
}

template <bool CPLX>
static cudaError_t occupancy_t(lmpk_ctx* ctx, int threads, int smem, int* occ) {
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
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, mpk_kernel<CPLX>, threads, smem);
}

// occupancy valid for both instantiations (complex uses more registers)
static int occupancy(lmpk_ctx* ctx, int threads, int smem, int* occ) {
  int o1 = 0, o2 = 0;
  cudaError_t e = occupancy_t<false>(ctx, threads, smem, &o1);
  if (e == cudaSuccess) e = occupancy_t<true>(ctx, threads, smem, &o2);
  if (e != cudaSuccess) {
    cudaGetLastError();  // do not leave a sticky status for later checks
    set_error("occupancy query failed: %s", cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  }
  *occ = std::min(o1, o2);
  return LMPK_OK;
}

template <bool CPLX>
static cudaError_t pipe_attr_t(lmpk_ctx* ctx, int smem, int* occ) {
  auto fn = mpk_pipe_kernel<CPLX, kPipeConsumers>;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  const int max_dyn = ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes);
  if (smem > max_dyn) {
    *occ = 0;
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, 32 * (kPipeConsumers + 1), smem);
}

template <bool CPLX>
static cudaError_t res_attr_t(lmpk_ctx* ctx, int smem, int* occ) {
  auto fn = mpk_res_kernel<CPLX, kPipeConsumers>;
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  const int max_dyn = ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes);
  if (smem > max_dyn) {
    *occ = 0;
    return cudaSuccess;
  }
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, fn, 32 * (kPipeConsumers + 1), smem);
}

static int res_occupancy(lmpk_ctx* ctx, int smem, int* occ) {
  int o1 = 0, o2 = 0;
  cudaError_t e = res_attr_t<false>(ctx, smem, &o1);
  if (e == cudaSuccess) e = res_attr_t<true>(ctx, smem, &o2);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("occupancy query failed: %s", cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  }
  *occ = std::min(o1, o2);
  return LMPK_OK;
}

static int pipe_occupancy(lmpk_ctx* ctx, int smem, int* occ) {
  int o1 = 0, o2 = 0;
  cudaError_t e = pipe_attr_t<false>(ctx, smem, &o1);
  if (e == cudaSuccess) e = pipe_attr_t<true>(ctx, smem, &o2);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("occupancy query failed: %s", cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  }
  *occ = std::min(o1, o2);
  return LMPK_OK;
}

// Partition the 32-row slices greedily into tiles whose block fits `cap`.
static void partition_slices(const std::vector<int32_t>& width, int64_t cap,
                             std::vector<int32_t>& tile_first, std::vector<int64_t>& tile_E) {
  const int32_t S = static_cast<int32_t>(width.size());
  tile_first.clear();
  tile_E.clear();
  int32_t s = 0;
  while (s < S) {
    int32_t ns = 0;
    int64_t E = 0;
    while (s + ns < S) {
      const int64_t e2 = E + int64_t(width[s + ns]) * 32;
      if (ns > 0 && blk_bytes(ns + 1, e2) > cap) break;
      E = e2;
      ++ns;
    }
    tile_first.push_back(s);
    tile_E.push_back(E);
    s += ns;
  }
  if (S == 0) {
    tile_first.push_back(0);
    tile_E.push_back(0);
  }
}

// max over t of the (p_m-1)-step forward dependency chain, via the prefix max
// of dep_hi (monotone, conservative).
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
      const int32_t nc = H[c];
      if (nc == c) break;
      c = nc;
    }
    worst = std::max(worst, c - t);
  }
  return worst;
}

}  // namespace lmpk

using namespace lmpk;

extern "C" int lmpk_tiling_destroy(lmpk_tiling* t) {
  if (!t) return LMPK_OK;
  cudaFree(t->d_tile_row);
  cudaFree(t->d_tile_ofs);
  cudaFree(t->d_tile_E);
  cudaFree(t->d_dep_lo);
  cudaFree(t->d_dep_hi);
  cudaFree(t->d_items);
  cudaFree(t->d_progress);
  cudaFree(t->d_blocks);
  delete t;
  return LMPK_OK;
}

// Tiles + tile-SELL-32 blocks + dependency ranges for block cap `cap` bytes.
static int build_tiling(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr,
                        const int32_t* col, const double* val, const std::vector<int32_t>& width,
                        int64_t cap, cudaStream_t st) {
  const int32_t S = static_cast<int32_t>(width.size());
  std::vector<int32_t> first;
  std::vector<int64_t> Es;
  partition_slices(width, cap, first, Es);
  const int32_t nt = static_cast<int32_t>(first.size());
  std::vector<int32_t> tile_row(nt + 1), tile_E(nt), slice_tile(std::max(S, 1)), slice_off(std::max(S, 1));
  std::vector<int64_t> tile_ofs(nt + 1);
  int64_t ofs = 0;
  int64_t maxb = 0;
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t s0 = first[t], s1 = (t + 1 < nt) ? first[t + 1] : S;
    tile_row[t] = std::min(s0 * 32, n);
    tile_E[t] = static_cast<int32_t>(Es[t]);
    tile_ofs[t] = ofs;
    const int64_t b = blk_bytes(s1 - s0, Es[t]);
    maxb = std::max(maxb, b);
    ofs += b;
    int32_t e = 0;
    for (int32_t s = s0; s < s1; ++s) {
      slice_tile[s] = t;
      slice_off[s] = e;
      e += width[s] * 32;
    }
  }
  tile_row[nt] = n;
  tile_ofs[nt] = ofs;
  T->h_tile_row = tile_row;
  T->block_bytes = ofs;
  T->max_block = static_cast<int32_t>(maxb);
  LMPK_TRY(dmalloc(&T->d_tile_row, nt + 1));
  LMPK_TRY(dmalloc(&T->d_tile_ofs, nt + 1));
  LMPK_TRY(dmalloc(&T->d_tile_E, nt));
  LMPK_TRY(dmalloc(&T->d_dep_lo, nt));
  LMPK_TRY(dmalloc(&T->d_dep_hi, nt));
  LMPK_TRY(dmalloc(&T->d_progress, nt));
  LMPK_TRY(dmalloc(&T->d_blocks, size_t(std::max<int64_t>(ofs, 128))));
  int32_t *d_slice_tile = nullptr, *d_slice_off = nullptr, *d_width = nullptr;
  LMPK_TRY(dmalloc(&d_slice_tile, std::max(S, 1)));
  LMPK_TRY(dmalloc(&d_slice_off, std::max(S, 1)));
  LMPK_TRY(dmalloc(&d_width, std::max(S, 1)));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_row, tile_row.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_ofs, tile_ofs.data(), (nt + 1) * 8, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_E, tile_E.data(), nt * 4, cudaMemcpyHostToDevice, st));
  if (S > 0) {
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_slice_tile, slice_tile.data(), size_t(S) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_slice_off, slice_off.data(), size_t(S) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_width, width.data(), size_t(S) * 4, cudaMemcpyHostToDevice, st));
  }
  LMPK_CHECK_CUDA(cudaMemsetAsync(T->d_progress, 0, size_t(nt) * 4, st));
  if (S > 0) {
    k_fill_blocks<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, val, S, d_slice_tile, d_slice_off,
                                                                 d_width, T->d_tile_row, T->d_tile_ofs,
                                                                 T->d_tile_E, T->d_blocks);
    launch_count_add(ctx, 1);
  }
  k_tile_deps<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(row_ptr, col, T->d_tile_row, nt, T->d_dep_lo,
                                                             T->d_dep_hi);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  T->h_dep_lo.resize(nt);
  T->h_dep_hi.resize(nt);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->h_dep_lo.data(), T->d_dep_lo, nt * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->h_dep_hi.data(), T->d_dep_hi, nt * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_slice_tile);
  cudaFree(d_slice_off);
  cudaFree(d_width);
  T->info.n_tiles = nt;
  T->info.block_bytes = ofs;
  return LMPK_OK;
}

extern "C" int lmpk_tiling_create(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                                  const double* val, int32_t p_m, const lmpk_tiling_params* params,
                                  lmpk_tiling** out, lmpk_tiling_info* info, void* stream) {
  LMPK_ARG_CHECK(ctx && out && row_ptr && col && val, "lmpk_tiling_create: NULL argument");
  LMPK_ARG_CHECK(p_m >= 1 && p_m <= LMPK_MAX_POWERS, "p_m must be in [1, %d]", LMPK_MAX_POWERS);
  LMPK_ARG_CHECK(n >= 0, "n must be >= 0");
  lmpk_tiling_params prm{};
  if (params) prm = *params;
  *out = nullptr;
  cudaStream_t st = as_stream(stream);
  int32_t h_nnz = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&h_nnz, row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
  const int32_t S = (n + 31) / 32;
  std::vector<int32_t> width(S);
  if (S > 0) {
    int32_t* d_w = nullptr;
    LMPK_TRY(dmalloc(&d_w, S));
    k_slice_width<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, n, S, d_w);
    launch_count_add(ctx, 1);
    LMPK_CHECK_CUDA(cudaMemcpyAsync(width.data(), d_w, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_w);
  } else {
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  int32_t max_row = 0;
  for (int32_t w : width) max_row = std::max(max_row, w);
  LMPK_ARG_CHECK(max_row <= 65535, "rows longer than 65535 entries are not supported by the tiled kernel");

  const bool want_stream = (prm.mode_flags & LMPK_FLAG_MODE_STREAM) != 0;
  const bool want_res = (prm.mode_flags & LMPK_FLAG_MODE_RESIDENT) != 0;
  const int threads = prm.threads > 0 ? prm.threads : kMaxThreads;
  LMPK_ARG_CHECK(threads % 32 == 0 && threads >= 64 && threads <= kMaxThreads,
                 "threads must be a multiple of 32 in [64, %d]", kMaxThreads);
  const int static_reserve = 1024 + 64;  // per-CTA driver reserve + static smem
  // candidates: (mode, ring/resident slots); both pipelined kernels run one
  // CTA per SM with one producer warp and kPipeConsumers consumer warps
  struct Cand {
    int mode, slots;
  };
  std::vector<Cand> cands;
  if (!want_stream) {
    if (prm.slots > 0)
      cands.push_back({1, std::min(prm.slots, kResMaxSlots)});
    else
      for (int r : {2, 3, 4, 6, 8}) cands.push_back({1, r});
  }
  if (!want_res) cands.push_back({2, prm.slots > 0 ? std::min(prm.slots, kPipeMaxSlots) : 3});
  lmpk_tiling* T = nullptr;
  int grid = 0, smem = 0, mode = 0, slots = 1;
  int32_t mfwd = 0, creach = 0;
  int64_t cap_used = 0;
  for (const Cand& cd : cands) {
    int64_t cap = (ctx->max_smem_block - 1024) / cd.slots;
    if (prm.tile_nnz_hint > 0) cap = std::min<int64_t>(cap, int64_t(prm.tile_nnz_hint) * 12 + 2048);
    cap &= ~int64_t(127);
    if (cap < 2048) continue;
    const int smem_need = static_cast<int>(cap * cd.slots);
    int occ = 0;
    if (cd.mode == 1)
      LMPK_TRY(res_occupancy(ctx, smem_need, &occ));
    else
      LMPK_TRY(pipe_occupancy(ctx, smem_need, &occ));
    if (occ < 1) continue;
    lmpk_tiling* cand = new lmpk_tiling();
    cand->ctx = ctx;
    cand->n = n;
    const int rc = build_tiling(ctx, cand, n, row_ptr, col, val, width, cap, st);
    if (rc != LMPK_OK) {
      lmpk_tiling_destroy(cand);
      return rc;
    }
    int32_t mf = 0;
    const int32_t cr = chain_reach(cand->h_dep_hi, p_m, &mf);
    const int g = ctx->sm_count;
    // resident: every held tile must fit its slot, and the dependency chain
    // of the oldest held tile must stay inside the held window
    if (cd.mode == 1 && !(cr < g * cd.slots - 1 && cand->max_block <= cap)) {
      lmpk_tiling_destroy(cand);
      continue;
    }
    T = cand;
    mode = cd.mode;
    grid = g;
    smem = smem_need;
    slots = cd.slots;
    mfwd = mf;
    creach = cr;
    cap_used = cap;
    break;
  }
  if (!T) {
    set_error("lmpk_tiling_create: no feasible tiling (mode flags 0x%x)", prm.mode_flags);
    return want_res ? LMPK_ERR_UNSUPPORTED : LMPK_ERR_ARG;
  }
  const int32_t nt = T->info.n_tiles;
  T->info.p_m = p_m;
  T->info.mode = mode;
  T->info.block = 32 * (kPipeConsumers + 1);
  T->slots = slots;
  (void)threads;
  T->info.smem_bytes = smem;
  T->info.tile_nnz_cap = static_cast<int32_t>(cap_used / 12);
  T->info.max_fwd_reach = mfwd;
  T->info.chain_reach = creach;
  T->info.max_row_nnz = max_row;
  T->info.nnz = h_nnz;
  T->info.grid = grid;
  if (mode == 2) {
    // skewed diagonal order key (t + p*M, p), M = D + slack; dependent items
    // land ~slack*p_m queue positions apart
    const int32_t slack = prm.queue_slack > 0 ? prm.queue_slack : std::max(1, (2 * grid + p_m - 1) / p_m);
    T->info.queue_slack = slack;
    const int64_t M = int64_t(std::max(mfwd, 0)) + slack;
    std::vector<int64_t> keys;
    keys.reserve(int64_t(nt) * p_m);
    for (int32_t t = 0; t < nt; ++t)
      for (int32_t p = 1; p <= p_m; ++p) keys.push_back(((t + p * M) << 8) | p);
    std::vector<int32_t> order(keys.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return keys[a] < keys[b]; });
    std::vector<int32_t> items(order.size());
    for (size_t i = 0; i < order.size(); ++i) {
      const int32_t t = order[i] / p_m, p = order[i] % p_m + 1;
      items[i] = (t << 7) | p;
    }
    LMPK_TRY(dmalloc(&T->d_items, items.size()));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_items, items.data(), items.size() * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
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

static int launch_mpk(lmpk_ctx* ctx, const lmpk_tiling* T, MpkParams& Pm, PowerCfgDev& C, bool cplx,
                      bool coop, int grid, int smem, cudaStream_t st) {
  void* args[] = {&Pm, &C};
  const bool pipe = Pm.mode != 1;
  const void* fn = pipe ? (cplx ? reinterpret_cast<const void*>(mpk_pipe_kernel<true, kPipeConsumers>)
                                : reinterpret_cast<const void*>(mpk_pipe_kernel<false, kPipeConsumers>))
                        : (cplx ? reinterpret_cast<const void*>(mpk_res_kernel<true, kPipeConsumers>)
                                : reinterpret_cast<const void*>(mpk_res_kernel<false, kPipeConsumers>));
  const int block = 32 * (kPipeConsumers + 1);
  cudaError_t e = coop ? cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, st)
                       : cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("mpk launch failed: %s (grid %d, block %d, smem %d)", cudaGetErrorString(e), grid, block,
              smem);
    return LMPK_ERR_CUDA;
  }
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

extern "C" int lmpk_mpk_run(lmpk_ctx* ctx, const lmpk_tiling* T, double* y, int64_t ldy, int32_t n_slots,
                            const lmpk_power_cfg* cfg, double* acc, int use_acc, int flags, void* stream) {
  LMPK_ARG_CHECK(ctx && T && cfg && y, "lmpk_mpk_run: NULL ctx/tiling/cfg/y");
  LMPK_ARG_CHECK(T->ctx == ctx, "tiling belongs to another ctx");
  const int32_t P = cfg->n_powers;
  const bool sweep = (flags & LMPK_FLAG_SWEEP) != 0;
  LMPK_ARG_CHECK(P >= 1 && P <= LMPK_MAX_POWERS, "n_powers must be in [1, %d]", LMPK_MAX_POWERS);
  LMPK_ARG_CHECK(sweep || P <= T->info.p_m, "n_powers %d exceeds the tiling's p_m %d", P, T->info.p_m);
  const bool cplx = (flags & LMPK_FLAG_COMPLEX) != 0;
  LMPK_ARG_CHECK(ldy >= int64_t(T->n) * (cplx ? 2 : 1), "ldy too small");
  LMPK_ARG_CHECK(!use_acc || acc != nullptr, "use_acc requires acc");
  LMPK_ARG_CHECK(!cplx || (reinterpret_cast<uintptr_t>(y) & 15) == 0, "complex y must be 16-byte aligned");
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
  MpkParams Pm;
  memset(&Pm, 0, sizeof(Pm));
  Pm.blocks = T->d_blocks;
  Pm.tile_ofs = T->d_tile_ofs;
  Pm.tile_E = T->d_tile_E;
  Pm.tile_row = T->d_tile_row;
  Pm.dep_lo = T->d_dep_lo;
  Pm.dep_hi = T->d_dep_hi;
  Pm.items = T->d_items;
  Pm.y = y;
  Pm.ldy = ldy;
  Pm.acc = acc;
  Pm.use_acc = use_acc ? 1 : 0;
  Pm.progress = Tm->d_progress;
  Pm.queue = reinterpret_cast<unsigned long long*>(ctx->queue_ctr);
  Pm.n_tiles = T->info.n_tiles;
  Pm.n_slots = T->slots;
  Pm.smem_cap = T->info.smem_bytes / T->slots;
  Pm.use_tma = (flags & LMPK_FLAG_NO_TMA) ? 0 : 1;
  Pm.err = ctx->err.dev;
  if (sweep) {
    // n_powers back-to-back, dependency-free passes (one launch per power)
    const int grid = std::min<int>(ctx->sm_count, T->info.n_tiles);
    // ring slots of the tiling's block cap (at least 2 when they fit)
    const int64_t avail = ctx->max_smem_block - 1024;
    const int64_t cap = T->max_block;
    int S = static_cast<int>(std::min<int64_t>(std::max<int64_t>(avail / std::max<int64_t>(cap, 1), 1), kPipeMaxSlots));
    const int smem = static_cast<int>(std::min<int64_t>(S * cap, avail));
    Pm.smem_cap = static_cast<int32_t>(smem / S) & ~127;
    Pm.n_slots = S;
    for (int i = 0; i < P; ++i) {
      PowerCfgDev Ci;
      memset(&Ci, 0, sizeof(Ci));
      Ci.out_slot[0] = C.out_slot[i];
      Ci.in_slot[0] = C.in_slot[i];
      Ci.prev_slot[0] = C.prev_slot[i];
      Ci.kernel[0] = C.kernel[i];
      Ci.coef_re[0] = C.coef_re[i];
      Ci.coef_im[0] = C.coef_im[i];
      Pm.mode = 3;
      Pm.n_powers = 1;
      Pm.n_items = T->info.n_tiles;
      Pm.queue_base = ctx->queue_base;
      Pm.epoch_base = 0;
      LMPK_TRY(launch_mpk(ctx, T, Pm, Ci, cplx, false, grid, smem, st));
    }
    return LMPK_OK;
  }
  ctx->epoch += 1;
  if (ctx->epoch >= (1u << 24)) {  // counter wrap: reset progress words
    LMPK_CHECK_CUDA(cudaMemsetAsync(Tm->d_progress, 0, size_t(T->info.n_tiles) * 4, st));
    ctx->epoch = 1;
  }
  Pm.epoch_base = ctx->epoch * kEpochStride;
  Pm.queue_base = ctx->queue_base;
  Pm.n_powers = P;
  Pm.mode = T->info.mode;
  Pm.n_items = T->info.n_tiles * T->info.p_m;
  LMPK_ARG_CHECK(Pm.mode == 1 || P == T->info.p_m,
                 "streaming tiling built for p_m=%d cannot run %d powers", T->info.p_m, P);
  const int grid = Pm.mode == 1 ? T->info.grid : std::min<int>(T->info.grid, Pm.n_items);
  LMPK_TRY(launch_mpk(ctx, T, Pm, C, cplx, Pm.mode == 1, grid, T->info.smem_bytes, st));
  // every successful grab takes one work unit; every grab sequence ends with
  // exactly one failing grab: one per CTA (streaming) or per resident slot
  const int64_t work = (Pm.mode == 1) ? T->info.n_tiles : Pm.n_items;
  const int64_t fails = (Pm.mode == 1) ? int64_t(grid) * T->slots : grid;
  ctx->queue_base += uint64_t(work + fails);
  return LMPK_OK;
}

// Host-side check after the caller synchronized the stream.
extern "C" int lmpk_ctx_check(lmpk_ctx* ctx, void* stream) {
  LMPK_ARG_CHECK(ctx != nullptr, "ctx is NULL");
  LMPK_CHECK_CUDA(cudaStreamSynchronize(as_stream(stream)));
  const int rc = ctx_check_device_error(ctx, "mpk");
  if (rc != LMPK_OK) {
    // the aborted launch left the queue counter inconsistent: reset it
    cudaMemset(ctx->queue_ctr, 0, 64);
    cudaDeviceSynchronize();
    ctx->queue_base = 0;
  }
  return rc;
}
