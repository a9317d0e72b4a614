// lean_kernel.cuh -- the "lean" ring walk: the level-blocked MPK of
// mpk_kernel.cuh (same items, progress words, producer and publisher) with a
// consumer body that spends its issue slots on the row sums only.
//
// Reference semantics: the per-row body of _walk (pkg/src/levelmpk/
// executor.py:127-147), rows summed in CRS storage order from +0.0 with
// separately rounded products and sums (csr.py:195-201), for every row of an
// item (tile, power); the item order and the dependency waits are those of the
// ring walk (mpk_kernel.cuh: skewed diagonal key, schedule.py:91-99).
//
// What changes against the ring kernel's compressed tile body:
//   * LEAN BLOCKS.  A tile's 32-row slices are re-ordered by width W (<= 8)
//     into UNITS: pairs of same-width slices (or one slice), each described
//     by one 16-byte record {col offset, value offset, W | flags, slice ids}.
//     A unit's body is compiled for its W -- no per-slice width records,
//     no mixed-width pairs, no per-lane length table in the hot loop.
//   * Lane-contiguous indices: lane i's int16 column offsets are Wc = 4 or 8
//     contiguous entries (one LDS.64 / LDS.128), its dictionary byte codes Wc
//     contiguous bytes (one LDS.32 / LDS.64); the dictionary sits at a fixed
//     offset of the slot, so a value is PRMT + LDS [code + slot].
//   * Padding without predication: a padding entry repeats the row's last
//     column with the value +0.0, so it adds +-0 to a running sum that is
//     never -0.0 (it starts at +0.0; a round-to-nearest sum is -0.0 only when
//     both terms are): bitwise the reference for finite operands.  A padded
//     unit whose row comes out NaN is recomputed with the row's true length
//     (a non-finite gathered operand could otherwise turn an Inf sum into
//     NaN) -- the rare slow path, off the hot loop.
//   * Static unit striding (warp w takes units w, w + NC, ... rotated by the
//     piece counter so the extra units move between warps): no shared
//     counter, no per-pair grab.
//   * Per-piece descriptors (tile, power, first row, rows, unit count) are
//     written once by the producer; a consumer's per-piece setup is a handful
//     of shared loads.
#pragma once
#include "mpk_kernel.cuh"

namespace lmpk {

#ifndef LMPK_LEAN_NC
#define LMPK_LEAN_NC 26
#endif
constexpr int kLeanConsumers = LMPK_LEAN_NC;
constexpr int kLeanHdr = 16;          // [nu, nrows, flags, 0]
constexpr int kLeanDict = 16;         // dictionary byte offset in the block
constexpr int kLeanRec = 16 + 256;    // first unit record
constexpr uint32_t kLeanPair = 1u << 8, kLeanPadded = 1u << 9, kLeanPattern = 1u << 10;

__host__ __device__ constexpr int lean_wc(int w) { return w <= 0 ? 0 : (w <= 4 ? 4 : 8); }
// bytes of one slice's column offsets / dictionary codes / raw values
__host__ __device__ constexpr int lean_col_bytes(int w) { return 64 * lean_wc(w); }
__host__ __device__ constexpr int lean_code_bytes(int w) { return 32 * lean_wc(w); }
__host__ __device__ constexpr int lean_raw_bytes(int w) { return 256 * (w < 0 ? 0 : w); }

struct LeanParams {
  const unsigned char* blocks;  // lean tile blocks
  const int64_t* ofs;           // [n_tiles + 1] byte offset of each lean block
  const uint8_t* rowlen;        // [n] row lengths (slow path only)
};

// ---------------------------------------------------------------- row sums
// Shared-memory reads by 32-bit address.  They are plain (non-volatile) asm
// so the scheduler may batch them; every address derives from the piece's
// base, which is an OUTPUT of the piece's mbarrier wait (lean_wait), so no
// read can move above the wait or be reused across pieces.
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
  uint4 v;
  asm("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds_v2(uint32_t a) {
  uint2 v;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_b8(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ int32_t lds_s16(uint32_t a) {
  int16_t v;
  asm("ld.shared.s16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_d(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
  double2 v;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// Lane's W column offsets (lane-contiguous Wc int16 at p).
template <int W>
__device__ __forceinline__ void lean_cols(uint32_t p, int32_t (&c)[W]) {
  if constexpr (lean_wc(W) == 8) {
    const uint4 v = lds_v4(p);
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < W; ++j) c[j] = (j & 1) ? (int32_t(w4[j >> 1]) >> 16) : int32_t(int16_t(w4[j >> 1] & 0xffffu));
  } else {
    const uint2 v = lds_v2(p);
    const uint32_t w2[2] = {v.x, v.y};
#pragma unroll
    for (int j = 0; j < W; ++j) c[j] = (j & 1) ? (int32_t(w2[j >> 1]) >> 16) : int32_t(int16_t(w2[j >> 1] & 0xffffu));
  }
}
// Lane's W dictionary values: byte codes (premultiplied by 8) at p, the
// dictionary at dict.
template <int W>
__device__ __forceinline__ void lean_dvals(uint32_t p, uint32_t dict, double (&v)[W]) {
  if constexpr (lean_wc(W) == 8) {
    const uint2 k = lds_v2(p);
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] = lds_d(dict + __byte_perm(j < 4 ? k.x : k.y, 0u, 0x4440u + uint32_t(j & 3)));
  } else {
    const uint32_t k = lds_u32(p);
#pragma unroll
    for (int j = 0; j < W; ++j) v[j] = lds_d(dict + __byte_perm(k, 0u, 0x4440u + uint32_t(j)));
  }
}
// raw values of lane's W entries, chunked (quads, pair, single; see chunk_entry)
template <int W>
__device__ __forceinline__ void lean_raw(uint32_t p, uint32_t lane, double (&v)[W]) {
  constexpr int Q = W >> 2, PR = (W >> 1) & 1, SG = W & 1;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double2 a = lds_d2(p + q * 1024 + lane * 32);
    const double2 b = lds_d2(p + q * 1024 + lane * 32 + 16);
    v[4 * q] = a.x, v[4 * q + 1] = a.y, v[4 * q + 2] = b.x, v[4 * q + 3] = b.y;
  }
  if constexpr (PR) {
    const double2 a = lds_d2(p + Q * 1024 + lane * 16);
    v[4 * Q] = a.x, v[4 * Q + 1] = a.y;
  }
  if constexpr (SG) v[W - 1] = lds_d(p + Q * 1024 + PR * 512 + lane * 8);
}

template <bool CPLX>
struct LeanX {
  using T = double;
};
template <>
struct LeanX<true> {
  using T = double2;
};

// gather of x[row + d] (row pointer rp = &x[row])
template <bool CPLX>
__device__ __forceinline__ typename LeanX<CPLX>::T lean_gather(const char* rp, int32_t d) {
  if constexpr (CPLX) {
    double2 v;
    asm("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(rp + int64_t(d) * 16));
    return v;
  } else {
    double v;
    asm("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(rp + int64_t(d) * 8));
    return v;
  }
}

template <bool CPLX>
struct LeanSum {
  double r, i;
};

template <int W, bool CPLX, bool EXACT>
__device__ __forceinline__ LeanSum<CPLX> lean_chain(const double (&v)[W], const typename LeanX<CPLX>::T (&x)[W]) {
  LeanSum<CPLX> s{0.0, 0.0};
#pragma unroll
  for (int j = 0; j < W; ++j) {
    if constexpr (CPLX) {
      s.r = madd<EXACT>(s.r, v[j], x[j].x);
      s.i = madd<EXACT>(s.i, v[j], x[j].y);
    } else {
      s.r = madd<EXACT>(s.r, v[j], x[j]);
    }
  }
  return s;
}

// One slice of width W: lane's row sum in storage order (real or complex x).
// cp/vp: lane's column-offset / code (or slice-base raw value) addresses.
template <int W, bool CPLX, bool EXACT, bool VD>
__device__ __forceinline__ LeanSum<CPLX> lean_slice(uint32_t cp, uint32_t vp, uint32_t dict, uint32_t lane,
                                                    const char* rp) {
  if constexpr (W == 0) {
    return LeanSum<CPLX>{0.0, 0.0};
  } else {
    int32_t c[W];
    lean_cols<W>(cp, c);
    typename LeanX<CPLX>::T x[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x[j] = lean_gather<CPLX>(rp, c[j]);
    double v[W];
    if constexpr (VD)
      lean_dvals<W>(vp, dict, v);
    else
      lean_raw<W>(vp, lane, v);
    return lean_chain<W, CPLX, EXACT>(v, x);
  }
}

// Two slices of the same width: every gather of both in flight at once.
template <int W, bool CPLX, bool EXACT, bool VD>
__device__ __forceinline__ void lean_pair(uint32_t cp0, uint32_t vp0, uint32_t cp1, uint32_t vp1, uint32_t dict,
                                          uint32_t lane, const char* rp0, const char* rp1, LeanSum<CPLX>& s0,
                                          LeanSum<CPLX>& s1) {
  if constexpr (W == 0) {
    s0 = s1 = LeanSum<CPLX>{0.0, 0.0};
  } else {
    int32_t c0[W], c1[W];
    lean_cols<W>(cp0, c0);
    lean_cols<W>(cp1, c1);
    typename LeanX<CPLX>::T x0[W], x1[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x0[j] = lean_gather<CPLX>(rp0, c0[j]);
#pragma unroll
    for (int j = 0; j < W; ++j) x1[j] = lean_gather<CPLX>(rp1, c1[j]);
    {
      double v[W];
      if constexpr (VD)
        lean_dvals<W>(vp0, dict, v);
      else
        lean_raw<W>(vp0, lane, v);
      s0 = lean_chain<W, CPLX, EXACT>(v, x0);
    }
    {
      double v[W];
      if constexpr (VD)
        lean_dvals<W>(vp1, dict, v);
      else
        lean_raw<W>(vp1, lane, v);
      s1 = lean_chain<W, CPLX, EXACT>(v, x1);
    }
  }
}

// Slow path of a padded row whose sum came out NaN: the row again with its
// true length (padding entries skipped), exactly as the reference sums it.
template <bool CPLX, bool EXACT, bool VD>
__device__ __noinline__ LeanSum<CPLX> lean_row_exact(uint32_t cp, uint32_t vp, uint32_t dict, uint32_t lane,
                                                     const char* rp, int w, int len) {
  LeanSum<CPLX> s{0.0, 0.0};
  const int Q = w >> 2, PR = (w >> 1) & 1;
  for (int j = 0; j < len; ++j) {
    const int32_t c = lds_s16(cp + 2 * j);
    double v;
    if constexpr (VD) {
      v = lds_d(dict + lds_b8(vp + j));
    } else {
      // vp is the slice's raw-value base here: chunk position of entry j
      uint32_t e;
      if (j < 4 * Q)
        e = uint32_t(j >> 2) * 128u + lane * 4u + uint32_t(j & 3);
      else if (PR && j < 4 * Q + 2)
        e = uint32_t(Q) * 128u + lane * 2u + uint32_t(j - 4 * Q);
      else
        e = uint32_t(Q) * 128u + (PR ? 64u : 0u) + lane;
      v = lds_d(vp + e * 8u);
    }
    const typename LeanX<CPLX>::T x = lean_gather<CPLX>(rp, c);
    if constexpr (CPLX) {
      s.r = madd<EXACT>(s.r, v, x.x);
      s.i = madd<EXACT>(s.i, v, x.y);
    } else {
      s.r = madd<EXACT>(s.r, v, x);
    }
  }
  return s;
}

__device__ __forceinline__ bool lean_nan(double a) { return a != a; }

// ---------------------------------------------------------------- epilogue
// Row r (tile-local lr) at power pt: plain store, or the Chebyshev step
// t = 2t - y_{p-2} and the accumulation acc += c t (executor.py:131-135).
template <bool CPLX, bool EXACT, bool GEN>
__device__ __forceinline__ void lean_store(const PowTab& pt, double* acc, bool use_acc, int64_t r, LeanSum<CPLX> s) {
  if constexpr (!CPLX) {
    double t = s.r;
    if constexpr (GEN) {
      if (pt.cheb) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(pt.ypv + r));
    }
    stg_f64(pt.yout + r, t);
    if constexpr (GEN) {
      if (use_acc) stg_f64(acc + r, madd<EXACT>(ld_cg(acc + r), pt.cre, t));
    }
  } else {
    double2 t = make_double2(s.r, s.i);
    const int64_t r2 = 2 * r;
    if constexpr (GEN) {
      if (pt.cheb) {
        t.x = __dsub_rn(__dmul_rn(2.0, t.x), ld_cg(pt.ypv + r2));
        t.y = __dsub_rn(__dmul_rn(2.0, t.y), ld_cg(pt.ypv + r2 + 1));
      }
    }
    stg_f64x2(pt.yout + r2, t);
    if constexpr (GEN) {
      if (use_acc) {
        const double ar = ld_cg(acc + r2), ai = ld_cg(acc + r2 + 1);
        const double pr = __dsub_rn(__dmul_rn(pt.cre, t.x), __dmul_rn(pt.cim, t.y));
        const double pim = __dadd_rn(__dmul_rn(pt.cre, t.y), __dmul_rn(pt.cim, t.x));
        stg_f64x2(acc + r2, make_double2(__dadd_rn(ar, pr), __dadd_rn(ai, pim)));
      }
    }
  }
}

// Lane's column-offset / code addresses of one slice.  Plain lean slices
// hold every lane's entries (lane-contiguous); PATTERN slices (dictionary
// tiles) hold the slice's distinct rows once -- [32 u8 row pattern ids]
// [P x 2Wc B offsets][P x Wc B codes] -- and a lane reads its pattern's record.
template <int W, bool VD>
__device__ __forceinline__ void lean_ptrs(uint32_t blk, uint32_t off, uint32_t np, bool pat, uint32_t lane,
                                          uint32_t& cp, uint32_t& vp, uint32_t vo) {
  if (VD && pat) {
    const uint32_t sl = blk + off;
    const uint32_t id = lds_b8(sl + lane);
    cp = sl + 32 + id * (2 * lean_wc(W));
    vp = sl + 32 + np * (2 * lean_wc(W)) + id * lean_wc(W);
  } else {
    cp = blk + off + lane * (2 * lean_wc(W));
    vp = VD ? blk + vo + lane * lean_wc(W) : blk + vo;
  }
}

// One unit of width W (compile time): a pair or a single slice.
// Record: plain {col off, value off, W | flags, slice ids}; pattern
// {slice a off, slice b off, W | flags | Pa << 16 | Pb << 24, slice ids}.
template <int W, bool CPLX, bool EXACT, bool VD, bool GEN>
__device__ __forceinline__ void lean_unit(uint32_t blk, uint4 rec, uint32_t lane, int32_t r0, int32_t nrows,
                                          const PowTab& pt, double* acc, bool use_acc, const uint8_t* rowlen) {
  constexpr int cw = CPLX ? 16 : 8;
  const uint32_t dict = blk + kLeanDict;
  const int32_t s0 = int32_t(rec.w & 0xffffu), s1 = int32_t(rec.w >> 16);
  const int32_t l0 = s0 * 32 + int32_t(lane), l1 = s1 * 32 + int32_t(lane);
  const bool pat = VD && (rec.z & kLeanPattern) != 0;
  // lanes past the tile (last slice) use the last valid lane's pattern: gather
  // around that row (their sums are discarded)
  const char* rp0 = pt.yin + int64_t(r0 + (pat ? min(l0, nrows - 1) : l0)) * cw;
  uint32_t cp0, vp0;
  lean_ptrs<W, VD>(blk, rec.x, (rec.z >> 16) & 255u, pat, lane, cp0, vp0, rec.y);
  const bool padded = (rec.z & kLeanPadded) != 0;
  if (rec.z & kLeanPair) {
    const char* rp1 = pt.yin + int64_t(r0 + (pat ? min(l1, nrows - 1) : l1)) * cw;
    uint32_t cp1, vp1;
    if (pat) {
      lean_ptrs<W, VD>(blk, rec.y, rec.z >> 24, true, lane, cp1, vp1, 0u);
    } else {
      cp1 = cp0 + lean_col_bytes(W);
      vp1 = vp0 + (VD ? lean_code_bytes(W) : lean_raw_bytes(W));
    }
    LeanSum<CPLX> a, b;
    lean_pair<W, CPLX, EXACT, VD>(cp0, vp0, cp1, vp1, dict, lane, rp0, rp1, a, b);
    if (padded) {
      if (lean_nan(a.r) || (CPLX && lean_nan(a.i)))
        if (l0 < nrows) a = lean_row_exact<CPLX, EXACT, VD>(cp0, vp0, dict, lane, rp0, W, rowlen[r0 + l0]);
      if (lean_nan(b.r) || (CPLX && lean_nan(b.i)))
        if (l1 < nrows) b = lean_row_exact<CPLX, EXACT, VD>(cp1, vp1, dict, lane, rp1, W, rowlen[r0 + l1]);
    }
    if (l0 < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l0), a);
    if (l1 < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l1), b);
  } else {
    LeanSum<CPLX> a = lean_slice<W, CPLX, EXACT, VD>(cp0, vp0, dict, lane, rp0);
    if (padded && (lean_nan(a.r) || (CPLX && lean_nan(a.i))))
      if (l0 < nrows) a = lean_row_exact<CPLX, EXACT, VD>(cp0, vp0, dict, lane, rp0, W, rowlen[r0 + l0]);
    if (l0 < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l0), a);
  }
}

// Wait for a piece and return its base address: the base is an asm output of
// the completed wait, so every shared read addressed from it stays below it.
__device__ __forceinline__ uint32_t lean_wait(uint64_t* bar, uint32_t parity, uint32_t base) {
  while (!mbar_try_wait_sleep(bar, parity, 1000000u)) {
  }
  uint32_t out;
  asm volatile("mov.u32 %0, %1;" : "=r"(out) : "r"(base) : "memory");
  return out;
}

// ---------------------------------------------------------------- kernel
// Same launch contract as mpk_ring_kernel (cooperative, one CTA per SM, a
// 2-piece ring): warp NC is the producer, warp NC + 1 the publisher.
template <bool CPLX, bool EXACT, bool VD, bool GEN, int NP>
__global__ void __launch_bounds__(32 * (kLeanConsumers + 2), 1)
    mpk_lean_kernel(MpkParams P, PowerCfgDev C, LeanParams L) {
  constexpr int NC = kLeanConsumers;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[NP], empty_bar[NP], done_bar[NP];
  __shared__ int32_t d_t[NP], d_p[NP], d_r0[NP], d_rows[NP];
  __shared__ uint32_t d_done[NP];
  __shared__ uint32_t trace_ctr;
  __shared__ PowTab s_pow[LMPK_MAX_POWERS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  build_powtab(s_pow, P, C);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NP; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
      mbar_init(&done_bar[i], 1);
      d_done[i] = 0;
    }
    trace_ctr = 0;
    fence_mbar_init();
  }
  __syncthreads();
  const int cap = P.smem_cap;
  if (warp == NC + 1) {
    // ------------------------------------------------ publisher (ring order)
    for (uint32_t k = 0;; ++k) {
      const int slot = int(k % NP);
      mbar_wait_sleep(&done_bar[slot], (k / NP) & 1);
      const int32_t t = d_t[slot], p = d_p[slot];
      __syncwarp();
      if (t < 0) break;
      if (lane == 0) {
        mbar_arrive(&empty_bar[slot]);
        st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
      }
      __syncwarp();
    }
  } else if (warp == NC) {
    // ------------------------------------------------ producer
    const int pm = (P.flags >> 8) & 3;
    const uint64_t pol = pm == 1 ? policy_evict_normal() : (pm == 3 ? policy_evict_last() : policy_evict_first());
    unsigned long long rounds = 0;
    uint32_t k = 0;
    bool abort = false;
    for (;;) {
      int32_t i = 0;
      if (lane == 0) i = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
      i = __shfl_sync(0xffffffffu, i, 0);
      if (i >= P.n_items || i < 0) break;
      const int32_t code = __ldg(P.items + i);
      const int32_t T = code >> 8, p = (code & 255) + 1;
      if (p > P.n_powers) continue;
      const int32_t m0 = __ldg(P.st_first + T), m1 = __ldg(P.st_first + T + 1);
      if (lane == 0) trace_ev(P, &trace_ctr, 1, 0, uint32_t(T) << 8 | uint32_t(p));
      if (p > 1 && !spin_deps(P, __ldg(P.st_lo + T), __ldg(P.st_hi + T), P.epoch_base + uint32_t(p - 1), &rounds)) {
        abort = true;
        break;
      }
      if (lane == 0) trace_ev(P, &trace_ctr, 4, 0, uint32_t(T) << 8 | uint32_t(p));
      for (int32_t m = m0; m < m1; ++m) {
        const int slot = int(k % NP);
        if (k >= uint32_t(NP) && !mbar_wait_bounded(&empty_bar[slot], (k / NP - 1) & 1, P)) {
          abort = true;
          break;
        }
        if (lane == 0) {
          const int64_t ofs = __ldg(L.ofs + m), bytes = __ldg(L.ofs + m + 1) - ofs;
          d_t[slot] = m;
          d_p[slot] = p;
          const int32_t r0 = __ldg(P.tile_row + m);
          d_r0[slot] = r0;
          d_rows[slot] = __ldg(P.tile_row + m + 1) - r0;
          trace_ev(P, &trace_ctr, 2, uint32_t(slot), uint32_t(m) << 8 | uint32_t(p));
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full_bar[slot], uint32_t(bytes));
          bulk_g2s(smem_raw + int64_t(slot) * cap, L.blocks + ofs, uint32_t(bytes), &full_bar[slot],
                   p == P.n_powers ? policy_evict_first() : pol);
        }
        __syncwarp();
        ++k;
      }
      if (abort) break;
    }
    if (lane == 0) {
      const int slot = int(k % NP);
      bool ok = true;
      if (k >= uint32_t(NP)) {
        unsigned long long t0 = globaltimer();
        while (!mbar_try_wait(&empty_bar[slot], (k / NP - 1) & 1)) {
          if (globaltimer() - t0 > kWatchdogNs || *(volatile unsigned long long*)(P.queue + 1) != 0ull) {
            ok = false;
            break;
          }
        }
      }
      if (ok) {
        d_t[slot] = -1;
        mbar_arrive(&full_bar[slot]);
      }
    }
    if (P.prof && lane == 0) atomicAdd(P.prof + 3, rounds);
  } else {
    // ------------------------------------------------ consumers
    const bool use_acc = P.use_acc != 0;
    const uint32_t ring = smem_u32(smem_raw);
    for (uint32_t k = 0;; ++k) {
      const int slot = int(k % NP);
      const uint32_t blk = lean_wait(&full_bar[slot], (k / NP) & 1, ring + uint32_t(slot) * uint32_t(cap));
      const int32_t t = d_t[slot];
      if (t < 0) {
        if (warp == 0 && lane == 0) mbar_arrive(&done_bar[slot]);
        break;
      }
      const int32_t p = d_p[slot], r0 = d_r0[slot], nrows = d_rows[slot];
      const int32_t nu = int32_t(lds_u32(blk));
      const PowTab& pt = s_pow[p - 1];
      if (lane == 0 && (warp == 0 || warp == NC - 1)) trace_ev(P, &trace_ctr, 10, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
      // static striding, rotated by the piece counter
      int32_t u = warp + int32_t(k % uint32_t(NC));
      if (u >= NC) u -= NC;
      for (; u < nu; u += NC) {
        const uint4 rec = lds_v4(blk + kLeanRec + uint32_t(u) * 16u);
        switch (rec.z & 15u) {
#define LMPK_LEAN_CASE(Wv) \
  case Wv: lean_unit<Wv, CPLX, EXACT, VD, GEN>(blk, rec, lane, r0, nrows, pt, P.acc, use_acc, L.rowlen); break;
          LMPK_LEAN_CASE(0)
          LMPK_LEAN_CASE(1)
          LMPK_LEAN_CASE(2)
          LMPK_LEAN_CASE(3)
          LMPK_LEAN_CASE(4)
          LMPK_LEAN_CASE(5)
          LMPK_LEAN_CASE(6)
          LMPK_LEAN_CASE(7)
          LMPK_LEAN_CASE(8)
#undef LMPK_LEAN_CASE
          default: break;
        }
      }
      __syncwarp();
      if (lane == 0 && (warp == 0 || warp == NC - 1)) trace_ev(P, &trace_ctr, 11, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
      uint32_t old = 0;
      if (lane == 0) old = atom_add_acqrel_cta_smem(&d_done[slot], 1u);
      if (__shfl_sync(0xffffffffu, old, 0) == uint32_t(NC - 1) && lane == 0) {
        trace_ev(P, &trace_ctr, 12, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
        d_done[slot] = 0;
        mbar_arrive(&done_bar[slot]);
      }
    }
  }
}

}  // namespace lmpk
