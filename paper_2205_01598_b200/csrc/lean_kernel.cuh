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
constexpr uint32_t kLeanSameVal = 1u << 11;  // pattern pair whose slices share one row of dictionary values
// same-value pair of two full, unpadded one-pattern slices (the interior of a grid): the unit body
// with every check resolved at build time (lean_unit's fast path)
constexpr uint32_t kLeanFast = 1u << 12;
// fast unit whose values are row (z >> 13) & 3 of the tile's value table (the free dictionary slots
// 8 (1 + row) ..: k_lean_vrows)
constexpr uint32_t kLeanVRow = 1u << 15;

__host__ __device__ constexpr int lean_wc(int w) { return w <= 0 ? 0 : (w <= 4 ? 4 : 8); }
// bytes of one slice's column offsets / dictionary codes / raw values
__host__ __device__ constexpr int lean_col_bytes(int w) { return 64 * lean_wc(w); }
__host__ __device__ constexpr int lean_code_bytes(int w) { return 32 * lean_wc(w); }
__host__ __device__ constexpr int lean_raw_bytes(int w) { return 256 * (w < 0 ? 0 : w); }

struct LeanParams {
  const unsigned char* blocks;  // lean tile blocks
  const int64_t* ofs;           // [n_tiles + 1] byte offset of each lean block
  const uint8_t* rowlen;        // [n] row lengths (slow path only)
  // x staging (mpk_xlean_kernel): per tile the runs of y_{p-1} its rows gather,
  // bulk-copied behind the block; column fields then hold (buffer index - lane)
  const int4* runs;             // [n_tiles * kLeanMaxRuns] {first entry, entries, buffer entry, 0}
  const int2* xinfo;            // [n_tiles] {runs, staged entries}
  int32_t xoff;                 // byte offset of the x buffer inside a piece
  int32_t np;                   // ring depth (pieces) of the staged kernel
  const int4* wl;               // per-CTA static work lists (2 x int4 per piece), or null: ticket queue
  const int32_t* wl_ptr;        // [grid + 1]
  int32_t pub_batch;            // pieces the publisher makes visible per gpu-scope fence (1..8)
};
constexpr int kLeanMaxRuns = 32;  // one bulk copy per producer lane

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

// Row pointer of the gathers: &x[row] in global memory, or (x staging) the
// 32-bit shared address of the lane's base entry in the piece's x buffer.
template <bool XS>
struct LeanRp {
  using T = const char*;
};
template <>
struct LeanRp<true> {
  using T = uint32_t;
};

// gather of x[row + d] (row pointer rp = &x[row])
template <bool CPLX, bool XS = false>
__device__ __forceinline__ typename LeanX<CPLX>::T lean_gather(typename LeanRp<XS>::T rp, int32_t d) {
  if constexpr (XS) {
    if constexpr (CPLX)
      return lds_d2(rp + uint32_t(d) * 16u);
    else
      return lds_d(rp + uint32_t(d) * 8u);
  } else if constexpr (CPLX) {
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
template <int W, bool CPLX, bool EXACT, bool VD, bool XS = false>
__device__ __forceinline__ LeanSum<CPLX> lean_slice(uint32_t cp, uint32_t vp, uint32_t dict, uint32_t lane,
                                                    typename LeanRp<XS>::T rp) {
  if constexpr (W == 0) {
    return LeanSum<CPLX>{0.0, 0.0};
  } else {
    int32_t c[W];
    lean_cols<W>(cp, c);
    typename LeanX<CPLX>::T x[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x[j] = lean_gather<CPLX, XS>(rp, c[j]);
    double v[W];
    if constexpr (VD)
      lean_dvals<W>(vp, dict, v);
    else
      lean_raw<W>(vp, lane, v);
    return lean_chain<W, CPLX, EXACT>(v, x);
  }
}

// Two slices of the same width: every gather of both in flight at once.
template <int W, bool CPLX, bool EXACT, bool VD, bool XS = false, bool SV = false>
__device__ __forceinline__ void lean_pair(uint32_t cp0, uint32_t vp0, uint32_t cp1, uint32_t vp1, uint32_t dict,
                                          uint32_t lane, typename LeanRp<XS>::T rp0, typename LeanRp<XS>::T rp1,
                                          LeanSum<CPLX>& s0, LeanSum<CPLX>& s1) {
  if constexpr (W == 0) {
    s0 = s1 = LeanSum<CPLX>{0.0, 0.0};
  } else {
    int32_t c0[W], c1[W];
    lean_cols<W>(cp0, c0);
    lean_cols<W>(cp1, c1);
    typename LeanX<CPLX>::T x0[W], x1[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x0[j] = lean_gather<CPLX, XS>(rp0, c0[j]);
#pragma unroll
    for (int j = 0; j < W; ++j) x1[j] = lean_gather<CPLX, XS>(rp1, c1[j]);
    if constexpr (SV) {  // kLeanSameVal: one row of dictionary values for both slices
      double v[W];
      lean_dvals<W>(vp0, dict, v);
      s0 = lean_chain<W, CPLX, EXACT>(v, x0);
      s1 = lean_chain<W, CPLX, EXACT>(v, x1);
    } else {
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
}

// Slow path of a padded row whose sum came out NaN: the row again with its
// true length (padding entries skipped), exactly as the reference sums it.
template <bool CPLX, bool EXACT, bool VD, bool XS = false>
__device__ __noinline__ LeanSum<CPLX> lean_row_exact(uint32_t cp, uint32_t vp, uint32_t dict, uint32_t lane,
                                                     typename LeanRp<XS>::T rp, int w, int len) {
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
    const typename LeanX<CPLX>::T x = lean_gather<CPLX, XS>(rp, c);
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

// The epilogue's own operands (y_{p-2} of the Chebyshev step, acc) are
// L1-prefetched BEFORE the gathers are issued, so their L2 / HBM latency
// overlaps the gathers' instead of following the row sum; lean_store_pf then
// loads them with plain L1-allocating loads.  (Loading them into registers up
// front does not work: under the 72-register cap ptxas sinks the loads below
// the row sum, and the Chebyshev subtraction took 35% of all stall samples.)
// Both vectors are written only by this row's items at other powers, which
// the item dependencies order, and the item's dependency acquire invalidated
// the L1 -- the argument that makes the gathers coherent.
template <bool CPLX, bool GEN>
__device__ __forceinline__ void lean_prefetch_epi(const PowTab& pt, const double* acc, bool use_acc, int64_t r,
                                                  bool valid) {
  if constexpr (GEN) {
    if (valid) {
      if (pt.cheb) asm volatile("prefetch.global.L1 [%0];" ::"l"(pt.ypv + (CPLX ? 2 : 1) * r));
      if (use_acc) asm volatile("prefetch.global.L1 [%0];" ::"l"(acc + (CPLX ? 2 : 1) * r));
    }
  }
}
template <bool CPLX, bool EXACT, bool GEN>
__device__ __forceinline__ void lean_store_pf(const PowTab& pt, double* acc, bool use_acc, int64_t r,
                                              LeanSum<CPLX> s) {
  if constexpr (!CPLX) {
    double t = s.r;
    if constexpr (GEN) {
      if (pt.cheb) t = __dsub_rn(__dmul_rn(2.0, t), ldg_f64(reinterpret_cast<const char*>(pt.ypv + r)));
    }
    stg_f64(pt.yout + r, t);
    if constexpr (GEN) {
      if (use_acc) stg_f64(acc + r, madd<EXACT>(ldg_f64(reinterpret_cast<const char*>(acc + r)), pt.cre, t));
    }
  } else {
    double2 t = make_double2(s.r, s.i);
    const int64_t r2 = 2 * r;
    if constexpr (GEN) {
      if (pt.cheb) {
        const double2 pv = ldg_f64x2(reinterpret_cast<const char*>(pt.ypv + r2));
        t.x = __dsub_rn(__dmul_rn(2.0, t.x), pv.x);
        t.y = __dsub_rn(__dmul_rn(2.0, t.y), pv.y);
      }
    }
    stg_f64x2(pt.yout + r2, t);
    if constexpr (GEN) {
      if (use_acc) {
        const double2 a = ldg_f64x2(reinterpret_cast<const char*>(acc + r2));
        const double pr = __dsub_rn(__dmul_rn(pt.cre, t.x), __dmul_rn(pt.cim, t.y));
        const double pim = __dadd_rn(__dmul_rn(pt.cre, t.y), __dmul_rn(pt.cim, t.x));
        stg_f64x2(acc + r2, make_double2(__dadd_rn(a.x, pr), __dadd_rn(a.y, pim)));
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
    const uint32_t id = np > 1u ? lds_b8(sl + lane) : 0u;  // one pattern (grid interior): no id
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
// XS (x staging): the column fields hold (x-buffer entry - lane) and the
// gathers read the piece's x buffer at shared address xb.
// the staged kernel keeps the L2 loads of lean_store (its gathers come from shared memory)
template <bool CPLX, bool EXACT, bool GEN, bool XS>
__device__ __forceinline__ void lean_store_u(const PowTab& pt, double* acc, bool use_acc, int64_t r, LeanSum<CPLX> s) {
  if constexpr (XS)
    lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, r, s);
  else
    lean_store_pf<CPLX, EXACT, GEN>(pt, acc, use_acc, r, s);
}

template <int W, bool CPLX, bool EXACT, bool VD, bool GEN, bool XS = false>
__device__ __forceinline__ void lean_unit(uint32_t blk, uint4 rec, uint32_t lane, int32_t r0, int32_t nrows,
                                          const PowTab& pt, double* acc, bool use_acc, const uint8_t* rowlen,
                                          uint32_t xb = 0) {
  constexpr int cw = CPLX ? 16 : 8;
  using RP = typename LeanRp<XS>::T;
  const uint32_t dict = blk + kLeanDict;
  const int32_t s0 = int32_t(rec.w & 0xffffu), s1 = int32_t(rec.w >> 16);
  const int32_t l0 = s0 * 32 + int32_t(lane), l1 = s1 * 32 + int32_t(lane);
  if constexpr (VD && !CPLX && !XS && W > 0) {
    // FAST units (kLeanFast, set by lean_build): a pattern pair of two full,
    // unpadded slices with one pattern each and the same dictionary indices.
    // No ids, no bounds, no NaN re-check, no per-slice branches: the ~100
    // instructions of unit set-up around the 95 of the pair itself (cfg2: 69%
    // of the units) shrink to the address arithmetic.
    if (rec.z & kLeanFast) {
      const char* q0 = pt.yin + int64_t(r0 + l0) * 8;
      const char* q1 = pt.yin + int64_t(r0 + l1) * 8;
      // two opaque bases: otherwise the compiler derives the second slice's
      // gather addresses from the first's with 64-bit add pairs instead of
      // one IMAD.WIDE per gather
      asm("" : "+l"(q0));
      asm("" : "+l"(q1));
      const uint32_t ca = blk + rec.x + 32u, cb = blk + rec.y + 32u;
      if constexpr (GEN) {
        lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l0), true);
        lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l1), true);
      }
      LeanSum<CPLX> a, b;
      if (rec.z & kLeanVRow) {
        // the seven values as broadcast LDS.128 from the tile's value table
        const uint32_t vr = dict + 64u * (1u + ((rec.z >> 13) & 3u));
        int32_t c0[W], c1[W];
        lean_cols<W>(ca, c0);
        lean_cols<W>(cb, c1);
        double x0[W], x1[W];
#pragma unroll
        for (int j = 0; j < W; ++j) x0[j] = lean_gather<false, false>(q0, c0[j]);
#pragma unroll
        for (int j = 0; j < W; ++j) x1[j] = lean_gather<false, false>(q1, c1[j]);
        double v[W];
#pragma unroll
        for (int j = 0; j + 1 < W; j += 2) {
          const double2 d = lds_d2(vr + 8u * uint32_t(j));
          v[j] = d.x, v[j + 1] = d.y;
        }
        if constexpr (W & 1) v[W - 1] = lds_d(vr + 8u * uint32_t(W - 1));
        a = lean_chain<W, CPLX, EXACT>(v, x0);
        b = lean_chain<W, CPLX, EXACT>(v, x1);
      } else {
        lean_pair<W, CPLX, EXACT, true, false, true>(ca, ca + 2u * uint32_t(lean_wc(W)), cb, 0u, dict, lane, q0, q1, a, b);
      }
      lean_store_pf<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l0), a);
      lean_store_pf<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l1), b);
      return;
    }
  }
  const bool pat = VD && (rec.z & kLeanPattern) != 0;
  // lanes past the tile (last slice) use the last valid lane's pattern: gather
  // around that row (their sums are discarded)
  RP rp0;
  if constexpr (XS)
    rp0 = xb + uint32_t(pat ? min(int32_t(lane), nrows - 1 - s0 * 32) : int32_t(lane)) * uint32_t(cw);
  else
    rp0 = pt.yin + int64_t(r0 + (pat ? min(l0, nrows - 1) : l0)) * cw;
  uint32_t cp0, vp0;
  lean_ptrs<W, VD>(blk, rec.x, (rec.z >> 16) & 255u, pat, lane, cp0, vp0, rec.y);
  const bool padded = (rec.z & kLeanPadded) != 0;
  if constexpr (!XS) lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l0), l0 < nrows);
  if (rec.z & kLeanPair) {
    if constexpr (!XS) lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l1), l1 < nrows);
    RP rp1;
    if constexpr (XS)
      rp1 = xb + uint32_t(pat ? min(int32_t(lane), nrows - 1 - s1 * 32) : int32_t(lane)) * uint32_t(cw);
    else
      rp1 = pt.yin + int64_t(r0 + (pat ? min(l1, nrows - 1) : l1)) * cw;
    if constexpr (!XS) {  // opaque bases: one IMAD.WIDE per gather (see the fast path)
      asm("" : "+l"(rp0));
      asm("" : "+l"(rp1));
    }
    uint32_t cp1, vp1;
    if (pat) {
      lean_ptrs<W, VD>(blk, rec.y, rec.z >> 24, true, lane, cp1, vp1, 0u);
    } else {
      cp1 = cp0 + lean_col_bytes(W);
      vp1 = vp0 + (VD ? lean_code_bytes(W) : lean_raw_bytes(W));
    }
    LeanSum<CPLX> a, b;
    if (VD && !CPLX && (rec.z & kLeanSameVal))
      lean_pair<W, CPLX, EXACT, VD, XS, VD && !CPLX>(cp0, vp0, cp1, vp1, dict, lane, rp0, rp1, a, b);
    else
      lean_pair<W, CPLX, EXACT, VD, XS>(cp0, vp0, cp1, vp1, dict, lane, rp0, rp1, a, b);
    if (padded) {
      if (lean_nan(a.r) || (CPLX && lean_nan(a.i)))
        if (l0 < nrows) a = lean_row_exact<CPLX, EXACT, VD, XS>(cp0, vp0, dict, lane, rp0, W, rowlen[r0 + l0]);
      if (lean_nan(b.r) || (CPLX && lean_nan(b.i)))
        if (l1 < nrows) b = lean_row_exact<CPLX, EXACT, VD, XS>(cp1, vp1, dict, lane, rp1, W, rowlen[r0 + l1]);
    }
    if (l0 < nrows) lean_store_u<CPLX, EXACT, GEN, XS>(pt, acc, use_acc, int64_t(r0 + l0), a);
    if (l1 < nrows) lean_store_u<CPLX, EXACT, GEN, XS>(pt, acc, use_acc, int64_t(r0 + l1), b);
  } else {
    LeanSum<CPLX> a = lean_slice<W, CPLX, EXACT, VD, XS>(cp0, vp0, dict, lane, rp0);
    if (padded && (lean_nan(a.r) || (CPLX && lean_nan(a.i))))
      if (l0 < nrows) a = lean_row_exact<CPLX, EXACT, VD, XS>(cp0, vp0, dict, lane, rp0, W, rowlen[r0 + l0]);
    if (l0 < nrows) lean_store_u<CPLX, EXACT, GEN, XS>(pt, acc, use_acc, int64_t(r0 + l0), a);
  }
}

// ---------------------------------------------------------------- DP units
// DIAGONAL-PRIVATE dictionary blocks (lean_vd == 2; built by dp_build in
// mpk_dp.cuh): matrices whose off-diagonal values come from one small global
// dictionary while the diagonal differs row by row -- a stencil plus a
// potential (the Anderson / Schroedinger operators of the paper's Chebyshev
// application).  Every slice is a pattern slice with 32-bit column offsets:
//   [32 u8 row pattern ids][P x Wc i32 (col - row)][P x Wc u8 codes]
//   [pad to 8][32 f64 private values (lane's diagonal entry)]
// A code is 8 x the dictionary index; kDpPriv marks the row's diagonal
// entry, whose value is the lane's private one.  The row sum itself is
// lean_chain in storage order, so EXACT mode stays bitwise the reference
// (executor.py:127-130, csr.py:195-201); padding entries carry the code of
// +0.0 and repeat the row's last column as in the lean blocks above.
constexpr uint32_t kDpPriv = 248u;
__host__ __device__ constexpr int dp_priv_off(int w, int np) { return (32 + 5 * lean_wc(w) * np + 7) & ~7; }
__host__ __device__ constexpr int dp_slice_bytes(int w, int np) {
  return w <= 0 ? 0 : ((dp_priv_off(w, np) + 256 + 15) & ~15);
}

// Lane's addresses in a DP slice: op = its pattern's offsets, kp = its
// pattern's codes, pd = (address of its private value) - dict - kDpPriv.
template <int W>
__device__ __forceinline__ void dp_ptrs(uint32_t sl, uint32_t np, uint32_t lane, uint32_t dict, uint32_t& op,
                                        uint32_t& kp, uint32_t& pd) {
  constexpr uint32_t WC = lean_wc(W);
  const uint32_t id = np > 1u ? lds_b8(sl + lane) : 0u;
  op = sl + 32u + id * (4u * WC);
  kp = sl + 32u + np * (4u * WC) + id * WC;
  pd = sl + ((32u + 5u * WC * np + 7u) & ~7u) + lane * 8u - dict - kDpPriv;
}
template <int W>
__device__ __forceinline__ void dp_cols(uint32_t op, int32_t (&c)[W]) {
  const uint4 a = lds_v4(op);
  const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int j = 0; j < (W < 4 ? W : 4); ++j) c[j] = int32_t(w4[j]);
  if constexpr (W > 4) {
    const uint4 b = lds_v4(op + 16);
    const uint32_t v4[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int j = 4; j < W; ++j) c[j] = int32_t(v4[j - 4]);
  }
}
template <int W>
__device__ __forceinline__ void dp_vals(uint32_t kp, uint32_t dict, uint32_t pd, double (&v)[W]) {
  uint32_t k0, k1 = 0u;
  if constexpr (lean_wc(W) == 8) {
    const uint2 k = lds_v2(kp);
    k0 = k.x, k1 = k.y;
  } else {
    k0 = lds_u32(kp);
  }
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const uint32_t code = __byte_perm(j < 4 ? k0 : k1, 0u, 0x4440u + uint32_t(j & 3));
    v[j] = lds_d(dict + code + (code == kDpPriv ? pd : 0u));
  }
}
template <bool CPLX, bool EXACT>
__device__ __noinline__ LeanSum<CPLX> dp_row_exact(uint32_t op, uint32_t kp, uint32_t dict, uint32_t pd,
                                                   const char* rp, int len) {
  LeanSum<CPLX> s{0.0, 0.0};
  for (int j = 0; j < len; ++j) {
    const int32_t c = int32_t(lds_u32(op + 4 * j));
    const uint32_t code = lds_b8(kp + j);
    const double v = lds_d(dict + code + (code == kDpPriv ? pd : 0u));
    const typename LeanX<CPLX>::T x = lean_gather<CPLX, false>(rp, c);
    if constexpr (CPLX) {
      s.r = madd<EXACT>(s.r, v, x.x);
      s.i = madd<EXACT>(s.i, v, x.y);
    } else {
      s.r = madd<EXACT>(s.r, v, x);
    }
  }
  return s;
}

// One slice of a DP unit (tile-local slice sidx at byte offset sl_off of the
// block, np distinct rows): prefetch of the epilogue operands, gathers, row
// sum, epilogue.
template <int W, bool CPLX, bool EXACT, bool GEN>
__device__ __forceinline__ void dp_single(uint32_t blk, uint32_t sl_off, uint32_t np, int32_t sidx, bool padded,
                                          uint32_t lane, int32_t r0, int32_t nrows, const PowTab& pt, double* acc,
                                          bool use_acc, const uint8_t* rowlen) {
  constexpr int cw = CPLX ? 16 : 8;
  const uint32_t dict = blk + kLeanDict;
  const int32_t l0 = sidx * 32 + int32_t(lane);
  // lanes past the tile use the last valid lane's pattern: gather around that row
  const char* rp0 = pt.yin + int64_t(r0 + min(l0, nrows - 1)) * cw;
  asm("" : "+l"(rp0));  // opaque base: one IMAD.WIDE per gather
  uint32_t op0, kp0, pd0;
  dp_ptrs<W>(blk + sl_off, np, lane, dict, op0, kp0, pd0);
  lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l0), l0 < nrows);
  int32_t c0[W];
  dp_cols<W>(op0, c0);
  typename LeanX<CPLX>::T x0[W];
#pragma unroll
  for (int j = 0; j < W; ++j) x0[j] = lean_gather<CPLX, false>(rp0, c0[j]);
  double v[W];
  dp_vals<W>(kp0, dict, pd0, v);
  LeanSum<CPLX> a = lean_chain<W, CPLX, EXACT>(v, x0);
  if (padded && (lean_nan(a.r) || (CPLX && lean_nan(a.i))))
    if (l0 < nrows) a = dp_row_exact<CPLX, EXACT>(op0, kp0, dict, pd0, rp0, rowlen[r0 + l0]);
  if (l0 < nrows) lean_store_pf<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l0), a);
}

// One DP unit of width W: rec = {slice a off, slice b off,
// W | flags | Pa << 16 | Pb << 24, slice ids} as for lean pattern units.
// Real vectors keep both slices of a pair in flight (2W gathers); complex
// vectors take a pair's slices one after the other (2W double2 gathers exceed
// the register budget; dp_build gives complex tilings single-slice units).
template <int W, bool CPLX, bool EXACT, bool GEN>
__device__ __forceinline__ void dp_unit(uint32_t blk, uint4 rec, uint32_t lane, int32_t r0, int32_t nrows,
                                        const PowTab& pt, double* acc, bool use_acc, const uint8_t* rowlen) {
  constexpr int cw = CPLX ? 16 : 8;
  const uint32_t dict = blk + kLeanDict;
  const int32_t s0 = int32_t(rec.w & 0xffffu), s1 = int32_t(rec.w >> 16);
  const int32_t l0 = s0 * 32 + int32_t(lane), l1 = s1 * 32 + int32_t(lane);
  const bool pair = (rec.z & kLeanPair) != 0;
  const bool padded = (rec.z & kLeanPadded) != 0;
  if constexpr (W == 0) {
    if (l0 < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l0), LeanSum<CPLX>{0.0, 0.0});
    if (pair && l1 < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l1), LeanSum<CPLX>{0.0, 0.0});
  } else if constexpr (CPLX) {
#pragma unroll 1
    for (int h = 0; h < (pair ? 2 : 1); ++h)
      dp_single<W, CPLX, EXACT, GEN>(blk, h ? rec.y : rec.x, h ? (rec.z >> 24) : ((rec.z >> 16) & 255u), h ? s1 : s0,
                                     padded, lane, r0, nrows, pt, acc, use_acc, rowlen);
  } else if (!pair) {
    dp_single<W, CPLX, EXACT, GEN>(blk, rec.x, (rec.z >> 16) & 255u, s0, padded, lane, r0, nrows, pt, acc, use_acc,
                                   rowlen);
  } else {
    const char* rp0 = pt.yin + int64_t(r0 + min(l0, nrows - 1)) * cw;
    const char* rp1 = pt.yin + int64_t(r0 + min(l1, nrows - 1)) * cw;
    asm("" : "+l"(rp0));  // opaque bases: one IMAD.WIDE per gather (see lean_unit's fast path)
    asm("" : "+l"(rp1));
    uint32_t op0, kp0, pd0, op1, kp1, pd1;
    dp_ptrs<W>(blk + rec.x, (rec.z >> 16) & 255u, lane, dict, op0, kp0, pd0);
    dp_ptrs<W>(blk + rec.y, rec.z >> 24, lane, dict, op1, kp1, pd1);
    lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l0), l0 < nrows);
    lean_prefetch_epi<CPLX, GEN>(pt, acc, use_acc, int64_t(r0 + l1), l1 < nrows);
    int32_t c0[W], c1[W];
    dp_cols<W>(op0, c0);
    dp_cols<W>(op1, c1);
    typename LeanX<CPLX>::T x0[W], x1[W];
#pragma unroll
    for (int j = 0; j < W; ++j) x0[j] = lean_gather<CPLX, false>(rp0, c0[j]);
#pragma unroll
    for (int j = 0; j < W; ++j) x1[j] = lean_gather<CPLX, false>(rp1, c1[j]);
    LeanSum<CPLX> a, b;
    {
      double v[W];
      dp_vals<W>(kp0, dict, pd0, v);
      a = lean_chain<W, CPLX, EXACT>(v, x0);
    }
    {
      double v[W];
      dp_vals<W>(kp1, dict, pd1, v);
      b = lean_chain<W, CPLX, EXACT>(v, x1);
    }
    if (padded) {
      if (lean_nan(a.r))
        if (l0 < nrows) a = dp_row_exact<CPLX, EXACT>(op0, kp0, dict, pd0, rp0, rowlen[r0 + l0]);
      if (lean_nan(b.r))
        if (l1 < nrows) b = dp_row_exact<CPLX, EXACT>(op1, kp1, dict, pd1, rp1, rowlen[r0 + l1]);
    }
    if (l0 < nrows) lean_store_pf<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l0), a);
    if (l1 < nrows) lean_store_pf<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + l1), b);
  }
}

// ---------------------------------------------------------------- XP units
// Staged dictionary tilings whose slices repeat few distinct rows (structured
// grids) use XP blocks: a unit is a run of m <= 4 consecutive slices.  Its
// data is one ROW RECORD per distinct row of the slice --
//   [Wc x i32: (x-buffer entry - lane) * entry bytes][Wc x f64: values]
// -- behind 32 u8 record ids when the rows differ; a UNIFORM unit (every row
// of every slice the same record, the interior of a grid) holds the one
// record and no ids, and its m slices reuse the registers: slice i gathers at
// the same fields + 32 i entries.  A row costs no index arithmetic beyond one
// add per gather and no dictionary lookups.
constexpr uint32_t kXpUniform = 1u << 8, kXpPadded = 1u << 9;
__host__ __device__ constexpr int xp_rec_bytes(int w) { return 12 * lean_wc(w); }

template <int W>
__device__ __forceinline__ void xp_load(uint32_t ra, int32_t (&c)[W], double (&v)[W]) {
  constexpr int WC = lean_wc(W);
  {
    const uint4 a = lds_v4(ra);
    const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 0; j < (W < 4 ? W : 4); ++j) c[j] = int32_t(w4[j]);
  }
  if constexpr (W > 4) {
    const uint4 a = lds_v4(ra + 16);
    const uint32_t w4[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int j = 4; j < W; ++j) c[j] = int32_t(w4[j - 4]);
  }
#pragma unroll
  for (int j = 0; j + 1 < W; j += 2) {
    const double2 d = lds_d2(ra + 4 * WC + 8 * j);
    v[j] = d.x, v[j + 1] = d.y;
  }
  if constexpr (W & 1) v[W - 1] = lds_d(ra + 4 * WC + 8 * (W - 1));
}

// gather at byte offset c from the lane's row pointer (x staging: shared)
template <bool CPLX, bool XS>
__device__ __forceinline__ typename LeanX<CPLX>::T xp_gather(typename LeanRp<XS>::T rp, int32_t c) {
  if constexpr (XS) {
    if constexpr (CPLX)
      return lds_d2(rp + uint32_t(c));
    else
      return lds_d(rp + uint32_t(c));
  } else if constexpr (CPLX) {
    double2 v;
    asm("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(rp + int64_t(c)));
    return v;
  } else {
    double v;
    asm("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(rp + int64_t(c)));
    return v;
  }
}

// slow path of a padded row whose sum came out NaN: the row's true length
template <bool CPLX, bool EXACT, bool XS>
__device__ __noinline__ LeanSum<CPLX> xp_row_exact(uint32_t ra, typename LeanRp<XS>::T rp, int wc, int len) {
  LeanSum<CPLX> s{0.0, 0.0};
  for (int j = 0; j < len; ++j) {
    const int32_t c = int32_t(lds_u32(ra + 4 * j));
    const double v = lds_d(ra + 4 * wc + 8 * j);
    const typename LeanX<CPLX>::T x = xp_gather<CPLX, XS>(rp, c);
    if constexpr (CPLX) {
      s.r = madd<EXACT>(s.r, v, x.x);
      s.i = madd<EXACT>(s.i, v, x.y);
    } else {
      s.r = madd<EXACT>(s.r, v, x);
    }
  }
  return s;
}

// rec = {data offset, first slice | m << 16, W | flags, records}.  XS: the
// fields are x-buffer offsets (gathers from shared memory at xb); otherwise
// (column - row) byte offsets and the gathers read y_{p-1} in global memory.
template <int W, bool CPLX, bool EXACT, bool GEN, bool XS = true>
__device__ __forceinline__ void xp_unit(uint32_t blk, uint4 rec, uint32_t lane, int32_t r0, int32_t nrows,
                                        const PowTab& pt, double* acc, bool use_acc, const uint8_t* rowlen,
                                        uint32_t xb) {
  constexpr uint32_t cw = CPLX ? 16u : 8u;
  const int32_t m = int32_t(rec.y >> 16);
  int32_t lr = int32_t(rec.y & 0xffffu) * 32 + int32_t(lane);  // tile-local row
  typename LeanRp<XS>::T rp;
  if constexpr (XS)
    rp = xb + lane * cw;
  else
    rp = pt.yin + int64_t(r0 + lr) * int64_t(cw);
  if constexpr (W == 0) {
    for (int32_t i = 0; i < m; ++i, lr += 32)
      if (lr < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + lr), LeanSum<CPLX>{0.0, 0.0});
  } else {
    uint32_t ra = blk + rec.x;
    if (!(rec.z & kXpUniform)) ra += 32u + lds_b8(ra + lane) * uint32_t(xp_rec_bytes(W));
    int32_t c[W];
    double v[W];
    xp_load<W>(ra, c, v);
    const bool padded = (rec.z & kXpPadded) != 0;
    for (int32_t i = 0; i < m; ++i) {
      typename LeanX<CPLX>::T x[W];
#pragma unroll
      for (int j = 0; j < W; ++j) x[j] = xp_gather<CPLX, XS>(rp, c[j]);
      LeanSum<CPLX> a = lean_chain<W, CPLX, EXACT>(v, x);
      if (padded && (lean_nan(a.r) || (CPLX && lean_nan(a.i))))
        if (lr < nrows) a = xp_row_exact<CPLX, EXACT, XS>(ra, rp, lean_wc(W), rowlen[r0 + lr]);
      if (lr < nrows) lean_store<CPLX, EXACT, GEN>(pt, acc, use_acc, int64_t(r0 + lr), a);
      rp += 32u * cw;
      lr += 32;
    }
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
template <bool CPLX, bool EXACT, bool VD, bool GEN, int NP, bool XP = false, bool DP = false>
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
      if (XP && lds_u32(blk + 8) == 2u) {
        // XP block (row records, units of up to 4 slices; the units are
        // binned per consumer warp at build time, bin starts at blk + 16)
        const uint32_t b2 = lds_u32(blk + 16u + 2u * uint32_t(u & ~1));
        const int32_t ub = (u & 1) ? int32_t(b2 >> 16) : int32_t(b2 & 0xffffu);
        const uint32_t e2 = lds_u32(blk + 16u + 2u * uint32_t((u + 1) & ~1));
        const int32_t ue = ((u + 1) & 1) ? int32_t(e2 >> 16) : int32_t(e2 & 0xffffu);
        for (int32_t q = ub; q < ue; ++q) {
          const uint4 rec = lds_v4(blk + kLeanRec + uint32_t(q) * 16u);
          switch (rec.z & 15u) {
#define LMPK_XP_CASE(Wv) \
  case Wv: xp_unit<Wv, CPLX, EXACT, GEN, false>(blk, rec, lane, r0, nrows, pt, P.acc, use_acc, L.rowlen, 0u); break;
            LMPK_XP_CASE(0)
            LMPK_XP_CASE(1)
            LMPK_XP_CASE(2)
            LMPK_XP_CASE(3)
            LMPK_XP_CASE(4)
            LMPK_XP_CASE(5)
            LMPK_XP_CASE(6)
            LMPK_XP_CASE(7)
            LMPK_XP_CASE(8)
#undef LMPK_XP_CASE
            default: break;
          }
        }
        u = nu;  // the lean loop below is skipped
      }
      // a warp's units of one piece come width class by width class (the
      // builder sorts them): a run of units of one width stays inside that
      // width's compiled body instead of going through the jump table again
      while (u < nu) {
        uint4 rec = lds_v4(blk + kLeanRec + uint32_t(u) * 16u);
        switch (rec.z & 15u) {
#define LMPK_LEAN_CASE(Wv)                                                                     \
  case Wv:                                                                                     \
    for (;;) {                                                                                 \
      if constexpr (DP)                                                                        \
        dp_unit<Wv, CPLX, EXACT, GEN>(blk, rec, lane, r0, nrows, pt, P.acc, use_acc, L.rowlen); \
      else                                                                                     \
        lean_unit<Wv, CPLX, EXACT, VD, GEN>(blk, rec, lane, r0, nrows, pt, P.acc, use_acc, L.rowlen); \
      u += NC;                                                                                 \
      if (u >= nu) break;                                                                      \
      rec = lds_v4(blk + kLeanRec + uint32_t(u) * 16u);                                        \
      if ((rec.z & 15u) != uint32_t(Wv)) break;                                                \
    }                                                                                          \
    break;
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
          default: u += NC; break;
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

// ---------------------------------------------------------------- staged kernel
// The lean walk with x staging: a piece is [lean block | x buffer].  The
// producer bulk-copies, behind the tile's block, the runs of y_{p-1} the tile's
// rows gather (LeanParams::runs, planned once per tiling by k_lean_xplan) --
// after the item's dependencies were acquired, with a generic->async proxy
// fence in between -- and the consumers gather from shared memory: an
// unaligned 32 x 8 B gather costs 2 shared-memory wavefronts instead of 3 L1
// tag lookups and never waits for an L1 miss.  Ring depth L.np (2..4, run
// time): the slot and its phase are stepped, not divided.
// Dependency wait of the staged kernel: progress[lo..hi] >= target with
// ACQUIRE loads (LDG.STRONG.GPU + CCTL.IVALL) instead of relaxed loads and a
// gpu-scope fence (MEMBAR.ALL.GPU: ~1 us on a busy SM, once per item): the
// data behind the flags is only read by the bulk copies issued afterwards.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool spin_deps_acq(const MpkParams& P, int32_t lo, int32_t hi, uint32_t target,
                                              unsigned long long* rounds) {
  const int lane = threadIdx.x & 31;
  unsigned long long t0 = 0;
  for (int spins = 0;; ++spins) {
    uint32_t m = 0xffffffffu;
    for (int32_t i = lo + lane; i <= hi; i += 32) m = min(m, ld_acquire_u32(P.progress + i));
    ++*rounds;
    if (__all_sync(0xffffffffu, m >= target)) return true;
    if (spins > 2) __nanosleep(64);
    if ((spins & 63) == 63) {
      const unsigned long long now = globaltimer();
      if (t0 == 0) t0 = now;
      const volatile unsigned long long* ab = P.queue + 1;
      bool stop = *ab != 0ull;
      if (!stop && now - t0 > kWatchdogNs) {
        if (lane == 0) {
          atomicExch(P.queue + 1, 1ull);
          *P.err = 1;
        }
        stop = true;
      }
      if (__any_sync(0xffffffffu, stop)) return false;
    }
  }
}

constexpr int kXleanRingMax = 4;
// NCV consumer warps and MINB CTAs per SM: (26, 1) or (12, 2) -- two CTAs per SM
// are two independent rings, so one CTA's hand-off gaps are the other's work.
constexpr int kXleanConsumers2 = 12;
template <bool CPLX, bool EXACT, bool VD, bool GEN, bool XP = false, int NCV = kLeanConsumers, int MINB = 1>
__global__ void __launch_bounds__(32 * (NCV + 2), MINB)
    mpk_xlean_kernel(MpkParams P, PowerCfgDev C, LeanParams L) {
  constexpr int NC = NCV;
  constexpr int NPM = kXleanRingMax;
  constexpr uint32_t cw = CPLX ? 16u : 8u;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NQ = 8;  // publish queue entries
  __shared__ uint64_t full_bar[NPM], empty_bar[NPM], done_bar[NQ], pq_free[NQ];
  __shared__ int32_t d_t[NPM], d_p[NPM], pq_t[NQ], pq_p[NQ];
  __shared__ uint32_t d_done[NPM];
  __shared__ uint32_t trace_ctr;
  __shared__ PowTab s_pow[LMPK_MAX_POWERS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  build_powtab(s_pow, P, C);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NPM; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
      d_done[i] = 0;
    }
    for (int i = 0; i < NQ; ++i) {
      mbar_init(&done_bar[i], 1);
      mbar_init(&pq_free[i], 1);
    }
    trace_ctr = 0;
    fence_mbar_init();
  }
  __syncthreads();
  const int NP = L.np;
  const uint32_t cap = uint32_t(P.smem_cap);
  const uint32_t ring = smem_u32(smem_raw);
  if (warp == NC + 1) {
    // ------------------------------------------------ publisher
    // The last consumer warp of a piece frees its slot itself and queues
    // (tile, power) here; the publisher makes every piece queued so far
    // visible with ONE gpu-scope fence (~1-2 us on a busy SM: per piece it
    // would cap the walk at one piece per fence) and relaxed flag stores.
    if (lane == 0) {
      uint32_t kk = 0;
      for (bool stop = false; !stop;) {
        mbar_wait_sleep(&done_bar[kk & (NQ - 1)], (kk / NQ) & 1u);
        const uint32_t k0 = kk++;
        while (kk - k0 < uint32_t(L.pub_batch) && mbar_try_wait(&done_bar[kk & (NQ - 1)], (kk / NQ) & 1u)) ++kk;
        fence_acq_rel_gpu();
        for (uint32_t q = k0; q < kk; ++q) {
          const int32_t t = pq_t[q & (NQ - 1)], p = pq_p[q & (NQ - 1)];
          mbar_arrive(&pq_free[q & (NQ - 1)]);
          if (t < 0) {
            stop = true;
            break;
          }
          st_relaxed_u32(P.progress + t, P.epoch_base + uint32_t(p));
        }
      }
    }
  } else if (warp == NC) {
    // ------------------------------------------------ producer
    const int pm = (P.flags >> 8) & 3;
    const uint64_t pol = pm == 1 ? policy_evict_normal() : (pm == 3 ? policy_evict_last() : policy_evict_first());
    const uint64_t xpol = policy_evict_normal();
    unsigned long long rounds = 0;
    int slot = 0;
    uint32_t ph = 0;
    bool wrapped = false, abort = false;
    if (L.wl) {
      // ---- static work list: 32 piece records per coalesced load; the runs
      // of the next piece are fetched while this one waits for its slot
      const int32_t w0 = __ldg(L.wl_ptr + blockIdx.x), w1 = __ldg(L.wl_ptr + blockIdx.x + 1);
      for (int32_t base = w0; base < w1 && !abort; base += 32) {
        int4 ra = make_int4(0, 0, 0, 0), rb = ra;
        if (base + lane < w1) {
          ra = __ldg(L.wl + 2 * int64_t(base + lane));
          rb = __ldg(L.wl + 2 * int64_t(base + lane) + 1);
        }
        const int32_t cnt = min(32, w1 - base);
        int4 rn = make_int4(0, 0, 0, 0);
        {
          const int32_t mf = __shfl_sync(0xffffffffu, ra.x, 0), nf = __shfl_sync(0xffffffffu, rb.w, 0) & 255;
          if (lane < nf) rn = __ldg(L.runs + int64_t(mf) * kLeanMaxRuns + lane);
        }
        for (int32_t j = 0; j < cnt; ++j) {
          const int32_t m = __shfl_sync(0xffffffffu, ra.x, j), pf = __shfl_sync(0xffffffffu, ra.y, j);
          const int32_t dlo = __shfl_sync(0xffffffffu, ra.z, j), dhi = __shfl_sync(0xffffffffu, ra.w, j);
          const uint32_t olo = uint32_t(__shfl_sync(0xffffffffu, rb.x, j)), ohi = uint32_t(__shfl_sync(0xffffffffu, rb.y, j));
          const int32_t bytes = __shfl_sync(0xffffffffu, rb.z, j), xw = __shfl_sync(0xffffffffu, rb.w, j);
          const int4 rc = rn;  // this piece's runs; fetch the next piece's
          if (j + 1 < cnt) {
            const int32_t mn = __shfl_sync(0xffffffffu, ra.x, j + 1), nn = __shfl_sync(0xffffffffu, rb.w, j + 1) & 255;
            if (lane < nn) rn = __ldg(L.runs + int64_t(mn) * kLeanMaxRuns + lane);
          }
          const int32_t p = pf & 255;
          if (p > P.n_powers) continue;
          if (pf & 256) {
            if (lane == 0) trace_ev(P, &trace_ctr, 1, 0, uint32_t(m) << 8 | uint32_t(p));
            if (p > 1 && !spin_deps_acq(P, dlo, dhi, P.epoch_base + uint32_t(p - 1), &rounds)) {
              abort = true;
              break;
            }
            // the bulk copies below read y_{p-1} through the async proxy
            asm volatile("fence.proxy.async.global;" ::: "memory");
            if (lane == 0) trace_ev(P, &trace_ctr, 4, 0, uint32_t(m) << 8 | uint32_t(p));
          }
          if (wrapped && !mbar_wait_bounded(&empty_bar[slot], ph ^ 1u, P)) {
            abort = true;
            break;
          }
          if (lane == 0) {
            d_t[slot] = m;
            d_p[slot] = p;
            trace_ev(P, &trace_ctr, 2, uint32_t(slot), uint32_t(m) << 8 | uint32_t(p));
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[slot], uint32_t(bytes) + uint32_t(xw >> 8) * cw);
            bulk_g2s_a(ring + uint32_t(slot) * cap, L.blocks + (int64_t(ohi) << 32 | int64_t(olo)), uint32_t(bytes),
                       &full_bar[slot], p == P.n_powers ? policy_evict_first() : pol);
          }
          __syncwarp();
          if (lane < (xw & 255))
            bulk_g2s_a(ring + uint32_t(slot) * cap + uint32_t(L.xoff) + uint32_t(rc.z) * cw,
                       s_pow[p - 1].yin + int64_t(rc.x) * int64_t(cw), uint32_t(rc.y) * cw, &full_bar[slot], xpol);
          __syncwarp();
          if (++slot == NP) slot = 0, ph ^= 1u, wrapped = true;
        }
      }
      // keep the ticket counter where the queue walk would leave it (the host
      // advances queue_base by n_items + grid per launch)
      if (lane == 0) {
        const int32_t mine = (P.n_items > int32_t(blockIdx.x)) ? (P.n_items - 1 - int32_t(blockIdx.x)) / int32_t(gridDim.x) + 1 : 0;
        atomicAdd(P.queue, static_cast<unsigned long long>(mine + 1));
      }
    } else
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
      if (p > 1 && !spin_deps_acq(P, __ldg(P.st_lo + T), __ldg(P.st_hi + T), P.epoch_base + uint32_t(p - 1), &rounds)) {
        abort = true;
        break;
      }
      // the bulk copies below read y_{p-1} through the async proxy
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (lane == 0) trace_ev(P, &trace_ctr, 4, 0, uint32_t(T) << 8 | uint32_t(p));
      const char* yin = s_pow[p - 1].yin;
      for (int32_t m = m0; m < m1; ++m) {
        if (wrapped && !mbar_wait_bounded(&empty_bar[slot], ph ^ 1u, P)) {
          abort = true;
          break;
        }
        const int2 xi = __ldg(L.xinfo + m);
        if (lane == 0) {
          const int64_t ofs = __ldg(L.ofs + m), bytes = __ldg(L.ofs + m + 1) - ofs;
          d_t[slot] = m;
          d_p[slot] = p;
          trace_ev(P, &trace_ctr, 2, uint32_t(slot), uint32_t(m) << 8 | uint32_t(p));
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&full_bar[slot], uint32_t(bytes) + uint32_t(xi.y) * cw);
          bulk_g2s_a(ring + uint32_t(slot) * cap, L.blocks + ofs, uint32_t(bytes), &full_bar[slot],
                     p == P.n_powers ? policy_evict_first() : pol);
        }
        __syncwarp();
        if (lane < xi.x) {
          const int4 rn = __ldg(L.runs + int64_t(m) * kLeanMaxRuns + lane);
          bulk_g2s_a(ring + uint32_t(slot) * cap + uint32_t(L.xoff) + uint32_t(rn.z) * cw,
                     yin + int64_t(rn.x) * int64_t(cw), uint32_t(rn.y) * cw, &full_bar[slot], xpol);
        }
        __syncwarp();
        if (++slot == NP) slot = 0, ph ^= 1u, wrapped = true;
      }
      if (abort) break;
    }
    if (lane == 0) {
      bool ok = true;
      if (wrapped) {
        unsigned long long t0 = globaltimer();
        while (!mbar_try_wait(&empty_bar[slot], ph ^ 1u)) {
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
    int slot = 0;
    uint32_t ph = 0, kk = 0;
    int32_t rot = warp;
    for (;;) {
      const uint32_t blk = lean_wait(&full_bar[slot], ph, ring + uint32_t(slot) * cap);
      const int32_t t = d_t[slot];
      if (t < 0) {
        if (warp == 0 && lane == 0) {
          const uint32_t q = kk & (NQ - 1);
          if (kk >= uint32_t(NQ)) mbar_wait(&pq_free[q], (kk / NQ - 1) & 1u);
          pq_t[q] = -1;
          mbar_arrive(&done_bar[q]);
        }
        break;
      }
      const int32_t p = d_p[slot];
      const uint4 hdr = lds_v4(blk);  // {units, rows, format, first row}
      const int32_t nu = int32_t(hdr.x), nrows = int32_t(hdr.y), r0 = int32_t(hdr.w);
      const uint32_t xb = blk + uint32_t(L.xoff);
      const PowTab& pt = s_pow[p - 1];
      if (lane == 0) trace_ev(P, &trace_ctr, 10, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
      // static striding, rotated piece by piece; XP tilings: a piece is an XP
      // block (header word 2 == 2) or a lean block
#define LMPK_XLEAN_LOOP(UNIT)                                        \
  for (int32_t u = rot; u < nu; u += NC) {                           \
    const uint4 rec = lds_v4(blk + kLeanRec + uint32_t(u) * 16u);    \
    switch (rec.z & 15u) {                                           \
      case 0: UNIT(0) break;                                         \
      case 1: UNIT(1) break;                                         \
      case 2: UNIT(2) break;                                         \
      case 3: UNIT(3) break;                                         \
      case 4: UNIT(4) break;                                         \
      case 5: UNIT(5) break;                                         \
      case 6: UNIT(6) break;                                         \
      case 7: UNIT(7) break;                                         \
      case 8: UNIT(8) break;                                         \
      default: break;                                                \
    }                                                                \
  }
#define LMPK_UNIT_XP(Wv) xp_unit<Wv, CPLX, EXACT, GEN>(blk, rec, lane, r0, nrows, pt, P.acc, use_acc, L.rowlen, xb);
#define LMPK_UNIT_LEAN(Wv) \
  lean_unit<Wv, CPLX, EXACT, VD, GEN, true>(blk, rec, lane, r0, nrows, pt, P.acc, use_acc, L.rowlen, xb);
      if (XP && hdr.z == 2u) {
        // XP blocks: the units are binned per consumer warp at build time
        // (longest-first onto the lightest bin); bin starts at blk + 16
        const uint32_t b2 = lds_u32(blk + 16u + 2u * uint32_t(rot & ~1));
        const int32_t ub = (rot & 1) ? int32_t(b2 >> 16) : int32_t(b2 & 0xffffu);
        const uint32_t e2 = lds_u32(blk + 16u + 2u * uint32_t((rot + 1) & ~1));
        const int32_t ue = ((rot + 1) & 1) ? int32_t(e2 >> 16) : int32_t(e2 & 0xffffu);
        for (int32_t u = ub; u < ue; ++u) {
          const uint4 rec = lds_v4(blk + kLeanRec + uint32_t(u) * 16u);
          switch (rec.z & 15u) {
            case 0: LMPK_UNIT_XP(0) break;
            case 1: LMPK_UNIT_XP(1) break;
            case 2: LMPK_UNIT_XP(2) break;
            case 3: LMPK_UNIT_XP(3) break;
            case 4: LMPK_UNIT_XP(4) break;
            case 5: LMPK_UNIT_XP(5) break;
            case 6: LMPK_UNIT_XP(6) break;
            case 7: LMPK_UNIT_XP(7) break;
            case 8: LMPK_UNIT_XP(8) break;
            default: break;
          }
        }
      } else {
        LMPK_XLEAN_LOOP(LMPK_UNIT_LEAN)
      }
#undef LMPK_UNIT_XP
#undef LMPK_UNIT_LEAN
#undef LMPK_XLEAN_LOOP
      if (++rot == NC) rot = 0;
      __syncwarp();
      if (lane == 0) trace_ev(P, &trace_ctr, 11, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
      uint32_t old = 0;
      if (lane == 0) old = atom_add_acqrel_cta_smem(&d_done[slot], 1u);
      if (__shfl_sync(0xffffffffu, old, 0) == uint32_t(NC - 1) && lane == 0) {
        // last warp of the piece: queue it for the publisher, free the slot
        trace_ev(P, &trace_ctr, 12, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
        d_done[slot] = 0;
        const uint32_t q = kk & (NQ - 1);
        if (kk >= uint32_t(NQ)) mbar_wait(&pq_free[q], (kk / NQ - 1) & 1u);
        pq_t[q] = t;
        pq_p[q] = p;
        mbar_arrive(&done_bar[q]);
        mbar_arrive(&empty_bar[slot]);
      }
      ++kk;
      if (++slot == NP) slot = 0, ph ^= 1u;
    }
  }
}

}  // namespace lmpk
