// mpk_kernel.cuh -- level-blocked matrix power kernel for sm_100a (device code;
// instantiated once per variant in mpk_k_*.cu, host side in mpk.cu).
//
// Reference: the diagonal Lp-diagram walk of pkg/src/levelmpk/schedule.py:91-99
// executed by the p2p walker _walk/_wait_all (executor.py:84-150) over the
// flat ExecPlan (plan.py:184-370).  The GPU form:
//
//   * the level-permuted matrix is cut into contiguous row TILES (multiples
//     of 32 rows) sized to the shared-memory budget and re-laid out once as
//     "tile-SELL-32" blocks.  Per 32-row slice of width w (its longest row)
//     the entries are stored in CHUNKS of 4, 2 and 1 entries (w = 4Q + 2P + S):
//     inside a chunk of c entries, lane i's c entries are contiguous, so one
//     LDS.128 fetches four column indices and two LDS.128 four values; the
//     warp reads each chunk as one conflict-free contiguous row of smem.
//     Each row is still summed in CRS storage order (padding is skipped), so
//     the bit-exact mode reproduces the reference bitwise;
//   * tile t's dependency range [dep_lo(t), dep_hi(t)] is the set of tiles
//     owning its column indices (level confinement, Eq. 4 of the paper,
//     keeps it narrow: a tile couples only to its own and adjacent levels);
//   * WORK ITEMS are (tile t, power group g): the powers gq+1 .. gq+q of one
//     tile, computed on ONE staged copy of the tile block (q = powers per
//     item).  Items are queued by the skewed diagonal key (t + g*M, g),
//     M = q*D + slack (D = max forward reach), which is topologically valid
//     and keeps the items of one key window inside the 126 MB L2: the block
//     is read from HBM once and re-staged from L2 once per group, i.e. the
//     matrix crosses the L2->SM path ceil(p_m/q) times instead of p_m times.
//     q = p_m is the fully SMEM-resident walk (one group), q = 1 the pure
//     streaming walk;
//   * a persistent grid (one CTA per SM: 1 producer warp + NC consumer warps)
//     holds R items in R shared-memory slots.  The producer grabs items in
//     queue order (one atomic ticket each), stages the block with one TMA
//     bulk copy, and polls the dependencies of every held item WITHOUT
//     blocking on any one of them (one batch of relaxed loads per round, then
//     one fence.acq_rel.gpu: acquire + L1 invalidation).  A ready (slot, p)
//     goes into a small smem work ring; consumer warps drain the ring with no
//     CTA-wide barrier, and the last warp to finish a (tile, power) publishes
//     the tile's epoch-tagged progress word with a gpu-scope release -- the
//     device form of conditions (A)/(B)/(C) (schedule.py:195-240).
//     Deadlock freedom: items are grabbed in queue order, so the oldest
//     unfinished item X always progresses if every item it transitively waits
//     on inside its group is held: at most G*(chain_q + 1) queue positions
//     after X (G groups per key, chain_q = (q-1)-step forward chain reach),
//     checked against grid*R when the tiling is planned;
//   * SWEEP (LMPK_FLAG_SWEEP): n_powers dependency-free passes, one launch
//     per power -- the blocking-free "k back-to-back SpMVs" baseline on the
//     same tiles and the same row kernel.
#pragma once
#include <string.h>

#include <algorithm>
#include <numeric>

#include "lmpk_internal.cuh"

namespace lmpk {

constexpr uint32_t kEpochStride = 128;  // > LMPK_MAX_POWERS
constexpr unsigned long long kWatchdogNs = 8ull * 1000 * 1000 * 1000;
#ifndef LMPK_MAXSLOTS
#define LMPK_MAXSLOTS 4
#endif
constexpr int kMaxSlots = LMPK_MAXSLOTS;
constexpr int kWorkRing = 8;
#ifndef LMPK_NC
#define LMPK_NC 24
#endif
constexpr int kConsumers = LMPK_NC;  // consumer warps per CTA (+1 producer warp)
#ifndef LMPK_RING_NC
#define LMPK_RING_NC 26
#endif
// ring walk: consumer warps per CTA (+ producer + publisher); 26 measured
// 1.5% faster than 24 on cfg2, 28 spills
constexpr int kRingConsumers = LMPK_RING_NC;
constexpr int kBlockThreads = 32 * (kConsumers + kMaxSlots);  // launched with NC + R warps

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
  const int32_t* rdep_ptr;   // ready-queue walk: tiles depending on tile t are
  const int32_t* rdep;       //   rdep[rdep_ptr[t] .. rdep_ptr[t+1])
  uint32_t* rcnt;            // [p_m][n_tiles] finished dependencies of (t, p+1)
  int32_t* rqueue;           // ready items (t << 8 | p), -1 = not yet written
  uint32_t* rctrl;           // [0] queue head, [32] queue tail, [64] next power-1 tile, [96] items done
  int32_t lead;              // ready walk: max power-1 lead (tiles) over the completed work
  int32_t n_tiles;
  const int32_t* tile_nseg;  // x-segments per tile (0: global columns)
  const int32_t* tile_xent;  // x-buffer entries per tile
  const int32_t* tile_mode;  // compressed block format per tile (kModeC16 | kModeDict | nd << 8), 0 = plain
  const int32_t* st_first;   // ring walk: super-tile -> first tile ([n_super + 1])
  const int32_t* st_lo;      // ring walk: dependency range of a super-tile, in tiles
  const int32_t* st_hi;
  const int32_t* items;  // packed (t << 8) | g in queue order (NULL: item i = tile i, g = 0)
  double* y;
  int64_t ldy;
  double* acc;
  int32_t use_acc;
  uint32_t* progress;
  unsigned long long* queue;  // [0] work counter, [1] abort flag
  unsigned long long queue_base;
  uint32_t epoch_base;
  int32_t n_items;
  int32_t n_powers;
  int32_t q;         // powers per item
  int32_t mode;      // 1 key-order group walk, 3 sweep (one power, no deps), 4 ready-queue walk (q = 1)
  int32_t smem_cap;  // bytes of one slot
  int32_t xoff;      // unused (the x buffer follows each tile's block in its slot)
  int32_t blk_cap;   // bytes of a slot available to the staged block
  int32_t xmode;     // 0 no x staging, 1 TMA (aligned vectors), 2 cooperative copy
  int32_t n_slots;   // R
  int32_t flags;     // LMPK_FLAG_* (NO_TMA, policy bits 8-9)
  int32_t ypol;      // y store L2 policy: 0 default, 1 evict_last, 2 evict_first (LMPK_YPOL)
  int* err;          // host-mapped
  unsigned long long* prof;  // optional phase counters (LMPK_PROFILE), else null
  uint4* trace;              // optional event trace (LMPK_TRACE), else null
};

// Trace events (kind): producer 1 fetched, 2 TMA issued, 3 staged, 4 deps
// ready, 5 pushed, 6 slot freed; consumer 10 item start, 11 item end, 12 last
// warp published.
__device__ __forceinline__ void trace_ev(const MpkParams& P, uint32_t* ctr, uint32_t kind, uint32_t slot,
                                         uint32_t item) {
  if (P.trace && blockIdx.x < kTraceCtas) {
    const uint32_t i = atomicAdd(ctr, 1u);
    if (i < uint32_t(kTraceEvents)) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      P.trace[blockIdx.x * kTraceEvents + i] =
          make_uint4(uint32_t(t), uint32_t(t >> 32), kind | (slot << 8) | ((threadIdx.x >> 5) << 16), item);
    }
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__host__ __device__ inline int64_t align16(int64_t b) { return (b + 15) & ~int64_t(15); }

// Block layout of a tile with ns slices, E entries (E = 32 * sum of widths)
// and nseg x-segments:
//   [rec int2 x ns] [lens uint16 x 32*ns] | align16 | [seg int4 x nseg]
//   [col int32 x E] [val f64 x E]
// rec[s] = {byte offset of slice s's first column index in the block,
//           w | wmin << 16} (w = longest row, wmin = shortest row).
// seg[j] = {first vector entry, entry count, local base, 0}: the tile's
// columns covered by even-aligned runs of the gathered vector.  When nseg > 0
// the columns are LOCAL indices into the slot's x buffer, which the producer
// fills with one bulk copy per run once the dependencies of a power are met
// (gathers then come from shared memory); nseg == 0 keeps global columns.
constexpr int kMaxSegs = 64;
#ifndef LMPK_TMA_SPLIT
#define LMPK_TMA_SPLIT 1
#endif
constexpr int kTmaSplit = LMPK_TMA_SPLIT;  // concurrent bulk copies per staged block
__host__ __device__ inline int64_t blk_seg_off(int32_t ns) { return align16(int64_t(ns) * 72); }
__host__ __device__ inline int64_t blk_col_off(int32_t ns, int32_t nseg) {
  return blk_seg_off(ns) + int64_t(nseg) * 16;
}
__host__ __device__ inline int64_t blk_bytes(int32_t ns, int64_t E, int32_t nseg) {
  return (blk_col_off(ns, nseg) + E * 12 + 127) & ~int64_t(127);
}

// Entry index of (lane, j) inside a slice of width w starting at entry `base`:
// quads first, then a pair, then a single entry.
__host__ __device__ inline int64_t chunk_entry(int64_t base, int w, int lane, int j) {
  const int Q = w >> 2;
  if (j < 4 * Q) return base + int64_t(j >> 2) * 128 + lane * 4 + (j & 3);
  const int r = j - 4 * Q;
  if ((w & 2) && r < 2) return base + int64_t(Q) * 128 + lane * 2 + r;
  return base + int64_t(Q) * 128 + ((w & 2) ? 64 : 0) + lane;
}

// ---------------------------------------------------------------- row kernel
// Gather sources of the row kernel: the vector in global memory (global
// columns) or the slot's x buffer in shared memory (local columns).
// row(r) / at(row, d): the entry at signed offset d from row r (compressed
// blocks), one IMAD.WIDE per gather instead of re-adding the row index.
struct GatherGlobal {
  const char* base;
  using Row = const char*;
  __device__ __forceinline__ Row row(int32_t r) const { return base + int64_t(r) * 8; }
  // one mad.wide per gather address (keeps the compiler from re-associating
  // base + 8 (row + d) into three integer ops)
  __device__ __forceinline__ double at(Row rp, int32_t d) const {
    const char* a;
    asm("mad.wide.s32 %0, %1, 8, %2;" : "=l"(a) : "r"(d), "l"(rp));
    return ldg_f64(a);
  }
  __device__ __forceinline__ double d(int32_t c) const { return ldg_f64(base + uint64_t(uint32_t(c)) * 8u); }
  __device__ __forceinline__ double2 d2(int32_t c) const {
    return ldg_f64x2(base + uint64_t(uint32_t(c)) * 16u);
  }
};
struct GatherSmem {
  uint32_t base;
  using Row = uint32_t;
  __device__ __forceinline__ Row row(int32_t r) const { return base + uint32_t(r) * 8u; }
  __device__ __forceinline__ double at(Row rp, int32_t d) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(rp + uint32_t(d) * 8u));
    return v;
  }
  __device__ __forceinline__ double d(int32_t c) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + uint32_t(c) * 8u));
    return v;
  }
  __device__ __forceinline__ double2 d2(int32_t c) const {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(base + uint32_t(c) * 16u));
    return v;
  }
};
// Per-power operands, built once per launch in shared memory (the consumers
// would otherwise re-derive them from the constant bank for every item).
struct PowTab {
  const char* yin;    // gathered vector y_{p-1}
  double* yout;       // y_p
  const double* ypv;  // y_{p-2} slot (Chebyshev)
  double cre, cim;    // acc coefficient
  int32_t general;    // Chebyshev step and/or accumulation
  int32_t cheb;
  uint64_t ypol;      // L2 cache policy of the y stores (0 = default)
};

template <bool EXACT>
__device__ __forceinline__ double madd(double t, double v, double x) {
  if constexpr (EXACT)
    return __dadd_rn(t, __dmul_rn(v, x));  // tmp = tmp + v*x, separately rounded
  else
    return __fma_rn(v, x, t);
}
// t = madd(t, v, x) only for entries j < len (the row's own length): one
// ISETP + predicated DFMA (or DMUL/DADD) instead of a select chain.
template <bool EXACT>
__device__ __forceinline__ void madd_if(double& t, double v, double x, int j, int len) {
  if constexpr (EXACT) {
    const double m = __dmul_rn(v, x);  // harmless for padding: only the add is predicated
    asm("{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %2, %3;\n\t@q add.rn.f64 %0, %0, %1;\n\t}"
        : "+d"(t)
        : "d"(m), "r"(j), "r"(len));
  } else {
    asm("{\n\t.reg .pred q;\n\tsetp.lt.s32 q, %3, %4;\n\t@q fma.rn.f64 %0, %1, %2, %0;\n\t}"
        : "+d"(t)
        : "d"(v), "d"(x), "r"(j), "r"(len));
  }
}
__device__ __forceinline__ void stg_f64(double* p, double v) {
  asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}
// y_p store with an optional L2 eviction-priority hint (pol != 0)
__device__ __forceinline__ void stg_y(double* p, double v, uint64_t pol) {
  if (pol)
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol));
  else
    asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ void stg_f64x2(double* p, double2 v) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y));
}

// Row sum of one slice of compile-time width W <= 8 (real vectors): all column
// loads, then all gathers, then the values and the ordered chain.  cb/vb are
// the slice's column/value byte offsets in the block, l4 = 4*lane.
template <int W, bool EXACT, bool FULL, class Blk, class G, int PROBE = 0>
__device__ __forceinline__ double slice_real_w(const Blk& B, uint32_t cb, uint32_t vb, uint32_t l4,
                                               const G& g, int len) {
  constexpr int Q = W >> 2, PR = (W >> 1) & 1, SG = W & 1;
  int32_t c[W];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int4 c4 = B.i4(cb + q * 512 + 4 * l4);
    c[4 * q] = c4.x;
    c[4 * q + 1] = c4.y;
    c[4 * q + 2] = c4.z;
    c[4 * q + 3] = c4.w;
  }
  if constexpr (PR) {
    const int2 c2 = B.i2(cb + Q * 512 + 2 * l4);
    c[4 * Q] = c2.x;
    c[4 * Q + 1] = c2.y;
  }
  if constexpr (SG) c[W - 1] = B.i1(cb + Q * 512 + PR * 256 + l4);
  double x[W];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    // PROBE (compute probe only): 1 = gathers confined to 8 KB, 2 = coalesced
    // gathers, 3 = no gathers
    if constexpr (PROBE == 1) c[j] &= 1023;
    if constexpr (PROBE == 2) c[j] = int32_t(l4 >> 2) + 32 * j;
    if constexpr (PROBE == 3)
      x[j] = __int_as_float(c[j]);
    else
      x[j] = g.d(c[j]);
  }
  double v[W];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double2 a = B.d2(vb + q * 1024 + 8 * l4), b = B.d2(vb + q * 1024 + 8 * l4 + 16);
    v[4 * q] = a.x;
    v[4 * q + 1] = a.y;
    v[4 * q + 2] = b.x;
    v[4 * q + 3] = b.y;
  }
  if constexpr (PR) {
    const double2 a = B.d2(vb + Q * 1024 + 4 * l4);
    v[4 * Q] = a.x;
    v[4 * Q + 1] = a.y;
  }
  if constexpr (SG) v[W - 1] = B.d1(vb + Q * 1024 + PR * 512 + 2 * l4);
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    if constexpr (FULL)
      t = madd<EXACT>(t, v[j], x[j]);
    else
      madd_if<EXACT>(t, v[j], x[j], j, len);
  }
  return t;
}

// Any width (real vectors): a loop over quads plus the pair/single tail.
template <bool EXACT, class Blk, class G>
__device__ __noinline__ double slice_real_any(const Blk& B, uint32_t cb, uint32_t vb, uint32_t l4,
                                              const G& g, int w, int len) {
  const int Q = w >> 2;
  double t = 0.0;
  for (int q = 0; q < Q; ++q) {
    const int4 c4 = B.i4(cb + q * 512 + 4 * l4);
    const double x0 = g.d(c4.x);
    const double x1 = g.d(c4.y);
    const double x2 = g.d(c4.z);
    const double x3 = g.d(c4.w);
    const double2 a = B.d2(vb + q * 1024 + 8 * l4), b = B.d2(vb + q * 1024 + 8 * l4 + 16);
    const int j = 4 * q;
    madd_if<EXACT>(t, a.x, x0, j, len);
    madd_if<EXACT>(t, a.y, x1, j + 1, len);
    madd_if<EXACT>(t, b.x, x2, j + 2, len);
    madd_if<EXACT>(t, b.y, x3, j + 3, len);
  }
  const int PR = (w >> 1) & 1;
  if (PR) {
    const int2 c2 = B.i2(cb + Q * 512 + 2 * l4);
    const double x0 = g.d(c2.x);
    const double x1 = g.d(c2.y);
    const double2 a = B.d2(vb + Q * 1024 + 4 * l4);
    madd_if<EXACT>(t, a.x, x0, 4 * Q, len);
    madd_if<EXACT>(t, a.y, x1, 4 * Q + 1, len);
  }
  if (w & 1) {
    const int32_t c = B.i1(cb + Q * 512 + PR * 256 + l4);
    const double x0 = g.d(c);
    const double a = B.d1(vb + Q * 1024 + PR * 512 + 2 * l4);
    madd_if<EXACT>(t, a, x0, w - 1, len);
  }
  return t;
}

// Complex vectors (real matrix): t += v * x per component, storage order.
template <bool EXACT, class Blk, class G>
__device__ __forceinline__ double2 slice_cplx(const Blk& B, uint32_t cb, uint32_t vb, uint32_t l4,
                                              const G& g, int w, int len) {
  double tr = 0.0, ti = 0.0;
  const int Q = w >> 2;
  for (int q = 0; q < Q; ++q) {
    const int4 c4 = B.i4(cb + q * 512 + 4 * l4);
    const double2 x0 = g.d2(c4.x);
    const double2 x1 = g.d2(c4.y);
    const double2 x2 = g.d2(c4.z);
    const double2 x3 = g.d2(c4.w);
    const double2 a = B.d2(vb + q * 1024 + 8 * l4), b = B.d2(vb + q * 1024 + 8 * l4 + 16);
    const int j = 4 * q;
    madd_if<EXACT>(tr, a.x, x0.x, j, len);
    madd_if<EXACT>(ti, a.x, x0.y, j, len);
    madd_if<EXACT>(tr, a.y, x1.x, j + 1, len);
    madd_if<EXACT>(ti, a.y, x1.y, j + 1, len);
    madd_if<EXACT>(tr, b.x, x2.x, j + 2, len);
    madd_if<EXACT>(ti, b.x, x2.y, j + 2, len);
    madd_if<EXACT>(tr, b.y, x3.x, j + 3, len);
    madd_if<EXACT>(ti, b.y, x3.y, j + 3, len);
  }
  const int PR = (w >> 1) & 1;
  if (PR) {
    const int2 c2 = B.i2(cb + Q * 512 + 2 * l4);
    const double2 x0 = g.d2(c2.x);
    const double2 x1 = g.d2(c2.y);
    const double2 a = B.d2(vb + Q * 1024 + 4 * l4);
    madd_if<EXACT>(tr, a.x, x0.x, 4 * Q, len);
    madd_if<EXACT>(ti, a.x, x0.y, 4 * Q, len);
    madd_if<EXACT>(tr, a.y, x1.x, 4 * Q + 1, len);
    madd_if<EXACT>(ti, a.y, x1.y, 4 * Q + 1, len);
  }
  if (w & 1) {
    const int32_t c = B.i1(cb + Q * 512 + PR * 256 + l4);
    const double2 x0 = g.d2(c);
    const double a = B.d1(vb + Q * 1024 + PR * 512 + 2 * l4);
    madd_if<EXACT>(tr, a, x0.x, w - 1, len);
    madd_if<EXACT>(ti, a, x0.y, w - 1, len);
  }
  return make_double2(tr, ti);
}

// Two slices of the same width W <= 8 at once (one warp): both slices'
// gathers are in flight together, so the second slice's L2 latency hides
// behind the first one's.
template <int W, bool EXACT, bool FULL, class Blk, class G>
__device__ __forceinline__ double2 slice_real_w2(const Blk& B, uint32_t cb0, uint32_t vb0, uint32_t cb1,
                                                 uint32_t vb1, uint32_t l4, const G& g, int len0,
                                                 int len1) {
  constexpr int Q = W >> 2, PR = (W >> 1) & 1, SG = W & 1;
  int32_t c0[W], c1[W];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int4 a = B.i4(cb0 + q * 512 + 4 * l4), b = B.i4(cb1 + q * 512 + 4 * l4);
    c0[4 * q] = a.x, c0[4 * q + 1] = a.y, c0[4 * q + 2] = a.z, c0[4 * q + 3] = a.w;
    c1[4 * q] = b.x, c1[4 * q + 1] = b.y, c1[4 * q + 2] = b.z, c1[4 * q + 3] = b.w;
  }
  if constexpr (PR) {
    const int2 a = B.i2(cb0 + Q * 512 + 2 * l4), b = B.i2(cb1 + Q * 512 + 2 * l4);
    c0[4 * Q] = a.x, c0[4 * Q + 1] = a.y;
    c1[4 * Q] = b.x, c1[4 * Q + 1] = b.y;
  }
  if constexpr (SG) {
    c0[W - 1] = B.i1(cb0 + Q * 512 + PR * 256 + l4);
    c1[W - 1] = B.i1(cb1 + Q * 512 + PR * 256 + l4);
  }
  double x0[W], x1[W];
#pragma unroll
  for (int j = 0; j < W; ++j) x0[j] = g.d(c0[j]);
#pragma unroll
  for (int j = 0; j < W; ++j) x1[j] = g.d(c1[j]);
  double t0 = 0.0, t1 = 0.0;
  {
    double v[W];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double2 a = B.d2(vb0 + q * 1024 + 8 * l4), b = B.d2(vb0 + q * 1024 + 8 * l4 + 16);
      v[4 * q] = a.x, v[4 * q + 1] = a.y, v[4 * q + 2] = b.x, v[4 * q + 3] = b.y;
    }
    if constexpr (PR) {
      const double2 a = B.d2(vb0 + Q * 1024 + 4 * l4);
      v[4 * Q] = a.x, v[4 * Q + 1] = a.y;
    }
    if constexpr (SG) v[W - 1] = B.d1(vb0 + Q * 1024 + PR * 512 + 2 * l4);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if constexpr (FULL)
        t0 = madd<EXACT>(t0, v[j], x0[j]);
      else
        madd_if<EXACT>(t0, v[j], x0[j], j, len0);
    }
  }
  {
    double v[W];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double2 a = B.d2(vb1 + q * 1024 + 8 * l4), b = B.d2(vb1 + q * 1024 + 8 * l4 + 16);
      v[4 * q] = a.x, v[4 * q + 1] = a.y, v[4 * q + 2] = b.x, v[4 * q + 3] = b.y;
    }
    if constexpr (PR) {
      const double2 a = B.d2(vb1 + Q * 1024 + 4 * l4);
      v[4 * Q] = a.x, v[4 * Q + 1] = a.y;
    }
    if constexpr (SG) v[W - 1] = B.d1(vb1 + Q * 1024 + PR * 512 + 2 * l4);
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if constexpr (FULL)
        t1 = madd<EXACT>(t1, v[j], x1[j]);
      else
        madd_if<EXACT>(t1, v[j], x1[j], j, len1);
    }
  }
  return make_double2(t0, t1);
}

template <bool EXACT, bool FULL, class Blk, class G>
__device__ __forceinline__ double2 slice_real_pair(const Blk& B, uint32_t cb0, uint32_t vb0, uint32_t cb1,
                                                   uint32_t vb1, uint32_t l4, const G& g, int w,
                                                   int len0, int len1) {
  switch (w) {
    case 1: return slice_real_w2<1, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    case 2: return slice_real_w2<2, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    case 3: return slice_real_w2<3, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    case 4: return slice_real_w2<4, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    case 5: return slice_real_w2<5, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    case 6: return slice_real_w2<6, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    case 7: return slice_real_w2<7, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
    default: return slice_real_w2<8, EXACT, FULL>(B, cb0, vb0, cb1, vb1, l4, g, len0, len1);
  }
}

template <bool EXACT, bool FULL, class Blk, class G, bool LONG = true>
__device__ __forceinline__ double slice_real(const Blk& B, uint32_t cb, uint32_t vb, uint32_t l4,
                                             const G& g, int w, int len) {
  switch (w) {
    case 1: return slice_real_w<1, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 2: return slice_real_w<2, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 3: return slice_real_w<3, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 4: return slice_real_w<4, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 5: return slice_real_w<5, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 6: return slice_real_w<6, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 7: return slice_real_w<7, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 8: return slice_real_w<8, EXACT, FULL>(B, cb, vb, l4, g, len);
    case 0: return 0.0;
    default:
      if constexpr (LONG)
        return slice_real_any<EXACT>(B, cb, vb, l4, g, w, FULL ? w : len);
      else
        return 0.0;  // the tiling has no slice wider than 8
  }
}

// Slice scheduling of one (tile, power) among the consumer warps: static
// striding (sched == kSchedStatic: warp w takes w, w + nwarps, ...) or dynamic
// grabs from a shared-memory counter (sched = its smem address), which keeps
// the warps balanced when a tile's slice count is not a multiple of the warp
// count (static striding always gives the low warps the extra slices).
constexpr uint32_t kSchedStatic = 0xffffffffu;
__device__ __forceinline__ int32_t sched_grab(uint32_t sched, uint32_t k) {
  uint32_t v = 0;
  if ((threadIdx.x & 31) == 0) asm volatile("atom.shared::cta.add.u32 %0, [%1], %2;" : "=r"(v) : "r"(sched), "r"(k) : "memory");
  return int32_t(__shfl_sync(0xffffffffu, v, 0));
}
__device__ __forceinline__ int32_t sched_first(uint32_t sched, int wid, uint32_t k) {
  return sched != kSchedStatic ? sched_grab(sched, k) : wid;
}
__device__ __forceinline__ int32_t sched_next(uint32_t sched, int32_t s, int step, uint32_t k) {
  return sched != kSchedStatic ? sched_grab(sched, k) : s + step;
}

// ---------------------------------------------------------------- compressed blocks
// Compressed tile block (tile_mode bit 0): the same slices, chunks and entry
// order as above, but
//   * columns are int16 offsets from the entry's own row (col - row): a
//     level-ordered matrix couples a row only to its own and the adjacent
//     levels, so the offsets stay within +-32767 for level widths up to that
//     (index compression in the style of CSR-DU, Kourtis et al. 2008);
//   * values are either raw f64, or (tile_mode bit 1) uint8 codes into a
//     per-tile dictionary of <= 32 distinct values (CSR-VI value indexing),
//     each code stored as its dictionary byte offset (index * 8).  Padding
//     entries (rows shorter than their slice) hold the value 0.0 -- the
//     dictionary always contains +0.0 -- and are skipped by the gathers.
//     The dictionary holds the exact bit patterns, so every product is the
//     same double as from the CRS arrays and the row sums stay bitwise equal.
// Layout: [rec int2 x ns] [lens u16 x 32 ns] | align16 | [dict f64 x nd]
//   | align16 | [col16 x E] | align16 | [code u8 x E  or  val f64 x E]
// rec[s] = {first entry of slice s (relative to the tile), w | wmin << 16}.
// Matrix bytes per entry: 3 (dictionary) or 10 (raw) instead of 12.
constexpr int kDictMax = 32;  // codes are stored premultiplied by 8 (dictionary byte offsets)
constexpr int32_t kModeC16 = 1, kModeDict = 2, kModeLong = 4;  // kModeLong: some slice has w > 8
// With x-segments (nseg > 0) the segment table (int4 x nseg, as in the plain
// layout) follows the lens, and the columns are LOCAL indices into the slot's
// x buffer, stored biased by -32768 (decoded as 32768 + int16).
constexpr int32_t kLocalBias = 32768;
__host__ __device__ inline int64_t cblk_dict_off(int32_t ns, int32_t nseg) {
  return align16(int64_t(ns) * 72) + int64_t(nseg) * 16;
}
__host__ __device__ inline int64_t cblk_col_off(int32_t ns, int32_t nd, int32_t nseg) {
  return align16(cblk_dict_off(ns, nseg) + int64_t(nd) * 8);
}
__host__ __device__ inline int64_t cblk_val_off(int32_t ns, int32_t nd, int64_t E, int32_t nseg) {
  return align16(cblk_col_off(ns, nd, nseg) + E * 2);
}
__host__ __device__ inline int64_t cblk_bytes(int32_t ns, int32_t nd, int64_t E, bool dict, int32_t nseg) {
  return (cblk_val_off(ns, nd, E, nseg) + E * (dict ? 1 : 8) + 127) & ~int64_t(127);
}
__device__ __forceinline__ int32_t sx16(int32_t v) { return (v << 16) >> 16; }

// Signed column offsets (col - row) of lane's W entries.
template <int W>
__device__ __forceinline__ void c16_offs(const SmemBlk& B, uint32_t cb, uint32_t lane, int32_t (&c)[W]) {
  constexpr int Q = W >> 2, PR = (W >> 1) & 1, SG = W & 1;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int2 v = B.i2(cb + q * 256 + lane * 8);
    c[4 * q] = sx16(v.x);
    c[4 * q + 1] = v.x >> 16;
    c[4 * q + 2] = sx16(v.y);
    c[4 * q + 3] = v.y >> 16;
  }
  if constexpr (PR) {
    const int32_t v = B.i1(cb + Q * 256 + lane * 4);
    c[4 * Q] = sx16(v);
    c[4 * Q + 1] = v >> 16;
  }
  if constexpr (SG) c[W - 1] = sx16(int32_t(B.u16(cb + Q * 256 + PR * 128 + lane * 2)));
}

// Values of lane's W entries: dictionary codes (VD) or raw f64.
template <int W, bool VD>
__device__ __forceinline__ void c16_vals(const SmemBlk& B, uint32_t vb, uint32_t lane, uint32_t dict,
                                         double (&v)[W]) {
  constexpr int Q = W >> 2, PR = (W >> 1) & 1, SG = W & 1;
  if constexpr (VD) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const uint32_t k = uint32_t(B.i1(vb + q * 128 + lane * 4));
      v[4 * q] = lds_f64(dict + (k & 255u));
      v[4 * q + 1] = lds_f64(dict + ((k >> 8) & 255u));
      v[4 * q + 2] = lds_f64(dict + ((k >> 16) & 255u));
      v[4 * q + 3] = lds_f64(dict + (k >> 24));
    }
    if constexpr (PR) {
      const uint32_t k = B.u16(vb + Q * 128 + lane * 2);
      v[4 * Q] = lds_f64(dict + (k & 255u));
      v[4 * Q + 1] = lds_f64(dict + (k >> 8));
    }
    if constexpr (SG) v[W - 1] = lds_f64(dict + B.u8(vb + Q * 128 + PR * 64 + lane));
  } else {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const double2 a = B.d2(vb + q * 1024 + lane * 32), b = B.d2(vb + q * 1024 + lane * 32 + 16);
      v[4 * q] = a.x, v[4 * q + 1] = a.y, v[4 * q + 2] = b.x, v[4 * q + 3] = b.y;
    }
    if constexpr (PR) {
      const double2 a = B.d2(vb + Q * 1024 + lane * 16);
      v[4 * Q] = a.x, v[4 * Q + 1] = a.y;
    }
    if constexpr (SG) v[W - 1] = B.d1(vb + Q * 1024 + PR * 512 + lane * 8);
  }
}

// Byte offsets of a compressed slice's column / value arrays (entry e_s).
struct CSlice {
  uint32_t cb, vb;
};
template <bool VD>
__device__ __forceinline__ CSlice cslice(uint32_t col_o, uint32_t val_o, uint32_t e_s) {
  return CSlice{col_o + e_s * 2u, val_o + e_s * (VD ? 1u : 8u)};
}

template <bool EXACT, bool FULL, int W>
__device__ __forceinline__ double chain(const double (&v)[W], const double (&x)[W], int len) {
  double t = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    if constexpr (FULL)
      t = madd<EXACT>(t, v[j], x[j]);
    else
      madd_if<EXACT>(t, v[j], x[j], j, len);
  }
  return t;
}

// One compressed slice of width W <= 8 (real vectors).
template <int W, bool EXACT, bool FULL, bool VD, class G, int PROBE = 0>
__device__ __forceinline__ double cslice_real_w(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row,
                                                uint32_t dict, const G& g, int len) {
  int32_t c[W];
  c16_offs<W>(B, a.cb, lane, c);
  double x[W];
  const typename G::Row rp = g.row(row);
#pragma unroll
  for (int j = 0; j < W; ++j) {
    // PROBE (compute probe only): 1 = gathers confined to 8 KB, 2 = coalesced, 3 = none
    if constexpr (PROBE == 1) x[j] = g.d((row + c[j]) & 1023);
    if constexpr (PROBE == 2) x[j] = g.d(int32_t(lane) + 32 * j);
    if constexpr (PROBE == 3) x[j] = __int_as_float(c[j]);
    if constexpr (PROBE == 0) x[j] = (FULL || j < len) ? g.at(rp, c[j]) : 0.0;
  }
  double v[W];
  c16_vals<W, VD>(B, a.vb, lane, dict, v);
  return chain<EXACT, true, W>(v, x, len);
}

// Two compressed slices of the same width W <= 8: all gathers in flight together.
template <int W, bool EXACT, bool FULL, bool VD, class G>
__device__ __forceinline__ double2 cslice_real_w2(const SmemBlk& B, CSlice a0, CSlice a1, uint32_t lane,
                                                  int32_t row0, int32_t row1, uint32_t dict, const G& g,
                                                  int len0, int len1) {
  int32_t c0[W], c1[W];
  c16_offs<W>(B, a0.cb, lane, c0);
  c16_offs<W>(B, a1.cb, lane, c1);
  double x0[W], x1[W];
  const typename G::Row rp0 = g.row(row0), rp1 = g.row(row1);
  // non-full slices: a padding entry gathers nothing (x = 0) and its stored
  // value is 0.0, so its product is +0 and t + 0 == t exactly (t starts at
  // +0.0 and a round-to-nearest sum is never -0.0 unless both terms are)
#pragma unroll
  for (int j = 0; j < W; ++j) x0[j] = (FULL || j < len0) ? g.at(rp0, c0[j]) : 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) x1[j] = (FULL || j < len1) ? g.at(rp1, c1[j]) : 0.0;
  double t0, t1;
  {
    double v[W];
    c16_vals<W, VD>(B, a0.vb, lane, dict, v);
    t0 = chain<EXACT, true, W>(v, x0, len0);
  }
  {
    double v[W];
    c16_vals<W, VD>(B, a1.vb, lane, dict, v);
    t1 = chain<EXACT, true, W>(v, x1, len1);
  }
  return make_double2(t0, t1);
}

// Any width (real or complex vectors), one entry at a time in chunk order.
template <bool CPLX, bool EXACT, bool VD, class G>
__device__ __noinline__ double2 cslice_any(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row, uint32_t dict,
                                           const G& g, int w, int len) {
  double tr = 0.0, ti = 0.0;
  const int Q = w >> 2, PR = (w >> 1) & 1;
  for (int j = 0; j < w; ++j) {
    uint32_t ec;  // entry offset inside the slice (chunk order of chunk_entry)
    if (j < 4 * Q)
      ec = uint32_t(j >> 2) * 128u + lane * 4u + uint32_t(j & 3);
    else if (PR && j < 4 * Q + 2)
      ec = uint32_t(Q) * 128u + lane * 2u + uint32_t(j - 4 * Q);
    else
      ec = uint32_t(Q) * 128u + (PR ? 64u : 0u) + lane;
    const int32_t c = row + sx16(int32_t(B.u16(a.cb + ec * 2u)));
    double v;
    if constexpr (VD)
      v = lds_f64(dict + B.u8(a.vb + ec));
    else
      v = B.d1(a.vb + ec * 8u);
    if constexpr (CPLX) {
      const double2 x = g.d2(c);
      madd_if<EXACT>(tr, v, x.x, j, len);
      madd_if<EXACT>(ti, v, x.y, j, len);
    } else {
      madd_if<EXACT>(tr, v, g.d(c), j, len);
    }
  }
  return make_double2(tr, ti);
}

// One chunk of n (4, 2 or 1) entries of a compressed slice: the lane's
// column offsets, values and gathers (padding entries j >= len gather
// nothing; their stored value is 0.0, so they add +0 exactly).
template <int NQ, bool VD>
__device__ __forceinline__ void c16_quads(const SmemBlk& B, uint32_t cb, uint32_t vb, uint32_t lane, uint32_t dict,
                                          int q0, int32_t (&c)[4 * NQ], double (&v)[4 * NQ]) {
#pragma unroll
  for (int u = 0; u < NQ; ++u) {
    const int2 cc = B.i2(cb + uint32_t(q0 + u) * 256u + lane * 8u);
    c[4 * u] = sx16(cc.x), c[4 * u + 1] = cc.x >> 16, c[4 * u + 2] = sx16(cc.y), c[4 * u + 3] = cc.y >> 16;
    if constexpr (VD) {
      const uint32_t k = uint32_t(B.i1(vb + uint32_t(q0 + u) * 128u + lane * 4u));
      v[4 * u] = lds_f64(dict + (k & 255u));
      v[4 * u + 1] = lds_f64(dict + ((k >> 8) & 255u));
      v[4 * u + 2] = lds_f64(dict + ((k >> 16) & 255u));
      v[4 * u + 3] = lds_f64(dict + (k >> 24));
    } else {
      const double2 a0 = B.d2(vb + uint32_t(q0 + u) * 1024u + lane * 32u);
      const double2 a1 = B.d2(vb + uint32_t(q0 + u) * 1024u + lane * 32u + 16u);
      v[4 * u] = a0.x, v[4 * u + 1] = a0.y, v[4 * u + 2] = a1.x, v[4 * u + 3] = a1.y;
    }
  }
}

// Long rows (w > 8, real vectors): quads two at a time (8 gathers in flight),
// then the pair / single tail; storage order throughout.
template <bool EXACT, bool VD, class G>
__device__ __forceinline__ double cslice_real_long(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row, uint32_t dict,
                                                const G& g, int w, int len) {
  const int Q = w >> 2, PR = (w >> 1) & 1;
  const typename G::Row rp = g.row(row);
  double t = 0.0;
  int q = 0;
  for (; q + 2 <= Q; q += 2) {
    int32_t c[8];
    double v[8], x[8];
    c16_quads<2, VD>(B, a.cb, a.vb, lane, dict, q, c, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = (4 * q + j < len) ? g.at(rp, c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) t = madd<EXACT>(t, v[j], x[j]);
  }
  if (q < Q) {
    int32_t c[4];
    double v[4], x[4];
    c16_quads<1, VD>(B, a.cb, a.vb, lane, dict, q, c, v);
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = (4 * q + j < len) ? g.at(rp, c[j]) : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) t = madd<EXACT>(t, v[j], x[j]);
  }
  const int j0 = 4 * Q;
  if (PR) {
    const int32_t cc = B.i1(a.cb + uint32_t(Q) * 256u + lane * 4u);
    double v0, v1;
    if constexpr (VD) {
      const uint32_t k = B.u16(a.vb + uint32_t(Q) * 128u + lane * 2u);
      v0 = lds_f64(dict + (k & 255u));
      v1 = lds_f64(dict + (k >> 8));
    } else {
      const double2 vv = B.d2(a.vb + uint32_t(Q) * 1024u + lane * 16u);
      v0 = vv.x, v1 = vv.y;
    }
    const double x0 = j0 < len ? g.at(rp, sx16(cc)) : 0.0;
    const double x1 = j0 + 1 < len ? g.at(rp, cc >> 16) : 0.0;
    t = madd<EXACT>(t, v0, x0);
    t = madd<EXACT>(t, v1, x1);
  }
  if (w & 1) {
    const int32_t cc = sx16(int32_t(B.u16(a.cb + uint32_t(Q) * 256u + uint32_t(PR) * 128u + lane * 2u)));
    double v0;
    if constexpr (VD)
      v0 = lds_f64(dict + B.u8(a.vb + uint32_t(Q) * 128u + uint32_t(PR) * 64u + lane));
    else
      v0 = B.d1(a.vb + uint32_t(Q) * 1024u + uint32_t(PR) * 512u + lane * 8u);
    const double x0 = w - 1 < len ? g.at(rp, cc) : 0.0;
    t = madd<EXACT>(t, v0, x0);
  }
  return t;
}

// Complex vectors, width W <= 8: all W complex gathers in flight at once.
template <int W, bool EXACT, bool VD, class G>
__device__ __forceinline__ double2 cslice_cplx_w(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row, uint32_t dict,
                                                 const G& g, int len) {
  int32_t c[W];
  c16_offs<W>(B, a.cb, lane, c);
  double2 x[W];
#pragma unroll
  for (int j = 0; j < W; ++j) x[j] = j < len ? g.d2(row + c[j]) : make_double2(0.0, 0.0);
  double v[W];
  c16_vals<W, VD>(B, a.vb, lane, dict, v);
  double tr = 0.0, ti = 0.0;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    tr = madd<EXACT>(tr, v[j], x[j].x);
    ti = madd<EXACT>(ti, v[j], x[j].y);
  }
  return make_double2(tr, ti);
}

// Complex vectors (real matrix), any width: a quad at a time (4 complex
// gathers in flight); storage order, re and im chains as the plain path.
template <bool EXACT, bool VD, class G>
__device__ __forceinline__ double2 cslice_cplx(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row, uint32_t dict,
                                            const G& g, int w, int len) {
  const int Q = w >> 2, PR = (w >> 1) & 1;
  double tr = 0.0, ti = 0.0;
  for (int q = 0; q < Q; ++q) {
    int32_t c[4];
    double v[4];
    c16_quads<1, VD>(B, a.cb, a.vb, lane, dict, q, c, v);
    double2 x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = (4 * q + j < len) ? g.d2(row + c[j]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      tr = madd<EXACT>(tr, v[j], x[j].x);
      ti = madd<EXACT>(ti, v[j], x[j].y);
    }
  }
  const int j0 = 4 * Q;
  for (int j = j0; j < w; ++j) {
    uint32_t ec;
    if (PR && j < j0 + 2)
      ec = uint32_t(Q) * 128u + lane * 2u + uint32_t(j - j0);
    else
      ec = uint32_t(Q) * 128u + (PR ? 64u : 0u) + lane;
    const int32_t c = row + sx16(int32_t(B.u16(a.cb + ec * 2u)));
    double v;
    if constexpr (VD)
      v = lds_f64(dict + B.u8(a.vb + ec));
    else
      v = B.d1(a.vb + ec * 8u);
    const double2 x = j < len ? g.d2(c) : make_double2(0.0, 0.0);
    tr = madd<EXACT>(tr, v, x.x);
    ti = madd<EXACT>(ti, v, x.y);
  }
  return make_double2(tr, ti);
}

template <bool EXACT, bool FULL, bool VD, bool LONG, class G>
__device__ __forceinline__ double cslice_real(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row,
                                              uint32_t dict, const G& g, int w, int len) {
  switch (w) {
    case 1: return cslice_real_w<1, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 2: return cslice_real_w<2, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 3: return cslice_real_w<3, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 4: return cslice_real_w<4, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 5: return cslice_real_w<5, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 6: return cslice_real_w<6, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 7: return cslice_real_w<7, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 8: return cslice_real_w<8, EXACT, FULL, VD>(B, a, lane, row, dict, g, len);
    case 0: return 0.0;
    default:
      // tiles without slices wider than 8 (tile_mode kModeLong clear) never get
      // here, and their kernel body carries no long-row code
      if constexpr (LONG)
        return cslice_real_long<EXACT, VD>(B, a, lane, row, dict, g, w, FULL ? w : len);
      else
        return 0.0;
  }
}

template <bool EXACT, bool FULL, bool VD, class G>
__device__ __forceinline__ double2 cslice_real_pair(const SmemBlk& B, CSlice a0, CSlice a1, uint32_t lane,
                                                    int32_t row0, int32_t row1, uint32_t dict, const G& g, int w,
                                                    int len0, int len1) {
  switch (w) {
    case 1: return cslice_real_w2<1, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    case 2: return cslice_real_w2<2, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    case 3: return cslice_real_w2<3, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    case 4: return cslice_real_w2<4, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    case 5: return cslice_real_w2<5, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    case 6: return cslice_real_w2<6, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    case 7: return cslice_real_w2<7, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
    default: return cslice_real_w2<8, EXACT, FULL, VD>(B, a0, a1, lane, row0, row1, dict, g, len0, len1);
  }
}

// One power step of one COMPRESSED tile (see tile_power for the contract).
// LOCAL: the columns index the slot's staged x buffer (G = GatherSmem).
// LONG: the tile has slices wider than 8 (long-row path compiled in).
template <bool CPLX, bool EXACT, bool GENERAL, bool VD, bool LOCAL = false, bool LONG = false, bool DYN = false,
          class G>
__device__ __forceinline__ void tile_power_c(const PowTab& pt, double* acc_base, bool use_acc, const SmemBlk& B,
                                             const G& g, int32_t r0, int32_t nrows, uint32_t E, int32_t nd,
                                             int32_t nseg, int wid, int nwarps, uint32_t sched = kSchedStatic) {
  const int32_t ns = (nrows + 31) >> 5;
  const uint32_t lens_o = uint32_t(ns) * 8;
  const uint32_t dict = B.a + uint32_t(cblk_dict_off(ns, nseg));
  const uint32_t col_o = uint32_t(cblk_col_off(ns, nd, nseg));
  const uint32_t val_o = uint32_t(cblk_val_off(ns, nd, E, nseg));
  const int32_t rb = LOCAL ? kLocalBias : r0 + int32_t(threadIdx.x & 31);  // decode base of lane's columns
  const uint32_t lane = threadIdx.x & 31;
  constexpr int cw = CPLX ? 2 : 1;
  double* yout = pt.yout + int64_t(r0) * cw;
  const double* ypv = pt.ypv + int64_t(r0) * cw;
  double* acc = acc_base + int64_t(r0) * cw;
  auto len_of = [&](int32_t s, int2 rec) -> int {
    const int w = rec.y & 0xffff;
    return int(uint32_t(rec.y) >> 16) == w ? w : int(B.u16(lens_o + uint32_t(s) * 64 + lane * 2));
  };
  if constexpr (!CPLX) {
    // lane-offset pointers: slice s of this lane is element s * 32
    double* yl = yout + lane;
    const double* pl = ypv + lane;
    double* al = acc + lane;
    auto epilogue = [&](int32_t s, double t) {
      if (s * 32 + int32_t(lane) < nrows) {
        const int32_t o = s * 32;
        if constexpr (GENERAL) {
          if (pt.cheb) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(pl + o));
          stg_f64(yl + o, t);
          if (use_acc) stg_f64(al + o, madd<EXACT>(ld_cg(al + o), pt.cre, t));
        } else {
          stg_f64(yl + o, t);
        }
      }
    };
    auto single = [&](int32_t s, int2 rec) -> double {
      const CSlice a = cslice<VD>(col_o, val_o, uint32_t(rec.x));
      const int w = rec.y & 0xffff;
      const int32_t row = LOCAL ? rb : rb + s * 32;
      if (int(uint32_t(rec.y) >> 16) == w) return cslice_real<EXACT, true, VD, LONG>(B, a, lane, row, dict, g, w, w);
      return cslice_real<EXACT, false, VD, LONG>(B, a, lane, row, dict, g, w, len_of(s, rec));
    };
    // slices s and s2 (dynamic grabs: s + 1; static: s + nwarps): a
    // same-width pair keeps both slices' gathers in flight.  One loop so the
    // body is inlined once (two call sites made ptxas outline it to a stack frame).
    const bool dyn = DYN || sched != kSchedStatic;  // DYN: the caller always provides a counter
    for (int32_t s = dyn ? sched_grab(sched, 2) : wid; s < ns; s = dyn ? sched_grab(sched, 2) : s + 2 * nwarps) {
      const int32_t s2 = dyn ? s + 1 : s + nwarps;
      const int2 rec0 = B.i2(uint32_t(s) * 8);
      if (s2 >= ns) {
        epilogue(s, single(s, rec0));
        break;
      }
      const int2 rec1 = B.i2(uint32_t(s2) * 8);
      const int w0 = rec0.y & 0xffff, w1 = rec1.y & 0xffff;
      if (w0 == w1 && uint32_t(w0 - 1) < 8u) {
        const bool full = (uint32_t(rec0.y) >> 16) == uint32_t(w0) && (uint32_t(rec1.y) >> 16) == uint32_t(w1);
        const CSlice a0 = cslice<VD>(col_o, val_o, uint32_t(rec0.x)), a1 = cslice<VD>(col_o, val_o, uint32_t(rec1.x));
        const int32_t row0 = LOCAL ? rb : rb + s * 32, row1 = LOCAL ? rb : rb + s2 * 32;
        double2 t;
        if (full)
          t = cslice_real_pair<EXACT, true, VD>(B, a0, a1, lane, row0, row1, dict, g, w0, w0, w0);
        else
          t = cslice_real_pair<EXACT, false, VD>(B, a0, a1, lane, row0, row1, dict, g, w0, len_of(s, rec0),
                                                 len_of(s2, rec1));
        epilogue(s, t.x);
        epilogue(s2, t.y);
      } else {
        epilogue(s, single(s, rec0));
        epilogue(s2, single(s2, rec1));
      }
    }
  } else {
    for (int32_t s = sched_grab(sched, 1); s < ns; s = sched_grab(sched, 1)) {
      const int2 rec = B.i2(uint32_t(s) * 8);
      const CSlice a = cslice<VD>(col_o, val_o, uint32_t(rec.x));
      const int w = rec.y & 0xffff;
      const int32_t lr = s * 32 + int32_t(lane);
      const int32_t crow = LOCAL ? rb : r0 + lr;
      const int clen = len_of(s, rec);
      double2 t;
      switch (w) {  // W <= 8: every complex gather of the row in flight at once
        case 1: t = cslice_cplx_w<1, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 2: t = cslice_cplx_w<2, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 3: t = cslice_cplx_w<3, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 4: t = cslice_cplx_w<4, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 5: t = cslice_cplx_w<5, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 6: t = cslice_cplx_w<6, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 7: t = cslice_cplx_w<7, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        case 8: t = cslice_cplx_w<8, EXACT, VD>(B, a, lane, crow, dict, g, clen); break;
        default: t = cslice_cplx<EXACT, VD>(B, a, lane, crow, dict, g, w, clen);
      }
      if (lr < nrows) {
        const int64_t r2 = 2 * int64_t(lr);
        if constexpr (GENERAL) {
          if (pt.cheb) {
            t.x = __dsub_rn(__dmul_rn(2.0, t.x), ld_cg(ypv + r2));
            t.y = __dsub_rn(__dmul_rn(2.0, t.y), ld_cg(ypv + r2 + 1));
          }
        }
        stg_f64x2(yout + r2, t);
        if constexpr (GENERAL) {
          if (use_acc) {
            const double ar = ld_cg(acc + r2), ai = ld_cg(acc + r2 + 1);
            const double pr = __dsub_rn(__dmul_rn(pt.cre, t.x), __dmul_rn(pt.cim, t.y));
            const double pim = __dadd_rn(__dmul_rn(pt.cre, t.y), __dmul_rn(pt.cim, t.x));
            stg_f64x2(acc + r2, make_double2(__dadd_rn(ar, pr), __dadd_rn(ai, pim)));
          }
        }
      }
    }
  }
}

// Dispatch one compressed tile on its format bits (tile_mode): GENERAL
// (Chebyshev / accumulation), dictionary or raw values, long rows.  Tiles
// with slices wider than 8 run in a separate non-inlined body (tile_c_long):
// inlining the long-row code into the walk kernels cost the W <= 8 path its
// register allocation (cfg2 0.50 -> 0.58 ms).
#define LMPK_TPC(GEN, VDV, LG) \
  tile_power_c<CPLX, EXACT, GEN, VDV, LOCAL, LG>(pt, acc, use_acc, B, g, r0, rows, E, nd, nseg, warp, nw, sch)
template <bool CPLX, bool EXACT, bool LOCAL, class G>
__device__ __noinline__ void tile_c_long(int32_t tmode, const PowTab& pt, double* acc, bool use_acc, const SmemBlk B,
                                         const G g, int32_t r0, int32_t rows, uint32_t E, int32_t nseg, int warp,
                                         int nw, uint32_t sch) {
  const int32_t nd = tmode >> 8;
  const bool vd = (tmode & kModeDict) != 0;
  if (pt.general) {
    if (vd) LMPK_TPC(true, true, true); else LMPK_TPC(true, false, true);
  } else {
    if (vd) LMPK_TPC(false, true, true); else LMPK_TPC(false, false, true);
  }
}
template <bool CPLX, bool EXACT, bool LOCAL, class G, bool HASLONG = true>
__device__ __forceinline__ void tile_c_dispatch(int32_t tmode, const PowTab& pt, double* acc, bool use_acc,
                                                const SmemBlk& B, const G& g, int32_t r0, int32_t rows, uint32_t E,
                                                int32_t nseg, int warp, int nw, uint32_t sch) {
  if constexpr (!CPLX && HASLONG) {
    if (tmode & kModeLong) {
      tile_c_long<CPLX, EXACT, LOCAL>(tmode, pt, acc, use_acc, B, g, r0, rows, E, nseg, warp, nw, sch);
      return;
    }
  }
  const int32_t nd = tmode >> 8;
  const bool vd = (tmode & kModeDict) != 0;
  if (pt.general) {
    if (vd) LMPK_TPC(true, true, false); else LMPK_TPC(true, false, false);
  } else {
    if (vd) LMPK_TPC(false, true, false); else LMPK_TPC(false, false, false);
  }
}
#undef LMPK_TPC

// One power step of one tile (rows r0 .. r0+nrows-1, E block entries): warps
// stride over the 32-row slices, lane = row.  GENERAL adds the Chebyshev
// three-term step and the accumulation; plain SpMV powers skip both.
template <bool CPLX, bool EXACT, bool GENERAL, class Blk, class G, bool LONG = true>
__device__ __forceinline__ void tile_power(const PowTab& pt, double* acc_base, bool use_acc, const Blk& B,
                                           const G& g, int32_t r0, int32_t nrows, uint32_t E, int32_t nseg,
                                           int wid, int nwarps, bool pairs = true, uint32_t sched = kSchedStatic) {
  const int32_t ns = (nrows + 31) >> 5;
  const uint32_t lens_o = uint32_t(ns) * 8;
  const uint32_t col_o = uint32_t(blk_col_off(ns, nseg));
  const uint32_t vdelta = col_o + E * 4 - 2 * col_o;  // vb = 2*cb + vdelta
  const int lane = threadIdx.x & 31;
  const uint32_t l4 = uint32_t(lane) * 4;
  constexpr int cw = CPLX ? 2 : 1;
  double* yout = pt.yout + int64_t(r0) * cw;
  const double* ypv = pt.ypv + int64_t(r0) * cw;
  double* acc = acc_base + int64_t(r0) * cw;
  if constexpr (!CPLX) {
    auto epilogue = [&](int32_t s, double t) {
      const int32_t lr = s * 32 + lane;
      if (lr < nrows) {
        if constexpr (GENERAL) {
          if (pt.cheb) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(ypv + lr));
          stg_y(yout + lr, t, pt.ypol);
          if (use_acc) stg_f64(acc + lr, madd<EXACT>(ld_cg(acc + lr), pt.cre, t));
        } else {
          stg_y(yout + lr, t, pt.ypol);
        }
      }
    };
    auto single = [&](int32_t s, int2 rec) -> double {
      const uint32_t cb = uint32_t(rec.x), vb = 2 * cb + vdelta;
      const int w = rec.y & 0xffff;
      if (int(uint32_t(rec.y) >> 16) == w) return slice_real<EXACT, true, Blk, G, LONG>(B, cb, vb, l4, g, w, w);
      const int len = int(B.u16(lens_o + uint32_t(s) * 64 + (l4 >> 1)));
      return slice_real<EXACT, false, Blk, G, LONG>(B, cb, vb, l4, g, w, len);
    };
    // warp `wid` owns slices wid, wid + nwarps, ...; it takes them two at a time
    for (int32_t s = sched_first(sched, wid, 2); s < ns; s = sched_next(sched, s, 2 * nwarps, 2)) {
      const int32_t s2 = sched != kSchedStatic ? s + 1 : s + nwarps;
      const int2 rec0 = B.i2(uint32_t(s) * 8);
      if (s2 >= ns) {
        epilogue(s, single(s, rec0));
        break;
      }
      const int2 rec1 = B.i2(uint32_t(s2) * 8);
      const int w0 = rec0.y & 0xffff, w1 = rec1.y & 0xffff;
      if (pairs && w0 == w1 && w0 >= 1 && w0 <= 8) {
        const bool full0 = int(uint32_t(rec0.y) >> 16) == w0, full1 = int(uint32_t(rec1.y) >> 16) == w1;
        const uint32_t cb0 = uint32_t(rec0.x), cb1 = uint32_t(rec1.x);
        double2 t;
        if (full0 && full1) {
          t = slice_real_pair<EXACT, true>(B, cb0, 2 * cb0 + vdelta, cb1, 2 * cb1 + vdelta, l4, g, w0, w0, w0);
        } else {
          const int len0 = full0 ? w0 : int(B.u16(lens_o + uint32_t(s) * 64 + (l4 >> 1)));
          const int len1 = full1 ? w1 : int(B.u16(lens_o + uint32_t(s2) * 64 + (l4 >> 1)));
          t = slice_real_pair<EXACT, false>(B, cb0, 2 * cb0 + vdelta, cb1, 2 * cb1 + vdelta, l4, g, w0, len0,
                                            len1);
        }
        epilogue(s, t.x);
        epilogue(s2, t.y);
      } else {
        epilogue(s, single(s, rec0));
        epilogue(s2, single(s2, rec1));
      }
    }
  } else {
  for (int32_t s = sched_first(sched, wid, 1); s < ns; s = sched_next(sched, s, nwarps, 1)) {
    const int2 rec = B.i2(uint32_t(s) * 8);
    const uint32_t cb = uint32_t(rec.x);
    const uint32_t vb = 2 * cb + vdelta;
    const int w = rec.y & 0xffff;
    const bool full = int(uint32_t(rec.y) >> 16) == w;
    const int32_t lr = s * 32 + lane;
    {
      const int len = full ? w : int(B.u16(lens_o + uint32_t(s) * 64 + (l4 >> 1)));
      double2 t = slice_cplx<EXACT>(B, cb, vb, l4, g, w, len);
      if (lr < nrows) {
        const int64_t r2 = 2 * int64_t(lr);
        if constexpr (GENERAL) {
          if (pt.cheb) {
            t.x = __dsub_rn(__dmul_rn(2.0, t.x), ld_cg(ypv + r2));
            t.y = __dsub_rn(__dmul_rn(2.0, t.y), ld_cg(ypv + r2 + 1));
          }
        }
        stg_f64x2(yout + r2, t);
        if constexpr (GENERAL) {
          if (use_acc) {
            // acc += (cre + i cim) * t with the products spelled out
            const double ar = ld_cg(acc + r2), ai = ld_cg(acc + r2 + 1);
            const double pr = __dsub_rn(__dmul_rn(pt.cre, t.x), __dmul_rn(pt.cim, t.y));
            const double pim = __dadd_rn(__dmul_rn(pt.cre, t.y), __dmul_rn(pt.cim, t.x));
            stg_f64x2(acc + r2, make_double2(__dadd_rn(ar, pr), __dadd_rn(ai, pim)));
          }
        }
      }
    }
  }
  }
}

// Fill the per-power table (all threads of the CTA, then __syncthreads).
__device__ __forceinline__ void build_powtab(PowTab* tab, const MpkParams& P, const PowerCfgDev& C) {
  for (int i = threadIdx.x; i < P.n_powers; i += blockDim.x) {
    PowTab e;
    e.yin = reinterpret_cast<const char*>(P.y + int64_t(C.in_slot[i]) * P.ldy);
    e.yout = P.y + int64_t(C.out_slot[i]) * P.ldy;
    e.ypv = P.y + int64_t(C.prev_slot[i]) * P.ldy;
    e.cre = C.coef_re[i];
    e.cim = C.coef_im[i];
    e.cheb = C.kernel[i] == LMPK_KERNEL_CHEB;
    e.general = e.cheb || P.use_acc;
    e.ypol = P.ypol == 1 ? policy_evict_last() : (P.ypol == 2 ? policy_evict_first() : 0ull);
    tab[i] = e;
  }
}

// ---------------------------------------------------------------- group walk kernel
// See the file header.  Warps 0..NC-1 are consumers; warp NC + r is the
// producer of slot r (r < R).  Each producer runs its slot's state machine on
// its own -- stage the block (TMA), wait for the dependencies of each power,
// push (slot, power) into the shared work ring, wait until the consumers
// freed the slot -- so a slow L2 round trip of one slot never delays another.
// Shared state per slot r: h_t (tile), h_last (last power of the held item),
// h_glb (block read from global memory), h_r0/h_rows/h_E (tile geometry),
// free_bar (completed by the consumer that finished the item's last power).

// mbarrier wait of a whole warp with the launch's abort flag / watchdog:
// lane 0 waits, the verdict is broadcast (warp-uniform), __syncwarp orders
// the other lanes' later shared-memory reads after the completed phase.
__device__ __forceinline__ bool mbar_wait_bounded(uint64_t* bar, uint32_t parity, const MpkParams& P) {
  int ok = 1;
  if ((threadIdx.x & 31) == 0) {
    unsigned long long t0 = 0;
    for (int spins = 0; !mbar_try_wait(bar, parity); ++spins) {
      if ((spins & 255) == 255) {
        const unsigned long long now = globaltimer();
        if (t0 == 0) t0 = now;
        const volatile unsigned long long* ab = P.queue + 1;
        if (*ab != 0ull) {
          ok = 0;
          break;
        }
        if (now - t0 > kWatchdogNs) {
          atomicExch(P.queue + 1, 1ull);
          *P.err = 2;
          ok = 0;
          break;
        }
      }
    }
  }
  ok = __shfl_sync(0xffffffffu, ok, 0);
  __syncwarp();
  return ok != 0;
}

// Experiment switches of the dependency wait (LMPK_ACQ, mpk.cu): acquire
// loads instead of relaxed loads + fence; no fence at all (measurement only:
// not a valid acquire pattern).
constexpr int kFlagNoAcqFence = 0x100000, kFlagAcqLoads = 0x200000;

// Spin until progress[lo..hi] >= target (one warp, all loads in flight per
// round); then one acquire fence (also invalidates L1 for the gathers).
// Returns false if the launch is aborting (abort flag or watchdog).
__device__ __forceinline__ bool spin_deps(const MpkParams& P, int32_t lo, int32_t hi, uint32_t target,
                                          unsigned long long* rounds) {
  const int lane = threadIdx.x & 31;
  unsigned long long t0 = 0;
  for (int spins = 0;; ++spins) {
    uint32_t m = 0xffffffffu;
    if (P.flags & kFlagAcqLoads) {
      for (int32_t i = lo + lane; i <= hi; i += 32) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.progress + i) : "memory");
        m = min(m, v);
      }
    } else {
      for (int32_t i = lo + lane; i <= hi; i += 32) m = min(m, ld_relaxed_u32(P.progress + i));
    }
    ++*rounds;
    if (__all_sync(0xffffffffu, m >= target)) {
      if (!(P.flags & (kFlagAcqLoads | kFlagNoAcqFence))) fence_acq_rel_gpu();
      return true;
    }
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

// x-segments of a slot whose vectors are not 16-byte aligned (no bulk copy):
// all consumer warps copy the runs with plain loads, then one named barrier.
template <bool CPLX, int NC>
__device__ __forceinline__ void copy_x_segments(const SmemBlk& B, const PowTab& pt, int32_t rows, int32_t nseg,
                                                uint32_t xb, int warp, int lane) {
  const int tid = warp * 32 + lane;
  const uint32_t seg_o = uint32_t(blk_seg_off((rows + 31) >> 5));
  const int cw = CPLX ? 2 : 1;
  const double* yin = reinterpret_cast<const double*>(pt.yin);
  for (int j = 0; j < nseg; ++j) {
    const int4 sg = B.i4(seg_o + uint32_t(j) * 16);
    for (int e = tid; e < sg.y * cw; e += NC * 32) {
      const double v = ld_cg(yin + int64_t(sg.x) * cw + e);
      asm volatile("st.shared.f64 [%0], %1;" ::"r"(xb + uint32_t(sg.z * cw + e) * 8u), "d"(v));
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
}

template <bool CPLX, bool EXACT, int NC>
__global__ void __launch_bounds__(32 * (NC + kMaxSlots), 1) mpk_group_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t tile_bar[kMaxSlots], free_bar[kMaxSlots], x_bar[kMaxSlots];
  __shared__ uint64_t full_bar[kWorkRing], empty_bar[kWorkRing];
  __shared__ int32_t w_slot[kWorkRing], w_p[kWorkRing];
  __shared__ uint32_t w_done[kWorkRing], w_ctr[kWorkRing];
  __shared__ uint32_t ring_ctr, prod_done, trace_ctr;
  __shared__ int32_t h_t[kMaxSlots], h_last[kMaxSlots], h_glb[kMaxSlots];
  __shared__ int32_t h_r0[kMaxSlots], h_rows[kMaxSlots], h_E[kMaxSlots], h_nseg[kMaxSlots], h_mode[kMaxSlots];
  __shared__ int32_t h_xoff[kMaxSlots];  // x buffer offset in the slot = the block's (128-aligned) size
  __shared__ int64_t h_ofs[kMaxSlots];
  __shared__ PowTab s_pow[LMPK_MAX_POWERS];
  const int R = P.n_slots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  build_powtab(s_pow, P, C);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kMaxSlots; ++i) {
      mbar_init(&tile_bar[i], 1);
      mbar_init(&free_bar[i], 1);
      mbar_init(&x_bar[i], 1);
    }
    for (int i = 0; i < kWorkRing; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], NC);
      w_done[i] = 0;
      w_ctr[i] = 0;
    }
    ring_ctr = 0;
    prod_done = 0;
    trace_ctr = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (warp >= NC) {
    // ------------------------------------------------ producer of slot r
    const int r = warp - NC;
    if (r >= R) return;
    const int pol_mode = (P.flags >> 8) & 3;
    const uint64_t pol_keep = pol_mode == 0 ? policy_evict_last()
                                            : (pol_mode == 1 ? policy_evict_normal() : policy_evict_first());
    const uint64_t pol_drop = policy_evict_first();
    const bool no_tma = (P.flags & LMPK_FLAG_NO_TMA) != 0;
    // q > 1: a grabbed item must be held at once (the deadlock-freedom window
    // counts grabbed items as held), so a ticket is taken only for a free
    // slot.  q == 1 items only wait for older items: prefetch one ahead.
    const bool prefetch = P.q == 1;
    unsigned long long p_rounds = 0, p_items = 0, p_tma = 0, p_dep = 0, p_free = 0, p_x = 0;
    const unsigned long long p_t0 = P.prof ? globaltimer() : 0;
    struct Next {
      int32_t t, first, last, r0, rows, E, lo, hi, nseg, xent, mode;
      int64_t ofs, bytes;
      bool valid;
    } nx;
    // Ready-queue walk: take a ready (t, p) if the queue has one, else start
    // the next power-1 tile; every enqueued item's dependencies are complete.
    auto fetch_ready = [&]() -> int32_t {  // item code, -1 exhausted, -2 abort
      int32_t code = -1;
      if (lane == 0) {
        const uint32_t total_q = uint32_t(P.n_tiles) * uint32_t(P.n_powers - 1);
        unsigned long long t0 = 0;
        // head / tail / next power-1 tile live on separate 128-byte lines
        uint32_t* q_head = P.rctrl;
        uint32_t* q_tail = P.rctrl + 32;
        uint32_t* q_p1 = P.rctrl + 64;
        for (int spins = 0;; ++spins) {
          const uint32_t h = ld_relaxed_u32(q_head), tl = ld_relaxed_u32(q_tail);
          if (h < tl) {
            // fetch-and-add dequeue: no CAS herd.  An index past the current
            // tail is a reservation of a future item; every index below
            // total_q is eventually enqueued, so waiting for it cannot
            // deadlock (this slot holds no work while it waits).
            const uint32_t idx = atomicAdd(q_head, 1u);
            if (idx >= total_q) break;  // all queue items are taken
            int32_t c;
            const unsigned long long tw = P.prof ? globaltimer() : 0;
            for (int w = 0; (c = ld_acquire_s32(P.rqueue + idx)) < 0; ++w) {
              if (w > 8) __nanosleep(64);
              if ((w & 1023) == 1023) {
                const unsigned long long now = globaltimer();
                if (t0 == 0) t0 = now;
                const volatile unsigned long long* ab = P.queue + 1;
                if (*ab != 0ull || now - t0 > kWatchdogNs) {
                  if (*ab == 0ull) {
                    atomicExch(P.queue + 1, 1ull);
                    *P.err = 3;
                  }
                  c = -2;
                  break;
                }
              }
            }
            if (P.prof) atomicAdd(P.prof + 10, globaltimer() - tw);
            code = c;
            if (P.prof && c >= 0) atomicAdd(P.prof + 14, 1ull);
            break;
          }
          // a new power-1 tile only within `lead` tiles of the completed
          // work (completed items / powers): keeps the walk's L2 window tight
          const uint32_t p1 = ld_relaxed_u32(q_p1);
          if (p1 < uint32_t(P.n_tiles) &&
              p1 < ld_relaxed_u32(P.rctrl + 96) / uint32_t(P.n_powers) + uint32_t(P.lead)) {
            const uint32_t i = atomicAdd(q_p1, 1u);
            if (i < uint32_t(P.n_tiles)) {
              code = int32_t(i << 8) | 1;
              if (P.prof) atomicAdd(P.prof + 15, 1ull);
              break;
            }
            continue;
          }
          if (h >= total_q) break;  // every item handed out
          if (P.prof) atomicAdd(P.prof + 13, 1ull);
          if (spins > 4) __nanosleep(64);
          if ((spins & 63) == 63) {
            const unsigned long long now = globaltimer();
            if (t0 == 0) t0 = now;
            const volatile unsigned long long* ab = P.queue + 1;
            if (*ab != 0ull) {
              code = -2;
              break;
            }
            if (now - t0 > kWatchdogNs) {
              atomicExch(P.queue + 1, 1ull);
              *P.err = 3;
              code = -2;
              break;
            }
          }
        }
        if (code >= 0 && (code & 255) > 1) fence_acq_rel_gpu();  // acquire the deps; invalidate L1
      }
      return __shfl_sync(0xffffffffu, code, 0);
    };
    auto fetch_next = [&]() {
      while (true) {
        int32_t i = 0;
        if (P.mode == 4) {
          const unsigned long long tf0 = P.prof ? globaltimer() : 0;
          const int32_t code = fetch_ready();
          if (P.prof && lane == 0) atomicAdd(P.prof + 0, globaltimer() - tf0);
          if (code < 0) {
            nx.valid = false;
            return;
          }
          const int32_t t = code >> 8;
          nx.t = t;
          nx.first = nx.last = code & 255;
          nx.ofs = __ldg(P.tile_ofs + t);
          nx.bytes = __ldg(P.tile_ofs + t + 1) - nx.ofs;
          nx.r0 = __ldg(P.tile_row + t);
          nx.rows = __ldg(P.tile_row + t + 1) - nx.r0;
          nx.E = __ldg(P.tile_E + t);
          nx.lo = nx.hi = t;
          nx.nseg = P.xmode ? __ldg(P.tile_nseg + t) : 0;
          nx.xent = nx.nseg ? __ldg(P.tile_xent + t) : 0;
          nx.mode = P.tile_mode ? __ldg(P.tile_mode + t) : 0;
          nx.valid = true;
          return;
        }
        if (lane == 0) i = int32_t(atomicAdd(P.queue, 1ull) - P.queue_base);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= P.n_items || i < 0) {
          nx.valid = false;
          return;
        }
        int32_t t = i, g = 0;
        if (P.items) {
          const int32_t code = __ldg(P.items + i);
          t = code >> 8;
          g = code & 255;
        }
        const int first = g * P.q + 1;
        if (first > P.n_powers) continue;  // fewer powers than planned
        nx.t = t;
        nx.first = first;
        nx.last = min(first + P.q - 1, P.n_powers);
        nx.ofs = __ldg(P.tile_ofs + t);
        nx.bytes = __ldg(P.tile_ofs + t + 1) - nx.ofs;
        nx.r0 = __ldg(P.tile_row + t);
        nx.rows = __ldg(P.tile_row + t + 1) - nx.r0;
        nx.E = __ldg(P.tile_E + t);
        nx.lo = __ldg(P.dep_lo + t);
        nx.hi = __ldg(P.dep_hi + t);
        nx.nseg = P.xmode ? __ldg(P.tile_nseg + t) : 0;
        nx.xent = nx.nseg ? __ldg(P.tile_xent + t) : 0;
        nx.mode = P.tile_mode ? __ldg(P.tile_mode + t) : 0;
        nx.valid = true;
        return;
      }
    };
    // Stage the x-segments of the gathered vector y_{p-1} into the slot's x
    // buffer (one bulk copy per segment, completion on x_bar[r]).  The
    // preceding acquire made the producers' stores visible to this thread;
    // the proxy fence orders them before the async-proxy reads.
    uint32_t xph = 0;
    const uint32_t slot_base = smem_u32(smem_raw) + uint32_t(r) * uint32_t(P.smem_cap);
    auto stage_x = [&](const char* yin, int32_t ns, int32_t nseg, int32_t xent, int32_t xoff) -> bool {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (lane == 0) mbar_arrive_expect_tx(&x_bar[r], uint32_t(xent) * 8u);
      __syncwarp();
      const uint32_t seg_o = slot_base + uint32_t(blk_seg_off(ns));
      const uint32_t xb = slot_base + uint32_t(xoff);
      for (int j = lane; j < nseg; j += 32) {
        const int4 sg = SmemBlk{seg_o}.i4(uint32_t(j) * 16);
        // even entry count: 16-byte granules (the extra entry is inside the
        // slot -- bulk copies run only for even ldy)
        bulk_g2s_a(xb + uint32_t(sg.z) * 8u, yin + int64_t(sg.x) * 8, uint32_t((sg.y + 1) & ~1) * 8u, &x_bar[r],
                   policy_evict_normal());
      }
      const bool ok = mbar_wait_bounded(&x_bar[r], xph & 1, P);
      ++xph;
      return ok;
    };
    auto push = [&](int p) {
      const unsigned long long tq0 = P.prof ? globaltimer() : 0;
      if (lane == 0) {
        const uint32_t k = atomicAdd(&ring_ctr, 1u);
        const int ws = int(k % kWorkRing);
        if (k >= kWorkRing) mbar_wait(&empty_bar[ws], (k / kWorkRing - 1) & 1);
        w_slot[ws] = r;
        w_p[ws] = p;
        mbar_arrive(&full_bar[ws]);
        if (P.prof) atomicAdd(P.prof + 1, globaltimer() - tq0);
      }
      __syncwarp();
    };
    uint32_t fills = 0, frees = 0;
    bool abort = false, tma_pending = false;
    fetch_next();
    while (nx.valid && !abort) {
      const Next cur = nx;
      const bool glb = no_tma || cur.bytes > P.blk_cap;
      const uint32_t tcode = uint32_t(cur.t) << 8 | uint32_t(cur.first);
      if (lane == 0) trace_ev(P, &trace_ctr, 1, r, tcode);
      if (lane == 0) {
        h_t[r] = cur.t;
        h_last[r] = cur.last;
        h_ofs[r] = cur.ofs;
        h_glb[r] = glb ? 1 : 0;
        h_r0[r] = cur.r0;
        h_rows[r] = cur.rows;
        h_E[r] = cur.E;
        h_nseg[r] = glb ? 0 : cur.nseg;
        h_mode[r] = glb ? 0 : cur.mode;
        h_xoff[r] = int32_t(cur.bytes);
        if (!glb) {
          fence_proxy_async_smem();
          mbar_arrive_expect_tx(&tile_bar[r], uint32_t(cur.bytes));
        }
      }
      __syncwarp();
      if (!glb) {
        // the block as kTmaSplit bulk copies (16-byte aligned pieces) on the
        // slot's one barrier; 4 or 8 concurrent pieces measured no faster
        // than one on cfg2 (the per-SM transfer is bandwidth-, not
        // request-bound), so LMPK_TMA_SPLIT defaults to 1
        const int64_t piece = ((cur.bytes + kTmaSplit - 1) / kTmaSplit + 15) & ~int64_t(15);
        const int64_t a = int64_t(lane) * piece, b = std::min<int64_t>(a + piece, cur.bytes);
        if (lane < kTmaSplit && b > a) {
          if (lane) fence_proxy_async_smem();
          bulk_g2s(smem_raw + int64_t(r) * P.smem_cap + a, P.blocks + cur.ofs + a, uint32_t(b - a), &tile_bar[r],
                   cur.last == P.n_powers ? pol_drop : pol_keep);
        }
      }
      if (lane == 0) trace_ev(P, &trace_ctr, 2, r, tcode);
      __syncwarp();
      tma_pending = !glb;
      ++p_items;
      for (int p = cur.first; p <= cur.last; ++p) {
        if (p > 1 && P.mode != 4) {
          const unsigned long long t0 = P.prof ? globaltimer() : 0;
          if (!spin_deps(P, cur.lo, cur.hi, P.epoch_base + uint32_t(p - 1), &p_rounds)) {
            abort = true;
            break;
          }
          if (P.prof) p_dep += globaltimer() - t0;
          if (lane == 0) trace_ev(P, &trace_ctr, 4, r, tcode);
        }
        if (tma_pending) {
          const unsigned long long t0 = P.prof ? globaltimer() : 0;
          const bool ok = mbar_wait_bounded(&tile_bar[r], fills & 1, P);
          ++fills;
          tma_pending = false;
          if (!ok) {
            abort = true;
            break;
          }
          if (P.prof) p_tma += globaltimer() - t0;
          if (lane == 0) trace_ev(P, &trace_ctr, 3, r, tcode);
        }
        if (P.xmode == 1 && !glb && cur.nseg > 0) {
          const unsigned long long t0 = P.prof ? globaltimer() : 0;
          if (!stage_x(s_pow[p - 1].yin, (cur.rows + 31) >> 5, cur.nseg, cur.xent, int32_t(cur.bytes))) {
            abort = true;
            break;
          }
          if (P.prof) p_x += globaltimer() - t0;
        }
        push(p);
        if (lane == 0) trace_ev(P, &trace_ctr, 5, r, tcode);
        if (p == cur.first && prefetch) {
          fetch_next();
          // warm L2 with the next item's block while this one computes: its
          // TMA then pays an L2 hit instead of an HBM round trip
          if (nx.valid && lane == 0 && !(no_tma || nx.bytes > P.blk_cap) && (P.flags & 0x4000) == 0)
            bulk_prefetch_l2(P.blocks + nx.ofs, uint32_t(nx.bytes));
        }
      }
      if (abort) break;
      const unsigned long long t0 = P.prof ? globaltimer() : 0;
      if (!mbar_wait_bounded(&free_bar[r], frees & 1, P)) {  // consumers finished the last power
        abort = true;
        break;
      }
      ++frees;
      if (lane == 0) trace_ev(P, &trace_ctr, 6, r, tcode);
      if (P.prof) p_free += globaltimer() - t0;
      if (!prefetch) fetch_next();
    }
    if (tma_pending && lane == 0) mbar_wait(&tile_bar[r], fills & 1);  // no TMA may land after exit
    if (P.prof && lane == 0) {
      atomicAdd(P.prof + 3, p_rounds);
      atomicAdd(P.prof + 5, globaltimer() - p_t0);
      atomicAdd(P.prof + 6, p_items);
      atomicAdd(P.prof + 7, p_tma);
      atomicAdd(P.prof + 8, p_dep);
      atomicAdd(P.prof + 9, p_free);
      atomicAdd(P.prof + 11, p_x);
    }
    // the last producer to finish posts the terminator (after every push)
    if (lane == 0 && atomicAdd(&prod_done, 1u) == uint32_t(R - 1)) {
      const uint32_t k = atomicAdd(&ring_ctr, 1u);
      const int ws = int(k % kWorkRing);
      if (k >= kWorkRing) mbar_wait(&empty_bar[ws], (k / kWorkRing - 1) & 1);
      w_slot[ws] = -1;
      mbar_arrive(&full_bar[ws]);
    }
  } else {
    // ------------------------------------------------ consumer warps: compute only
    unsigned long long n_it = 0;
    for (int k = 0;; ++k) {
      const int ws = k % kWorkRing;
      mbar_wait_sleep(&full_bar[ws], uint32_t(k / kWorkRing) & 1);
      const int r = w_slot[ws];
      if (r < 0) break;
      const int p = w_p[ws];
      const int32_t t = h_t[r];
      const int32_t r0 = h_r0[r], rows = h_rows[r];
      if (lane == 0 && (warp == 0 || warp == NC - 1)) trace_ev(P, &trace_ctr, 10, r, uint32_t(t) << 8 | uint32_t(p));
      const uint32_t E = uint32_t(h_E[r]);
      const PowTab& pt = s_pow[p - 1];
      const uint32_t sch = (P.flags & 0x8000) ? kSchedStatic : smem_u32(&w_ctr[ws]);
      const bool use_acc = P.use_acc != 0;
      const int32_t nseg = h_nseg[r];
      const int32_t tmode = h_mode[r];
      // separate inlined copies so each sees a known address space (LDS vs
      // LDG); plain SpMV powers take the epilogue without Chebyshev/acc
      if (!h_glb[r]) {
        const uint32_t sb = smem_u32(smem_raw) + uint32_t(r) * uint32_t(P.smem_cap);
        const SmemBlk B{sb};
        const bool pairs = (P.flags & 0x800) == 0;  // internal A/B switch
        if (tmode != 0) {
          if (!CPLX && nseg > 0) {  // x staging is planned for real-vector tilings only
            const uint32_t xb = sb + uint32_t(h_xoff[r]);
            if (P.xmode == 2) copy_x_segments<CPLX, NC>(B, pt, rows, nseg, xb, warp, lane);
            const GatherSmem G{xb};
            if constexpr (!CPLX) {
            tile_c_dispatch<CPLX, EXACT, true>(tmode, pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, sch);
            }
          } else {
            tile_c_dispatch<CPLX, EXACT, false>(tmode, pt, P.acc, use_acc, B, GatherGlobal{pt.yin}, r0, rows, E, 0,
                                                warp, NC, sch);
          }
        } else if (nseg > 0) {
          const uint32_t xb = sb + uint32_t(h_xoff[r]);
          if (P.xmode == 2) copy_x_segments<CPLX, NC>(B, pt, rows, nseg, xb, warp, lane);
          const GatherSmem G{xb};
          if (pt.general)
            tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, pairs, sch);
          else
            tile_power<CPLX, EXACT, false>(pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, pairs, sch);
        } else {
          const GatherGlobal G{pt.yin};
          if (pt.general)
            tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, pairs, sch);
          else
            tile_power<CPLX, EXACT, false>(pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, pairs, sch);
        }
      } else {
        tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, GlbBlk{P.blocks + h_ofs[r]}, GatherGlobal{pt.yin}, r0,
                                      rows, E, 0, warp, NC, true, sch);
      }
      __syncwarp();
      ++n_it;
      if (lane == 0 && (warp == 0 || warp == NC - 1)) trace_ev(P, &trace_ctr, 11, r, uint32_t(t) << 8 | uint32_t(p));
      uint32_t old = 0;
      if (lane == 0) old = atom_add_acqrel_cta_smem(&w_done[ws], 1u);
      const bool last = __shfl_sync(0xffffffffu, old, 0) == uint32_t(NC - 1);
      if (last) {
        // this warp finished (t, p) last: every warp's rows are stored and
        // every warp is done reading the slot.  Free the slot and the ring
        // entry FIRST (CTA-scope releases), then publish at gpu scope -- the
        // release fence of the publish waits for this warp's global stores
        // (~1.4 us) and must not delay the refill.
        if (lane == 0) {
          trace_ev(P, &trace_ctr, 12, r, uint32_t(t) << 8 | uint32_t(p));
          const int last_p = h_last[r];
          w_done[ws] = 0;
          w_ctr[ws] = 0;
          if (p == last_p) mbar_arrive(&free_bar[r]);  // release.cta: the slot may be refilled
          mbar_arrive(&empty_bar[ws]);
        }
        if (P.mode == 4) {
          if (p < P.n_powers) {
            // count (t, p) towards each dependent (u, p+1); the increment that
            // completes u's dependency range enqueues (u, p+1)
            __syncwarp();
            fence_acq_rel_gpu();
            const int32_t a = __ldg(P.rdep_ptr + t), b = __ldg(P.rdep_ptr + t + 1);
            for (int32_t i = a + lane; i < b; i += 32) {
              const int32_t u = __ldg(P.rdep + i);
              const uint32_t target = uint32_t(__ldg(P.dep_hi + u) - __ldg(P.dep_lo + u) + 1);
              const uint32_t prev = atom_add_acqrel_gpu(P.rcnt + int64_t(p) * P.n_tiles + u, 1u);
              if (prev + 1 == target) {
                const uint32_t idx = atomicAdd(P.rctrl + 32, 1u);
                st_release_s32(P.rqueue + idx, (u << 8) | (p + 1));
              }
            }
          }
          if (lane == 0) atomicAdd(P.rctrl + 96, 1u);
        } else if (P.mode != 3 && lane == 0) {
          st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
        }
      } else if (lane == 0) {
        mbar_arrive(&empty_bar[ws]);
      }
    }
    if (P.prof && lane == 0) atomicAdd(P.prof + 2, n_it);
  }
}


// ---------------------------------------------------------------- ring walk kernel
// Streaming walk with a ring of shared-memory pieces (the default plan for
// compressed tilings).  The tiles are small ("pieces", one ring slot each);
// a WORK ITEM is (super-tile T = a run of consecutive tiles, power p), queued
// by the same skewed diagonal key as above in super-tile units.  One producer
// warp takes an item, waits for its dependencies (the tiles of
// [st_lo(T), st_hi(T)] at power p-1), then streams T's tiles through the ring
// with one TMA bulk copy each, running ahead of the consumers by up to the
// ring depth -- across item boundaries, so neither the TMA latency nor the
// next item's dependency wait leaves the consumers idle.  All NC consumer
// warps share each piece (slices strided by warp, no CTA barrier); the last
// warp to finish a piece hands it to a publisher warp, which frees the slot
// and publishes the tile's progress word (gpu-scope release, cumulative over
// the consumers' stores through the CTA-scope acq_rel chain), so dependents
// wait on exactly the tiles they read and no consumer pays the release fence.
// Deadlock freedom: an item depends only on items with smaller keys (M > D),
// each producer processes its items in ticket order, and the pieces of a
// started item never wait on anything but ring space, which the CTA's own
// consumers free unconditionally.
constexpr int kRingMax = 16;
// HASLONG = false: the tiling has no slice wider than 8, and the kernel body
// carries no long-row code at all (it cost the W <= 8 path its registers).
// UNIFORM = 1 (2): every tile is a compressed dictionary (raw-value) tile of
// width <= 8 without x-staging (cfg2: dictionary; cfg5: raw): the consumers
// carry only that one tile body, which measured 3% faster on cfg2 than the
// general kernel (better register allocation of the hot loop).
// UNIFORM = 3: as 1, for plain powers only (no Chebyshev step, no accumulation).
template <bool CPLX, bool EXACT, int NC, bool HASLONG, int UNIFORM = 0>
__global__ void __launch_bounds__(32 * (NC + 2), 1) mpk_ring_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t full_bar[kRingMax], empty_bar[kRingMax], done_bar[kRingMax];
  __shared__ int32_t d_t[kRingMax], d_p[kRingMax], d_r0[kRingMax], d_rows[kRingMax], d_E[kRingMax];
  __shared__ int32_t d_mode[kRingMax], d_glb[kRingMax], d_nseg[kRingMax], d_xoff[kRingMax];
  __shared__ int64_t d_ofs[kRingMax];
  __shared__ uint32_t d_done[kRingMax], d_ctr[kRingMax];
  __shared__ uint32_t trace_ctr;
  __shared__ PowTab s_pow[LMPK_MAX_POWERS];
  // the plain dictionary kernel runs only with the default 2-piece ring (the
  // host checks), so its ring index arithmetic is shifts, not divisions
  const int NP = UNIFORM == 3 ? 2 : P.n_slots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  build_powtab(s_pow, P, C);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kRingMax; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
      mbar_init(&done_bar[i], 1);
      d_done[i] = 0;
      d_ctr[i] = 0;
    }
    trace_ctr = 0;
    fence_mbar_init();
  }
  __syncthreads();
  const uint32_t ring_base = smem_u32(smem_raw);
  if (warp == NC + 1) {
    // ------------------------------------------------ publisher: pieces in ring order
    for (uint32_t k = 0;; ++k) {
      const int slot = int(k % uint32_t(NP));
      mbar_wait_sleep(&done_bar[slot], (k / uint32_t(NP)) & 1);
      const int32_t t = d_t[slot], p = d_p[slot];
      __syncwarp();
      if (t < 0) break;  // terminator (forwarded by the consumers)
      if (lane == 0) {
        mbar_arrive(&empty_bar[slot]);  // descriptors read: the slot may be refilled
        st_release_u32(P.progress + t, P.epoch_base + uint32_t(p));
      }
      __syncwarp();
    }
  } else if (warp == NC) {
    // ------------------------------------------------ producer
    // block L2 policy (run flag bits 8-9): 0 (default) / 2 evict_first -- the
    // blocks' 8-power reuse window exceeds L2, so keeping them only evicts the
    // gathered vectors (measured: 0.51 vs 0.53 ms on cfg2) -- 1 normal, 3 last
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
      if (p > 1 && !spin_deps(P, __ldg(P.st_lo + T), __ldg(P.st_hi + T), P.epoch_base + uint32_t(p - 1), &rounds)) {
        abort = true;
        break;
      }
      if (lane == 0) trace_ev(P, &trace_ctr, 4, 0, uint32_t(T) << 8 | uint32_t(p));
      for (int32_t m = m0; m < m1; ++m) {
        const int slot = int(k % uint32_t(NP));
        if (k >= uint32_t(NP) && !mbar_wait_bounded(&empty_bar[slot], (k / uint32_t(NP) - 1) & 1, P)) {
          abort = true;
          break;
        }
        if (lane == 0) {
          const int64_t ofs = __ldg(P.tile_ofs + m), bytes = __ldg(P.tile_ofs + m + 1) - ofs;
          const bool glb = bytes > P.smem_cap;
          d_t[slot] = m;
          d_p[slot] = p;
          d_r0[slot] = __ldg(P.tile_row + m);
          d_rows[slot] = __ldg(P.tile_row + m + 1) - d_r0[slot];
          d_E[slot] = __ldg(P.tile_E + m);
          d_mode[slot] = glb ? 0 : (P.tile_mode ? __ldg(P.tile_mode + m) : 0);
          d_glb[slot] = glb ? 1 : 0;
          d_ofs[slot] = ofs;
          const int32_t nseg = (glb || !P.xmode) ? 0 : __ldg(P.tile_nseg + m);
          d_nseg[slot] = nseg;
          d_xoff[slot] = int32_t(bytes);  // the x buffer follows the block
          trace_ev(P, &trace_ctr, 2, uint32_t(slot), uint32_t(m) << 8 | uint32_t(p));
          if (!glb) {
            const uint32_t xbytes = (nseg > 0 && P.xmode == 1) ? uint32_t(__ldg(P.tile_xent + m)) * 8u : 0u;
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&full_bar[slot], uint32_t(bytes) + xbytes);
            bulk_g2s(smem_raw + int64_t(slot) * P.smem_cap, P.blocks + ofs, uint32_t(bytes), &full_bar[slot],
                     p == P.n_powers ? policy_evict_first() : pol);
          } else {
            mbar_arrive(&full_bar[slot]);
          }
        }
        __syncwarp();
        // x staging: the runs of y_{p-1} this piece gathers, bulk-copied after
        // the item's dependencies were acquired (segment table read from the
        // block in global memory: the staged copy may not have landed yet)
        const int32_t nseg = __shfl_sync(0xffffffffu, lane == 0 ? d_nseg[slot] : 0, 0);
        if (nseg > 0 && P.xmode == 1) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          const int64_t ofs = __ldg(P.tile_ofs + m);
          const int32_t rows = __ldg(P.tile_row + m + 1) - __ldg(P.tile_row + m);
          const int4* seg = reinterpret_cast<const int4*>(P.blocks + ofs + blk_seg_off((rows + 31) >> 5));
          const uint32_t xb = ring_base + uint32_t(slot) * uint32_t(P.smem_cap) +
                              uint32_t(__ldg(P.tile_ofs + m + 1) - ofs);
          const char* yin = s_pow[p - 1].yin;
          for (int j = lane; j < nseg; j += 32) {
            const int4 sg = __ldg(seg + j);
            bulk_g2s_a(xb + uint32_t(sg.z) * 8u, yin + int64_t(sg.x) * 8, uint32_t((sg.y + 1) & ~1) * 8u,
                       &full_bar[slot], policy_evict_normal());
          }
        }
        __syncwarp();
        ++k;
      }
      if (abort) break;
    }
    // terminator (after every piece): consumers stop at a slot with t = -1
    if (lane == 0) {
      const int slot = int(k % uint32_t(NP));
      bool ok = true;
      if (k >= uint32_t(NP)) {
        // bounded like every other wait; on abort the consumers may never free it
        unsigned long long t0 = globaltimer();
        while (!mbar_try_wait(&empty_bar[slot], (k / uint32_t(NP) - 1) & 1)) {
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
    for (uint32_t k = 0;; ++k) {
      const int slot = int(k % uint32_t(NP));
      mbar_wait_sleep(&full_bar[slot], (k / uint32_t(NP)) & 1);
      const int32_t t = d_t[slot];
      if (t < 0) {
        if (warp == 0 && lane == 0) mbar_arrive(&done_bar[slot]);  // stop the publisher
        break;
      }
      const int32_t p = d_p[slot], r0 = d_r0[slot], rows = d_rows[slot], tmode = d_mode[slot];
      const uint32_t E = uint32_t(d_E[slot]);
      const PowTab& pt = s_pow[p - 1];
      const uint32_t sch = (P.flags & 0x8000) ? kSchedStatic : smem_u32(&d_ctr[slot]);
      if (lane == 0 && (warp == 0 || warp == NC - 1)) trace_ev(P, &trace_ctr, 10, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
      const int32_t nseg = d_nseg[slot];
      if constexpr (UNIFORM != 0) {
        const SmemBlk B{ring_base + uint32_t(slot) * uint32_t(P.smem_cap)};
        const GatherGlobal G{pt.yin};
        constexpr bool VDU = UNIFORM != 2;
        if constexpr (UNIFORM == 3)
          tile_power_c<CPLX, EXACT, false, true, false, false, true>(pt, P.acc, use_acc, B, G, r0, rows, E,
                                                                      tmode >> 8, 0, warp, NC, smem_u32(&d_ctr[slot]));
        else if (pt.general)
          tile_power_c<CPLX, EXACT, true, VDU>(pt, P.acc, use_acc, B, G, r0, rows, E, tmode >> 8, 0, warp, NC, sch);
        else
          tile_power_c<CPLX, EXACT, false, VDU>(pt, P.acc, use_acc, B, G, r0, rows, E, tmode >> 8, 0, warp, NC, sch);
      } else if (!CPLX && nseg > 0) {
        // gathers from the staged x runs (local columns)
        const SmemBlk B{ring_base + uint32_t(slot) * uint32_t(P.smem_cap)};
        const uint32_t xb = B.a + uint32_t(d_xoff[slot]);
        if (P.xmode == 2) copy_x_segments<CPLX, NC>(B, pt, rows, nseg, xb, warp, lane);
        const GatherSmem G{xb};
        if constexpr (!CPLX) {
          if (tmode == 0) {
            if (pt.general)
              tile_power<CPLX, EXACT, true, SmemBlk, decltype(G), HASLONG>(pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, true, sch);
            else
              tile_power<CPLX, EXACT, false, SmemBlk, decltype(G), HASLONG>(pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, true, sch);
          } else tile_c_dispatch<CPLX, EXACT, true, GatherSmem, HASLONG>(tmode, pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, sch);
        }
      } else if (!d_glb[slot]) {
        const SmemBlk B{ring_base + uint32_t(slot) * uint32_t(P.smem_cap)};
        const GatherGlobal G{pt.yin};
        if (tmode != 0) {
          tile_c_dispatch<CPLX, EXACT, false, GatherGlobal, HASLONG>(tmode, pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, sch);
        } else {
          if (pt.general)
            tile_power<CPLX, EXACT, true, SmemBlk, decltype(G), HASLONG>(pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, true, sch);
          else
            tile_power<CPLX, EXACT, false, SmemBlk, decltype(G), HASLONG>(pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, true, sch);
        }
      } else if constexpr (HASLONG) {  // oversize tiles exist only with slices far wider than 8
        tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, GlbBlk{P.blocks + d_ofs[slot]}, GatherGlobal{pt.yin}, r0,
                                      rows, E, 0, warp, NC, true, sch);
      }
      __syncwarp();
      if (lane == 0 && (warp == 0 || warp == NC - 1)) trace_ev(P, &trace_ctr, 11, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
      uint32_t old = 0;
      if (lane == 0) old = atom_add_acqrel_cta_smem(&d_done[slot], 1u);
      if (__shfl_sync(0xffffffffu, old, 0) == uint32_t(NC - 1) && lane == 0) {
        // last warp on this piece: every warp's rows are stored and nobody
        // reads the slot any more -- hand it to the publisher
        d_done[slot] = 0;
        d_ctr[slot] = 0;
        trace_ev(P, &trace_ctr, 12, uint32_t(slot), uint32_t(t) << 8 | uint32_t(p));
        mbar_arrive(&done_bar[slot]);
      }
    }
  }
}

}  // namespace lmpk
