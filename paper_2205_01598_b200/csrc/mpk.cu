// mpk.cu -- level-blocked matrix power kernel for sm_100a.
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
  int32_t xoff;      // byte offset of the x buffer inside a slot
  int32_t blk_cap;   // bytes of a slot available to the staged block
  int32_t xmode;     // 0 no x staging, 1 TMA (aligned vectors), 2 cooperative copy
  int32_t n_slots;   // R
  int32_t flags;     // LMPK_FLAG_* (NO_TMA, policy bits 8-9)
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
struct GatherGlobal {
  const char* base;
  __device__ __forceinline__ double d(int32_t c) const { return ldg_f64(base + uint64_t(uint32_t(c)) * 8u); }
  __device__ __forceinline__ double2 d2(int32_t c) const {
    return ldg_f64x2(base + uint64_t(uint32_t(c)) * 16u);
  }
};
struct GatherSmem {
  uint32_t base;
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

template <bool EXACT, bool FULL, class Blk, class G>
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
    default: return slice_real_any<EXACT>(B, cb, vb, l4, g, w, FULL ? w : len);
  }
}

// ---------------------------------------------------------------- compressed blocks
// Compressed tile block (tile_mode bit 0): the same slices, chunks and entry
// order as above, but
//   * columns are int16 offsets from the entry's own row (col - row): a
//     level-ordered matrix couples a row only to its own and the adjacent
//     levels, so the offsets stay within +-32767 for level widths up to that
//     (index compression in the style of CSR-DU, Kourtis et al. 2008);
//   * values are either raw f64, or (tile_mode bit 1) uint8 codes into a
//     per-tile dictionary of <= 256 distinct values (CSR-VI value indexing).
//     The dictionary holds the exact bit patterns, so every product is the
//     same double as from the CRS arrays and the row sums stay bitwise equal.
// Layout: [rec int2 x ns] [lens u16 x 32 ns] | align16 | [dict f64 x nd]
//   | align16 | [col16 x E] | align16 | [code u8 x E  or  val f64 x E]
// rec[s] = {first entry of slice s (relative to the tile), w | wmin << 16}.
// Matrix bytes per entry: 3 (dictionary) or 10 (raw) instead of 12.
constexpr int kDictMax = 256;
constexpr int32_t kModeC16 = 1, kModeDict = 2;
__host__ __device__ inline int64_t cblk_dict_off(int32_t ns) { return align16(int64_t(ns) * 72); }
__host__ __device__ inline int64_t cblk_col_off(int32_t ns, int32_t nd) {
  return align16(cblk_dict_off(ns) + int64_t(nd) * 8);
}
__host__ __device__ inline int64_t cblk_val_off(int32_t ns, int32_t nd, int64_t E) {
  return align16(cblk_col_off(ns, nd) + E * 2);
}
__host__ __device__ inline int64_t cblk_bytes(int32_t ns, int32_t nd, int64_t E, bool dict) {
  return (cblk_val_off(ns, nd, E) + E * (dict ? 1 : 8) + 127) & ~int64_t(127);
}
__device__ __forceinline__ int32_t sx16(int32_t v) { return (v << 16) >> 16; }

// Column indices of lane's W entries (row = the lane's row).
template <int W>
__device__ __forceinline__ void c16_cols(const SmemBlk& B, uint32_t cb, uint32_t lane, int32_t row,
                                         int32_t (&c)[W]) {
  constexpr int Q = W >> 2, PR = (W >> 1) & 1, SG = W & 1;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int2 v = B.i2(cb + q * 256 + lane * 8);
    c[4 * q] = row + sx16(v.x);
    c[4 * q + 1] = row + (v.x >> 16);
    c[4 * q + 2] = row + sx16(v.y);
    c[4 * q + 3] = row + (v.y >> 16);
  }
  if constexpr (PR) {
    const int32_t v = B.i1(cb + Q * 256 + lane * 4);
    c[4 * Q] = row + sx16(v);
    c[4 * Q + 1] = row + (v >> 16);
  }
  if constexpr (SG) c[W - 1] = row + sx16(int32_t(B.u16(cb + Q * 256 + PR * 128 + lane * 2)));
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
      v[4 * q] = lds_f64(dict + (k & 255u) * 8u);
      v[4 * q + 1] = lds_f64(dict + ((k >> 8) & 255u) * 8u);
      v[4 * q + 2] = lds_f64(dict + ((k >> 16) & 255u) * 8u);
      v[4 * q + 3] = lds_f64(dict + (k >> 24) * 8u);
    }
    if constexpr (PR) {
      const uint32_t k = B.u16(vb + Q * 128 + lane * 2);
      v[4 * Q] = lds_f64(dict + (k & 255u) * 8u);
      v[4 * Q + 1] = lds_f64(dict + (k >> 8) * 8u);
    }
    if constexpr (SG) v[W - 1] = lds_f64(dict + B.u8(vb + Q * 128 + PR * 64 + lane) * 8u);
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
template <int W, bool EXACT, bool FULL, bool VD, class G>
__device__ __forceinline__ double cslice_real_w(const SmemBlk& B, CSlice a, uint32_t lane, int32_t row,
                                                uint32_t dict, const G& g, int len) {
  int32_t c[W];
  c16_cols<W>(B, a.cb, lane, row, c);
  double x[W];
#pragma unroll
  for (int j = 0; j < W; ++j) x[j] = g.d(c[j]);
  double v[W];
  c16_vals<W, VD>(B, a.vb, lane, dict, v);
  return chain<EXACT, FULL, W>(v, x, len);
}

// Two compressed slices of the same width W <= 8: all gathers in flight together.
template <int W, bool EXACT, bool FULL, bool VD, class G>
__device__ __forceinline__ double2 cslice_real_w2(const SmemBlk& B, CSlice a0, CSlice a1, uint32_t lane,
                                                  int32_t row0, int32_t row1, uint32_t dict, const G& g,
                                                  int len0, int len1) {
  int32_t c0[W], c1[W];
  c16_cols<W>(B, a0.cb, lane, row0, c0);
  c16_cols<W>(B, a1.cb, lane, row1, c1);
  double x0[W], x1[W];
#pragma unroll
  for (int j = 0; j < W; ++j) x0[j] = g.d(c0[j]);
#pragma unroll
  for (int j = 0; j < W; ++j) x1[j] = g.d(c1[j]);
  double t0, t1;
  {
    double v[W];
    c16_vals<W, VD>(B, a0.vb, lane, dict, v);
    t0 = chain<EXACT, FULL, W>(v, x0, len0);
  }
  {
    double v[W];
    c16_vals<W, VD>(B, a1.vb, lane, dict, v);
    t1 = chain<EXACT, FULL, W>(v, x1, len1);
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
      v = lds_f64(dict + B.u8(a.vb + ec) * 8u);
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

template <bool EXACT, bool FULL, bool VD, class G>
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
    default: return cslice_any<false, EXACT, VD>(B, a, lane, row, dict, g, w, FULL ? w : len).x;
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
template <bool CPLX, bool EXACT, bool GENERAL, bool VD, class G>
__device__ __forceinline__ void tile_power_c(const PowTab& pt, double* acc_base, bool use_acc, const SmemBlk& B,
                                             const G& g, int32_t r0, int32_t nrows, uint32_t E, int32_t nd,
                                             int wid, int nwarps) {
  const int32_t ns = (nrows + 31) >> 5;
  const uint32_t lens_o = uint32_t(ns) * 8;
  const uint32_t dict = B.a + uint32_t(cblk_dict_off(ns));
  const uint32_t col_o = uint32_t(cblk_col_off(ns, nd));
  const uint32_t val_o = uint32_t(cblk_val_off(ns, nd, E));
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
    auto epilogue = [&](int32_t s, double t) {
      const int32_t lr = s * 32 + int32_t(lane);
      if (lr < nrows) {
        if constexpr (GENERAL) {
          if (pt.cheb) t = __dsub_rn(__dmul_rn(2.0, t), ld_cg(ypv + lr));
          stg_f64(yout + lr, t);
          if (use_acc) stg_f64(acc + lr, madd<EXACT>(ld_cg(acc + lr), pt.cre, t));
        } else {
          stg_f64(yout + lr, t);
        }
      }
    };
    auto single = [&](int32_t s, int2 rec) -> double {
      const CSlice a = cslice<VD>(col_o, val_o, uint32_t(rec.x));
      const int w = rec.y & 0xffff;
      const int32_t row = r0 + s * 32 + int32_t(lane);
      if (int(uint32_t(rec.y) >> 16) == w) return cslice_real<EXACT, true, VD>(B, a, lane, row, dict, g, w, w);
      return cslice_real<EXACT, false, VD>(B, a, lane, row, dict, g, w, len_of(s, rec));
    };
    for (int32_t s = wid; s < ns; s += 2 * nwarps) {
      const int32_t s2 = s + nwarps;
      const int2 rec0 = B.i2(uint32_t(s) * 8);
      if (s2 >= ns) {
        epilogue(s, single(s, rec0));
        break;
      }
      const int2 rec1 = B.i2(uint32_t(s2) * 8);
      const int w0 = rec0.y & 0xffff, w1 = rec1.y & 0xffff;
      if (w0 == w1 && w0 >= 1 && w0 <= 8) {
        const bool full0 = int(uint32_t(rec0.y) >> 16) == w0, full1 = int(uint32_t(rec1.y) >> 16) == w1;
        const CSlice a0 = cslice<VD>(col_o, val_o, uint32_t(rec0.x)), a1 = cslice<VD>(col_o, val_o, uint32_t(rec1.x));
        const int32_t row0 = r0 + s * 32 + int32_t(lane), row1 = r0 + s2 * 32 + int32_t(lane);
        double2 t;
        if (full0 && full1)
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
    for (int32_t s = wid; s < ns; s += nwarps) {
      const int2 rec = B.i2(uint32_t(s) * 8);
      const CSlice a = cslice<VD>(col_o, val_o, uint32_t(rec.x));
      const int w = rec.y & 0xffff;
      const int32_t lr = s * 32 + int32_t(lane);
      double2 t = cslice_any<true, EXACT, VD>(B, a, lane, r0 + lr, dict, g, w, len_of(s, rec));
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

// One power step of one tile (rows r0 .. r0+nrows-1, E block entries): warps
// stride over the 32-row slices, lane = row.  GENERAL adds the Chebyshev
// three-term step and the accumulation; plain SpMV powers skip both.
template <bool CPLX, bool EXACT, bool GENERAL, class Blk, class G>
__device__ __forceinline__ void tile_power(const PowTab& pt, double* acc_base, bool use_acc, const Blk& B,
                                           const G& g, int32_t r0, int32_t nrows, uint32_t E, int32_t nseg,
                                           int wid, int nwarps, bool pairs = true) {
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
          stg_f64(yout + lr, t);
          if (use_acc) stg_f64(acc + lr, madd<EXACT>(ld_cg(acc + lr), pt.cre, t));
        } else {
          stg_f64(yout + lr, t);
        }
      }
    };
    auto single = [&](int32_t s, int2 rec) -> double {
      const uint32_t cb = uint32_t(rec.x), vb = 2 * cb + vdelta;
      const int w = rec.y & 0xffff;
      if (int(uint32_t(rec.y) >> 16) == w) return slice_real<EXACT, true>(B, cb, vb, l4, g, w, w);
      const int len = int(B.u16(lens_o + uint32_t(s) * 64 + (l4 >> 1)));
      return slice_real<EXACT, false>(B, cb, vb, l4, g, w, len);
    };
    // warp `wid` owns slices wid, wid + nwarps, ...; it takes them two at a time
    for (int32_t s = wid; s < ns; s += 2 * nwarps) {
      const int32_t s2 = s + nwarps;
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
  for (int32_t s = wid; s < ns; s += nwarps) {
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

// Spin until progress[lo..hi] >= target (one warp, all loads in flight per
// round); then one acquire fence (also invalidates L1 for the gathers).
// Returns false if the launch is aborting (abort flag or watchdog).
__device__ __forceinline__ bool spin_deps(const MpkParams& P, int32_t lo, int32_t hi, uint32_t target,
                                          unsigned long long* rounds) {
  const int lane = threadIdx.x & 31;
  unsigned long long t0 = 0;
  for (int spins = 0;; ++spins) {
    uint32_t m = 0xffffffffu;
    for (int32_t i = lo + lane; i <= hi; i += 32) m = min(m, ld_relaxed_u32(P.progress + i));
    ++*rounds;
    if (__all_sync(0xffffffffu, m >= target)) {
      fence_acq_rel_gpu();
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

template <bool CPLX, bool EXACT, int NC>
__global__ void __launch_bounds__(32 * (NC + kMaxSlots), 1) mpk_group_kernel(MpkParams P, PowerCfgDev C) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t tile_bar[kMaxSlots], free_bar[kMaxSlots], x_bar[kMaxSlots];
  __shared__ uint64_t full_bar[kWorkRing], empty_bar[kWorkRing];
  __shared__ int32_t w_slot[kWorkRing], w_p[kWorkRing];
  __shared__ uint32_t w_done[kWorkRing];
  __shared__ uint32_t ring_ctr, prod_done, trace_ctr;
  __shared__ int32_t h_t[kMaxSlots], h_last[kMaxSlots], h_glb[kMaxSlots];
  __shared__ int32_t h_r0[kMaxSlots], h_rows[kMaxSlots], h_E[kMaxSlots], h_nseg[kMaxSlots], h_mode[kMaxSlots];
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
    auto stage_x = [&](const char* yin, int32_t ns, int32_t nseg, int32_t xent) -> bool {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (lane == 0) mbar_arrive_expect_tx(&x_bar[r], uint32_t(xent) * 8u);
      __syncwarp();
      const uint32_t seg_o = slot_base + uint32_t(blk_seg_off(ns));
      const uint32_t xb = slot_base + uint32_t(P.xoff);
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
          if (!stage_x(s_pow[p - 1].yin, (cur.rows + 31) >> 5, cur.nseg, cur.xent)) {
            abort = true;
            break;
          }
          if (P.prof) p_x += globaltimer() - t0;
        }
        push(p);
        if (lane == 0) trace_ev(P, &trace_ctr, 5, r, tcode);
        if (p == cur.first && prefetch) fetch_next();
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
          const GatherGlobal G{pt.yin};
          const int32_t nd = tmode >> 8;
          if (tmode & kModeDict) {
            if (pt.general)
              tile_power_c<CPLX, EXACT, true, true>(pt, P.acc, use_acc, B, G, r0, rows, E, nd, warp, NC);
            else
              tile_power_c<CPLX, EXACT, false, true>(pt, P.acc, use_acc, B, G, r0, rows, E, nd, warp, NC);
          } else {
            if (pt.general)
              tile_power_c<CPLX, EXACT, true, false>(pt, P.acc, use_acc, B, G, r0, rows, E, nd, warp, NC);
            else
              tile_power_c<CPLX, EXACT, false, false>(pt, P.acc, use_acc, B, G, r0, rows, E, nd, warp, NC);
          }
        } else if (nseg > 0) {
          const uint32_t xb = sb + uint32_t(P.xoff);
          if (P.xmode == 2) {
            // vectors not 16-byte aligned: all consumer warps copy the
            // segments (plain loads), then one named barrier
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
          const GatherSmem G{xb};
          if (pt.general)
            tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, pairs);
          else
            tile_power<CPLX, EXACT, false>(pt, P.acc, use_acc, B, G, r0, rows, E, nseg, warp, NC, pairs);
        } else {
          const GatherGlobal G{pt.yin};
          if (pt.general)
            tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, pairs);
          else
            tile_power<CPLX, EXACT, false>(pt, P.acc, use_acc, B, G, r0, rows, E, 0, warp, NC, pairs);
        }
      } else {
        tile_power<CPLX, EXACT, true>(pt, P.acc, use_acc, GlbBlk{P.blocks + h_ofs[r]}, GatherGlobal{pt.yin}, r0,
                                      rows, E, 0, warp, NC);
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

// ---------------------------------------------------------------- tiling kernels
// per slice: longest row (width), shortest row (padding-free prefix) and,
// when fit16 != NULL, whether every entry's column offset col - row fits int16
__global__ void k_slice_width(const int32_t* row_ptr, const int32_t* col, int32_t n, int32_t n_slices,
                              int32_t* width, int32_t* wmin, uint8_t* fit16) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int32_t r = s * 32 + lane;
  const int32_t a = r < n ? __ldg(row_ptr + r) : 0;
  const int len = r < n ? __ldg(row_ptr + r + 1) - a : 0;
  const int w = __reduce_max_sync(0xffffffffu, len);
  const int m = __reduce_min_sync(0xffffffffu, len);
  if (fit16) {
    bool ok = true;
    for (int j = 0; j < len; ++j) {
      const int32_t d = __ldg(col + a + j) - r;
      ok = ok && d >= -32768 && d <= 32767;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) fit16[s] = ok ? 1 : 0;
  }
  if (lane == 0) {
    width[s] = w;
    wmin[s] = m;
  }
}

// Per-tile value dictionary (one CTA per listed tile): the distinct bit
// patterns of the tile's CRS values, sorted ascending, or nd = -1 if there
// are more than kDictMax.  Open-addressing hash set in shared memory.
constexpr int kDictHash = 1024;
__global__ void __launch_bounds__(256) k_tile_dict(const int32_t* row_ptr, const double* val, const int32_t* tile_row,
                                                   const int32_t* list, int32_t n_list, uint64_t* dict_out,
                                                   int32_t* nd_out) {
  __shared__ unsigned long long keys[kDictHash];
  __shared__ uint32_t state[kDictHash];
  __shared__ unsigned long long packed[kDictMax];
  __shared__ uint32_t count, overflow, npk;
  const int32_t li = blockIdx.x;
  if (li >= n_list) return;
  const int32_t t = list[li];
  for (int i = threadIdx.x; i < kDictHash; i += blockDim.x) state[i] = 0;
  if (threadIdx.x == 0) count = overflow = npk = 0;
  __syncthreads();
  const int32_t e0 = row_ptr[tile_row[t]], e1 = row_ptr[tile_row[t + 1]];
  volatile uint32_t* vs = state;
  volatile unsigned long long* vk = keys;
  for (int32_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    if (*(volatile uint32_t*)&overflow) break;
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(__ldg(val + e)));
    uint32_t h = uint32_t((bits * 0x9E3779B97F4A7C15ull) >> 54);
    for (;;) {
      const uint32_t st = vs[h];
      if (st == 2) {
        if (vk[h] == bits) break;
        h = (h + 1) & (kDictHash - 1);
      } else if (st == 0) {
        if (atomicCAS(&state[h], 0u, 1u) == 0u) {
          vk[h] = bits;
          __threadfence_block();
          atomicExch(&state[h], 2u);
          if (atomicAdd(&count, 1u) >= uint32_t(kDictMax)) atomicExch(&overflow, 1u);
          break;
        }
      }  // st == 1: another thread is writing this key, re-read
    }
  }
  __syncthreads();
  if (overflow) {
    if (threadIdx.x == 0) nd_out[li] = -1;
    return;
  }
  for (int i = threadIdx.x; i < kDictHash; i += blockDim.x)
    if (state[i] == 2) packed[atomicAdd(&npk, 1u)] = keys[i];
  __syncthreads();
  const uint32_t nd = npk;
  for (uint32_t j = threadIdx.x; j < nd; j += blockDim.x) {
    const unsigned long long k = packed[j];
    uint32_t rank = 0;
    for (uint32_t i = 0; i < nd; ++i) rank += packed[i] < k;
    dict_out[int64_t(li) * kDictMax + rank] = k;
  }
  if (threadIdx.x == 0) nd_out[li] = int32_t(nd);
}

// one warp per slice: slice record, row lengths and the chunked entries.
// Tiles with x-segments get local columns (index into the tile's x buffer);
// the warp of a tile's first slice also writes the tile's segment table.
__global__ void k_fill_blocks(const int32_t* row_ptr, const int32_t* col, const double* val,
                              int32_t n_slices, const int32_t* slice_tile, const int32_t* slice_off,
                              const int32_t* width, const int32_t* wmin, const int32_t* tile_row,
                              const int64_t* tile_ofs, const int32_t* tile_E, const int32_t* seg_ptr,
                              const int4* segs, const int32_t* tile_mode, const int32_t* tile_dict,
                              const uint64_t* dict_tab, unsigned char* blocks) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int32_t t = slice_tile[s];
  const int32_t r0 = tile_row[t], r1 = tile_row[t + 1];
  const int32_t ns = (r1 - r0 + 31) >> 5;
  const int32_t ls = s - (r0 >> 5);
  const int32_t mode = tile_mode ? tile_mode[t] : 0;
  if (mode != 0) {
    // compressed block (see cblk_*): int16 column offsets, dictionary codes or raw values
    const int32_t nd = mode >> 8;
    const bool vd = (mode & kModeDict) != 0;
    unsigned char* blk = blocks + tile_ofs[t];
    const int32_t E = tile_E[t];
    const uint64_t* dict = vd ? dict_tab + int64_t(tile_dict[t]) * kDictMax : nullptr;
    if (ls == 0 && vd)
      for (int j = lane; j < nd; j += 32) reinterpret_cast<uint64_t*>(blk + cblk_dict_off(ns))[j] = dict[j];
    int16_t* c16 = reinterpret_cast<int16_t*>(blk + cblk_col_off(ns, nd));
    unsigned char* vbase = blk + cblk_val_off(ns, nd, E);
    const int32_t base = slice_off[s];
    const int32_t r = s * 32 + lane;
    const bool valid = r < r1;
    const int32_t a = valid ? row_ptr[r] : 0;
    const int len = valid ? row_ptr[r + 1] - a : 0;
    const int w = width[s];
    if (lane == 0) reinterpret_cast<int2*>(blk)[ls] = make_int2(base, w | (wmin[s] << 16));
    reinterpret_cast<uint16_t*>(blk + int64_t(ns) * 8)[ls * 32 + lane] = uint16_t(len);
    // padding: the row's last column (own row if empty; r0 for lanes past the tile)
    int32_t pad = valid ? 0 : r0 - r;
    for (int j = 0; j < w; ++j) {
      const int64_t e = chunk_entry(base, w, lane, j);
      int32_t d = pad;
      double v = 0.0;
      if (j < len) {
        d = col[a + j] - r;
        v = val[a + j];
        pad = d;
      }
      c16[e] = int16_t(d);
      if (vd) {
        uint8_t code = 0;
        if (j < len) {
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
          int lo = 0, hi = nd - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (dict[mid] < bits)
              lo = mid + 1;
            else
              hi = mid;
          }
          code = uint8_t(lo);
        }
        vbase[e] = code;
      } else {
        reinterpret_cast<double*>(vbase)[e] = v;
      }
    }
    return;
  }
  const int32_t sg0 = seg_ptr ? seg_ptr[t] : 0;
  const int32_t nseg = seg_ptr ? seg_ptr[t + 1] - sg0 : 0;
  unsigned char* blk = blocks + tile_ofs[t];
  int2* rec = reinterpret_cast<int2*>(blk);
  uint16_t* lens = reinterpret_cast<uint16_t*>(blk + int64_t(ns) * 8);
  const int64_t co = blk_col_off(ns, nseg);
  const int32_t E = tile_E[t];
  int32_t* cols = reinterpret_cast<int32_t*>(blk + co);
  double* vals = reinterpret_cast<double*>(blk + co + int64_t(E) * 4);
  if (ls == 0)
    for (int j = lane; j < nseg; j += 32)
      reinterpret_cast<int4*>(blk + blk_seg_off(ns))[j] = segs[sg0 + j];
  const int32_t base = slice_off[s];
  const int32_t r = s * 32 + lane;
  const bool valid = r < r1;
  const int32_t a = valid ? row_ptr[r] : 0;
  const int len = valid ? row_ptr[r + 1] - a : 0;
  const int w = width[s];
  if (lane == 0) rec[ls] = make_int2(int32_t(co + int64_t(base) * 4), w | (wmin[s] << 16));
  lens[ls * 32 + lane] = uint16_t(len);
  // local index of a global column: its segment (binary search) + offset
  auto local = [&](int32_t c) -> int32_t {
    if (nseg == 0) return c;
    int lo = 0, hi = nseg - 1;  // last segment with start <= c
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (segs[sg0 + mid].x <= c)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int4 g = segs[sg0 + lo];
    return g.z + (c - g.x);
  };
  const int32_t pad = local(valid ? r : r0);  // harmless in-range index, never accumulated
  for (int j = 0; j < w; ++j) {
    const int64_t e = chunk_entry(base, w, lane, j);
    if (j < len) {
      cols[e] = local(col[a + j]);
      vals[e] = val[a + j];
    } else {
      cols[e] = (j == 0 || !valid) ? pad : local(col[a + len - 1]);
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

static const void* group_fn(bool cplx, bool exact) {
  if (cplx)
    return exact ? reinterpret_cast<const void*>(mpk_group_kernel<true, true, kConsumers>)
                 : reinterpret_cast<const void*>(mpk_group_kernel<true, false, kConsumers>);
  return exact ? reinterpret_cast<const void*>(mpk_group_kernel<false, true, kConsumers>)
               : reinterpret_cast<const void*>(mpk_group_kernel<false, false, kConsumers>);
}

// Largest dynamic smem one group-kernel CTA may use (all instantiations), and
// the occupancy at `smem` bytes (min over instantiations).
static int group_occupancy(lmpk_ctx* ctx, int smem, int* occ) {
  *occ = 1 << 20;
  for (int c = 0; c < 2; ++c)
    for (int x = 0; x < 2; ++x) {
      const void* fn = group_fn(c != 0, x != 0);
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, fn);
      const int max_dyn = ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes);
      if (e == cudaSuccess && smem > max_dyn) {
        *occ = 0;
        return LMPK_OK;
      }
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
      int o = 0;
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, kBlockThreads, smem);
      if (e != cudaSuccess) {
        cudaGetLastError();  // do not leave a sticky status for later checks
        set_error("occupancy query failed: %s", cudaGetErrorString(e));
        return LMPK_ERR_CUDA;
      }
      *occ = std::min(*occ, o);
    }
  return LMPK_OK;
}

// Largest static shared memory over the group-kernel instantiations.
static int group_static_smem(int* out) {
  int mx = 0;
  for (int c = 0; c < 2; ++c)
    for (int x = 0; x < 2; ++x) {
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, group_fn(c != 0, x != 0));
      if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaFuncGetAttributes failed: %s", cudaGetErrorString(e));
        return LMPK_ERR_CUDA;
      }
      mx = std::max(mx, static_cast<int>(fa.sharedSizeBytes));
    }
  *out = mx;
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
      if (ns > 0 && blk_bytes(ns + 1, e2, 0) > cap) break;
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

// max over t of the (steps)-step forward dependency chain, via the prefix max
// of dep_hi (monotone, conservative).
static int32_t chain_reach(const std::vector<int32_t>& dep_hi, int32_t steps, int32_t* max_fwd) {
  const int32_t nt = static_cast<int32_t>(dep_hi.size());
  std::vector<int32_t> H(nt);
  int32_t run = 0, mf = 0;
  for (int32_t t = 0; t < nt; ++t) {
    run = std::max(run, dep_hi[t]);
    H[t] = run;
    mf = std::max(mf, dep_hi[t] - t);
  }
  if (max_fwd) *max_fwd = mf;
  int32_t worst = 0;
  for (int32_t t = 0; t < nt; ++t) {
    int32_t c = t;
    for (int32_t j = 0; j < steps; ++j) {
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
  cudaFree(t->d_tile_nseg);
  cudaFree(t->d_tile_xent);
  cudaFree(t->d_tile_mode);
  cudaFree(t->d_rdep_ptr);
  cudaFree(t->d_rdep);
  cudaFree(t->d_rcnt);
  cudaFree(t->d_rqueue);
  cudaFree(t->d_rctrl);
  cudaFree(t->d_items);
  cudaFree(t->d_progress);
  cudaFree(t->d_blocks);
  delete t;
  return LMPK_OK;
}

// x-segments of every tile (host): the tile's distinct columns, as runs of
// the gathered vector merged across gaps <= `gap`, each run's start rounded
// down to an even entry (16-byte aligned bulk copies) and its local base
// rounded up to even.  At most kMaxSegs runs (the gap doubles until they
// fit); a tile whose runs exceed `xcap` entries or whose column span is huge
// keeps global columns (nseg = 0).  Returns per tile nseg/xent and the runs.
static void plan_segments(const std::vector<int32_t>& rp, const std::vector<int32_t>& col,
                          const std::vector<int32_t>& tile_row, const std::vector<uint8_t>& allow, int32_t n,
                          int64_t xcap, std::vector<int32_t>& seg_ptr, std::vector<int4>& segs,
                          std::vector<int32_t>& xent) {
  const int32_t nt = static_cast<int32_t>(tile_row.size()) - 1;
  seg_ptr.assign(nt + 1, 0);
  xent.assign(nt, 0);
  segs.clear();
  std::vector<uint8_t> mark;
  std::vector<int2> runs;
  for (int32_t t = 0; t < nt; ++t) {
    seg_ptr[t] = static_cast<int32_t>(segs.size());
    const int64_t e0 = rp[tile_row[t]], e1 = rp[tile_row[t + 1]];
    if (e1 == e0 || xcap <= 0 || !allow[t]) continue;
    int32_t mn = INT32_MAX, mx = -1;
    for (int64_t e = e0; e < e1; ++e) {
      mn = std::min(mn, col[e]);
      mx = std::max(mx, col[e]);
    }
    const int64_t span = int64_t(mx) - mn + 1;
    if (span > (int64_t(1) << 22)) continue;
    mark.assign(span, 0);
    for (int64_t e = e0; e < e1; ++e) mark[col[e] - mn] = 1;
    for (int32_t gap = 8;; gap *= 2) {
      runs.clear();
      for (int64_t i = 0; i < span;) {
        if (!mark[i]) {
          ++i;
          continue;
        }
        int64_t j = i;
        while (j < span && mark[j]) ++j;
        const int32_t a = int32_t((mn + i) & ~int64_t(1));
        const int32_t b = int32_t(std::min<int64_t>(mn + j, n));
        if (!runs.empty() && a - runs.back().y <= gap)
          runs.back().y = std::max(runs.back().y, b);
        else
          runs.push_back(make_int2(a, b));
        i = j;
      }
      if (static_cast<int>(runs.size()) <= kMaxSegs) break;
    }
    int64_t lb = 0;
    for (const int2& g : runs) lb += (g.y - g.x + 1) & ~1;
    if (lb > xcap) continue;
    lb = 0;
    for (const int2& g : runs) {
      const int32_t cnt = g.y - g.x;
      segs.push_back(make_int4(g.x, cnt, int32_t(lb), 0));
      lb += (cnt + 1) & ~1;
    }
    xent[t] = int32_t(lb);
  }
  seg_ptr[nt] = static_cast<int32_t>(segs.size());
}

// Greedy partition of slices [s0, s1) into tiles whose block cost(ns, E) fits
// `cap` bytes and whose entries stay <= e_cap (a tile holds >= 1 slice).
template <class Cost>
static void partition_range(const std::vector<int32_t>& width, int32_t s0, int32_t s1, int64_t cap, int64_t e_cap,
                            Cost cost, std::vector<int32_t>& first, std::vector<int64_t>& Es) {
  int32_t s = s0;
  while (s < s1) {
    int32_t ns = 0;
    int64_t E = 0;
    while (s + ns < s1) {
      const int64_t e2 = E + int64_t(width[s + ns]) * 32;
      if (ns > 0 && (cost(ns + 1, e2) > cap || e2 > e_cap)) break;
      E = e2;
      ++ns;
    }
    first.push_back(s);
    Es.push_back(E);
    s += ns;
  }
}

// Tiles + chunked tile-SELL-32 blocks + dependency ranges for block cap `cap`
// bytes.  With fit16 (compressed tiling), runs of slices whose column offsets
// fit int16 become compressed tiles: first partitioned for the dictionary
// format (3 B/entry), then every tile with more than kDictMax distinct values
// is re-partitioned for raw values (10 B/entry); the other slices stay plain.
static int build_tiling(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr,
                        const int32_t* col, const double* val, const std::vector<int32_t>& width,
                        const int32_t* d_wmin, int64_t cap, const std::vector<int32_t>* h_rp,
                        const std::vector<int32_t>* h_col, int64_t xcap, const std::vector<uint8_t>* fit16,
                        int64_t e_cap, cudaStream_t st) {
  const int32_t S = static_cast<int32_t>(width.size());
  std::vector<int32_t> first;
  std::vector<int64_t> Es;
  std::vector<int32_t> tmode;   // per tile: 0 plain, else kModeC16 [| kModeDict | nd << 8]
  std::vector<int32_t> tdict;   // per tile: index into the dictionary table (dict tiles)
  uint64_t* d_dict_tab = nullptr;
  int32_t* d_tile_dict = nullptr;
  auto plain_cost = [](int32_t ns, int64_t E) { return blk_bytes(ns, E, 0); };
  if (fit16 && S > 0) {
    auto dict_cost = [](int32_t ns, int64_t E) { return cblk_bytes(ns, kDictMax, E, true); };
    auto raw_cost = [](int32_t ns, int64_t E) { return cblk_bytes(ns, 0, E, false); };
    // pass 1: runs of equal fit16, compressed runs cut for the dictionary format
    std::vector<int32_t> f1;
    std::vector<int64_t> E1;
    std::vector<uint8_t> c1;
    for (int32_t s = 0; s < S;) {
      int32_t e = s;
      while (e < S && (*fit16)[e] == (*fit16)[s]) ++e;
      const size_t before = f1.size();
      if ((*fit16)[s])
        partition_range(width, s, e, cap, e_cap, dict_cost, f1, E1);
      else
        partition_range(width, s, e, cap, INT64_MAX, plain_cost, f1, E1);
      c1.resize(f1.size(), (*fit16)[s]);
      (void)before;
      s = e;
    }
    const int32_t n1 = static_cast<int32_t>(f1.size());
    // dictionaries of the compressed pass-1 tiles (on the device)
    std::vector<int32_t> row1(n1 + 1), list;
    for (int32_t t = 0; t < n1; ++t) {
      row1[t] = std::min(f1[t] * 32, n);
      if (c1[t]) list.push_back(t);
    }
    row1[n1] = n;
    const int32_t nl = static_cast<int32_t>(list.size());
    std::vector<int32_t> nd(nl, -1);
    if (nl > 0) {
      int32_t *d_row1 = nullptr, *d_list = nullptr, *d_nd = nullptr;
      LMPK_TRY(dmalloc(&d_row1, n1 + 1));
      LMPK_TRY(dmalloc(&d_list, nl));
      LMPK_TRY(dmalloc(&d_nd, nl));
      LMPK_TRY(dmalloc(&d_dict_tab, size_t(nl) * kDictMax));
      LMPK_CHECK_CUDA(cudaMemcpyAsync(d_row1, row1.data(), size_t(n1 + 1) * 4, cudaMemcpyHostToDevice, st));
      LMPK_CHECK_CUDA(cudaMemcpyAsync(d_list, list.data(), size_t(nl) * 4, cudaMemcpyHostToDevice, st));
      k_tile_dict<<<nl, 256, 0, st>>>(row_ptr, val, d_row1, d_list, nl, d_dict_tab, d_nd);
      launch_count_add(ctx, 1);
      LMPK_CHECK_CUDA(cudaGetLastError());
      LMPK_CHECK_CUDA(cudaMemcpyAsync(nd.data(), d_nd, size_t(nl) * 4, cudaMemcpyDeviceToHost, st));
      LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
      cudaFree(d_row1);
      cudaFree(d_list);
      cudaFree(d_nd);
    }
    // pass 2: final tiles
    for (int32_t t = 0, li = 0; t < n1; ++t) {
      const int32_t s0 = f1[t], s1 = t + 1 < n1 ? f1[t + 1] : S;
      if (!c1[t]) {
        first.push_back(s0);
        Es.push_back(E1[t]);
        tmode.push_back(0);
        tdict.push_back(-1);
        continue;
      }
      const int32_t k = nd[li];
      if (k >= 0 && dict_cost(s1 - s0, E1[t]) <= cap) {
        first.push_back(s0);
        Es.push_back(E1[t]);
        tmode.push_back(kModeC16 | kModeDict | (k << 8));
        tdict.push_back(li);
      } else {
        const size_t b = first.size();
        partition_range(width, s0, s1, cap, e_cap, raw_cost, first, Es);
        for (size_t i = b; i < first.size(); ++i) {
          const int32_t a0 = first[i], a1 = i + 1 < first.size() ? first[i + 1] : s1;
          // a single slice too large for a slot stays plain (read from global)
          tmode.push_back(raw_cost(a1 - a0, Es[i]) <= cap ? kModeC16 : 0);
          tdict.push_back(-1);
        }
      }
      ++li;
    }
  } else {
    partition_slices(width, cap, first, Es);
    tmode.assign(first.size(), 0);
    tdict.assign(first.size(), -1);
  }
  const int32_t nt = static_cast<int32_t>(first.size());
  std::vector<int32_t> tile_row(nt + 1), tile_E(nt), slice_tile(std::max(S, 1)), slice_off(std::max(S, 1));
  std::vector<int64_t> tile_ofs(nt + 1);
  for (int32_t t = 0; t < nt; ++t) tile_row[t] = std::min(first[t] * 32, n);
  tile_row[nt] = n;
  // x-segments (real-vector tilings only)
  std::vector<int32_t> seg_ptr, xent;
  std::vector<int4> segs;
  if (h_rp && h_col && xcap > 0) {
    // only tiles whose block is staged in shared memory can use an x buffer
    std::vector<uint8_t> allow(nt);
    for (int32_t t = 0; t < nt; ++t) {
      const int32_t s1 = (t + 1 < nt) ? first[t + 1] : S;
      allow[t] = tmode[t] == 0 && blk_bytes(s1 - first[t], Es[t], 0) <= cap;
    }
    plan_segments(*h_rp, *h_col, tile_row, allow, n, xcap, seg_ptr, segs, xent);
  }
  int64_t ofs = 0;
  int64_t maxb = 0;
  int32_t n_comp = 0, n_dict = 0;
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t s0 = first[t], s1 = (t + 1 < nt) ? first[t + 1] : S;
    tile_E[t] = static_cast<int32_t>(Es[t]);
    tile_ofs[t] = ofs;
    const int32_t nseg = seg_ptr.empty() ? 0 : seg_ptr[t + 1] - seg_ptr[t];
    const int64_t b = tmode[t] ? cblk_bytes(s1 - s0, tmode[t] >> 8, Es[t], (tmode[t] & kModeDict) != 0)
                               : blk_bytes(s1 - s0, Es[t], nseg);
    n_comp += tmode[t] != 0;
    n_dict += (tmode[t] & kModeDict) != 0;
    maxb = std::max(maxb, b);
    ofs += b;
    int32_t e = 0;
    for (int32_t s = s0; s < s1; ++s) {
      slice_tile[s] = t;
      slice_off[s] = e;
      e += width[s] * 32;
    }
  }
  tile_ofs[nt] = ofs;
  T->info.compressed_tiles = n_comp;
  T->info.dict_tiles = n_dict;
  if (n_comp > 0) {
    LMPK_TRY(dmalloc(&T->d_tile_mode, nt));
    LMPK_TRY(dmalloc(&d_tile_dict, nt));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_mode, tmode.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_tile_dict, tdict.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
  }
  T->h_tile_row = tile_row;
  T->block_bytes = ofs;
  T->max_block = static_cast<int32_t>(std::min<int64_t>(maxb, INT32_MAX));
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
  // per-tile x-segment counts / entries (all zero without staging)
  std::vector<int32_t> tile_nseg(nt, 0);
  if (!seg_ptr.empty())
    for (int32_t t = 0; t < nt; ++t) tile_nseg[t] = seg_ptr[t + 1] - seg_ptr[t];
  if (xent.empty()) xent.assign(nt, 0);
  LMPK_TRY(dmalloc(&T->d_tile_nseg, nt));
  LMPK_TRY(dmalloc(&T->d_tile_xent, nt));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_nseg, tile_nseg.data(), nt * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_tile_xent, xent.data(), nt * 4, cudaMemcpyHostToDevice, st));
  int32_t* d_seg_ptr = nullptr;
  int4* d_segs = nullptr;
  if (!segs.empty()) {
    LMPK_TRY(dmalloc(&d_seg_ptr, nt + 1));
    LMPK_TRY(dmalloc(&d_segs, segs.size()));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_seg_ptr, seg_ptr.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_segs, segs.data(), segs.size() * 16, cudaMemcpyHostToDevice, st));
  }
  int64_t staged = 0, xmax = 0;
  for (int32_t t = 0; t < nt; ++t) {
    staged += tile_nseg[t] > 0;
    xmax = std::max<int64_t>(xmax, xent[t]);
  }
  T->staged_tiles = static_cast<int32_t>(staged);
  T->max_xent = static_cast<int32_t>(xmax);
  if (S > 0) {
    k_fill_blocks<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, val, S, d_slice_tile, d_slice_off,
                                                                 d_width, d_wmin, T->d_tile_row, T->d_tile_ofs,
                                                                 T->d_tile_E, d_seg_ptr, d_segs, T->d_tile_mode,
                                                                 d_tile_dict, d_dict_tab, T->d_blocks);
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
  cudaFree(d_seg_ptr);
  cudaFree(d_segs);
  cudaFree(d_tile_dict);
  cudaFree(d_dict_tab);
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
  LMPK_ARG_CHECK(prm.slots >= 0 && prm.slots <= kMaxSlots, "slots must be in [0, %d]", kMaxSlots);
  LMPK_ARG_CHECK(prm.powers_per_item >= 0 && prm.powers_per_item <= p_m,
                 "powers_per_item must be in [0, p_m]");
  *out = nullptr;
  cudaStream_t st = as_stream(stream);
  int32_t h_nnz = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&h_nnz, row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
  const int32_t S = (n + 31) / 32;
  std::vector<int32_t> width(S);
  int32_t* d_w = nullptr;
  int32_t* d_wmin = nullptr;
  uint8_t* d_fit = nullptr;
  LMPK_TRY(dmalloc(&d_w, std::max(S, 1)));
  LMPK_TRY(dmalloc(&d_wmin, std::max(S, 1)));
  LMPK_TRY(dmalloc(&d_fit, std::max(S, 1)));
  struct Guard {
    int32_t *a, *b;
    uint8_t* c;
    ~Guard() {
      cudaFree(a);
      cudaFree(b);
      cudaFree(c);
    }
  } guard{d_w, d_wmin, d_fit};
  // compressed blocks (int16 column offsets + value dictionary): opt-in via
  // LMPK_FLAG_COMPRESS or LMPK_COMPRESS=1; not with unstaged blocks or x staging
  bool compress = (prm.mode_flags & LMPK_FLAG_COMPRESS) != 0;
  if (const char* e = getenv("LMPK_COMPRESS")) compress = atoi(e) != 0;
  if (prm.mode_flags & LMPK_FLAG_NO_TMA) compress = false;
  std::vector<uint8_t> fit16;
  if (S > 0) {
    k_slice_width<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, n, S, d_w, d_wmin,
                                                               compress ? d_fit : nullptr);
    launch_count_add(ctx, 1);
    LMPK_CHECK_CUDA(cudaMemcpyAsync(width.data(), d_w, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
    if (compress) {
      fit16.resize(S);
      LMPK_CHECK_CUDA(cudaMemcpyAsync(fit16.data(), d_fit, size_t(S), cudaMemcpyDeviceToHost, st));
    }
  }
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  int32_t max_row = 0;
  for (int32_t w : width) max_row = std::max(max_row, w);
  LMPK_ARG_CHECK(max_row <= 65535, "rows longer than 65535 entries are not supported by the tiled kernel");

  const bool want_stream = (prm.mode_flags & LMPK_FLAG_MODE_STREAM) != 0;
  const bool want_res = (prm.mode_flags & LMPK_FLAG_MODE_RESIDENT) != 0;
  LMPK_ARG_CHECK(!(want_stream && want_res), "MODE_STREAM and MODE_RESIDENT are exclusive");
  // candidates (q powers per item, R slots), first feasible wins
  struct Cand {
    int q, slots;
  };
  std::vector<Cand> cands;
  const int R0 = prm.slots > 0 ? prm.slots : 0;
  if (want_res) {
    if (R0)
      cands.push_back({p_m, R0});
    else
      for (int r : {2, 3, 4}) cands.push_back({p_m, r});
  } else if (want_stream || prm.powers_per_item > 0) {
    const int q = prm.powers_per_item > 0 ? prm.powers_per_item : 1;
    cands.push_back({q, R0 ? R0 : 2});
    if (!R0) cands.push_back({q, 3});
  } else {
    // default plan: pure streaming (measured fastest on the cfg2 stencil:
    // 1.07 ms vs 1.46 ms for q = 2 and 1.80 ms fully resident)
    cands.push_back({1, R0 ? R0 : 2});
  }
  lmpk_tiling* T = nullptr;
  int grid = 0, smem = 0, slots = 1, q_used = 1;
  int32_t mfwd = 0, creach = 0;
  int64_t cap_used = 0, xoff_used = 0;
  int static_smem = 0;
  LMPK_TRY(group_static_smem(&static_smem));
  // the driver reserves 1 KB per CTA; the rest of the SM's smem is the budget
  const int64_t per_cta = std::min<int64_t>(ctx->max_smem_sm - 1024 - static_smem,
                                            ctx->max_smem_block - static_smem);
  // LMPK_FLAG_NO_TMA in the tiling's mode flags: blocks are streamed from
  // global memory, so the slots need no shared memory and R is free
  const bool unstaged = (prm.mode_flags & LMPK_FLAG_NO_TMA) != 0;
  // x-segment staging (real-vector tilings, opt-in): a slot is [block | x
  // buffer]; LMPK_XFRAC = percent of the slot for the x buffer (default 0 =
  // off: measured slower on cfg2 -- 1.36 vs 0.99 ms at 25%)
  int xfrac = 0;
  if (const char* e = getenv("LMPK_XFRAC")) xfrac = std::max(0, std::min(60, atoi(e)));
  const bool xstage = !compress && !unstaged && !(prm.mode_flags & LMPK_FLAG_COMPLEX) && xfrac > 0 && n > 0;
  std::vector<int32_t> h_rp, h_col;
  if (xstage) {
    h_rp.resize(size_t(n) + 1);
    h_col.resize(size_t(h_nnz));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(h_rp.data(), row_ptr, (size_t(n) + 1) * 4, cudaMemcpyDeviceToHost, st));
    if (h_nnz > 0)
      LMPK_CHECK_CUDA(cudaMemcpyAsync(h_col.data(), col, size_t(h_nnz) * 4, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  // LMPK_SLOT_KB caps a slot (experiments: smaller slots leave the rest of
  // the SM's unified L1/shared memory to the gathers)
  int64_t slot_cap = INT64_MAX;
  if (const char* e = getenv("LMPK_SLOT_KB")) slot_cap = std::max(4, atoi(e)) * int64_t(1024);
  for (const Cand& cd : cands) {
    const int64_t slot = std::min<int64_t>(unstaged ? per_cta / 2 : per_cta / cd.slots, slot_cap) & ~int64_t(127);
    int64_t xbytes = xstage ? (slot * xfrac / 100) & ~int64_t(127) : 0;
    int64_t cap = slot - xbytes - (xstage ? kMaxSegs * 16 : 0);
    if (prm.tile_nnz_hint > 0 && !compress) cap = std::min<int64_t>(cap, int64_t(prm.tile_nnz_hint) * 12 + 2048);
    const int64_t e_cap = (compress && prm.tile_nnz_hint > 0) ? int64_t(prm.tile_nnz_hint) : INT64_MAX;
    cap &= ~int64_t(127);
    if (cap < 2048) continue;
    const int64_t xoff = xstage ? cap + kMaxSegs * 16 : 0;
    const int smem_need = unstaged ? 0 : static_cast<int>(xstage ? xoff + xbytes : cap * cd.slots / cd.slots);
    int occ = 0;
    LMPK_TRY(group_occupancy(ctx, unstaged ? 0 : smem_need * cd.slots, &occ));
    if (occ < 1) continue;
    lmpk_tiling* cand = new lmpk_tiling();
    cand->ctx = ctx;
    cand->n = n;
    const int rc = build_tiling(ctx, cand, n, row_ptr, col, val, width, d_wmin, cap, xstage ? &h_rp : nullptr,
                                xstage ? &h_col : nullptr, xbytes / 8, compress ? &fit16 : nullptr, e_cap, st);
    if (rc != LMPK_OK) {
      lmpk_tiling_destroy(cand);
      return rc;
    }
    int32_t mf = 0;
    const int32_t cr = chain_reach(cand->h_dep_hi, cd.q - 1, &mf);
    const int g = ctx->sm_count;
    const int64_t G = (p_m + cd.q - 1) / cd.q;
    // the oldest unfinished item needs the next G*(cr+1) queue positions
    // held (q > 1 grabs a ticket only for a free slot)
    const bool ok = (cd.q == 1 || int64_t(g) * cd.slots >= G * (int64_t(cr) + 1) + 1) &&
                    (cd.q == 1 || unstaged || cand->max_block <= cap + (xstage ? kMaxSegs * 16 : 0));
    if (!ok) {
      lmpk_tiling_destroy(cand);
      continue;
    }
    T = cand;
    grid = g;
    smem = unstaged ? 0 : smem_need * cd.slots;
    slots = cd.slots;
    q_used = cd.q;
    mfwd = mf;
    creach = chain_reach(cand->h_dep_hi, p_m - 1, nullptr);
    cap_used = cap;
    xoff_used = xoff;
    break;
  }
  if (!T) {
    set_error("lmpk_tiling_create: no feasible tiling (mode flags 0x%x, powers_per_item %d)", prm.mode_flags,
              prm.powers_per_item);
    return want_res ? LMPK_ERR_UNSUPPORTED : LMPK_ERR_ARG;
  }
  const int32_t nt = T->info.n_tiles;
  if (nt >= (1 << 23)) {
    lmpk_tiling_destroy(T);
    set_error("too many tiles (%d)", nt);
    return LMPK_ERR_UNSUPPORTED;
  }
  T->info.p_m = p_m;
  T->info.mode = q_used == p_m ? 1 : 2;
  T->info.block = 32 * (kConsumers + slots);
  T->slots = slots;
  T->info.smem_bytes = smem;
  T->info.tile_nnz_cap = static_cast<int32_t>(cap_used / 12);
  T->info.max_fwd_reach = mfwd;
  T->info.chain_reach = creach;
  T->info.max_row_nnz = max_row;
  T->info.nnz = h_nnz;
  T->info.grid = grid;
  T->info.powers_per_item = q_used;
  T->info.slots = slots;
  T->xoff = xoff_used;
  T->info.x_staged_tiles = T->staged_tiles;
  // skewed diagonal key (t + g*M, g), M = q*D + slack
  const int32_t G = (p_m + q_used - 1) / q_used;
  // default slack ~1.5 * (items in flight) / G: measured optimum on cfg2
  const int32_t slack = prm.queue_slack > 0 ? prm.queue_slack : std::max(1, (3 * grid * slots) / (2 * G));
  T->info.queue_slack = G > 1 ? slack : 0;
  const int64_t M = int64_t(q_used) * std::max(mfwd, 0) + slack;
  std::vector<int64_t> keys;
  keys.reserve(int64_t(nt) * G);
  for (int32_t t = 0; t < nt; ++t)
    for (int32_t g = 0; g < G; ++g) keys.push_back(((t + g * M) << 8) | g);
  std::vector<int32_t> order(keys.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return keys[a] < keys[b]; });
  std::vector<int32_t> items(order.size());
  for (size_t i = 0; i < order.size(); ++i) {
    const int32_t t = order[i] / G, g = order[i] % G;
    items[i] = (t << 8) | g;
  }
  T->n_items = static_cast<int32_t>(items.size());
  // reverse dependencies for the ready-queue walk (q = 1): u depends on t
  // iff t lies in [dep_lo(u), dep_hi(u)]
  if (q_used == 1) {
    std::vector<int32_t> cnt(nt + 1, 0);
    for (int32_t u = 0; u < nt; ++u)
      for (int32_t t = T->h_dep_lo[u]; t <= T->h_dep_hi[u]; ++t) ++cnt[t + 1];
    for (int32_t t = 0; t < nt; ++t) cnt[t + 1] += cnt[t];
    std::vector<int32_t> rdep(std::max(cnt[nt], 1)), fill(cnt.begin(), cnt.end() - 1);
    for (int32_t u = 0; u < nt; ++u)
      for (int32_t t = T->h_dep_lo[u]; t <= T->h_dep_hi[u]; ++t) rdep[fill[t]++] = u;
    LMPK_TRY(dmalloc(&T->d_rdep_ptr, nt + 1));
    LMPK_TRY(dmalloc(&T->d_rdep, rdep.size()));
    LMPK_TRY(dmalloc(&T->d_rcnt, size_t(p_m) * nt));
    LMPK_TRY(dmalloc(&T->d_rqueue, size_t(p_m) * nt));
    LMPK_TRY(dmalloc(&T->d_rctrl, 128));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_rdep_ptr, cnt.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_rdep, rdep.data(), rdep.size() * 4, cudaMemcpyHostToDevice, st));
  }
  LMPK_TRY(dmalloc(&T->d_items, items.size()));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_items, items.data(), items.size() * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
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

static int launch_group(lmpk_ctx* ctx, MpkParams& Pm, PowerCfgDev& C, bool cplx, bool exact, bool coop,
                        int grid, int smem, cudaStream_t st) {
  void* args[] = {&Pm, &C};
  const void* fn = group_fn(cplx, exact);
  const int block = 32 * (kConsumers + Pm.n_slots);
  // shared-memory carveout: just what the slots need, so the rest of the
  // unified L1 serves the gathers (the driver rounds up to a supported split)
  {
    static int last[4] = {-1, -1, -1, -1};
    const int idx = (cplx ? 2 : 0) + (exact ? 1 : 0);
    int stat = 0;
    LMPK_TRY(group_static_smem(&stat));
    const int per_sm = std::max(1, ctx->max_smem_sm);
    const int pct = std::min(100, int((int64_t(smem + stat + 1024) * 100 + per_sm - 1) / per_sm));
    if (last[idx] != pct) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
      if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("carveout: %s", cudaGetErrorString(e));
        return LMPK_ERR_CUDA;
      }
      last[idx] = pct;
    }
  }
  cudaError_t e = coop ? cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, st)
                       : cudaLaunchKernel(fn, dim3(grid), dim3(block), args, smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("mpk launch failed: %s (grid %d, block %d, smem %d)", cudaGetErrorString(e), grid, block, smem);
    return LMPK_ERR_CUDA;
  }
  launch_count_add(ctx, 1);
  // every slot producer ends its grab sequence with exactly one failing grab
  // (the ready-queue walk does not use the ticket counter)
  if (Pm.mode != 4) ctx->queue_base += uint64_t(Pm.n_items) + uint64_t(grid) * uint64_t(Pm.n_slots);
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
  const bool exact = (flags & LMPK_FLAG_EXACT) != 0;
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
  Pm.y = y;
  Pm.ldy = ldy;
  Pm.acc = use_acc ? acc : y;  // never dereferenced without use_acc
  Pm.use_acc = use_acc ? 1 : 0;
  Pm.progress = Tm->d_progress;
  Pm.queue = reinterpret_cast<unsigned long long*>(ctx->queue_ctr);
  Pm.n_slots = T->slots;
  Pm.smem_cap = T->info.smem_bytes / T->slots;
  Pm.xoff = static_cast<int32_t>(T->xoff);
  Pm.blk_cap = T->xoff > 0 ? Pm.xoff : Pm.smem_cap;
  Pm.tile_nseg = T->d_tile_nseg;
  Pm.tile_xent = T->d_tile_xent;
  Pm.tile_mode = T->d_tile_mode;
  LMPK_ARG_CHECK(!T->d_tile_mode || !(flags & LMPK_FLAG_NO_TMA),
                 "LMPK_FLAG_NO_TMA cannot read a compressed tiling (build it without LMPK_FLAG_COMPRESS)");
  if (T->staged_tiles > 0) {
    LMPK_ARG_CHECK(!cplx, "this tiling stages real x-segments; build it with LMPK_FLAG_COMPLEX in "
                          "mode_flags for complex vectors");
    LMPK_ARG_CHECK(!(flags & LMPK_FLAG_NO_TMA), "LMPK_FLAG_NO_TMA needs a tiling built with LMPK_FLAG_NO_TMA");
    // bulk copies need 16-byte aligned vector slots; otherwise the consumers copy
    const bool aligned = (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (ldy & 1) == 0;
    Pm.xmode = aligned ? 1 : 2;
  }
  Pm.flags = flags;
  Pm.err = ctx->err.dev;
  Pm.prof = ctx->prof;
  Pm.trace = (ctx->prof && ctx->prof_words > 16) ? reinterpret_cast<uint4*>(ctx->prof + 16) : nullptr;
  const int grid = T->info.grid;
  if (sweep) {
    // n_powers back-to-back, dependency-free passes (one launch per power)
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
      Pm.items = nullptr;
      Pm.q = 1;
      Pm.n_powers = 1;
      Pm.n_items = T->info.n_tiles;
      Pm.queue_base = ctx->queue_base;
      Pm.epoch_base = 0;
      LMPK_TRY(launch_group(ctx, Pm, Ci, cplx, exact, false, std::min(grid, T->info.n_tiles),
                            (flags & LMPK_FLAG_NO_TMA) ? 0 : T->info.smem_bytes, st));
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
  Pm.mode = 1;
  Pm.items = T->d_items;
  Pm.q = T->info.powers_per_item;
  Pm.n_items = T->n_items;
  Pm.n_tiles = T->info.n_tiles;
  if (Pm.q == 1 && T->d_rcnt && (flags & LMPK_FLAG_READY_QUEUE)) {
    // ready-queue walk (opt-in; measured slower than the skewed-key walk on
    // cfg2: 1.56 vs 1.02 ms -- exposed TMA and per-item atomics):
    // reset the counters, the queue and its cursors
    Pm.mode = 4;
    Pm.rdep_ptr = T->d_rdep_ptr;
    Pm.rdep = T->d_rdep;
    Pm.rcnt = T->d_rcnt;
    Pm.rqueue = T->d_rqueue;
    Pm.rctrl = T->d_rctrl;
    const size_t nt = size_t(T->info.n_tiles);
    LMPK_CHECK_CUDA(cudaMemsetAsync(T->d_rcnt, 0, size_t(P) * nt * 4, st));
    LMPK_CHECK_CUDA(cudaMemsetAsync(T->d_rqueue, 0xff, size_t(P) * nt * 4, st));
    LMPK_CHECK_CUDA(cudaMemsetAsync(T->d_rctrl, 0, 128 * 4, st));
    Pm.lead = int32_t(std::min<int64_t>(int64_t(T->info.max_fwd_reach) * P + T->info.queue_slack, INT32_MAX / 2));
  }
  // co-residency of all CTAs is part of the deadlock-freedom argument.
  // LMPK_FLAG_NO_TMA: blocks are streamed from global memory by the
  // consumers, so no slot buffers -- the unified L1 is left to the gathers.
  const bool no_tma = (flags & LMPK_FLAG_NO_TMA) != 0;
  return launch_group(ctx, Pm, C, cplx, exact, true, grid, no_tma ? 0 : T->info.smem_bytes, st);
}

// ---------------------------------------------------------------- compute probe
// Each CTA stages tile blockIdx.x once and runs the row kernel `iters` times
// (power 1 into slot 1) with no cross-CTA synchronisation: the attainable
// per-SM rate of the tile kernel itself.
template <bool EXACT, int MODE>
__global__ void k_probe_compute(MpkParams P, PowerCfgDev C, int iters, int n_tiles) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  __shared__ PowTab s_pow[1];
  build_powtab(s_pow, P, C);
  const int32_t t = blockIdx.x % n_tiles;
  const int64_t ofs = P.tile_ofs[t], bytes = P.tile_ofs[t + 1] - ofs;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const bool staged = bytes <= P.smem_cap;
  if (threadIdx.x == 0) {
    if (staged) {
      mbar_arrive_expect_tx(&bar, uint32_t(bytes));
      bulk_g2s(smem_raw, P.blocks + ofs, uint32_t(bytes), &bar, policy_evict_normal());
    } else {
      mbar_arrive_expect_tx(&bar, 0);
    }
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  const int32_t r0 = P.tile_row[t], rows = P.tile_row[t + 1] - r0;
  const uint32_t E = uint32_t(P.tile_E[t]);
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE == 0) {
      if (staged)
        tile_power<false, EXACT, false>(s_pow[0], P.acc, false, SmemBlk{smem_u32(smem_raw)},
                                        GatherGlobal{s_pow[0].yin}, r0, rows, E, 0, wid, nw);
      else
        tile_power<false, EXACT, true>(s_pow[0], P.acc, false, GlbBlk{P.blocks + ofs}, GatherGlobal{s_pow[0].yin},
                                       r0, rows, E, 0, wid, nw);
    } else {
      // MODE 1..3: width-7 full slices only, single-slice path with the
      // gather variant of slice_real_w<..., PROBE = MODE>
      if (!staged) return;
      const SmemBlk B{smem_u32(smem_raw)};
      const int32_t ns = (rows + 31) >> 5;
      const uint32_t col_o = uint32_t(blk_col_off(ns, 0));
      const uint32_t vdelta = col_o + E * 4 - 2 * col_o;
      double* yout = s_pow[0].yout + r0;
      for (int32_t s = wid; s < ns; s += nw) {
        const int2 rec = B.i2(uint32_t(s) * 8);
        if ((rec.y & 0xffff) != 7 || (int(uint32_t(rec.y) >> 16) != 7)) continue;
        const uint32_t cb = uint32_t(rec.x);
        const double v = slice_real_w<7, EXACT, true, SmemBlk, GatherGlobal, MODE>(
            B, cb, 2 * cb + vdelta, uint32_t(lane) * 4, GatherGlobal{s_pow[0].yin}, 7);
        stg_f64(yout + s * 32 + lane, v);
      }
    }
  }
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

// ns per 1000 nonzeros per SM of the tile kernel alone (see k_probe_compute).
// flags: LMPK_FLAG_EXACT selects the separately rounded chain.
extern "C" int lmpk_probe_tile_compute(lmpk_ctx* ctx, const lmpk_tiling* T, double* y, int64_t ldy,
                                       int iters, int threads, int ctas_per_sm, double* ns_per_knnz) {
  LMPK_ARG_CHECK(ctx && T && y && ns_per_knnz, "probe: NULL argument");
  const bool exact = (ctas_per_sm & 0x100) != 0;
  const int mode = (ctas_per_sm >> 12) & 7;
  ctas_per_sm &= 0xff;
  MpkParams Pm;
  memset(&Pm, 0, sizeof(Pm));
  Pm.blocks = T->d_blocks;
  Pm.tile_ofs = T->d_tile_ofs;
  Pm.tile_E = T->d_tile_E;
  Pm.tile_row = T->d_tile_row;
  Pm.y = y;
  Pm.acc = y;
  Pm.ldy = ldy;
  Pm.smem_cap = T->max_block;
  Pm.n_powers = 1;
  PowerCfgDev C;
  memset(&C, 0, sizeof(C));
  C.out_slot[0] = 1;
  C.in_slot[0] = 0;
  const int smem = T->max_block;
  void (*fn)(MpkParams, PowerCfgDev, int, int) = nullptr;
  switch (mode) {
    case 1: fn = exact ? k_probe_compute<true, 1> : k_probe_compute<false, 1>; break;
    case 2: fn = exact ? k_probe_compute<true, 2> : k_probe_compute<false, 2>; break;
    case 3: fn = exact ? k_probe_compute<true, 3> : k_probe_compute<false, 3>; break;
    default: fn = exact ? k_probe_compute<true, 0> : k_probe_compute<false, 0>; break;
  }
  LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->max_smem_block - 1024));
  const int grid = ctx->sm_count * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fn<<<grid, threads, smem>>>(Pm, C, 1, T->info.n_tiles);
  cudaEventRecord(a);
  fn<<<grid, threads, smem>>>(Pm, C, iters, T->info.n_tiles);
  cudaEventRecord(b);
  LMPK_CHECK_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  LMPK_CHECK_CUDA(cudaGetLastError());
  // nnz processed: each CTA one tile per iteration
  const double avg_nnz = double(T->info.nnz) / std::max(1, T->info.n_tiles);
  const double nnz = avg_nnz * grid * iters;
  *ns_per_knnz = (ms * 1e6) * ctx->sm_count / (nnz / 1000.0);
  return LMPK_OK;
}
