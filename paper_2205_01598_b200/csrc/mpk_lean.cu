// mpk_lean.cu -- host side of the lean ring walk (lean_kernel.cuh): the lean
// block builder (width-sorted units, lane-contiguous indices) and the launch.
#include "lean_kernel.cuh"

namespace lmpk {

const void* mpk_lean_fn_r_e(bool vd, bool gen, int np, bool xp);
const void* mpk_lean_fn_r_f(bool vd, bool gen, int np, bool xp);
const void* mpk_lean_fn_c_e(bool vd, int np, bool xp);
const void* mpk_lean_fn_c_f(bool vd, int np, bool xp);
const void* mpk_dp_fn_r_e(bool gen, int np);
const void* mpk_dp_fn_r_f(bool gen, int np);
const void* mpk_dp_fn_c_e(int np);
const void* mpk_dp_fn_c_f(int np);
const void* mpk_xlean_fn_r_e(bool vd, bool gen, bool xp, int ctas);
const void* mpk_xlean_fn_r_f(bool vd, bool gen, bool xp, int ctas);
const void* mpk_xlean_fn_c_e(bool vd, bool xp, int ctas);
const void* mpk_xlean_fn_c_f(bool vd, bool xp, int ctas);

// Sorted-slice descriptor for the fill kernel: global slice, tile, the
// slice's column / value byte offsets inside the tile's lean block (pattern
// slices: the slice's offset in col_off), its pattern count, pattern flag.
struct LeanSliceDesc {
  int32_t s, t, col_off, val_off, np, pat, pad0, pad1;
};

// Lane's Wc entries of slice s in the lean representation: int16 column
// offsets (padding repeats the row's last column -- own row if empty; lanes
// past the tile copy the last valid lane) and dictionary byte codes (vd) or
// raw values.  With x staging (truns != nullptr: the tile's runs, sorted by
// first entry) a column field is (x-buffer entry of the column - lane), and
// empty rows / lanes past the tile point at buffer entry 0.  Returns the row
// length (-1 for lanes past the tile).
__device__ __forceinline__ int lean_entries(const int32_t* row_ptr, const int32_t* col, const double* val,
                                            int32_t s, int32_t r1, int w, int lane, const uint64_t* dict, int nd,
                                            bool vd, int32_t (&off)[8], uint32_t (&code)[8], double (&v)[8],
                                            const int4* truns = nullptr, int nrun = 0) {
  const int wc = lean_wc(w);
  const int32_t r = s * 32 + lane;
  const bool valid = r < r1;
  const int32_t a = valid ? row_ptr[r] : 0;
  const int len = valid ? row_ptr[r + 1] - a : 0;
  int32_t pad = (valid && !truns) ? 0 : -lane;
  for (int j = 0; j < 8; ++j) {
    int32_t o = pad;
    double x = 0.0;
    if (j < len) {
      const int32_t c = col[a + j];
      if (truns) {
        int lo = 0, hi = nrun - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (truns[mid].x <= c)
            lo = mid;
          else
            hi = mid - 1;
        }
        o = truns[lo].z + (c - truns[lo].x) - lane;
      } else {
        o = c - r;
      }
      x = val[a + j];
      pad = o;
    }
    off[j] = (j < w) ? o : 0;
    v[j] = (j < w) ? x : 0.0;
    code[j] = 0;
    if (vd && j < w) {
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
      int lo = 0, hi = nd - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (dict[mid] < bits)
          lo = mid + 1;
        else
          hi = mid;
      }
      code[j] = uint32_t(lo * 8);
    }
  }
  (void)wc;
  return valid ? len : -1;
}

// ---------------------------------------------------------------- x staging plan
// One CTA per tile: the columns the tile's rows read, as runs of whole
// 16-entry granules (16-byte aligned bulk copies), single-granule gaps
// filled.  runs[t * kLeanMaxRuns + i] = {first entry, entries, first buffer
// entry, 0}; xinfo[t] = {runs, staged entries}, or {-1, 0} when the tile's
// column window exceeds the bitmap or needs more than kLeanMaxRuns copies.
// n_even = n rounded up to even: the last run ends there (real vectors: the
// copy stays a multiple of 16 bytes; the launch checks ldy >= n_even).
constexpr int kXGran = 16;
constexpr int kXWords = 1024;  // bitmap words: 32768 granules = 512K columns
constexpr int kXThreads = 256;
__global__ void __launch_bounds__(kXThreads) k_lean_xplan(const int32_t* row_ptr, const int32_t* col,
                                                          const int32_t* tile_row, int32_t nt, int32_t n_even,
                                                          int4* runs, int2* xinfo) {
  __shared__ uint32_t bm[kXWords];
  __shared__ int32_t s_min, s_max;
  __shared__ int32_t sc[3][kXThreads / 32];
  __shared__ int32_t r_start[kLeanMaxRuns], r_rank[kLeanMaxRuns], r_end[kLeanMaxRuns];
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (t >= nt) return;
  const int32_t e0 = row_ptr[tile_row[t]], e1 = row_ptr[tile_row[t + 1]];
  if (tid == 0) s_min = INT32_MAX, s_max = -1;
  for (int i = tid; i < kXWords; i += kXThreads) bm[i] = 0u;
  __syncthreads();
  int32_t mn = INT32_MAX, mx = -1;
  for (int32_t e = e0 + tid; e < e1; e += kXThreads) {
    const int32_t c = col[e];
    mn = min(mn, c);
    mx = max(mx, c);
  }
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    atomicMin(&s_min, mn);
    atomicMax(&s_max, mx);
  }
  __syncthreads();
  if (s_max < 0) {  // no entries: nothing to stage
    if (tid == 0) xinfo[t] = make_int2(0, 0);
    return;
  }
  const int32_t g0 = s_min / kXGran, ng = s_max / kXGran - g0 + 1;
  if (ng > kXWords * 32) {
    if (tid == 0) xinfo[t] = make_int2(-1, 0);
    return;
  }
  for (int32_t e = e0 + tid; e < e1; e += kXThreads) {
    const int32_t g = col[e] / kXGran - g0;
    atomicOr(&bm[g >> 5], 1u << (g & 31));
  }
  __syncthreads();
  // fill single-granule gaps; thread i owns words [4i, 4i + 4)
  uint32_t w[4];
  {
    uint32_t o[6];
    for (int q = 0; q < 6; ++q) {
      const int i = 4 * tid - 1 + q;
      o[q] = (i >= 0 && i < kXWords) ? bm[i] : 0u;
    }
    for (int q = 0; q < 4; ++q) {
      const uint32_t up = (o[q + 1] << 1) | (o[q] >> 31), dn = (o[q + 1] >> 1) | (o[q + 2] << 31);
      w[q] = o[q + 1] | (up & dn);
    }
  }
  __syncthreads();
  for (int q = 0; q < 4; ++q) bm[4 * tid + q] = w[q];
  __syncthreads();
  // per thread: granules, run starts, run ends of its words
  uint32_t st[4], en[4];
  int32_t pc = 0, ns = 0, ne = 0;
  for (int q = 0; q < 4; ++q) {
    const int i = 4 * tid + q;
    const uint32_t prev = i > 0 ? bm[i - 1] >> 31 : 0u, next = i + 1 < kXWords ? bm[i + 1] & 1u : 0u;
    st[q] = w[q] & ~((w[q] << 1) | prev);
    en[q] = w[q] & ~((w[q] >> 1) | (next << 31));
    pc += __popc(w[q]);
    ns += __popc(st[q]);
    ne += __popc(en[q]);
  }
  // block exclusive scan of (pc, ns, ne)
  int32_t v3[3] = {pc, ns, ne}, ex[3], tot[3];
  for (int k = 0; k < 3; ++k) {
    int32_t x = v3[k];
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sc[k][wid] = x;
    ex[k] = x - v3[k];
  }
  __syncthreads();
  for (int k = 0; k < 3; ++k) {
    int32_t base = 0, all = 0;
    for (int j = 0; j < kXThreads / 32; ++j) {
      if (j < wid) base += sc[k][j];
      all += sc[k][j];
    }
    ex[k] += base;
    tot[k] = all;
  }
  const int32_t nrun = tot[1];
  if (nrun > kLeanMaxRuns) {
    if (tid == 0) xinfo[t] = make_int2(-1, 0);
    return;
  }
  int32_t rank = ex[0], si = ex[1], ei = ex[2];
  for (int q = 0; q < 4; ++q) {
    const int32_t gbase = (4 * tid + q) * 32;
    uint32_t m = st[q];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      r_start[si] = gbase + b;
      r_rank[si] = rank + __popc(w[q] & ((1u << b) - 1u));
      ++si;
    }
    m = en[q];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      r_end[ei++] = gbase + b + 1;
    }
    rank += __popc(w[q]);
  }
  __syncthreads();
  if (tid < nrun) {
    const int32_t a = (g0 + r_start[tid]) * kXGran;
    const int32_t b = min((g0 + r_end[tid]) * kXGran, n_even);
    runs[int64_t(t) * kLeanMaxRuns + tid] = make_int4(a, b - a, r_rank[tid] * kXGran, 0);
  }
  if (tid == 0) {
    int32_t total = 0;
    for (int i = 0; i < nrun; ++i) total += min((g0 + r_end[i]) * kXGran, n_even) - (g0 + r_start[i]) * kXGran;
    xinfo[t] = make_int2(nrun, total);
  }
}

// Pattern id of every lane of a slice (exact comparison of the lane's offset
// and code words against every lower lane's); lanes past the tile take the
// last valid lane's pattern.  Returns (pid, pattern count).
__device__ __forceinline__ int2 lean_pattern_ids(const int32_t (&off)[8], const uint32_t (&code)[8], int len,
                                                 int lane) {
  uint32_t wd[6];
#pragma unroll
  for (int q = 0; q < 4; ++q) wd[q] = (uint32_t(off[2 * q]) & 0xffffu) | (uint32_t(off[2 * q + 1]) << 16);
  wd[4] = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
  wd[5] = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
  const uint32_t validm = __ballot_sync(0xffffffffu, len >= 0);
  const int last = 31 - __clz(validm);
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const uint32_t t = __shfl_sync(0xffffffffu, wd[q], last);  // every lane takes part
    if (len < 0) wd[q] = t;
  }
  int first = lane;
  for (int j = 0; j < 32; ++j) {
    bool eq = true;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const uint32_t o = __shfl_sync(0xffffffffu, wd[q], j);  // no short circuit: every lane shuffles
      eq = eq & (o == wd[q]);
    }
    if (eq && j < first) first = j;
  }
  const uint32_t leaders = __ballot_sync(0xffffffffu, first == lane);
  const int pid = __popc(leaders & ((1u << first) - 1u));
  return make_int2(pid, __popc(leaders));
}

// ---------------------------------------------------------------- XP blocks (staged dictionary tilings)
// Record ids of a slice's rows for the XP format: like lean_pattern_ids, but
// lanes past the tile keep their own (entry 0) record instead of copying the
// last valid lane's, so no lane ever addresses outside the x buffer.
__device__ __forceinline__ int2 xp_pattern_ids(const int32_t (&off)[8], const uint32_t (&code)[8], int lane) {
  uint32_t wd[10];
#pragma unroll
  for (int q = 0; q < 8; ++q) wd[q] = uint32_t(off[q]);
  wd[8] = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
  wd[9] = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
  int first = lane;
  for (int j = 0; j < 32; ++j) {
    bool eq = true;
#pragma unroll
    for (int q = 0; q < 10; ++q) {
      const uint32_t o = __shfl_sync(0xffffffffu, wd[q], j);
      eq = eq & (o == wd[q]);
    }
    if (eq && j < first) first = j;
  }
  const uint32_t leaders = __ballot_sync(0xffffffffu, first == lane);
  return make_int2(__popc(leaders & ((1u << first) - 1u)), __popc(leaders));
}

// one warp per slice (natural order): out[s] = {distinct rows, continues}:
// continues = the slice and its predecessor in the same tile are uniform, of
// one width, and every field of this slice is the predecessor's + 32 entries.
__global__ void k_xp_scan(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t S,
                          const int32_t* slice_tile, const int32_t* tile_first, const int32_t* width,
                          const int32_t* tile_row, const int32_t* tile_dict, const int32_t* tile_nd,
                          const uint64_t* dict_tab, const int4* runs, const int2* xinfo, int32_t shift,
                          int2* out) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  const int32_t t = slice_tile[s];
  const int w = width[s];
  const uint64_t* dict = dict_tab + int64_t(tile_dict[t]) * kDictMax;
  const int4* tr = runs ? runs + int64_t(t) * kLeanMaxRuns : nullptr;
  const int nr = runs ? xinfo[t].x : 0;
  int32_t off[8];
  uint32_t code[8];
  double v[8];
  lean_entries(row_ptr, col, val, s, tile_row[t + 1], w, lane, dict, tile_nd[t], true, off, code, v, tr, nr);
  const int2 pp = xp_pattern_ids(off, code, lane);
  int cont = 0;
  if (pp.y == 1 && s > tile_first[t] && width[s - 1] == w) {  // warp-uniform branch
    int32_t off1[8];
    uint32_t code1[8];
    lean_entries(row_ptr, col, val, s - 1, tile_row[t + 1], w, lane, dict, tile_nd[t], true, off1, code1, v, tr, nr);
    const int2 p1 = xp_pattern_ids(off1, code1, lane);
    bool same = p1.y == 1;
    for (int j = 0; j < 8; ++j) same = same && (j >= w || (off[j] == off1[j] + shift && code[j] == code1[j]));
    cont = same ? 1 : 0;
  }
  if (lane == 0) out[s] = make_int2(pp.y, cont);
}

struct XpUnitDesc {
  int32_t s, t, data_off, np, uniform, pad0, pad1, pad2;
};

// one warp per unit: the unit's row records (and ids) from its first slice
__global__ void k_xp_fill(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n_desc,
                          const XpUnitDesc* desc, const int32_t* width, const int32_t* tile_row,
                          const int64_t* lean_ofs, const int32_t* tile_dict, const int32_t* tile_nd,
                          const uint64_t* dict_tab, const int4* runs, const int2* xinfo, int cw,
                          unsigned char* lean) {
  const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_desc) return;
  const XpUnitDesc d = desc[i];
  const int w = width[d.s];
  if (w == 0) return;
  const int wc = lean_wc(w);
  int32_t off[8];
  uint32_t code[8];
  double v[8];
  lean_entries(row_ptr, col, val, d.s, tile_row[d.t + 1], w, lane, dict_tab + int64_t(tile_dict[d.t]) * kDictMax,
               tile_nd[d.t], true, off, code, v, runs ? runs + int64_t(d.t) * kLeanMaxRuns : nullptr,
               runs ? xinfo[d.t].x : 0);
  const int2 pp = xp_pattern_ids(off, code, lane);
  unsigned char* data = lean + lean_ofs[d.t] + d.data_off;
  unsigned char* rec = data;
  bool writer = lane == 0;
  if (!d.uniform) {
    data[lane] = uint8_t(pp.x);
    rec = data + 32 + pp.x * xp_rec_bytes(w);
    writer = lane == __ffs(__match_any_sync(0xffffffffu, pp.x)) - 1;
  }
  if (writer) {
    int32_t* cp = reinterpret_cast<int32_t*>(rec);
    double* vp = reinterpret_cast<double*>(rec + 4 * wc);
    for (int j = 0; j < wc; ++j) {
      cp[j] = j < w ? off[j] * cw : 0;
      vp[j] = j < w ? v[j] : 0.0;
    }
  }
}

// one warp per tile: header {nu, nrows, 2, 0} and the unit records
__global__ void k_xp_head(int32_t nt, const int32_t* tile_row, const int64_t* lean_ofs, const int32_t* rec_ptr,
                          const uint4* recs, const uint8_t* take, const uint16_t* bins, const int32_t* bin_ptr,
                          unsigned char* lean) {
  const int32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nt || !take[t]) return;
  if (lane < kLeanConsumers + 2)
    reinterpret_cast<uint16_t*>(lean + lean_ofs[t] + 16)[lane] = bins[bin_ptr[t] + lane];
  unsigned char* blk = lean + lean_ofs[t];
  const int32_t u0 = rec_ptr[t], nu = rec_ptr[t + 1] - u0;
  if (lane == 0) *reinterpret_cast<int4*>(blk) = make_int4(nu, tile_row[t + 1] - tile_row[t], 2, tile_row[t]);
  for (int u = lane; u < nu; u += 32) reinterpret_cast<uint4*>(blk + kLeanRec)[u] = recs[u0 + u];
}

// pass 1 (dictionary tilings): pattern count of every slice
// (natural slice order: slice i of tile slice_tile[i]); sig_out[i] = the
// slice's dictionary indices (5 bits per entry) when it holds one pattern
__global__ void k_lean_patterns(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n_desc,
                                const int32_t* slice_tile, const int32_t* width, const int32_t* tile_row,
                                const int32_t* tile_dict, const int32_t* tile_nd, const uint64_t* dict_tab,
                                int32_t* np_out, uint64_t* sig_out, const int4* runs, const int2* xinfo) {
  const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_desc) return;
  LeanSliceDesc d{};
  d.s = i;
  d.t = slice_tile[i];
  const int w = width[d.s];
  int32_t off[8];
  uint32_t code[8];
  double v[8];
  const int len = lean_entries(row_ptr, col, val, d.s, tile_row[d.t + 1], w, lane,
                               dict_tab + int64_t(tile_dict[d.t]) * kDictMax, tile_nd[d.t], true, off, code, v,
                               runs ? runs + int64_t(d.t) * kLeanMaxRuns : nullptr, runs ? xinfo[d.t].x : 0);
  const int2 pp = lean_pattern_ids(off, code, len, lane);
  if (lane == 0) {
    np_out[i] = pp.y;
    uint64_t sig = 0;
    for (int j = 0; j < 8; ++j) sig |= uint64_t(code[j] >> 3) << (5 * j);
    sig_out[i] = sig;
  }
}

// one warp per sorted slice: plain lean slices -- lane-contiguous offsets
// (Wc entries) and codes (Wc bytes) or chunked raw values; pattern slices --
// [32 u8 row pattern ids][P x 2Wc B offsets][P x Wc B codes].
__global__ void k_lean_fill(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n_desc,
                            const LeanSliceDesc* desc, const int32_t* width, const int32_t* tile_row,
                            const int64_t* lean_ofs, const int32_t* tile_dict, const int32_t* tile_nd,
                            const uint64_t* dict_tab, int vd, unsigned char* lean, const int4* runs,
                            const int2* xinfo) {
  const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_desc) return;
  const LeanSliceDesc d = desc[i];
  const int w = width[d.s];
  const int wc = lean_wc(w);
  unsigned char* blk = lean + lean_ofs[d.t];
  const uint64_t* dict = vd ? dict_tab + int64_t(tile_dict[d.t]) * kDictMax : nullptr;
  int32_t off[8];
  uint32_t code[8];
  double v[8];
  const int len = lean_entries(row_ptr, col, val, d.s, tile_row[d.t + 1], w, lane, dict, vd ? tile_nd[d.t] : 0,
                               vd != 0, off, code, v, runs ? runs + int64_t(d.t) * kLeanMaxRuns : nullptr,
                               runs ? xinfo[d.t].x : 0);
  if (d.pat) {
    const int2 pp = lean_pattern_ids(off, code, len, lane);
    unsigned char* sl = blk + d.col_off;
    sl[lane] = uint8_t(pp.x);
    const bool leader = lane == __ffs(__match_any_sync(0xffffffffu, pp.x)) - 1;
    if (leader && len >= 0) {
      int16_t* cp = reinterpret_cast<int16_t*>(sl + 32) + pp.x * wc;
      unsigned char* kp = sl + 32 + d.np * 2 * wc + pp.x * wc;
      for (int j = 0; j < wc; ++j) {
        cp[j] = int16_t(off[j]);
        kp[j] = uint8_t(code[j]);
      }
    }
    return;
  }
  int16_t* cp = reinterpret_cast<int16_t*>(blk + d.col_off) + lane * wc;
  for (int j = 0; j < wc; ++j) {
    cp[j] = int16_t(off[j]);
    if (vd)
      blk[d.val_off + lane * wc + j] = uint8_t(code[j]);
    else if (j < w)
      reinterpret_cast<double*>(blk + d.val_off)[chunk_entry(0, w, lane, j)] = v[j];
  }
}

// one warp per tile: header {nu, nrows, vd, 0}, the dictionary (fixed slot
// offset kLeanDict) and the unit records.
__global__ void k_lean_head(int32_t nt, const int32_t* tile_row, const int64_t* lean_ofs, const int32_t* rec_ptr,
                            const uint4* recs, const int32_t* tile_dict, const int32_t* tile_nd,
                            const uint64_t* dict_tab, int vd, unsigned char* lean) {
  const int32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nt) return;
  unsigned char* blk = lean + lean_ofs[t];
  const int32_t u0 = rec_ptr[t], nu = rec_ptr[t + 1] - u0;
  if (lane == 0)
    *reinterpret_cast<int4*>(blk) = make_int4(nu, tile_row[t + 1] - tile_row[t], vd, tile_row[t]);
  uint64_t* dst = reinterpret_cast<uint64_t*>(blk + kLeanDict);
  const int nd = vd ? tile_nd[t] : 0;
  dst[lane] = lane < nd ? dict_tab[int64_t(tile_dict[t]) * kDictMax + lane] : 0ull;
  for (int u = lane; u < nu; u += 32) reinterpret_cast<uint4*>(blk + kLeanRec)[u] = recs[u0 + u];
}

// Value rows of the fast units: a tile whose dictionary holds <= 8 values has
// 24 free dictionary slots; up to three rows of 8 doubles go there, row r =
// the values of index signature vsig[3 t + r] (5 bits per entry), so a fast
// unit reads its seven values as four broadcast LDS.128 instead of a code word
// and seven dictionary lookups.  One warp per tile, after k_lean_head.
__global__ void k_lean_vrows(int32_t nt, const int64_t* lean_ofs, const uint64_t* vsig, unsigned char* lean) {
  const int32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nt || lane >= 24) return;
  const int r = lane >> 3, j = lane & 7;
  const uint64_t sg = vsig[int64_t(t) * 3 + r];
  if (sg == ~0ull) return;
  uint64_t* dict = reinterpret_cast<uint64_t*>(lean + lean_ofs[t] + kLeanDict);
  dict[8 * (1 + r) + j] = dict[(sg >> (5 * j)) & 31u];
}

__global__ void k_rowlen(const int32_t* row_ptr, int32_t n, uint8_t* out) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = uint8_t(min(255, row_ptr[r + 1] - row_ptr[r]));
}

template <typename T>
static int lmalloc(T** p, size_t count) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaMalloc(%zu) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    return LMPK_ERR_NOMEM;
  }
  return LMPK_OK;
}

// Lean block bytes of slices [s0, s1) in the plain lean layout (the tiling
// cost bound: a lean block must fit the slot like the compressed block it
// mirrors; pattern blocks are never larger).
int64_t lean_tile_bytes(const std::vector<int32_t>& width, int32_t s0, int32_t s1, bool vd) {
  int64_t cols = 0, vals = 0;
  for (int32_t s = s0; s < s1; ++s) {
    cols += lean_col_bytes(width[s]);
    vals += vd ? lean_code_bytes(width[s]) : lean_raw_bytes(width[s]);
  }
  const int64_t ns = s1 - s0;
  return (align16(align16(kLeanRec + 16 * ns) + cols) + vals + 127) & ~int64_t(127);
}
static int64_t pattern_slice_bytes(int w, int np) { return w <= 0 ? 0 : align16(32 + int64_t(3) * lean_wc(w) * np); }

// x-staging plan of a tile partition (device tile_row, nt tiles): runs and
// per-tile {runs, entries} into freshly allocated device arrays; *max_entries
// = the largest buffer, or -1 when some tile cannot be staged.
int lean_xplan(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col, const int32_t* d_tile_row,
               int32_t nt, bool cplx, int4** d_runs, int2** d_xinfo, int32_t* max_entries, cudaStream_t st) {
  *d_runs = nullptr;
  *d_xinfo = nullptr;
  *max_entries = -1;
  LMPK_TRY(lmalloc(d_runs, size_t(nt) * kLeanMaxRuns));
  LMPK_TRY(lmalloc(d_xinfo, nt));
  // real vectors: the last run may end at n rounded up to even (16-byte copies)
  k_lean_xplan<<<nt, kXThreads, 0, st>>>(row_ptr, col, d_tile_row, nt, cplx ? n : ((n + 1) & ~1), *d_runs, *d_xinfo);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  std::vector<int2> xi(nt);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(xi.data(), *d_xinfo, size_t(nt) * sizeof(int2), cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  int32_t mx = 0;
  for (int32_t t = 0; t < nt; ++t) {
    if (xi[t].x < 0 || xi[t].y > 32000) {  // int16 column fields hold (entry - lane)
      mx = -1;
      break;
    }
    mx = std::max(mx, xi[t].y);
  }
  *max_entries = mx;
  return LMPK_OK;
}

// Shared memory the staged kernel may use for its ring (static part and the
// driver's reserve left out).
// CTAs per SM of the staged kernel: 1 x 26 consumer warps, or (LMPK_XLEAN_CTAS=2)
// 2 x 12 -- two independent rings per SM
int lean_xs_ctas() {
  const char* e = getenv("LMPK_XLEAN_CTAS");
  return e != nullptr && atoi(e) == 2 ? 2 : 1;
}
int64_t lean_xs_budget(const lmpk_ctx* ctx) {
  if (lean_xs_ctas() == 2) return (int64_t(ctx->max_smem_sm) - 2 * (1024 + 6144)) / 2;
  return int64_t(ctx->max_smem_block) - 6144;
}
// x staging is opt-in (LMPK_XLEAN=1): on the BASELINE shapes the unstaged walk
// over XP blocks measured faster (the shallow ring of [block | x]
// pieces leaves the consumers idle ~40% of the time)
bool lean_xs_wanted() {
  const char* e = getenv("LMPK_XLEAN");
  return e != nullptr && atoi(e) != 0 && getenv("LMPK_NO_XLEAN") == nullptr;
}

// Builds the lean blocks of a compressed tiling whose tiles all have width
// <= 8 and one value format (all dictionary or all raw).  `first` are the
// tiles' first slices; tmode/tdict/d_dict_tab as in build_tiling.  Dictionary
// tiles whose slices repeat few distinct rows (structured grids) store each
// slice's distinct rows once (pattern slices) when that is smaller.
// want_xs: stage the gathered runs of y_{p-1} in shared memory (xlean kernel)
// when every tile's x buffer fits next to its block at ring depth >= 2; the
// column fields then hold buffer entries, so slices whose offsets do not fit
// int16 (plain tiles) are lean tiles too.
int lean_build(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr, const int32_t* col,
               const double* val, const std::vector<int32_t>& first, const std::vector<int32_t>& width,
               const int32_t* d_wmin, const std::vector<int32_t>& tmode, const std::vector<int32_t>& tdict,
               const uint64_t* d_dict_tab, const int32_t* d_width, int64_t cap, bool want_xs, bool cplx,
               cudaStream_t st) {
  const int32_t nt = static_cast<int32_t>(first.size());
  const int32_t S = static_cast<int32_t>(width.size());
  if (nt == 0 || S == 0 || getenv("LMPK_NO_LEAN")) return LMPK_OK;
  for (int32_t s = 0; s < S; ++s)
    if (width[s] > 8) return LMPK_OK;
  PhaseTimer pt(st);
  int vd = -1;
  bool any_plain = false;
  for (int32_t t = 0; t < nt; ++t) {
    if (tmode[t] & kModeLong) return LMPK_OK;
    if (!tmode[t]) any_plain = true;
    const int v = (tmode[t] & kModeDict) ? 1 : 0;
    if (vd >= 0 && v != vd) return LMPK_OK;
    vd = v;
  }
  if (any_plain && !want_xs) return LMPK_OK;
  // ---- x staging plan and feasibility (against the plain lean block bound)
  int4* d_runs = nullptr;
  int2* d_xinfo = nullptr;
  bool xs = false;
  int32_t x_piece = 0;
  if (want_xs) {
    int32_t mx = -1;
    LMPK_TRY(lean_xplan(ctx, n, row_ptr, col, T->d_tile_row, nt, cplx, &d_runs, &d_xinfo, &mx, st));
    if (mx >= 0) {
      int64_t plain_max = 0;
      for (int32_t t = 0; t < nt; ++t)
        plain_max = std::max(plain_max, lean_tile_bytes(width, first[t], t + 1 < nt ? first[t + 1] : S, vd == 1));
      x_piece = int32_t((int64_t(mx) * (cplx ? 16 : 8) + 127) & ~int64_t(127));
      xs = 2 * (((plain_max + 127) & ~int64_t(127)) + x_piece) <= lean_xs_budget(ctx);
    }
    if (!xs) {
      cudaFree(d_runs);
      cudaFree(d_xinfo);
      d_runs = nullptr;
      d_xinfo = nullptr;
      if (any_plain) return LMPK_OK;
    }
  }
  const bool try_pat = vd == 1 && getenv("LMPK_NO_PATTERN") == nullptr;
  std::vector<int32_t> wmin(S);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(wmin.data(), d_wmin, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
  std::vector<int32_t> nd(nt), slice_tile(S);
  for (int32_t t = 0; t < nt; ++t) {
    nd[t] = tmode[t] >> 8;
    for (int32_t s = first[t]; s < (t + 1 < nt ? first[t + 1] : S); ++s) slice_tile[s] = t;
  }
  int32_t *d_tdict = nullptr, *d_nd = nullptr, *d_np = nullptr;
  LeanSliceDesc* d_desc = nullptr;
  LMPK_TRY(tmp_alloc(&d_tdict, nt, st));
  LMPK_TRY(tmp_alloc(&d_nd, nt, st));
  LMPK_TRY(tmp_alloc(&d_desc, S, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_tdict, tdict.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_nd, nd.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
  const int ctas = xs ? lean_xs_ctas() : 1;
  const int nc = ctas == 2 ? kXleanConsumers2 : kLeanConsumers;  // consumer warps per CTA
  // ---- XP blocks (staged dictionary tilings): units = runs of <= 4 slices.
  // A tile takes the XP format when its block stays under xp_limit (tiles of
  // many distinct rows -- grid corners -- keep the compact lean format).
  std::vector<uint8_t> xp_take(nt, 0);
  std::vector<int64_t> xp_bytes(nt, 0);
  std::vector<int32_t> xp_rec_ptr(nt + 1, 0);
  std::vector<uint4> xp_recs;
  std::vector<XpUnitDesc> xp_desc;
  std::vector<uint16_t> xp_bins;  // per XP tile: kLeanConsumers + 2 bin starts (u16)
  std::vector<int32_t> xp_bin_ptr(nt, -1);
  int64_t xp_uniform = 0;
  bool any_xp = false;
  // (unstaged walk: opt-in with LMPK_XP=1 -- its units keep only one slice's
  // gathers in flight and measured slower than the lean pairs)
  if (vd == 1 && !any_plain && getenv("LMPK_NO_XP") == nullptr && (xs || (getenv("LMPK_XP") && atoi(getenv("LMPK_XP"))))) {
    int32_t *d_stile = nullptr, *d_tfirst = nullptr;
    int2* d_scan = nullptr;
    LMPK_TRY(tmp_alloc(&d_stile, S, st));
    LMPK_TRY(tmp_alloc(&d_tfirst, nt, st));
    LMPK_TRY(tmp_alloc(&d_scan, S, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_stile, slice_tile.data(), size_t(S) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_tfirst, first.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
    k_xp_scan<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, val, S, d_stile, d_tfirst, d_width,
                                                            T->d_tile_row, d_tdict, d_nd, d_dict_tab, d_runs,
                                                            d_xinfo, xs ? 32 : 0, d_scan);
    launch_count_add(ctx, 1);
    std::vector<int2> scan(S);
    LMPK_CHECK_CUDA(cudaMemcpyAsync(scan.data(), d_scan, size_t(S) * sizeof(int2), cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    tmp_free(d_stile, st);
    tmp_free(d_tfirst, st);
    tmp_free(d_scan, st);
    int run_max = 4;
    if (const char* e = getenv("LMPK_XP_RUN")) run_max = std::max(1, std::min(8, atoi(e)));
    // staged: the block shares a piece with the x buffer; unstaged: 4 pieces
    // must leave the unified L1 room for the gathers
    int64_t xp_limit = xs ? 16384 : 32768;
    if (const char* e = getenv("LMPK_XP_LIMIT")) xp_limit = std::max(1024, atoi(e));
    xp_recs.reserve(S);
    xp_desc.reserve(S);
    for (int32_t t = 0; t < nt; ++t) {
      const int32_t s0 = first[t], s1 = t + 1 < nt ? first[t + 1] : S;
      xp_rec_ptr[t] = static_cast<int32_t>(xp_recs.size());
      // units first (their count fixes where the data starts), then offsets
      const size_t u0 = xp_recs.size();
      int64_t uni_rows = 0;
      for (int32_t sl = s0; sl < s1;) {
        const int w = width[sl];
        int32_t m = 1;
        const bool uni = scan[sl].x == 1 || w == 0;
        if (uni)
          while (m < run_max && sl + m < s1 && ((w == 0 && width[sl + m] == 0) || (w > 0 && scan[sl + m].y))) ++m;
        bool padded = false;
        for (int32_t q = 0; q < m; ++q) padded = padded || wmin[sl + q] < w;
        uint4 r;
        r.x = 0;
        r.y = uint32_t(sl - s0) | (uint32_t(m) << 16);
        r.z = uint32_t(w) | (uni ? kXpUniform : 0u) | (padded ? kXpPadded : 0u);
        r.w = uint32_t(scan[sl].x);
        xp_recs.push_back(r);
        xp_desc.push_back(XpUnitDesc{sl, t, 0, scan[sl].x, uni ? 1 : 0, 0, 0, 0});
        uni_rows += uni ? m : 0;
        sl += m;
      }
      const int64_t nu = int64_t(xp_recs.size() - u0);
      int64_t off = align16(kLeanRec + 16 * nu);
      for (size_t u = u0; u < xp_recs.size(); ++u) {
        const int w = int(xp_recs[u].z & 15u);
        xp_recs[u].x = uint32_t(off);
        xp_desc[u].data_off = int32_t(off);
        if (w > 0)
          off += (xp_recs[u].z & kXpUniform) ? xp_rec_bytes(w) : align16(32 + int64_t(xp_recs[u].w) * xp_rec_bytes(w));
      }
      const int64_t bytes = (off + 127) & ~int64_t(127);
      if (bytes <= xp_limit) {
        // bins: longest unit first onto the lightest consumer warp
        {
          const size_t cntu = xp_recs.size() - u0;
          std::vector<int32_t> idx(cntu), binof(cntu), load(nc, 0);
          std::iota(idx.begin(), idx.end(), 0);
          auto cost = [&](int32_t i) {
            const uint4& r = xp_recs[u0 + i];
            const int32_t m = int32_t(r.y >> 16);
            return (r.z & kXpUniform) ? 2 + 3 * m : 6;  // record loads + per-slice work
          };
          std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return cost(a) > cost(b); });
          for (int32_t i : idx) {
            int best = 0;
            for (int b = 1; b < nc; ++b)
              if (load[b] < load[best]) best = b;
            binof[i] = best;
            load[best] += cost(i);
          }
          std::vector<uint4> r2;
          std::vector<XpUnitDesc> d2;
          std::vector<uint16_t> starts(kLeanConsumers + 2, 0);
          for (int b = 0; b < nc; ++b) {
            starts[b] = uint16_t(r2.size());
            for (size_t i = 0; i < cntu; ++i)
              if (binof[i] == b) {
                r2.push_back(xp_recs[u0 + i]);
                d2.push_back(xp_desc[u0 + i]);
              }
          }
          for (int b = nc; b < kLeanConsumers + 2; ++b) starts[b] = uint16_t(r2.size());
          std::copy(r2.begin(), r2.end(), xp_recs.begin() + u0);
          std::copy(d2.begin(), d2.end(), xp_desc.begin() + u0);
          xp_bins.insert(xp_bins.end(), starts.begin(), starts.end());
        }
        xp_take[t] = 1;
        xp_bin_ptr[t] = int32_t(xp_bins.size()) - (kLeanConsumers + 2);
        xp_bytes[t] = bytes;
        xp_uniform += uni_rows;
        any_xp = true;
      } else {  // the tile keeps the lean format: drop its XP units
        xp_recs.resize(u0);
        xp_desc.resize(u0);
      }
    }
    xp_rec_ptr[nt] = static_cast<int32_t>(xp_recs.size());
  }
  // pass 1: pattern counts per slice (natural slice order)
  std::vector<int32_t> np(S, 32);
  std::vector<uint64_t> sig(S, 0);  // dictionary indices of one-pattern slices (same-value pairs)
  const bool no_sameval = getenv("LMPK_NO_SAMEVAL") != nullptr;  // A/B switches (tools/sameval_ab.py)
  const bool no_fast = getenv("LMPK_NO_FAST") != nullptr;
  const bool no_vrow = getenv("LMPK_NO_VROW") != nullptr;
  std::vector<uint64_t> vsig(size_t(nt) * 3, ~0ull);
  if (try_pat) {
    int32_t* d_st = nullptr;
    uint64_t* d_sig = nullptr;
    LMPK_TRY(tmp_alloc(&d_np, S, st));
    LMPK_TRY(tmp_alloc(&d_st, S, st));
    LMPK_TRY(tmp_alloc(&d_sig, S, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_st, slice_tile.data(), size_t(S) * 4, cudaMemcpyHostToDevice, st));
    k_lean_patterns<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, val, S, d_st, d_width,
                                                                  T->d_tile_row, d_tdict, d_nd, d_dict_tab, d_np, d_sig,
                                                                  d_runs, d_xinfo);
    launch_count_add(ctx, 1);
    LMPK_CHECK_CUDA(cudaMemcpyAsync(np.data(), d_np, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(sig.data(), d_sig, size_t(S) * 8, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    tmp_free(d_st, st);
    tmp_free(d_sig, st);
  }
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  pt.mark("  lean: plan + pattern pass");
  std::vector<int64_t> ofs(nt + 1, 0);
  std::vector<int32_t> rec_ptr(nt + 1, 0);
  std::vector<uint4> recs;
  std::vector<LeanSliceDesc> desc;
  desc.reserve(S);
  recs.reserve(S);
  std::vector<int32_t> order;
  int64_t max_bytes = 0;
  int32_t n_pat = 0;
  // staged tiles: same-width slices pair up only when that still leaves every
  // consumer warp a unit (shared-memory gathers need no second slice in flight)
  int pair_min = 0;
  if (xs) {
    pair_min = 2 * nc;
    if (const char* e = getenv("LMPK_XLEAN_PAIR")) pair_min = atoi(e) ? 0 : INT32_MAX;
  }
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t s0 = first[t], s1 = t + 1 < nt ? first[t + 1] : S;
    if (xp_take[t]) {  // XP tile: its block is written by k_xp_fill / k_xp_head below
      rec_ptr[t] = static_cast<int32_t>(recs.size());
      max_bytes = std::max(max_bytes, xp_bytes[t]);
      ofs[t + 1] = ofs[t] + xp_bytes[t];
      continue;
    }
    // width classes 0..8, full slices first inside a class (counting sort)
    const int32_t ns = s1 - s0;
    {
      int32_t cnt[19] = {0};
      for (int32_t s = s0; s < s1; ++s) ++cnt[2 * width[s] + (wmin[s] < width[s] ? 1 : 0) + 1];
      for (int q = 0; q < 18; ++q) cnt[q + 1] += cnt[q];
      order.resize(ns);
      for (int32_t s = s0; s < s1; ++s) order[cnt[2 * width[s] + (wmin[s] < width[s] ? 1 : 0)]++] = s;
    }
    const bool pairing = ns >= pair_min;
    int32_t nu = 0;
    for (int32_t i = 0; i < ns;) {
      const bool pair = pairing && i + 1 < ns && width[order[i + 1]] == width[order[i]];
      ++nu;
      i += pair ? 2 : 1;
    }
    const int64_t plain_bytes = lean_tile_bytes(width, s0, s1, vd == 1);
    int64_t pat_bytes = INT64_MAX;
    if (try_pat) {
      pat_bytes = align16(kLeanRec + 16 * int64_t(nu));
      for (int32_t s = s0; s < s1; ++s) pat_bytes += pattern_slice_bytes(width[s], np[s]);
      pat_bytes = (pat_bytes + 127) & ~int64_t(127);
    }
    const bool pat = pat_bytes < plain_bytes;
    const int64_t bytes = pat ? pat_bytes : plain_bytes;
    if (bytes > cap) return LMPK_OK;  // cannot happen with the lean-aware tiling cost
    n_pat += pat ? 1 : 0;
    max_bytes = std::max(max_bytes, bytes);
    std::vector<int32_t> c_of(ns), v_of(ns);
    int64_t co = align16(kLeanRec + 16 * int64_t(nu));
    if (pat) {
      for (int32_t i = 0; i < ns; ++i) {
        const int w = width[order[i]];
        c_of[i] = int32_t(co);
        v_of[i] = 0;
        desc.push_back(LeanSliceDesc{order[i], t, int32_t(co), 0, np[order[i]], 1, 0, 0});
        co += pattern_slice_bytes(w, np[order[i]]);
      }
    } else {
      int64_t cols = 0;
      for (int32_t s = s0; s < s1; ++s) cols += lean_col_bytes(width[s]);
      int64_t vo = align16(co + cols);
      for (int32_t i = 0; i < ns; ++i) {
        const int w = width[order[i]];
        c_of[i] = int32_t(co);
        v_of[i] = int32_t(vo);
        desc.push_back(LeanSliceDesc{order[i], t, int32_t(co), int32_t(vo), 0, 0, 0, 0});
        co += lean_col_bytes(w);
        vo += vd ? lean_code_bytes(w) : lean_raw_bytes(w);
      }
    }
    rec_ptr[t] = static_cast<int32_t>(recs.size());
    uint64_t trow[3] = {~0ull, ~0ull, ~0ull};  // value rows of this tile (k_lean_vrows)
    const bool vrow_ok = pat && nd[t] <= 8 && !no_vrow;
    for (int32_t i = 0; i < ns;) {
      const int32_t sa = order[i];
      const bool pair = pairing && i + 1 < ns && width[order[i + 1]] == width[sa];
      const int32_t sb = pair ? order[i + 1] : sa;
      const int w = width[sa];
      const bool padded = wmin[sa] < w || (pair && wmin[sb] < w);
      uint4 r;
      r.x = uint32_t(c_of[i]);
      r.y = pat ? uint32_t(pair ? c_of[i + 1] : 0) : uint32_t(v_of[i]);
      r.z = uint32_t(w) | (pair ? kLeanPair : 0u) | (padded ? kLeanPadded : 0u);
      if (pat && w > 0) {
        r.z |= kLeanPattern | (uint32_t(np[sa]) << 16) | (uint32_t(pair ? np[sb] : 0) << 24);
        // both slices one pattern with the same dictionary indices: the values are read once
        if (pair && np[sa] == 1 && np[sb] == 1 && sig[sa] == sig[sb] && !no_sameval) {
          r.z |= kLeanSameVal;
          // both slices full (only the matrix's last slice can be partial) and unpadded: fast unit
          if (!padded && !xs && (int64_t(sa) + 1) * 32 <= n && (int64_t(sb) + 1) * 32 <= n && !no_fast) {
            r.z |= kLeanFast;
            if (vrow_ok) {  // the pair's values as a row of the tile's value table
              int q = 0;
              while (q < 3 && trow[q] != ~0ull && trow[q] != sig[sa]) ++q;
              if (q < 3) {
                trow[q] = sig[sa];
                r.z |= kLeanVRow | (uint32_t(q) << 13);
              }
            }
          }
        }
      }
      r.w = uint32_t(sa - s0) | (uint32_t(sb - s0) << 16);
      recs.push_back(r);
      i += pair ? 2 : 1;
    }
    vsig[size_t(t) * 3] = trow[0], vsig[size_t(t) * 3 + 1] = trow[1], vsig[size_t(t) * 3 + 2] = trow[2];
    ofs[t + 1] = ofs[t] + bytes;
  }
  rec_ptr[nt] = static_cast<int32_t>(recs.size());
  pt.mark("  lean: host units");
  const int64_t total = ofs[nt];
  int64_t* d_ofs = nullptr;
  unsigned char* d_lean = nullptr;
  uint8_t* d_rowlen = nullptr;
  int32_t* d_rec_ptr = nullptr;
  uint4* d_recs = nullptr;
  LMPK_TRY(lmalloc(&d_ofs, nt + 1));
  LMPK_TRY(lmalloc(&d_lean, size_t(total)));
  LMPK_TRY(lmalloc(&d_rowlen, size_t(std::max(n, 1))));
  LMPK_TRY(tmp_alloc(&d_rec_ptr, nt + 1, st));
  LMPK_TRY(tmp_alloc(&d_recs, recs.size(), st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_lean, 0, size_t(total), st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_ofs, ofs.data(), size_t(nt + 1) * 8, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_rec_ptr, rec_ptr.data(), size_t(nt + 1) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_recs, recs.data(), recs.size() * 16, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_desc, desc.data(), desc.size() * sizeof(LeanSliceDesc), cudaMemcpyHostToDevice,
                                  st));
  const int32_t nds = static_cast<int32_t>(desc.size());
  if (nds > 0)
    k_lean_fill<<<div_up(int64_t(nds) * 32, 256), 256, 0, st>>>(row_ptr, col, val, nds, d_desc, d_width,
                                                                T->d_tile_row, d_ofs, d_tdict, d_nd, d_dict_tab, vd,
                                                                d_lean, d_runs, d_xinfo);
  k_lean_head<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(nt, T->d_tile_row, d_ofs, d_rec_ptr, d_recs, d_tdict,
                                                             d_nd, d_dict_tab, vd, d_lean);
  k_rowlen<<<div_up(std::max(n, 1), 256), 256, 0, st>>>(row_ptr, n, d_rowlen);
  uint64_t* d_vsig = nullptr;
  if (vd == 1) {
    LMPK_TRY(tmp_alloc(&d_vsig, vsig.size(), st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_vsig, vsig.data(), vsig.size() * 8, cudaMemcpyHostToDevice, st));
    k_lean_vrows<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(nt, d_ofs, d_vsig, d_lean);
    launch_count_add(ctx, 1);
  }
  launch_count_add(ctx, 3);
  LMPK_CHECK_CUDA(cudaGetLastError());
  int32_t* d_xrec_ptr = nullptr;
  uint4* d_xrecs = nullptr;
  XpUnitDesc* d_udesc = nullptr;
  uint8_t* d_take = nullptr;
  uint16_t* d_bins = nullptr;
  int32_t* d_bin_ptr = nullptr;
  if (any_xp) {
    LMPK_TRY(tmp_alloc(&d_xrec_ptr, nt + 1, st));
    LMPK_TRY(tmp_alloc(&d_xrecs, xp_recs.size(), st));
    LMPK_TRY(tmp_alloc(&d_udesc, xp_desc.size(), st));
    LMPK_TRY(tmp_alloc(&d_take, nt, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_xrec_ptr, xp_rec_ptr.data(), size_t(nt + 1) * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_xrecs, xp_recs.data(), xp_recs.size() * 16, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_udesc, xp_desc.data(), xp_desc.size() * sizeof(XpUnitDesc),
                                    cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_take, xp_take.data(), size_t(nt), cudaMemcpyHostToDevice, st));
    const int32_t nxu = static_cast<int32_t>(xp_desc.size());
    if (nxu > 0)
      k_xp_fill<<<div_up(int64_t(nxu) * 32, 256), 256, 0, st>>>(row_ptr, col, val, nxu, d_udesc, d_width,
                                                              T->d_tile_row, d_ofs, d_tdict, d_nd, d_dict_tab,
                                                              d_runs, d_xinfo, cplx ? 16 : 8, d_lean);
    LMPK_TRY(tmp_alloc(&d_bins, xp_bins.size(), st));
    LMPK_TRY(tmp_alloc(&d_bin_ptr, nt, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_bins, xp_bins.data(), xp_bins.size() * 2, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_bin_ptr, xp_bin_ptr.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
    k_xp_head<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(nt, T->d_tile_row, d_ofs, d_xrec_ptr, d_xrecs, d_take,
                                                             d_bins, d_bin_ptr, d_lean);
    launch_count_add(ctx, 2);
    LMPK_CHECK_CUDA(cudaGetLastError());
  }
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  tmp_free(d_xrec_ptr, st);
  tmp_free(d_xrecs, st);
  tmp_free(d_udesc, st);
  tmp_free(d_take, st);
  tmp_free(d_bins, st);
  tmp_free(d_bin_ptr, st);
  tmp_free(d_vsig, st);
  tmp_free(d_rec_ptr, st);
  tmp_free(d_recs, st);
  tmp_free(d_desc, st);
  tmp_free(d_tdict, st);
  tmp_free(d_nd, st);
  tmp_free(d_np, st);
  pt.mark("  lean: alloc + fill + frees");
  T->d_lean = d_lean;
  T->d_lean_ofs = d_ofs;
  T->d_rowlen = d_rowlen;
  T->lean_vd = vd;
  T->lean_bytes = total;
  T->h_lean_ofs = ofs;
  T->lean_piece = static_cast<int32_t>((max_bytes + 127) & ~int64_t(127));
  T->info.lean_bytes = total;
  T->info.lean_pattern_tiles = n_pat;
  T->lean_xp = any_xp ? 1 : 0;
  if (any_xp) T->info.lean_pattern_tiles = static_cast<int32_t>(xp_uniform);
  T->info.lean_xstaged = any_xp ? 3 : 0;  // 3: XP blocks, gathers from global memory
  if (xs) {
    T->lean_xs = 1;
    T->lean_cplx = cplx ? 1 : 0;
    T->lean_xoff = T->lean_piece;
    T->lean_piece += x_piece;
    int np_ring = int(std::min<int64_t>(kXleanRingMax, lean_xs_budget(ctx) / T->lean_piece));
    if (const char* e = getenv("LMPK_XLEAN_NP")) np_ring = std::max(2, std::min(np_ring, atoi(e)));
    T->lean_np = np_ring;
    T->lean_ctas = ctas;
    T->d_lean_runs = d_runs;
    T->d_lean_xinfo = d_xinfo;
    T->h_lean_xinfo.resize(nt);
    LMPK_CHECK_CUDA(cudaMemcpy(T->h_lean_xinfo.data(), d_xinfo, size_t(nt) * sizeof(int2), cudaMemcpyDeviceToHost));
    T->lean_xp = any_xp ? 1 : 0;
    if (any_xp) T->info.lean_pattern_tiles = static_cast<int32_t>(xp_uniform);
    T->info.lean_xstaged = any_xp ? 2 : 1;
    T->info.lean_ring = np_ring;
    T->info.lean_piece = T->lean_piece;
  }
  return LMPK_OK;
}

// Static work lists of the staged kernel: item i of the queue (key order)
// belongs to CTA i mod grid; a CTA's list holds one 32-byte record per piece
//   {tile, power | first-piece flag << 8, dep lo, dep hi}
//   {block offset lo, hi, block bytes, runs | staged entries << 8}
// so its producer streams the list with coalesced loads (32 pieces per round
// trip) instead of a ticket atomic and four dependent loads per item.
int lean_worklist(lmpk_tiling* T, const std::vector<int32_t>& items, const std::vector<int32_t>& st_first,
                  const std::vector<int32_t>& lo, const std::vector<int32_t>& hi, int grid, cudaStream_t st) {
  if (!T->lean_xs || grid < 1 || getenv("LMPK_NO_WORKLIST")) return LMPK_OK;
  std::vector<std::vector<int4>> lists(grid);
  for (size_t i = 0; i < items.size(); ++i) {
    const int32_t sup = items[i] >> 8, p = (items[i] & 255) + 1;
    std::vector<int4>& l = lists[i % size_t(grid)];
    for (int32_t m = st_first[sup]; m < st_first[sup + 1]; ++m) {
      const int64_t o = T->h_lean_ofs[m], bytes = T->h_lean_ofs[m + 1] - o;
      const int2 xi = T->h_lean_xinfo[m];
      l.push_back(make_int4(m, p | (m == st_first[sup] ? 256 : 0), lo[sup], hi[sup]));
      l.push_back(make_int4(int32_t(uint32_t(o & 0xffffffffll)), int32_t(o >> 32), int32_t(bytes),
                            xi.x | (xi.y << 8)));
    }
  }
  std::vector<int32_t> ptr(grid + 1, 0);
  std::vector<int4> flat;
  for (int c = 0; c < grid; ++c) {
    ptr[c + 1] = ptr[c] + int32_t(lists[c].size() / 2);
    flat.insert(flat.end(), lists[c].begin(), lists[c].end());
  }
  LMPK_TRY(lmalloc(&T->d_lean_wl, flat.size()));
  LMPK_TRY(lmalloc(&T->d_lean_wl_ptr, grid + 1));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_lean_wl, flat.data(), flat.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_lean_wl_ptr, ptr.data(), size_t(grid + 1) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  T->lean_wl_grid = grid;
  return LMPK_OK;
}

void lean_free(lmpk_tiling* T) {
  cudaFree(T->d_lean_wl);
  cudaFree(T->d_lean_wl_ptr);
  T->d_lean_wl = nullptr;
  T->d_lean_wl_ptr = nullptr;
  T->lean_wl_grid = 0;
  cudaFree(T->d_lean);
  cudaFree(T->d_lean_ofs);
  cudaFree(T->d_rowlen);
  cudaFree(T->d_lean_runs);
  cudaFree(T->d_lean_xinfo);
  T->d_lean_runs = nullptr;
  T->d_lean_xinfo = nullptr;
  T->lean_xs = 0;
  T->lean_xp = 0;
  T->d_lean = nullptr;
  T->d_lean_ofs = nullptr;
  T->d_rowlen = nullptr;
  T->lean_vd = -1;
}

// Whether the staged kernel can run on these vectors: bulk copies need
// 16-byte aligned runs (real vectors: an even slot stride that also covers the
// rounded-up last run) and the x buffer was sized for real or complex entries.
bool lean_xs_runnable(const lmpk_tiling* T, const double* y, int64_t ldy, bool cplx) {
  if (!T->lean_xs) return true;
  if ((T->lean_cplx != 0) != cplx) return false;
  if (reinterpret_cast<uintptr_t>(y) % 16 != 0 || (ldy & 1)) return false;
  if (!cplx && ldy < ((int64_t(T->n) + 1) & ~int64_t(1))) return false;
  return true;
}

// Launch of the lean kernel for a ring tiling with lean blocks (same
// MpkParams as launch_ring; smem = the ring's pieces).
int launch_lean(lmpk_ctx* ctx, const lmpk_tiling* T, MpkParams& Pm, PowerCfgDev& C, bool cplx, bool exact, bool gen,
                int grid, cudaStream_t st) {
  const int ctas = T->lean_xs ? std::max(1, T->lean_ctas) : 1;
  grid *= ctas;
  const bool wl = T->lean_xs && T->lean_wl_grid == grid;
  LeanParams L{T->d_lean,    T->d_lean_ofs, T->d_rowlen, T->d_lean_runs,
               T->d_lean_xinfo, T->lean_xoff, T->lean_np, wl ? T->d_lean_wl : nullptr,
               wl ? T->d_lean_wl_ptr : nullptr, 1};
  if (const char* e = getenv("LMPK_XLEAN_PUB")) L.pub_batch = std::max(1, std::min(8, atoi(e)));
  void* args[] = {&Pm, &C, &L};
  const bool vd = T->lean_vd == 1;
  // ring depth: 4 pieces when the lean blocks are small (pattern tiles), so
  // the producer runs further ahead of dependency waits; the pieces hold the
  // largest lean block and the rest of the unified L1/shared memory caches
  // the gathers
  const int piece = T->lean_piece > 0 ? T->lean_piece : T->piece;
  int np = (4 * int64_t(piece) + 8192 <= ctx->max_smem_block) ? 4 : 2;
  if (const char* e = getenv("LMPK_LEAN_NP")) np = atoi(e) == 4 && 4 * int64_t(piece) + 8192 <= ctx->max_smem_block ? 4 : 2;
  const void* fn;
  if (T->lean_vd == 2) {  // DP blocks (diagonal-private dictionary)
    // pieces beyond 32 KB run a ring of 2: four would leave the gathers no L1
    // (cfg5, 48 KB pieces: 2.40 vs 2.59 ms per step)
    if (piece > 32 * 1024 && getenv("LMPK_LEAN_NP") == nullptr) np = 2;
    fn = cplx ? (exact ? mpk_dp_fn_c_e(np) : mpk_dp_fn_c_f(np)) : (exact ? mpk_dp_fn_r_e(gen, np) : mpk_dp_fn_r_f(gen, np));
  } else if (T->lean_xs) {
    np = T->lean_np;
    const bool xp = T->lean_xp != 0;
    fn = cplx ? (exact ? mpk_xlean_fn_c_e(vd, xp, ctas) : mpk_xlean_fn_c_f(vd, xp, ctas))
              : (exact ? mpk_xlean_fn_r_e(vd, gen, xp, ctas) : mpk_xlean_fn_r_f(vd, gen, xp, ctas));
  } else {
    const bool xp = T->lean_xp != 0;
    fn = cplx ? (exact ? mpk_lean_fn_c_e(vd, np, xp) : mpk_lean_fn_c_f(vd, np, xp))
              : (exact ? mpk_lean_fn_r_e(vd, gen, np, xp) : mpk_lean_fn_r_f(vd, gen, np, xp));
  }
  const int smem = np * piece;
  {
    static const void* seen[64];
    static int nseen = 0;
    bool known = false;
    for (int i = 0; i < nseen; ++i) known = known || seen[i] == fn;
    if (!known) {
      cudaFuncAttributes fa;
      LMPK_CHECK_CUDA(cudaFuncGetAttributes(&fa, fn));
      LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes)));
      if (nseen < 64) seen[nseen++] = fn;
    }
    // carveout: just what the pieces need, the rest of the unified
    // L1/shared memory caches the gathers (staged kernel: the y_{p-2} / acc
    // reads and the stores)
    cudaFuncAttributes fa;
    LMPK_CHECK_CUDA(cudaFuncGetAttributes(&fa, fn));
    const int per_sm = std::max(1, ctx->max_smem_sm);
    int pct = std::min(100, int((int64_t(smem + int(fa.sharedSizeBytes) + 1024) * ctas * 100 + per_sm - 1) / per_sm));
    if (const char* e = getenv("LMPK_LEAN_CARVE")) pct = std::max(0, std::min(100, atoi(e)));
    LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  }
  Pm.smem_cap = piece;
  const int nthreads = 32 * ((ctas == 2 ? kXleanConsumers2 : kLeanConsumers) + 2);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(nthreads), args, smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("mpk lean launch failed: %s (grid %d, smem %d)", cudaGetErrorString(e), grid, smem);
    return LMPK_ERR_CUDA;
  }
  launch_count_add(ctx, 1);
  ctx->queue_base += uint64_t(Pm.n_items) + uint64_t(grid);
  return LMPK_OK;
}

}  // namespace lmpk
