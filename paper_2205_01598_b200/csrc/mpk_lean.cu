// mpk_lean.cu -- host side of the lean ring walk (lean_kernel.cuh): the lean
// block builder (width-sorted units, lane-contiguous indices) and the launch.
#include "lean_kernel.cuh"

namespace lmpk {

const void* mpk_lean_fn_r_e(bool vd, bool gen, int np);
const void* mpk_lean_fn_r_f(bool vd, bool gen, int np);
const void* mpk_lean_fn_c_e(bool vd, int np);
const void* mpk_lean_fn_c_f(bool vd, int np);

// Sorted-slice descriptor for the fill kernel: global slice, tile, the
// slice's column / value byte offsets inside the tile's lean block (pattern
// slices: the slice's offset in col_off), its pattern count, pattern flag.
struct LeanSliceDesc {
  int32_t s, t, col_off, val_off, np, pat, pad0, pad1;
};

// Lane's Wc entries of slice s in the lean representation: int16 column
// offsets (padding repeats the row's last column -- own row if empty; lanes
// past the tile copy the last valid lane) and dictionary byte codes (vd) or
// raw values.  Returns the row length (-1 for lanes past the tile).
__device__ __forceinline__ int lean_entries(const int32_t* row_ptr, const int32_t* col, const double* val,
                                            int32_t s, int32_t r1, int w, int lane, const uint64_t* dict, int nd,
                                            bool vd, int32_t (&off)[8], uint32_t (&code)[8], double (&v)[8]) {
  const int wc = lean_wc(w);
  const int32_t r = s * 32 + lane;
  const bool valid = r < r1;
  const int32_t a = valid ? row_ptr[r] : 0;
  const int len = valid ? row_ptr[r + 1] - a : 0;
  int32_t pad = valid ? 0 : -lane;
  for (int j = 0; j < 8; ++j) {
    int32_t o = pad;
    double x = 0.0;
    if (j < len) {
      o = col[a + j] - r;
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

// pass 1 (dictionary tilings): pattern count of every slice
__global__ void k_lean_patterns(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n_desc,
                                const LeanSliceDesc* desc, const int32_t* width, const int32_t* tile_row,
                                const int32_t* tile_dict, const int32_t* tile_nd, const uint64_t* dict_tab,
                                int32_t* np_out) {
  const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_desc) return;
  const LeanSliceDesc d = desc[i];
  const int w = width[d.s];
  int32_t off[8];
  uint32_t code[8];
  double v[8];
  const int len = lean_entries(row_ptr, col, val, d.s, tile_row[d.t + 1], w, lane,
                               dict_tab + int64_t(tile_dict[d.t]) * kDictMax, tile_nd[d.t], true, off, code, v);
  const int2 pp = lean_pattern_ids(off, code, len, lane);
  if (lane == 0) np_out[i] = pp.y;
}

// one warp per sorted slice: plain lean slices -- lane-contiguous offsets
// (Wc entries) and codes (Wc bytes) or chunked raw values; pattern slices --
// [32 u8 row pattern ids][P x 2Wc B offsets][P x Wc B codes].
__global__ void k_lean_fill(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n_desc,
                            const LeanSliceDesc* desc, const int32_t* width, const int32_t* tile_row,
                            const int64_t* lean_ofs, const int32_t* tile_dict, const int32_t* tile_nd,
                            const uint64_t* dict_tab, int vd, unsigned char* lean) {
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
                               vd != 0, off, code, v);
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
    *reinterpret_cast<int4*>(blk) = make_int4(nu, tile_row[t + 1] - tile_row[t], vd, 0);
  uint64_t* dst = reinterpret_cast<uint64_t*>(blk + kLeanDict);
  const int nd = vd ? tile_nd[t] : 0;
  dst[lane] = lane < nd ? dict_tab[int64_t(tile_dict[t]) * kDictMax + lane] : 0ull;
  for (int u = lane; u < nu; u += 32) reinterpret_cast<uint4*>(blk + kLeanRec)[u] = recs[u0 + u];
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

// Builds the lean blocks of a compressed tiling whose tiles all have width
// <= 8 and one value format (all dictionary or all raw).  `first` are the
// tiles' first slices; tmode/tdict/d_dict_tab as in build_tiling.  Dictionary
// tiles whose slices repeat few distinct rows (structured grids) store each
// slice's distinct rows once (pattern slices) when that is smaller.
int lean_build(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr, const int32_t* col,
               const double* val, const std::vector<int32_t>& first, const std::vector<int32_t>& width,
               const int32_t* d_wmin, const std::vector<int32_t>& tmode, const std::vector<int32_t>& tdict,
               const uint64_t* d_dict_tab, const int32_t* d_width, int64_t cap, cudaStream_t st) {
  const int32_t nt = static_cast<int32_t>(first.size());
  const int32_t S = static_cast<int32_t>(width.size());
  if (nt == 0 || S == 0 || getenv("LMPK_NO_LEAN")) return LMPK_OK;
  int vd = -1;
  for (int32_t t = 0; t < nt; ++t) {
    if (!tmode[t] || (tmode[t] & kModeLong)) return LMPK_OK;
    const int v = (tmode[t] & kModeDict) ? 1 : 0;
    if (vd >= 0 && v != vd) return LMPK_OK;
    vd = v;
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
  LMPK_TRY(lmalloc(&d_tdict, nt));
  LMPK_TRY(lmalloc(&d_nd, nt));
  LMPK_TRY(lmalloc(&d_desc, S));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_tdict, tdict.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_nd, nd.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
  // pass 1: pattern counts per slice (natural slice order)
  std::vector<int32_t> np(S, 32);
  if (try_pat) {
    std::vector<LeanSliceDesc> nat(S);
    for (int32_t s = 0; s < S; ++s) nat[s] = LeanSliceDesc{s, slice_tile[s], 0, 0, 0, 0, 0, 0};
    LMPK_TRY(lmalloc(&d_np, S));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_desc, nat.data(), size_t(S) * sizeof(LeanSliceDesc), cudaMemcpyHostToDevice, st));
    k_lean_patterns<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, val, S, d_desc, d_width,
                                                                  T->d_tile_row, d_tdict, d_nd, d_dict_tab, d_np);
    launch_count_add(ctx, 1);
    LMPK_CHECK_CUDA(cudaMemcpyAsync(np.data(), d_np, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
  }
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> ofs(nt + 1, 0);
  std::vector<int32_t> rec_ptr(nt + 1, 0);
  std::vector<uint4> recs;
  std::vector<LeanSliceDesc> desc;
  desc.reserve(S);
  recs.reserve(S);
  std::vector<int32_t> order;
  int64_t max_bytes = 0;
  int32_t n_pat = 0;
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t s0 = first[t], s1 = t + 1 < nt ? first[t + 1] : S;
    // width classes 0..8, full slices first inside a class
    order.clear();
    for (int w = 0; w <= 8; ++w)
      for (int pad = 0; pad < 2; ++pad)
        for (int32_t s = s0; s < s1; ++s)
          if (width[s] == w && ((wmin[s] < w) ? 1 : 0) == pad) order.push_back(s);
    const int32_t ns = s1 - s0;
    int32_t nu = 0;
    for (int32_t i = 0; i < ns;) {
      const bool pair = i + 1 < ns && width[order[i + 1]] == width[order[i]];
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
    for (int32_t i = 0; i < ns;) {
      const int32_t sa = order[i];
      const bool pair = i + 1 < ns && width[order[i + 1]] == width[sa];
      const int32_t sb = pair ? order[i + 1] : sa;
      const int w = width[sa];
      const bool padded = wmin[sa] < w || (pair && wmin[sb] < w);
      uint4 r;
      r.x = uint32_t(c_of[i]);
      r.y = pat ? uint32_t(pair ? c_of[i + 1] : 0) : uint32_t(v_of[i]);
      r.z = uint32_t(w) | (pair ? kLeanPair : 0u) | (padded ? kLeanPadded : 0u);
      if (pat && w > 0)
        r.z |= kLeanPattern | (uint32_t(np[sa]) << 16) | (uint32_t(pair ? np[sb] : 0) << 24);
      r.w = uint32_t(sa - s0) | (uint32_t(sb - s0) << 16);
      recs.push_back(r);
      i += pair ? 2 : 1;
    }
    ofs[t + 1] = ofs[t] + bytes;
  }
  rec_ptr[nt] = static_cast<int32_t>(recs.size());
  const int64_t total = ofs[nt];
  int64_t* d_ofs = nullptr;
  unsigned char* d_lean = nullptr;
  uint8_t* d_rowlen = nullptr;
  int32_t* d_rec_ptr = nullptr;
  uint4* d_recs = nullptr;
  LMPK_TRY(lmalloc(&d_ofs, nt + 1));
  LMPK_TRY(lmalloc(&d_lean, size_t(total)));
  LMPK_TRY(lmalloc(&d_rowlen, size_t(std::max(n, 1))));
  LMPK_TRY(lmalloc(&d_rec_ptr, nt + 1));
  LMPK_TRY(lmalloc(&d_recs, recs.size()));
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_lean, 0, size_t(total), st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_ofs, ofs.data(), size_t(nt + 1) * 8, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_rec_ptr, rec_ptr.data(), size_t(nt + 1) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_recs, recs.data(), recs.size() * 16, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_desc, desc.data(), desc.size() * sizeof(LeanSliceDesc), cudaMemcpyHostToDevice,
                                  st));
  const int32_t nds = static_cast<int32_t>(desc.size());
  k_lean_fill<<<div_up(int64_t(nds) * 32, 256), 256, 0, st>>>(row_ptr, col, val, nds, d_desc, d_width,
                                                              T->d_tile_row, d_ofs, d_tdict, d_nd, d_dict_tab, vd,
                                                              d_lean);
  k_lean_head<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(nt, T->d_tile_row, d_ofs, d_rec_ptr, d_recs, d_tdict,
                                                             d_nd, d_dict_tab, vd, d_lean);
  k_rowlen<<<div_up(std::max(n, 1), 256), 256, 0, st>>>(row_ptr, n, d_rowlen);
  launch_count_add(ctx, 3);
  LMPK_CHECK_CUDA(cudaGetLastError());
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_rec_ptr);
  cudaFree(d_recs);
  cudaFree(d_desc);
  cudaFree(d_tdict);
  cudaFree(d_nd);
  cudaFree(d_np);
  T->d_lean = d_lean;
  T->d_lean_ofs = d_ofs;
  T->d_rowlen = d_rowlen;
  T->lean_vd = vd;
  T->lean_bytes = total;
  T->lean_piece = static_cast<int32_t>((max_bytes + 127) & ~int64_t(127));
  T->info.lean_bytes = total;
  T->info.lean_pattern_tiles = n_pat;
  return LMPK_OK;
}

void lean_free(lmpk_tiling* T) {
  cudaFree(T->d_lean);
  cudaFree(T->d_lean_ofs);
  cudaFree(T->d_rowlen);
  T->d_lean = nullptr;
  T->d_lean_ofs = nullptr;
  T->d_rowlen = nullptr;
  T->lean_vd = -1;
}

// Launch of the lean kernel for a ring tiling with lean blocks (same
// MpkParams as launch_ring; smem = the two pieces).
int launch_lean(lmpk_ctx* ctx, const lmpk_tiling* T, MpkParams& Pm, PowerCfgDev& C, bool cplx, bool exact, bool gen,
                int grid, cudaStream_t st) {
  LeanParams L{T->d_lean, T->d_lean_ofs, T->d_rowlen};
  void* args[] = {&Pm, &C, &L};
  const bool vd = T->lean_vd == 1;
  // ring depth: 4 pieces when the lean blocks are small (pattern tiles), so
  // the producer runs further ahead of dependency waits; the pieces hold the
  // largest lean block and the rest of the unified L1/shared memory caches
  // the gathers
  const int piece = T->lean_piece > 0 ? T->lean_piece : T->piece;
  int np = (4 * int64_t(piece) + 8192 <= ctx->max_smem_block) ? 4 : 2;
  if (const char* e = getenv("LMPK_LEAN_NP")) np = atoi(e) == 4 && 4 * int64_t(piece) + 8192 <= ctx->max_smem_block ? 4 : 2;
  const void* fn = cplx ? (exact ? mpk_lean_fn_c_e(vd, np) : mpk_lean_fn_c_f(vd, np))
                        : (exact ? mpk_lean_fn_r_e(vd, gen, np) : mpk_lean_fn_r_f(vd, gen, np));
  const int smem = np * piece;
  {
    static const void* seen[32];
    static int nseen = 0;
    bool known = false;
    for (int i = 0; i < nseen; ++i) known = known || seen[i] == fn;
    if (!known) {
      cudaFuncAttributes fa;
      LMPK_CHECK_CUDA(cudaFuncGetAttributes(&fa, fn));
      LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes)));
      if (nseen < 32) seen[nseen++] = fn;
    }
    // carveout: just what the two pieces need, the rest of the unified
    // L1/shared memory caches the gathers
    cudaFuncAttributes fa;
    LMPK_CHECK_CUDA(cudaFuncGetAttributes(&fa, fn));
    const int per_sm = std::max(1, ctx->max_smem_sm);
    int pct = std::min(100, int((int64_t(smem + int(fa.sharedSizeBytes) + 1024) * 100 + per_sm - 1) / per_sm));
    if (const char* e = getenv("LMPK_LEAN_CARVE")) pct = std::max(0, std::min(100, atoi(e)));
    LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
  }
  Pm.smem_cap = piece;
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(32 * (kLeanConsumers + 2)), args, smem, st);
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
