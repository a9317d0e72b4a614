// mpk_lean.cu -- host side of the lean ring walk (lean_kernel.cuh): the lean
// block builder (width-sorted units, lane-contiguous indices) and the launch.
#include "lean_kernel.cuh"

namespace lmpk {

const void* mpk_lean_fn_r(bool exact, bool vd, bool gen);
const void* mpk_lean_fn_c(bool exact, bool vd);

// Sorted-slice descriptor for the fill kernel: global slice, tile, the
// slice's column / value byte offsets inside the tile's lean block, width.
struct LeanSliceDesc {
  int32_t s, t, col_off, val_off;
};

// one warp per sorted slice: lane = row; int16 column offsets (lane-
// contiguous, Wc entries), dictionary byte codes (Wc bytes) or raw values
// (chunked).  Padding repeats the row's last column (own row if empty; the
// slice's first row for lanes past the tile) with the value +0.0.
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
  const int32_t r1 = tile_row[d.t + 1];
  const int32_t r = d.s * 32 + lane;
  const bool valid = r < r1;
  const int32_t a = valid ? row_ptr[r] : 0;
  const int len = valid ? row_ptr[r + 1] - a : 0;
  const uint64_t* dict = vd ? dict_tab + int64_t(tile_dict[d.t]) * kDictMax : nullptr;
  const int nd = vd ? tile_nd[d.t] : 0;
  int16_t* cp = reinterpret_cast<int16_t*>(blk + d.col_off) + lane * wc;
  int32_t pad = valid ? 0 : -lane;
  for (int j = 0; j < wc; ++j) {
    int32_t off = pad;
    double v = 0.0;
    if (j < len) {
      off = col[a + j] - r;
      v = val[a + j];
      pad = off;
    }
    cp[j] = int16_t(j < w ? off : 0);
    if (vd) {
      const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
      int lo = 0, hi = nd - 1;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (dict[mid] < bits)
          lo = mid + 1;
        else
          hi = mid;
      }
      blk[d.val_off + lane * wc + j] = uint8_t(j < w ? lo * 8 : 0);
    } else if (j < w) {
      reinterpret_cast<double*>(blk + d.val_off)[chunk_entry(0, w, lane, j)] = v;
    }
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

// Lean block bytes of slices [s0, s1) (the tiling cost bound: a lean block
// must fit the slot like the compressed block it mirrors).
int64_t lean_tile_bytes(const std::vector<int32_t>& width, int32_t s0, int32_t s1, bool vd) {
  int64_t cols = 0, vals = 0;
  for (int32_t s = s0; s < s1; ++s) {
    cols += lean_col_bytes(width[s]);
    vals += vd ? lean_code_bytes(width[s]) : lean_raw_bytes(width[s]);
  }
  const int64_t ns = s1 - s0;
  return (align16(align16(kLeanRec + 16 * ns) + cols) + vals + 127) & ~int64_t(127);
}

// Builds the lean blocks of a compressed tiling whose tiles all have width
// <= 8 and one value format (all dictionary or all raw).  `first` are the
// tiles' first slices; tmode/tdict/d_dict_tab as in build_tiling.
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
  std::vector<int32_t> wmin(S);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(wmin.data(), d_wmin, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> ofs(nt + 1, 0);
  std::vector<int32_t> rec_ptr(nt + 1, 0);
  std::vector<uint4> recs;
  std::vector<LeanSliceDesc> desc;
  desc.reserve(S);
  recs.reserve(S);
  std::vector<int32_t> order;
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t s0 = first[t], s1 = t + 1 < nt ? first[t + 1] : S;
    const int64_t bytes = lean_tile_bytes(width, s0, s1, vd == 1);
    if (bytes > cap) return LMPK_OK;  // cannot happen with the lean-aware tiling cost
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
    int64_t co = align16(kLeanRec + 16 * int64_t(nu));
    int64_t cols = 0;
    for (int32_t s = s0; s < s1; ++s) cols += lean_col_bytes(width[s]);
    int64_t vo = align16(co + cols);
    std::vector<int32_t> c_of(ns), v_of(ns);
    for (int32_t i = 0; i < ns; ++i) {
      const int w = width[order[i]];
      c_of[i] = int32_t(co);
      v_of[i] = int32_t(vo);
      desc.push_back(LeanSliceDesc{order[i], t, int32_t(co), int32_t(vo)});
      co += lean_col_bytes(w);
      vo += vd ? lean_code_bytes(w) : lean_raw_bytes(w);
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
      r.y = uint32_t(v_of[i]);
      r.z = uint32_t(w) | (pair ? kLeanPair : 0u) | (padded ? kLeanPadded : 0u);
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
  int32_t *d_rec_ptr = nullptr, *d_tdict = nullptr, *d_nd = nullptr;
  uint4* d_recs = nullptr;
  LeanSliceDesc* d_desc = nullptr;
  LMPK_TRY(lmalloc(&d_ofs, nt + 1));
  LMPK_TRY(lmalloc(&d_lean, size_t(total)));
  LMPK_TRY(lmalloc(&d_rowlen, size_t(std::max(n, 1))));
  LMPK_TRY(lmalloc(&d_rec_ptr, nt + 1));
  LMPK_TRY(lmalloc(&d_recs, recs.size()));
  LMPK_TRY(lmalloc(&d_desc, desc.size()));
  LMPK_TRY(lmalloc(&d_tdict, nt));
  LMPK_TRY(lmalloc(&d_nd, nt));
  std::vector<int32_t> nd(nt);
  for (int32_t t = 0; t < nt; ++t) nd[t] = tmode[t] >> 8;
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_lean, 0, size_t(total), st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_ofs, ofs.data(), size_t(nt + 1) * 8, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_rec_ptr, rec_ptr.data(), size_t(nt + 1) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_recs, recs.data(), recs.size() * 16, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_desc, desc.data(), desc.size() * 16, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_tdict, tdict.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_nd, nd.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st));
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
  T->d_lean = d_lean;
  T->d_lean_ofs = d_ofs;
  T->d_rowlen = d_rowlen;
  T->lean_vd = vd;
  T->lean_bytes = total;
  T->info.lean_bytes = total;
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
  const void* fn = cplx ? mpk_lean_fn_c(exact, vd) : mpk_lean_fn_r(exact, vd, gen);
  const int smem = 2 * T->piece;
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
  Pm.smem_cap = T->piece;
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
