// mpk_dp.cuh -- builder of DP (diagonal-private dictionary) tilings; included
// by mpk.cu.  The device format and its consumer body are in lean_kernel.cuh
// ("DP units").
//
// Reference: the matrix the walker reads is the level-permuted CRS matrix of
// prepare (pkg/src/levelmpk/executor.py:269-282); the tiles are the GPU form
// of the plan's row ranges (plan.py:184-370).  A DP tiling re-lays that
// matrix out for operators of the form "stencil + potential" (Anderson model,
// pkg/src/levelmpk/stencils.py gen_anderson_3d; the Chebyshev propagation of
// cheb.py:162-246): the off-diagonal values of the WHOLE matrix come from one
// dictionary of <= 31 values, each row keeps its diagonal entry as a private
// 8-byte value, and a 32-row slice stores each distinct (column offsets,
// codes) row once.  cfg5 (128^3, 14.7 M nonzeros): 152 MB of ring blocks
// become ~30 MB, which stay in L2 across the powers of a batch.
#pragma once

namespace lmpk {

constexpr int kDpDictMax = 31;   // dictionary entries (code 31 * 8 = kDpPriv is the private marker)
constexpr int kDpRowsPerCta = 8192;

// Sorted-slice descriptor of the fill kernel: global slice, tile, the slice's
// byte offset inside the tile's block, its pattern count.
struct DpSliceDesc {
  int32_t s, t, col_off, val_off, np, pat, pad0, pad1;
};

__global__ void k_dp_rowlen(const int32_t* row_ptr, int32_t n, uint8_t* out) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) out[r] = uint8_t(min(255, row_ptr[r + 1] - row_ptr[r]));
}

// Hash-set insert shared by the dictionary kernels (state: 0 empty, 1 being
// written, 2 valid).  Returns false once more than `cap` keys were inserted.
__device__ __forceinline__ void dp_set_insert(uint32_t* state, unsigned long long* keys, uint32_t* count,
                                              uint32_t* overflow, uint32_t cap, unsigned long long bits) {
  volatile uint32_t* vs = state;
  volatile unsigned long long* vk = keys;
  uint32_t h = uint32_t((bits * 0x9E3779B97F4A7C15ull) >> 54);
  for (;;) {
    if (*(volatile uint32_t*)overflow) return;
    const uint32_t st = vs[h];
    if (st == 2) {
      if (vk[h] == bits) return;
      h = (h + 1) & (kDictHash - 1);
    } else if (st == 0) {
      if (atomicCAS(&state[h], 0u, 1u) == 0u) {
        vk[h] = bits;
        __threadfence_block();
        atomicExch(&state[h], 2u);
        if (atomicAdd(count, 1u) >= cap) atomicExch(overflow, 1u);
        return;
      }
    }  // st == 1: another thread is writing this key, re-read
  }
}

// One CTA per kDpRowsPerCta rows: the distinct bit patterns of the rows'
// OFF-DIAGONAL values (col != row), unsorted, or nd = -1 beyond kDictMax.
// flags[0] is set when a row holds its diagonal column twice.
__global__ void __launch_bounds__(256) k_dp_dict(const int32_t* row_ptr, const int32_t* col, const double* val,
                                                 int32_t n, uint64_t* dict_out, int32_t* nd_out, int32_t* flags) {
  __shared__ unsigned long long keys[kDictHash];
  __shared__ uint32_t state[kDictHash];
  __shared__ uint32_t count, overflow, npk;
  for (int i = threadIdx.x; i < kDictHash; i += blockDim.x) state[i] = 0;
  if (threadIdx.x == 0) count = overflow = npk = 0;
  __syncthreads();
  const int32_t ra = blockIdx.x * kDpRowsPerCta, rb = min(n, ra + kDpRowsPerCta);
  for (int32_t r = ra + int32_t(threadIdx.x); r < rb; r += blockDim.x) {
    const int32_t a = row_ptr[r], b = row_ptr[r + 1];
    int nd = 0;
    for (int32_t e = a; e < b; ++e) {
      if (col[e] == r) {
        ++nd;
        continue;
      }
      dp_set_insert(state, keys, &count, &overflow, uint32_t(kDictMax),
                    static_cast<unsigned long long>(__double_as_longlong(val[e])));
    }
    if (nd > 1) atomicExch(flags, 1);
  }
  __syncthreads();
  if (overflow) {
    if (threadIdx.x == 0) nd_out[blockIdx.x] = -1;
    return;
  }
  for (int i = threadIdx.x; i < kDictHash; i += blockDim.x)
    if (state[i] == 2) dict_out[int64_t(blockIdx.x) * kDictMax + atomicAdd(&npk, 1u)] = keys[i];
  __syncthreads();
  if (threadIdx.x == 0) nd_out[blockIdx.x] = int32_t(npk);
}

// Lane's entries of slice s in the DP representation: 32-bit column offsets
// (col - row; padding repeats the row's last column, own row if empty), codes
// (8 x dictionary index, kDpPriv for the diagonal entry; padding: the code of
// +0.0, which is dictionary entry 0) and the private (diagonal) value.
// Returns the row length, -1 for lanes past the matrix.
__device__ __forceinline__ int dp_entries(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t s,
                                          int32_t n, int w, int lane, const uint64_t* dict, int nd,
                                          int32_t (&off)[8], uint32_t (&code)[8], double& priv) {
  const int32_t r = s * 32 + lane;
  const bool valid = r < n;
  const int32_t a = valid ? row_ptr[r] : 0;
  const int len = valid ? row_ptr[r + 1] - a : 0;
  int32_t pad = 0;
  priv = 0.0;
  for (int j = 0; j < 8; ++j) {
    int32_t o = pad;
    uint32_t k = 0;
    if (j < len) {
      const int32_t c = col[a + j];
      const double x = val[a + j];
      o = c - r;
      pad = o;
      if (c == r) {
        k = kDpPriv;
        priv = x;
      } else {
        const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
        int lo = 0, hi = nd - 1;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (dict[mid] < bits)
            lo = mid + 1;
          else
            hi = mid;
        }
        k = uint32_t(lo * 8);
      }
    }
    off[j] = (j < w) ? o : 0;
    code[j] = (j < w) ? k : 0u;
  }
  return valid ? len : -1;
}

// Pattern id of every lane of a DP slice (exact comparison of the 8 offset
// words and the 2 code words against every lower lane's); lanes past the
// matrix take the last valid lane's pattern.  Returns (pid, pattern count).
__device__ __forceinline__ int2 dp_pattern_ids(int32_t (&off)[8], uint32_t (&code)[8], int len, int lane) {
  uint32_t wd[10];
#pragma unroll
  for (int q = 0; q < 8; ++q) wd[q] = uint32_t(off[q]);
  wd[8] = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
  wd[9] = code[4] | (code[5] << 8) | (code[6] << 16) | (code[7] << 24);
  const uint32_t validm = __ballot_sync(0xffffffffu, len >= 0);
  const int last = 31 - __clz(validm);
#pragma unroll
  for (int q = 0; q < 10; ++q) {
    const uint32_t t = __shfl_sync(0xffffffffu, wd[q], last);  // every lane takes part
    if (len < 0) wd[q] = t;
  }
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

// pass 1: pattern count of every slice (one warp per slice)
__global__ void k_dp_patterns(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n, int32_t S,
                              const int32_t* width, const uint64_t* dict, int nd, int32_t* np_out) {
  const int32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= S) return;
  int32_t off[8];
  uint32_t code[8];
  double priv;
  const int len = dp_entries(row_ptr, col, val, s, n, width[s], lane, dict, nd, off, code, priv);
  const int2 pp = dp_pattern_ids(off, code, len, lane);
  if (lane == 0) np_out[s] = pp.y;
}

// pass 2: one warp per sorted slice writes [ids][offsets][codes][private]
__global__ void k_dp_fill(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t n, int32_t n_desc,
                          const DpSliceDesc* desc, const int32_t* width, const int64_t* lean_ofs,
                          const uint64_t* dict, int nd, unsigned char* lean) {
  const int32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_desc) return;
  const DpSliceDesc d = desc[i];
  const int w = width[d.s];
  if (w <= 0) return;
  const int wc = lean_wc(w);
  int32_t off[8];
  uint32_t code[8];
  double priv;
  const int len = dp_entries(row_ptr, col, val, d.s, n, w, lane, dict, nd, off, code, priv);
  const int2 pp = dp_pattern_ids(off, code, len, lane);
  unsigned char* sl = lean + lean_ofs[d.t] + d.col_off;
  sl[lane] = uint8_t(pp.x);
  const bool leader = lane == __ffs(__match_any_sync(0xffffffffu, pp.x)) - 1;
  if (leader && len >= 0) {
    int32_t* cp = reinterpret_cast<int32_t*>(sl + 32) + pp.x * wc;
    unsigned char* kp = sl + 32 + d.np * 4 * wc + pp.x * wc;
    for (int j = 0; j < wc; ++j) {
      cp[j] = off[j];
      kp[j] = uint8_t(code[j]);
    }
  }
  reinterpret_cast<double*>(sl + dp_priv_off(w, d.np))[lane] = priv;
}

// one warp per tile: header {nu, nrows, 2, first row}, the global dictionary
// at kLeanDict and the unit records
__global__ void k_dp_head(int32_t nt, const int32_t* tile_row, const int64_t* lean_ofs, const int32_t* rec_ptr,
                          const uint4* recs, const uint64_t* dict, int nd, unsigned char* lean) {
  const int32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= nt) return;
  unsigned char* blk = lean + lean_ofs[t];
  const int32_t u0 = rec_ptr[t], nu = rec_ptr[t + 1] - u0;
  if (lane == 0) *reinterpret_cast<int4*>(blk) = make_int4(nu, tile_row[t + 1] - tile_row[t], 2, tile_row[t]);
  reinterpret_cast<uint64_t*>(blk + kLeanDict)[lane] = lane < nd ? dict[lane] : 0ull;
  for (int u = lane; u < nu; u += 32) reinterpret_cast<uint4*>(blk + kLeanRec)[u] = recs[u0 + u];
}

// Whether a DP tiling should be tried: rows of <= 8 entries whose values do
// not already fit the per-tile dictionaries of the lean blocks (sampled), and
// LMPK_NO_DP unset.
static bool dp_wanted(int32_t max_row, bool dictish) {
  if (getenv("LMPK_NO_DP")) return false;
  if (const char* e = getenv("LMPK_DP"))
    if (atoi(e) == 2) return max_row >= 1 && max_row <= 8;  // forced (tests): also when a plain dictionary fits
  return max_row >= 1 && max_row <= 8 && !dictish;
}

// Builds a DP tiling of the matrix, or leaves *out == nullptr when the
// matrix is not eligible (off-diagonal values beyond one dictionary, a
// duplicated diagonal column, a block beyond the piece).  The tiling carries
// no ring blocks (d_blocks): walk and sweep both run the lean kernel.
static int dp_build(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col, const double* val,
                    const std::vector<int32_t>& width, const int32_t* d_width, const int32_t* d_wmin, bool cplx,
                    cudaStream_t st, lmpk_tiling** out) {
  *out = nullptr;
  const int32_t S = static_cast<int32_t>(width.size());
  if (S == 0 || n == 0) return LMPK_OK;
  PhaseTimer pt(st);
  // ---- global off-diagonal dictionary
  const int32_t nc = div_up(n, kDpRowsPerCta);
  uint64_t* d_part = nullptr;
  int32_t *d_nd = nullptr, *d_flag = nullptr;
  LMPK_TRY(tmp_alloc(&d_part, size_t(nc) * kDictMax, st));
  LMPK_TRY(tmp_alloc(&d_nd, nc, st));
  LMPK_TRY(tmp_alloc(&d_flag, 1, st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_flag, 0, 4, st));
  k_dp_dict<<<nc, 256, 0, st>>>(row_ptr, col, val, n, d_part, d_nd, d_flag);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  std::vector<uint64_t> part(size_t(nc) * kDictMax);
  std::vector<int32_t> pnd(nc);
  int32_t flag = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(part.data(), d_part, part.size() * 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(pnd.data(), d_nd, size_t(nc) * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&flag, d_flag, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  tmp_free(d_part, st);
  tmp_free(d_nd, st);
  tmp_free(d_flag, st);
  if (flag) return LMPK_OK;
  std::vector<uint64_t> dict{0ull};  // +0.0, the padding value, is entry 0 (smallest bit pattern)
  for (int32_t c = 0; c < nc; ++c) {
    if (pnd[c] < 0) return LMPK_OK;
    for (int32_t i = 0; i < pnd[c]; ++i) dict.push_back(part[size_t(c) * kDictMax + i]);
    std::sort(dict.begin(), dict.end());
    dict.erase(std::unique(dict.begin(), dict.end()), dict.end());
    if (dict.size() > size_t(kDpDictMax)) return LMPK_OK;
  }
  const int nd = static_cast<int>(dict.size());
  pt.mark("  dp: dictionary");
  uint64_t* d_dict = nullptr;
  int32_t* d_np = nullptr;
  LMPK_TRY(tmp_alloc(&d_dict, 32, st));
  LMPK_TRY(tmp_alloc(&d_np, S, st));
  struct Guard {
    std::vector<void*> p;
    cudaStream_t s;
    ~Guard() {
      for (void* q : p) tmp_free(q, s);
    }
  } guard;
  guard.s = st;
  guard.p = {d_dict, d_np};
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_dict, dict.data(), size_t(nd) * 8, cudaMemcpyHostToDevice, st));
  // ---- pass 1: distinct rows per slice
  k_dp_patterns<<<div_up(int64_t(S) * 32, 256), 256, 0, st>>>(row_ptr, col, val, n, S, d_width, d_dict, nd, d_np);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  std::vector<int32_t> np(S), wmin(S);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(np.data(), d_np, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(wmin.data(), d_wmin, size_t(S) * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  pt.mark("  dp: pattern pass");
  // ---- tiles: consecutive slices up to the piece cap.  Complex tilings: 48 KB
  // pieces (cfg5: ~3.7K rows, 570 tiles, a ring of 2) measured best (2.40 ms
  // per Chebyshev step; 32 KB and a ring of 4: 2.44, 64 KB: 2.65;
  // tools/cfg5_sweep.py).  Real tilings: 32 KB and a ring of 4 (cfg5's matrix,
  // real MPK k = 8: 0.142 ms against 0.153 at 48 KB; tools/lean_ab.py)
  int64_t cap = (cplx ? 48 : 32) * 1024;
  if (const char* e = getenv("LMPK_DP_TILE_KB")) cap = std::max(4, std::min(100, atoi(e))) * int64_t(1024);
  std::vector<int32_t> first;
  {
    int64_t bytes = 0;
    int32_t ns = 0;
    for (int32_t s = 0; s < S; ++s) {
      const int64_t sb = dp_slice_bytes(width[s], np[s]);
      if (kLeanRec + 16 + sb + 256 > cap) return LMPK_OK;
      if (ns == 0 || kLeanRec + 16 * int64_t(ns + 1) + 16 + bytes + sb + 128 > cap || ns >= 65535) {
        first.push_back(s);
        bytes = 0;
        ns = 0;
      }
      bytes += sb;
      ++ns;
    }
  }
  const int32_t nt = static_cast<int32_t>(first.size());
  // complex vectors: single-slice units (a pair's 2W double2 gathers exceed the registers)
  bool pairing = !cplx;
  if (const char* e = getenv("LMPK_DP_PAIR")) pairing = !cplx && atoi(e) != 0;
  std::vector<int64_t> ofs(nt + 1, 0);
  std::vector<int32_t> rec_ptr(nt + 1, 0), tile_row(nt + 1), tile_E(nt), order;
  std::vector<uint4> recs;
  std::vector<DpSliceDesc> desc;
  recs.reserve(S);
  desc.reserve(S);
  int64_t max_bytes = 0;
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t s0 = first[t], s1 = t + 1 < nt ? first[t + 1] : S, ns = s1 - s0;
    tile_row[t] = std::min(s0 * 32, n);
    int64_t E = 0;
    for (int32_t s = s0; s < s1; ++s) E += int64_t(width[s]) * 32;
    tile_E[t] = static_cast<int32_t>(E);
    {  // width classes 0..8, full slices first inside a class (counting sort)
      int32_t cnt[19] = {0};
      for (int32_t s = s0; s < s1; ++s) ++cnt[2 * width[s] + (wmin[s] < width[s] ? 1 : 0) + 1];
      for (int q = 0; q < 18; ++q) cnt[q + 1] += cnt[q];
      order.resize(ns);
      for (int32_t s = s0; s < s1; ++s) order[cnt[2 * width[s] + (wmin[s] < width[s] ? 1 : 0)]++] = s;
    }
    int32_t nu = 0;
    for (int32_t i = 0; i < ns;) {
      const bool pair = pairing && i + 1 < ns && width[order[i + 1]] == width[order[i]];
      ++nu;
      i += pair ? 2 : 1;
    }
    int64_t co = align16(kLeanRec + 16 * int64_t(nu));
    std::vector<int32_t> c_of(ns);
    for (int32_t i = 0; i < ns; ++i) {
      const int32_t s = order[i];
      c_of[i] = int32_t(co);
      desc.push_back(DpSliceDesc{s, t, int32_t(co), 0, np[s], 1, 0, 0});
      co += dp_slice_bytes(width[s], np[s]);
    }
    const int64_t bytes = (co + 127) & ~int64_t(127);
    max_bytes = std::max(max_bytes, bytes);
    rec_ptr[t] = static_cast<int32_t>(recs.size());
    for (int32_t i = 0; i < ns;) {
      const int32_t sa = order[i];
      const bool pair = pairing && i + 1 < ns && width[order[i + 1]] == width[sa];
      const int32_t sb = pair ? order[i + 1] : sa;
      const int w = width[sa];
      const bool padded = wmin[sa] < w || (pair && wmin[sb] < w);
      uint4 r;
      r.x = uint32_t(c_of[i]);
      r.y = uint32_t(pair ? c_of[i + 1] : 0);
      r.z = uint32_t(w) | (pair ? kLeanPair : 0u) | (padded ? kLeanPadded : 0u) | kLeanPattern |
            (uint32_t(np[sa]) << 16) | (uint32_t(pair ? np[sb] : 0) << 24);
      r.w = uint32_t(sa - s0) | (uint32_t(sb - s0) << 16);
      recs.push_back(r);
      i += pair ? 2 : 1;
    }
    ofs[t + 1] = ofs[t] + bytes;
  }
  tile_row[nt] = n;
  rec_ptr[nt] = static_cast<int32_t>(recs.size());
  if (max_bytes > cap) return LMPK_OK;
  pt.mark("  dp: host tiles + units");
  // ---- the tiling object
  lmpk_tiling* T = new lmpk_tiling();
  T->ctx = ctx;
  T->n = n;
  const int64_t total = ofs[nt];
  int32_t* d_rec_ptr = nullptr;
  uint4* d_recs = nullptr;
  DpSliceDesc* d_desc = nullptr;
#define LMPK_DP_TRY(...)                \
  do {                                  \
    const int rc_ = (__VA_ARGS__);      \
    if (rc_ != LMPK_OK) {               \
      lmpk_tiling_destroy(T);           \
      return rc_;                       \
    }                                   \
  } while (0)
  LMPK_DP_TRY(tmp_alloc(&d_rec_ptr, nt + 1, st));
  guard.p.push_back(d_rec_ptr);
  LMPK_DP_TRY(tmp_alloc(&d_recs, recs.size(), st));
  guard.p.push_back(d_recs);
  LMPK_DP_TRY(tmp_alloc(&d_desc, desc.size(), st));
  guard.p.push_back(d_desc);
  LMPK_DP_TRY(dmalloc(&T->d_tile_row, nt + 1));
  LMPK_DP_TRY(dmalloc(&T->d_tile_E, nt));
  LMPK_DP_TRY(dmalloc(&T->d_dep_lo, nt));
  LMPK_DP_TRY(dmalloc(&T->d_dep_hi, nt));
  LMPK_DP_TRY(dmalloc(&T->d_progress, nt));
  LMPK_DP_TRY(dmalloc(&T->d_lean_ofs, nt + 1));
  LMPK_DP_TRY(dmalloc(&T->d_lean, size_t(total)));
  LMPK_DP_TRY(dmalloc(&T->d_rowlen, size_t(n)));
  auto cuda_ok = [&](cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LMPK_OK;
    cudaGetLastError();
    set_error("dp_build: %s failed: %s", what, cudaGetErrorString(e));
    return LMPK_ERR_CUDA;
  };
  LMPK_DP_TRY(cuda_ok(cudaMemsetAsync(T->d_lean, 0, size_t(total), st), "memset"));
  LMPK_DP_TRY(cuda_ok(cudaMemsetAsync(T->d_progress, 0, size_t(nt) * 4, st), "memset"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(T->d_tile_row, tile_row.data(), size_t(nt + 1) * 4, cudaMemcpyHostToDevice, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(T->d_tile_E, tile_E.data(), size_t(nt) * 4, cudaMemcpyHostToDevice, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(T->d_lean_ofs, ofs.data(), size_t(nt + 1) * 8, cudaMemcpyHostToDevice, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(d_rec_ptr, rec_ptr.data(), size_t(nt + 1) * 4, cudaMemcpyHostToDevice, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(d_recs, recs.data(), recs.size() * 16, cudaMemcpyHostToDevice, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(d_desc, desc.data(), desc.size() * sizeof(DpSliceDesc), cudaMemcpyHostToDevice, st), "copy"));
  const int32_t nds = static_cast<int32_t>(desc.size());
  k_dp_fill<<<div_up(int64_t(nds) * 32, 256), 256, 0, st>>>(row_ptr, col, val, n, nds, d_desc, d_width, T->d_lean_ofs,
                                                            d_dict, nd, T->d_lean);
  k_dp_head<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(nt, T->d_tile_row, T->d_lean_ofs, d_rec_ptr, d_recs, d_dict,
                                                           nd, T->d_lean);
  k_dp_rowlen<<<div_up(n, 256), 256, 0, st>>>(row_ptr, n, T->d_rowlen);
  k_tile_deps<<<div_up(int64_t(nt) * 32, 256), 256, 0, st>>>(row_ptr, col, T->d_tile_row, nt, T->d_dep_lo, T->d_dep_hi);
  launch_count_add(ctx, 4);
  LMPK_DP_TRY(cuda_ok(cudaGetLastError(), "launch"));
  T->h_tile_row = tile_row;
  T->h_dep_lo.resize(nt);
  T->h_dep_hi.resize(nt);
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(T->h_dep_lo.data(), T->d_dep_lo, size_t(nt) * 4, cudaMemcpyDeviceToHost, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaMemcpyAsync(T->h_dep_hi.data(), T->d_dep_hi, size_t(nt) * 4, cudaMemcpyDeviceToHost, st), "copy"));
  LMPK_DP_TRY(cuda_ok(cudaStreamSynchronize(st), "sync"));
#undef LMPK_DP_TRY
  pt.mark("  dp: alloc + fill + deps");
  T->lean_vd = 2;
  T->lean_bytes = total;
  T->h_lean_ofs = ofs;
  T->lean_piece = static_cast<int32_t>((max_bytes + 127) & ~int64_t(127));
  T->max_block = T->lean_piece;
  T->block_bytes = 0;
  T->info.n_tiles = nt;
  T->info.block_bytes = total;  // the DP blocks are the only copy of the matrix
  T->info.lean_bytes = total;
  T->info.compressed_tiles = nt;
  T->info.dict_tiles = nt;
  T->info.lean_pattern_tiles = nt;
  T->info.dp_tiles = nt;
  *out = T;
  return LMPK_OK;
}

}  // namespace lmpk
