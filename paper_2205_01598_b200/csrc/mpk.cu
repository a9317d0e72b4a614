// mpk.cu -- host side of the level-blocked MPK: tiling, block layout, launch.
// The device code is in mpk_kernel.cuh (header comment there).
#include "lean_kernel.cuh"

namespace lmpk {

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
  // entry e0 - 1 stands for +0.0, the padding value every dictionary holds
  for (int32_t e = e0 - 1 + int32_t(threadIdx.x); e < e1; e += blockDim.x) {
    if (*(volatile uint32_t*)&overflow) break;
    const unsigned long long bits =
        e < e0 ? 0ull : static_cast<unsigned long long>(__double_as_longlong(__ldg(val + e)));
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
    const int32_t sg0 = seg_ptr ? seg_ptr[t] : 0;
    const int32_t nseg = seg_ptr ? seg_ptr[t + 1] - sg0 : 0;
    if (ls == 0) {
      for (int j = lane; j < nseg; j += 32) reinterpret_cast<int4*>(blk + blk_seg_off(ns))[j] = segs[sg0 + j];
      if (vd)
        for (int j = lane; j < nd; j += 32) reinterpret_cast<uint64_t*>(blk + cblk_dict_off(ns, nseg))[j] = dict[j];
    }
    // x-segments: the local index of a global column (binary search over the runs)
    auto local = [&](int32_t c) -> int32_t {
      int lo = 0, hi = nseg - 1;
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
    int16_t* c16 = reinterpret_cast<int16_t*>(blk + cblk_col_off(ns, nd, nseg));
    unsigned char* vbase = blk + cblk_val_off(ns, nd, E, nseg);
    const int32_t base = slice_off[s];
    const int32_t r = s * 32 + lane;
    const bool valid = r < r1;
    const int32_t a = valid ? row_ptr[r] : 0;
    const int len = valid ? row_ptr[r + 1] - a : 0;
    const int w = width[s];
    if (lane == 0) reinterpret_cast<int2*>(blk)[ls] = make_int2(base, w | (wmin[s] << 16));
    reinterpret_cast<uint16_t*>(blk + int64_t(ns) * 8)[ls * 32 + lane] = uint16_t(len);
    // padding: the row's last column (own row if empty; r0 for lanes past the
    // tile; local index 0 with x-segments)
    int32_t pad = nseg ? -kLocalBias : (valid ? 0 : r0 - r);
    for (int j = 0; j < w; ++j) {
      const int64_t e = chunk_entry(base, w, lane, j);
      int32_t d = pad;
      double v = 0.0;
      if (j < len) {
        d = nseg ? local(col[a + j]) - kLocalBias : col[a + j] - r;
        v = val[a + j];
        pad = d;
      }
      c16[e] = int16_t(d);
      if (vd) {
        uint8_t code = 0;
        {  // padding (j >= len) looks up +0.0 (v == 0.0 here)
          const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
          int lo = 0, hi = nd - 1;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (dict[mid] < bits)
              lo = mid + 1;
            else
              hi = mid;
          }
          code = uint8_t(lo * 8);  // dictionary byte offset
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

// lean ring walk (mpk_lean.cu)
int64_t lean_tile_bytes(const std::vector<int32_t>& width, int32_t s0, int32_t s1, bool vd);
int lean_build(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr, const int32_t* col,
               const double* val, const std::vector<int32_t>& first, const std::vector<int32_t>& width,
               const int32_t* d_wmin, const std::vector<int32_t>& tmode, const std::vector<int32_t>& tdict,
               const uint64_t* d_dict_tab, const int32_t* d_width, int64_t cap, bool want_xs, bool cplx,
               cudaStream_t st);
int lean_xplan(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col, const int32_t* d_tile_row,
               int32_t nt, bool cplx, int4** d_runs, int2** d_xinfo, int32_t* max_entries, cudaStream_t st);
int64_t lean_xs_budget(const lmpk_ctx* ctx);
bool lean_xs_wanted();
bool lean_xs_runnable(const lmpk_tiling* T, const double* y, int64_t ldy, bool cplx);
int lean_worklist(lmpk_tiling* T, const std::vector<int32_t>& items, const std::vector<int32_t>& st_first,
                  const std::vector<int32_t>& lo, const std::vector<int32_t>& hi, int grid, cudaStream_t st);
void lean_free(lmpk_tiling* T);
int launch_lean(lmpk_ctx* ctx, const lmpk_tiling* T, MpkParams& Pm, PowerCfgDev& C, bool cplx, bool exact, bool gen,
                int grid, cudaStream_t st);

// one explicit instantiation per variant (mpk_k_*.cu: separate, parallel TUs)
const void* mpk_group_fn_re();
const void* mpk_group_fn_rf();
const void* mpk_group_fn_ce();
const void* mpk_group_fn_cf();
const void* mpk_ring_fn_re(bool has_long);
const void* mpk_ring_fn_rf(bool has_long);
const void* mpk_ring_fn_ce(bool has_long);
const void* mpk_ring_fn_cf(bool has_long);
const void* mpk_ring_fn_re_uniform(int u);
const void* mpk_ring_fn_rf_uniform(int u);
const void* mpk_ring_fn_ce_uniform(int u);
const void* mpk_ring_fn_cf_uniform(int u);
// uniform: 0 general kernel, 1 all tiles dictionary (w <= 8), 2 all tiles raw compressed (w <= 8)
static const void* ring_fn(bool cplx, bool exact, bool has_long = true, int uniform = 0) {
  if (uniform && !has_long) {
    if (cplx) return exact ? mpk_ring_fn_ce_uniform(uniform) : mpk_ring_fn_cf_uniform(uniform);
    return exact ? mpk_ring_fn_re_uniform(uniform) : mpk_ring_fn_rf_uniform(uniform);
  }
  if (cplx) return exact ? mpk_ring_fn_ce(has_long) : mpk_ring_fn_cf(has_long);
  return exact ? mpk_ring_fn_re(has_long) : mpk_ring_fn_rf(has_long);
}
// Occupancy of the ring kernel (all instantiations) at `smem` dynamic bytes.
static int ring_occupancy(lmpk_ctx* ctx, int smem, int* occ) {
  *occ = 1 << 20;
  for (int c = 0; c < 4; ++c)
    for (int x = 0; x < 2; ++x) {
      const void* fn = ring_fn((c & 1) != 0, x != 0, c >= 2);
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, fn);
      if (e == cudaSuccess && smem > ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes)) {
        *occ = 0;
        return LMPK_OK;
      }
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes));
      int o = 0;
      if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, 32 * (kRingConsumers + 2), smem);
      if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("occupancy query failed: %s", cudaGetErrorString(e));
        return LMPK_ERR_CUDA;
      }
      *occ = std::min(*occ, o);
    }
  return LMPK_OK;
}
static const void* group_fn(bool cplx, bool exact) {
  if (cplx) return exact ? mpk_group_fn_ce() : mpk_group_fn_cf();
  return exact ? mpk_group_fn_re() : mpk_group_fn_rf();
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

// Largest static shared memory over the group- and ring-kernel instantiations.
static int group_static_smem(int* out) {
  int mx = 0;
  for (int c = 0; c < 4; ++c)
    for (int x = 0; x < 2; ++x) {
      cudaFuncAttributes fa;
      cudaError_t e = cudaFuncGetAttributes(&fa, c < 2 ? group_fn(c != 0, x != 0) : ring_fn(c == 3, x != 0, true));
      if (e == cudaSuccess && c >= 2) {
        cudaFuncAttributes fb;
        e = cudaFuncGetAttributes(&fb, ring_fn(c == 3, x != 0, false));
        fa.sharedSizeBytes = std::max(fa.sharedSizeBytes, fb.sharedSizeBytes);
        for (int u = 1; u <= (c == 3 ? 2 : 3) && e == cudaSuccess; ++u) {
          e = cudaFuncGetAttributes(&fb, ring_fn(c == 3, x != 0, false, u));
          fa.sharedSizeBytes = std::max(fa.sharedSizeBytes, fb.sharedSizeBytes);
        }
      }
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
  cudaFree(t->d_st_first);
  cudaFree(t->d_st_lo);
  cudaFree(t->d_st_hi);
  cudaFree(t->d_rdep_ptr);
  cudaFree(t->d_rdep);
  cudaFree(t->d_rcnt);
  cudaFree(t->d_rqueue);
  cudaFree(t->d_rctrl);
  cudaFree(t->d_items);
  cudaFree(t->d_progress);
  cudaFree(t->d_blocks);
  lean_free(t);
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
                          const std::vector<int64_t>& xcap, std::vector<int32_t>& seg_ptr,
                          std::vector<int4>& segs, std::vector<int32_t>& xent) {
  const int32_t nt = static_cast<int32_t>(tile_row.size()) - 1;
  seg_ptr.assign(nt + 1, 0);
  xent.assign(nt, 0);
  segs.clear();
  std::vector<uint8_t> mark;
  std::vector<int2> runs;
  for (int32_t t = 0; t < nt; ++t) {
    seg_ptr[t] = static_cast<int32_t>(segs.size());
    const int64_t e0 = rp[tile_row[t]], e1 = rp[tile_row[t + 1]];
    if (e1 == e0 || xcap[t] <= 0 || !allow[t]) continue;
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
    if (lb > xcap[t]) continue;
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
// Distinct gathered columns of the slices added so far (x-staged tilings):
// the slot must hold the tile's block AND its x buffer.
struct XCounter {
  const std::vector<int32_t>* rp = nullptr;
  const std::vector<int32_t>* col = nullptr;
  int32_t n = 0;
  std::vector<uint8_t> mark;
  std::vector<int32_t> touched;
  size_t add(int32_t s) {  // slice s; returns the undo mark
    const size_t b = touched.size();
    const int32_t r0 = s * 32, r1 = std::min(n, r0 + 32);
    for (int64_t e = (*rp)[r0]; e < (*rp)[r1]; ++e) {
      const int32_t c = (*col)[e];
      if (!mark[c]) {
        mark[c] = 1;
        touched.push_back(c);
      }
    }
    return b;
  }
  void undo(size_t b) {
    while (touched.size() > b) {
      mark[touched.back()] = 0;
      touched.pop_back();
    }
  }
  void reset() { undo(0); }
  // x buffer bytes of the current tile (+3% for the runs' gaps and parity
  // rounding) plus the segment table
  int64_t bytes() const { return ((int64_t(touched.size()) * 8 * 103 / 100 + 64 + 127) & ~int64_t(127)) + kMaxSegs * 16; }
};

template <class Cost>
static void partition_range(const std::vector<int32_t>& width, int32_t s0, int32_t s1, int64_t cap, int64_t e_cap,
                            Cost cost, std::vector<int32_t>& first, std::vector<int64_t>& Es,
                            XCounter* xc = nullptr, int32_t ns_cap = INT32_MAX) {
  int32_t s = s0;
  while (s < s1) {
    int32_t ns = 0;
    int64_t E = 0;
    if (xc) xc->reset();
    while (s + ns < s1) {
      const int64_t e2 = E + int64_t(width[s + ns]) * 32;
      const size_t u = xc ? xc->add(s + ns) : 0;
      const int64_t need = cost(s, ns + 1, e2) + (xc ? xc->bytes() : 0);
      if (ns > 0 && (need > cap || e2 > e_cap || ns >= ns_cap)) {
        if (xc) xc->undo(u);
        break;
      }
      E = e2;
      ++ns;
    }
    first.push_back(s);
    Es.push_back(E);
    s += ns;
  }
  if (xc) xc->reset();
}

// Tiles + chunked tile-SELL-32 blocks + dependency ranges for block cap `cap`
// bytes.  With fit16 (compressed tiling), runs of slices whose column offsets
// fit int16 become compressed tiles: first partitioned for the dictionary
// format (3 B/entry), then every tile with more than kDictMax distinct values
// is re-partitioned for raw values (10 B/entry); the other slices stay plain.
static int build_tiling(lmpk_ctx* ctx, lmpk_tiling* T, int32_t n, const int32_t* row_ptr,
                        const int32_t* col, const double* val, const std::vector<int32_t>& width,
                        const int32_t* d_wmin, int64_t cap, const std::vector<int32_t>* h_rp,
                        const std::vector<int32_t>* h_col, bool xstage, const std::vector<uint8_t>* fit16,
                        int64_t e_cap, cudaStream_t st, int32_t xs_slices = 0, bool cplx = false) {
  // xs_slices > 0: the lean walk stages x (lean_build): tiles hold at most
  // that many slices, so a tile's block and x buffer share one ring piece
  const int32_t ns_cap = xs_slices > 0 ? xs_slices : INT32_MAX;
  const int32_t S = static_cast<int32_t>(width.size());
  PhaseTimer pt(st);
  std::vector<int32_t> first;
  std::vector<int64_t> Es;
  std::vector<int32_t> tmode;   // per tile: 0 plain, else kModeC16 [| kModeDict | nd << 8]
  std::vector<int32_t> tdict;   // per tile: index into the dictionary table (dict tiles)
  uint64_t* d_dict_tab = nullptr;
  int32_t* d_tile_dict = nullptr;
  auto plain_cost = [](int32_t, int32_t ns, int64_t E) { return blk_bytes(ns, E, 0); };
  // x staging: a slot holds [block | x buffer] (per-tile split, see XCounter)
  XCounter xcnt;
  XCounter* xc = nullptr;
  if (xstage && h_rp && h_col) {
    xcnt.rp = h_rp;
    xcnt.col = h_col;
    xcnt.n = n;
    xcnt.mark.assign(size_t(n) + 1, 0);
    xc = &xcnt;
  }
  if (fit16 && S > 0) {
    // a compressed tile must also fit the slot as a lean block (lean_kernel.cuh)
    std::vector<int64_t> pre_d(S + 1, 0), pre_r(S + 1, 0);
    for (int32_t s = 0; s < S; ++s) {
      const int w = std::min(width[s], 9);
      pre_d[s + 1] = pre_d[s] + lean_col_bytes(w) + lean_code_bytes(w);
      pre_r[s + 1] = pre_r[s] + lean_col_bytes(w) + lean_raw_bytes(w);
    }
    auto lean_cost = [&](const std::vector<int64_t>& pre, int32_t s0, int32_t ns) {
      return (int64_t(kLeanRec) + 16 * int64_t(ns) + pre[s0 + ns] - pre[s0] + 127) & ~int64_t(127);
    };
    auto dict_cost = [&](int32_t s0, int32_t ns, int64_t E) {
      return std::max(cblk_bytes(ns, kDictMax, E, true, 0), lean_cost(pre_d, s0, ns));
    };
    auto raw_cost = [&](int32_t s0, int32_t ns, int64_t E) {
      return std::max(cblk_bytes(ns, 0, E, false, 0), lean_cost(pre_r, s0, ns));
    };
    // pass 1: runs of equal fit16, compressed runs cut for the dictionary format
    std::vector<int32_t> f1;
    std::vector<int64_t> E1;
    std::vector<uint8_t> c1;
    for (int32_t s = 0; s < S;) {
      int32_t e = s;
      while (e < S && (*fit16)[e] == (*fit16)[s]) ++e;
      const size_t before = f1.size();
      if ((*fit16)[s])
        partition_range(width, s, e, cap, e_cap, dict_cost, f1, E1, xc, ns_cap);
      else
        partition_range(width, s, e, cap, INT64_MAX, plain_cost, f1, E1, xc, ns_cap);
      c1.resize(f1.size(), (*fit16)[s]);
      (void)before;
      s = e;
    }
    const int32_t n1 = static_cast<int32_t>(f1.size());
    pt.mark("partition pass 1");
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
      LMPK_TRY(tmp_alloc(&d_row1, n1 + 1, st));
      LMPK_TRY(tmp_alloc(&d_list, nl, st));
      LMPK_TRY(tmp_alloc(&d_nd, nl, st));
      LMPK_TRY(tmp_alloc(&d_dict_tab, size_t(nl) * kDictMax, st));
      LMPK_CHECK_CUDA(cudaMemcpyAsync(d_row1, row1.data(), size_t(n1 + 1) * 4, cudaMemcpyHostToDevice, st));
      LMPK_CHECK_CUDA(cudaMemcpyAsync(d_list, list.data(), size_t(nl) * 4, cudaMemcpyHostToDevice, st));
      k_tile_dict<<<nl, 256, 0, st>>>(row_ptr, val, d_row1, d_list, nl, d_dict_tab, d_nd);
      launch_count_add(ctx, 1);
      LMPK_CHECK_CUDA(cudaGetLastError());
      LMPK_CHECK_CUDA(cudaMemcpyAsync(nd.data(), d_nd, size_t(nl) * 4, cudaMemcpyDeviceToHost, st));
      LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
      tmp_free(d_row1, st);
      tmp_free(d_list, st);
      tmp_free(d_nd, st);
    }
    pt.mark("tile dictionaries");
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
      if (k >= 0 && dict_cost(s0, s1 - s0, E1[t]) <= cap) {
        first.push_back(s0);
        Es.push_back(E1[t]);
        tmode.push_back(kModeC16 | kModeDict | (k << 8));
        tdict.push_back(li);
      } else {
        const size_t b = first.size();
        partition_range(width, s0, s1, cap, e_cap, raw_cost, first, Es, xc, ns_cap);
        for (size_t i = b; i < first.size(); ++i) {
          const int32_t a0 = first[i], a1 = i + 1 < first.size() ? first[i + 1] : s1;
          // a single slice too large for a slot stays plain (read from global)
          tmode.push_back(raw_cost(a0, a1 - a0, Es[i]) <= cap ? kModeC16 : 0);
          tdict.push_back(-1);
        }
      }
      ++li;
    }
  } else {
    if (xc)
      partition_range(width, 0, S, cap, INT64_MAX, plain_cost, first, Es, xc);
    else
      partition_slices(width, cap, first, Es);
    tmode.assign(first.size(), 0);
    tdict.assign(first.size(), -1);
  }
  const int32_t nt = static_cast<int32_t>(first.size());
  pt.mark("partition pass 2");
  // compressed tiles with slices wider than 8 take the long-row kernel body
  for (int32_t t = 0; t < nt; ++t) {
    if (!tmode[t]) continue;
    const int32_t s1 = t + 1 < nt ? first[t + 1] : S;
    for (int32_t sl = first[t]; sl < s1; ++sl)
      if (width[sl] > 8) {
        tmode[t] |= kModeLong;
        break;
      }
  }
  std::vector<int32_t> tile_row(nt + 1), tile_E(nt), slice_tile(std::max(S, 1)), slice_off(std::max(S, 1));
  std::vector<int64_t> tile_ofs(nt + 1);
  for (int32_t t = 0; t < nt; ++t) tile_row[t] = std::min(first[t] * 32, n);
  tile_row[nt] = n;
  // x-segments (real-vector tilings only)
  std::vector<int32_t> seg_ptr, xent;
  std::vector<int4> segs;
  if (xc) {
    // the x buffer follows the block in the slot: what the block leaves
    std::vector<uint8_t> allow(nt);
    std::vector<int64_t> xcap(nt);
    for (int32_t t = 0; t < nt; ++t) {
      const int32_t s1 = (t + 1 < nt) ? first[t + 1] : S;
      const int64_t b = tmode[t] ? cblk_bytes(s1 - first[t], tmode[t] >> 8, Es[t], (tmode[t] & kModeDict) != 0, kMaxSegs)
                                 : blk_bytes(s1 - first[t], Es[t], kMaxSegs);
      allow[t] = b <= cap;
      xcap[t] = (cap - b) / 8;
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
    const int64_t b = tmode[t] ? cblk_bytes(s1 - s0, tmode[t] >> 8, Es[t], (tmode[t] & kModeDict) != 0, nseg)
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
    LMPK_TRY(tmp_alloc(&d_tile_dict, nt, st));
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
  LMPK_TRY(tmp_alloc(&d_slice_tile, std::max(S, 1), st));
  LMPK_TRY(tmp_alloc(&d_slice_off, std::max(S, 1), st));
  LMPK_TRY(tmp_alloc(&d_width, std::max(S, 1), st));
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
    LMPK_TRY(tmp_alloc(&d_seg_ptr, nt + 1, st));
    LMPK_TRY(tmp_alloc(&d_segs, segs.size(), st));
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
  pt.mark("alloc + fill blocks + deps");
  if ((n_comp == nt || (xs_slices > 0 && n_comp > 0)) && !xc) {
    std::vector<int32_t> tfirst(first.begin(), first.begin() + nt);
    LMPK_TRY(lean_build(ctx, T, n, row_ptr, col, val, tfirst, width, d_wmin, tmode, tdict, d_dict_tab, d_width, cap,
                        xs_slices > 0, cplx, st));
  }
  pt.mark("lean build");
  T->h_dep_lo.resize(nt);
  T->h_dep_hi.resize(nt);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->h_dep_lo.data(), T->d_dep_lo, nt * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->h_dep_hi.data(), T->d_dep_hi, nt * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  tmp_free(d_slice_tile, st);
  tmp_free(d_slice_off, st);
  tmp_free(d_width, st);
  tmp_free(d_seg_ptr, st);
  tmp_free(d_segs, st);
  tmp_free(d_tile_dict, st);
  tmp_free(d_dict_tab, st);
  T->info.n_tiles = nt;
  T->info.block_bytes = ofs;
  pt.mark("geometry D2H + frees");
  return LMPK_OK;
}

#include "mpk_dp.cuh"

// Ring walk: super-tiles (runs of consecutive tiles of ~tile_nnz_hint
// nonzeros, default 32K: cfg2's ~34K-nonzero tiles become one super-tile
// each, 0.447 vs 0.470 ms for the former 64K default that paired them; cfg5
// unchanged (309 vs 313 us), cfg1 67 -> 50 us; LMPK_SUPER_NNZ overrides), their
// dependency ranges in tiles, and the items
// (T, power) in skewed diagonal key order (T + g*M, g), M = D + slack with D
// the max forward reach in super-tiles: every dependency of an item has a
// smaller key (deadlock freedom, see mpk_ring_kernel).
static int finish_ring_tiling(lmpk_ctx* ctx, lmpk_tiling* T, int32_t p_m, const lmpk_tiling_params& prm,
                              lmpk_tiling_info* info, lmpk_tiling** out, cudaStream_t st) {
  const int32_t nt = T->info.n_tiles;
  int64_t target = 32768;
  // complex vectors double the bytes a tile touches: items of one tile keep
  // the window of blocks and vectors between a tile's consecutive powers
  // smaller (cfg5 complex Chebyshev step 3.91 -> 3.47 ms, tools/cfg5_sweep.py)
  if (prm.mode_flags & LMPK_FLAG_COMPLEX) target = 8192;
  if (prm.tile_nnz_hint > 0) target = prm.tile_nnz_hint;
  else if (const char* e = getenv("LMPK_SUPER_NNZ")) target = std::max(1, atoi(e));
  std::vector<int32_t> tE(nt);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(tE.data(), T->d_tile_E, size_t(nt) * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  std::vector<int32_t> first{0}, sup(nt);
  int64_t acc = 0;
  for (int32_t t = 0; t < nt; ++t) {
    sup[t] = static_cast<int32_t>(first.size()) - 1;
    acc += tE[t];
    if (acc >= target && t + 1 < nt) {
      first.push_back(t + 1);
      acc = 0;
    }
  }
  first.push_back(nt);
  const int32_t ns = static_cast<int32_t>(first.size()) - 1;
  std::vector<int32_t> lo(ns), hi(ns);
  int32_t D = 0;
  for (int32_t s = 0; s < ns; ++s) {
    int32_t a = first[s], b = first[s + 1] - 1;
    for (int32_t t = first[s]; t < first[s + 1]; ++t) {
      a = std::min(a, T->h_dep_lo[t]);
      b = std::max(b, T->h_dep_hi[t]);
    }
    lo[s] = a;
    hi[s] = b;
    D = std::max(D, sup[b] - s);
  }
  const int32_t G = p_m;
  // ~5 x (items in flight) / G keys: measured 1% faster than 3x on cfg2 (0.498 vs 0.504 ms)
  // lean tilings whose blocks are L2-resident anyway (pattern slices: cfg2 23.6 MB)
  // take 4x the spacing: nothing is lost to the longer reuse distance and the
  // dependency waits all but vanish (cfg2 0.381 -> 0.371 ms, tools/xlean_sweep.py SLACK)
  const int32_t mult = (T->d_lean && T->lean_bytes < (int64_t(48) << 20)) ? 20 : 5;
  int32_t slack = prm.queue_slack > 0 ? prm.queue_slack : std::max(1, (mult * T->info.grid) / G);
  if (const char* e = getenv("LMPK_RING_SLACK")) slack = std::max(1, atoi(e));  // experiments (tools/cfg5_sweep.py)
  T->info.queue_slack = G > 1 ? slack : 0;
  T->info.max_fwd_reach = D;
  T->info.super_tiles = ns;
  const int64_t M = int64_t(D) + slack;
  // power passes: the powers run in passes of qp consecutive powers, each
  // pass a diagonal wavefront of its own (key pass * BIG + s + (g mod qp) M):
  // fewer powers in flight shrink the window of blocks and vectors the L2
  // must hold between a tile's consecutive powers
  int32_t qp = G;
  if (const char* e = getenv("LMPK_PASS_POWERS")) qp = std::max(1, std::min(G, atoi(e)));
  const int64_t BIG = int64_t(ns) + int64_t(qp) * M + 1;
  std::vector<int64_t> keys;
  keys.reserve(int64_t(ns) * G);
  for (int32_t s = 0; s < ns; ++s)
    for (int32_t g = 0; g < G; ++g) keys.push_back((((g / qp) * BIG + s + (g % qp) * M) << 8) | g);
  std::vector<int32_t> order(keys.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return keys[a] < keys[b]; });
  std::vector<int32_t> items(order.size());
  for (size_t i = 0; i < order.size(); ++i) items[i] = ((order[i] / G) << 8) | (order[i] % G);
  T->n_items = static_cast<int32_t>(items.size());
  T->h_items = items;
  T->h_st_first = first;
  LMPK_TRY(dmalloc(&T->d_items, items.size()));
  LMPK_TRY(dmalloc(&T->d_st_first, ns + 1));
  LMPK_TRY(dmalloc(&T->d_st_lo, ns));
  LMPK_TRY(dmalloc(&T->d_st_hi, ns));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_items, items.data(), items.size() * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_st_first, first.data(), (ns + 1) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_st_lo, lo.data(), ns * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(T->d_st_hi, hi.data(), ns * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  LMPK_TRY(lean_worklist(T, items, first, lo, hi, T->info.grid * std::max(1, T->lean_ctas), st));
  (void)ctx;
  if (info) *info = T->info;
  *out = T;
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
  // default plan (no mode flag, no q): the ring walk over compressed tiles,
  // measured fastest on every BASELINE shape; LMPK_FLAG_PLAIN
  // keeps it on plain tile-SELL-32 blocks
  const bool default_plan = !(prm.mode_flags & (LMPK_FLAG_MODE_STREAM | LMPK_FLAG_MODE_RESIDENT | LMPK_FLAG_NO_TMA)) &&
                            prm.powers_per_item == 0;
  bool ring = (prm.mode_flags & LMPK_FLAG_RING) != 0 || default_plan;
  if (const char* e = getenv("LMPK_RING")) ring = atoi(e) != 0;
  if ((prm.mode_flags & (LMPK_FLAG_MODE_RESIDENT | LMPK_FLAG_NO_TMA)) || prm.powers_per_item > 1) ring = false;
  LMPK_ARG_CHECK(prm.slots >= 0 && prm.slots <= (ring ? kRingMax : kMaxSlots), "slots must be in [0, %d]",
                 ring ? kRingMax : kMaxSlots);
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
  LMPK_TRY(tmp_alloc(&d_w, std::max(S, 1), st));
  LMPK_TRY(tmp_alloc(&d_wmin, std::max(S, 1), st));
  LMPK_TRY(tmp_alloc(&d_fit, std::max(S, 1), st));
  struct Guard {
    int32_t *a, *b;
    uint8_t* c;
    cudaStream_t s;
    ~Guard() {
      tmp_free(a, s);
      tmp_free(b, s);
      tmp_free(c, s);
    }
  } guard{d_w, d_wmin, d_fit, st};
  // compressed blocks (int16 column offsets + value dictionary): opt-in via
  // LMPK_FLAG_COMPRESS or LMPK_COMPRESS=1; not with unstaged blocks or x staging
  bool compress = (prm.mode_flags & LMPK_FLAG_COMPRESS) != 0 ||
                  (default_plan && !(prm.mode_flags & LMPK_FLAG_PLAIN));
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
  PhaseTimer ptc(st);
  ptc.mark("slice widths (sync only)");
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
  } else if (ring) {
    cands.push_back({1, R0 ? R0 : 2});  // ring depth (pieces): 2 x ~113 KB measured best on cfg2
    if (!R0) cands.push_back({1, 3});
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
  const bool xstage = !unstaged && !(prm.mode_flags & LMPK_FLAG_COMPLEX) && xfrac > 0 && n > 0;
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
  // Lean x staging (ring tilings of matrices with rows <= 8 entries, the
  // default): tiles are capped at R rows so that a tile's lean block and the
  // runs of y_{p-1} its rows gather share one ring piece (lean_build).  R is
  // the largest candidate whose x buffers (k_lean_xplan on a fixed-R grid)
  // leave room for the blocks at ring depth 2; the block estimate takes the
  // dictionary format when the first rows hold <= kDictMax distinct values.
  int32_t xs_slices = 0;
  int64_t xs_bcap = 0;
  const bool cplx_t = (prm.mode_flags & LMPK_FLAG_COMPLEX) != 0;
  if (ring && compress && !xstage && max_row >= 1 && max_row <= 8 && n > 0 && lean_xs_wanted()) {
    bool dictish = false;
    {
      const int32_t ns = std::min<int32_t>(h_nnz, 32768);
      std::vector<double> hv(ns);
      if (ns > 0) LMPK_CHECK_CUDA(cudaMemcpyAsync(hv.data(), val, size_t(ns) * 8, cudaMemcpyDeviceToHost, st));
      LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
      std::vector<uint64_t> bits(ns);
      if (ns > 0) memcpy(bits.data(), hv.data(), size_t(ns) * 8);
      std::sort(bits.begin(), bits.end());
      dictish = std::unique(bits.begin(), bits.end()) - bits.begin() <= kDictMax;
    }
    std::vector<int32_t> rows_c{1664, 832, 416};
    if (const char* e = getenv("LMPK_XLEAN_ROWS")) rows_c = {std::max(32, atoi(e) & ~31)};
    const int64_t slice_b = 16 + lean_col_bytes(max_row) + (dictish ? lean_code_bytes(max_row) : lean_raw_bytes(max_row));
    for (int32_t R : rows_c) {
      const int32_t ntf = (n + R - 1) / R;
      std::vector<int32_t> trow(ntf + 1);
      for (int32_t t = 0; t <= ntf; ++t) trow[t] = std::min<int64_t>(int64_t(t) * R, n);
      int32_t* d_trow = nullptr;
      LMPK_TRY(dmalloc(&d_trow, ntf + 1));
      LMPK_CHECK_CUDA(cudaMemcpyAsync(d_trow, trow.data(), size_t(ntf + 1) * 4, cudaMemcpyHostToDevice, st));
      int4* d_runs = nullptr;
      int2* d_xinfo = nullptr;
      int32_t mx = -1;
      const int rc = lean_xplan(ctx, n, row_ptr, col, d_trow, ntf, cplx_t, &d_runs, &d_xinfo, &mx, st);
      cudaFree(d_trow);
      cudaFree(d_runs);
      cudaFree(d_xinfo);
      if (rc != LMPK_OK) return rc;
      if (mx < 0) continue;
      // 12% headroom: the real tiles are cut by bytes too and need not sit on the R grid
      const int64_t xb = ((int64_t(mx) * (cplx_t ? 16 : 8) * 112 / 100) + 127) & ~int64_t(127);
      const int64_t bcap = (lean_xs_budget(ctx) / 2 - xb) & ~int64_t(127);
      if (bcap < kLeanRec + int64_t(R / 32) * slice_b + 256) continue;
      xs_slices = R / 32;
      xs_bcap = bcap;
      break;
    }
  }
  // DP tiling (mpk_dp.cuh): rows of <= 8 entries whose values defeat the
  // per-tile dictionaries -- or whose column offsets defeat int16 -- but whose
  // off-diagonal values come from one small global dictionary (stencil +
  // potential: cfg5's Anderson operator; constant stencils on periodic grids)
  if (default_plan && ring && compress && !xstage && !unstaged && xs_slices == 0 && n > 0 && prm.slots == 0 &&
      prm.tile_nnz_hint == 0 && max_row >= 1 && max_row <= 8) {
    bool dictish = false;
    {
      const int32_t ns = std::min<int32_t>(h_nnz, 32768);
      std::vector<uint64_t> bits(ns);
      if (ns > 0) LMPK_CHECK_CUDA(cudaMemcpyAsync(bits.data(), val, size_t(ns) * 8, cudaMemcpyDeviceToHost, st));
      LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
      std::sort(bits.begin(), bits.end());
      dictish = std::unique(bits.begin(), bits.end()) - bits.begin() <= kDictMax;
    }
    // a value set that fits the per-tile dictionaries keeps the lean blocks --
    // unless some slice's column offsets exceed int16 (periodic grids: those
    // tiles would stay plain and the tiling would lose its lean blocks)
    bool any_unfit = false;
    for (uint8_t f : fit16) any_unfit = any_unfit || f == 0;
    if (dp_wanted(max_row, dictish && !any_unfit)) {
      lmpk_tiling* D = nullptr;
      LMPK_TRY(dp_build(ctx, n, row_ptr, col, val, width, d_w, d_wmin, cplx_t, st, &D));
      if (D) {
        D->info.p_m = p_m;
        D->info.mode = 3;
        D->info.block = 32 * (kLeanConsumers + 2);
        D->ring = true;
        D->piece = D->lean_piece;
        D->slots = 2;
        D->info.smem_bytes = 2 * D->lean_piece;
        D->info.tile_nnz_cap = 0;
        D->info.chain_reach = chain_reach(D->h_dep_hi, p_m - 1, nullptr);
        D->info.max_row_nnz = max_row;
        D->info.nnz = h_nnz;
        D->info.grid = ctx->sm_count;
        D->info.powers_per_item = 1;
        D->info.slots = 2;
        ptc.mark("dp_build");
        const int rc = finish_ring_tiling(ctx, D, p_m, prm, info, out, st);
        if (rc != LMPK_OK) lmpk_tiling_destroy(D);
        ptc.mark("finish_ring_tiling");
        return rc;
      }
    }
  }
  for (const Cand& cd : cands) {
    const int64_t slot = std::min<int64_t>(unstaged ? per_cta / 2 : per_cta / cd.slots, slot_cap) & ~int64_t(127);
    int64_t cap = slot;  // with x staging the slot holds [block | x buffer] (build_tiling)
    // ring: tile_nnz_hint sizes the super-tiles, the tiles fill one piece
    if (prm.tile_nnz_hint > 0 && !compress && !ring)
      cap = std::min<int64_t>(cap, int64_t(prm.tile_nnz_hint) * 12 + 2048);
    const int64_t e_cap = (compress && !ring && prm.tile_nnz_hint > 0) ? int64_t(prm.tile_nnz_hint) : INT64_MAX;
    if (xs_slices > 0) cap = std::min(cap, xs_bcap);
    cap &= ~int64_t(127);
    if (cap < 2048) continue;
    const int64_t xoff = 0;
    const int smem_need = unstaged ? 0 : static_cast<int>(cap);
    int occ = 0;
    if (ring)
      LMPK_TRY(ring_occupancy(ctx, smem_need * cd.slots, &occ));
    else
      LMPK_TRY(group_occupancy(ctx, unstaged ? 0 : smem_need * cd.slots, &occ));
    if (occ < 1) continue;
    lmpk_tiling* cand = new lmpk_tiling();
    cand->ctx = ctx;
    cand->n = n;
    const int rc = build_tiling(ctx, cand, n, row_ptr, col, val, width, d_wmin, cap, xstage ? &h_rp : nullptr,
                                xstage ? &h_col : nullptr, xstage, compress ? &fit16 : nullptr, e_cap, st,
                                xs_slices, cplx_t);
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
                    (cd.q == 1 || unstaged || cand->max_block <= cap);
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
  T->info.mode = ring ? 3 : (q_used == p_m ? 1 : 2);
  T->info.block = ring ? 32 * (kRingConsumers + 2) : 32 * (kConsumers + slots);
  T->ring = ring;
  T->piece = static_cast<int32_t>(cap_used);
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
  ptc.mark("candidates / build_tiling");
  if (ring) {
    const int rc = finish_ring_tiling(ctx, T, p_m, prm, info, out, st);
    ptc.mark("finish_ring_tiling");
    return rc;
  }
  // skewed diagonal key (t + g*M, g), M = q*D + slack
  const int32_t G = (p_m + q_used - 1) / q_used;
  // default slack ~3 * (items in flight) / G: the dependency of an item must
  // have left the queue >= ~2 item durations earlier (measured on cfg2)
  const int32_t slack = prm.queue_slack > 0 ? prm.queue_slack : std::max(1, (3 * grid * slots) / G);
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
  T->h_items = items;
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

// The item queue as (tile, first power, powers) triples in queue order: ring
// tilings expand a super-tile item into its tiles; the group walk's items
// cover powers_per_item consecutive powers of one tile.
extern "C" int lmpk_tiling_items(const lmpk_tiling* t, int32_t* out, int64_t cap, int64_t* n_out) {
  LMPK_ARG_CHECK(t != nullptr && n_out != nullptr, "lmpk_tiling_items: NULL argument");
  const int32_t q = t->ring ? 1 : std::max(1, t->info.powers_per_item);
  int64_t k = 0;
  for (int32_t it : t->h_items) {
    const int32_t s = it >> 8, g = it & 0xff;
    const int32_t t0 = t->ring ? t->h_st_first[s] : s, t1 = t->ring ? t->h_st_first[s + 1] : s + 1;
    const int32_t p0 = g * q + 1, np_ = std::min(q, t->info.p_m - g * q);
    for (int32_t tt = t0; tt < t1; ++tt, ++k)
      if (out && k < cap) {
        out[3 * k] = tt;
        out[3 * k + 1] = p0;
        out[3 * k + 2] = np_;
      }
  }
  *n_out = k;
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
    static bool dyn_set[4] = {false, false, false, false};
    const int di = (cplx ? 2 : 0) + (exact ? 1 : 0);
    if (!dyn_set[di]) {  // a ring tiling's sweep may be this kernel's first launch
      cudaFuncAttributes fa;
      LMPK_CHECK_CUDA(cudaFuncGetAttributes(&fa, fn));
      LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes)));
      dyn_set[di] = true;
    }
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

static int launch_ring(lmpk_ctx* ctx, MpkParams& Pm, PowerCfgDev& C, bool cplx, bool exact, bool has_long,
                       int uniform, int grid, int smem, cudaStream_t st) {
  void* args[] = {&Pm, &C};
  const void* fn = ring_fn(cplx, exact, has_long, uniform);
  {
    static int last[32];
    static bool init = false;
    if (!init) {
      for (int& v : last) v = -1;
      init = true;
    }
    const int idx = uniform * 8 + (has_long ? 4 : 0) + (cplx ? 2 : 0) + (exact ? 1 : 0);
    cudaFuncAttributes fa;
    LMPK_CHECK_CUDA(cudaFuncGetAttributes(&fa, fn));
    static bool dyn_set[32] = {};
    if (!dyn_set[idx]) {  // every variant may be launched without an occupancy query first
      LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           ctx->max_smem_block - static_cast<int>(fa.sharedSizeBytes)));
      dyn_set[idx] = true;
    }
    const int per_sm = std::max(1, ctx->max_smem_sm);
    const int pct = std::min(100, int((int64_t(smem + int(fa.sharedSizeBytes) + 1024) * 100 + per_sm - 1) / per_sm));
    if (last[idx] != pct) {
      LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct));
      last[idx] = pct;
    }
  }
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(32 * (kRingConsumers + 2)), args, smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("mpk ring launch failed: %s (grid %d, smem %d)", cudaGetErrorString(e), grid, smem);
    return LMPK_ERR_CUDA;
  }
  launch_count_add(ctx, 1);
  // the producer ends with exactly one failing grab
  ctx->queue_base += uint64_t(Pm.n_items) + uint64_t(grid);
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
  Pm.blk_cap = Pm.smem_cap;
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
  if (const char* e = getenv("LMPK_ACQ")) Pm.flags |= atoi(e) == 0 ? kFlagNoAcqFence : (atoi(e) == 1 ? kFlagAcqLoads : 0);
  if (const char* e = getenv("LMPK_YPOL")) Pm.ypol = atoi(e);
  Pm.err = ctx->err.dev;
  Pm.prof = ctx->prof;
  Pm.trace = (ctx->prof && ctx->prof_words > 16) ? reinterpret_cast<uint4*>(ctx->prof + 16) : nullptr;
  const int grid = T->info.grid;
  if (T->ring) {
    Pm.st_first = T->d_st_first;
    Pm.st_lo = T->d_st_lo;
    Pm.st_hi = T->d_st_hi;
    Pm.smem_cap = T->piece;
    Pm.blk_cap = T->piece;
  }
  if (sweep && T->lean_vd == 2) {
    // DP tilings hold lean blocks only: a sweep is one lean launch per power
    // over the power-1 items (no dependencies), each with an epoch of its own
    for (int i = 0; i < P; ++i) {
      PowerCfgDev Ci;
      memset(&Ci, 0, sizeof(Ci));
      Ci.out_slot[0] = C.out_slot[i];
      Ci.in_slot[0] = C.in_slot[i];
      Ci.prev_slot[0] = C.prev_slot[i];
      Ci.kernel[0] = C.kernel[i];
      Ci.coef_re[0] = C.coef_re[i];
      Ci.coef_im[0] = C.coef_im[i];
      ctx->epoch += 1;
      if (ctx->epoch >= (1u << 24)) {
        ctx->epoch = 1;
        ctx->wrap_gen += 1;
      }
      if (Tm->wrap_gen != ctx->wrap_gen) {
        LMPK_CHECK_CUDA(cudaMemsetAsync(Tm->d_progress, 0, size_t(T->info.n_tiles) * 4, st));
        Tm->wrap_gen = ctx->wrap_gen;
      }
      Pm.epoch_base = ctx->epoch * kEpochStride;
      Pm.queue_base = ctx->queue_base;
      Pm.n_powers = 1;
      Pm.mode = 1;
      Pm.items = T->d_items;
      Pm.q = 1;
      Pm.n_items = T->n_items;
      Pm.n_tiles = T->info.n_tiles;
      LMPK_TRY(launch_lean(ctx, T, Pm, Ci, cplx, exact, use_acc || Ci.kernel[0] != LMPK_KERNEL_SPMV, grid, st));
    }
    return LMPK_OK;
  }
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
      if (T->ring) Pm.n_slots = std::min(T->slots, kMaxSlots);  // the sweep runs on the group kernel
      LMPK_TRY(launch_group(ctx, Pm, Ci, cplx, exact, false, std::min(grid, T->info.n_tiles),
                            (flags & LMPK_FLAG_NO_TMA) ? 0 : (T->ring ? Pm.n_slots * T->piece : T->info.smem_bytes),
                            st));
    }
    return LMPK_OK;
  }
  ctx->epoch += 1;
  if (ctx->epoch >= (1u << 24)) {  // counter wrap: a new generation of epochs
    ctx->epoch = 1;
    ctx->wrap_gen += 1;
  }
  // a tiling whose progress words predate the last wrap (possibly many
  // launches of other tilings ago) would hold tags up to 2^31 that pass
  // every wait of the new generation: clear them first
  if (Tm->wrap_gen != ctx->wrap_gen) {
    LMPK_CHECK_CUDA(cudaMemsetAsync(Tm->d_progress, 0, size_t(T->info.n_tiles) * 4, st));
    Tm->wrap_gen = ctx->wrap_gen;
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
  if (T->ring) {
    LMPK_ARG_CHECK(!(flags & (LMPK_FLAG_NO_TMA | LMPK_FLAG_READY_QUEUE)),
                   "the ring walk has no unstaged / ready-queue variant");
    // a kernel carrying one tile body when every tile has the same format
    int uniform = 0;
    if (T->staged_tiles == 0 && getenv("LMPK_NO_UNIFORM_KERNEL") == nullptr) {
      bool plain = !use_acc;
      for (int i = 0; i < P; ++i) plain = plain && C.kernel[i] == LMPK_KERNEL_SPMV;
      if (T->info.dict_tiles == T->info.n_tiles)
        uniform = (plain && !cplx && T->slots == 2) ? 3 : 1;  // the plain kernel assumes the 2-piece ring
      else if (T->info.compressed_tiles == T->info.n_tiles && T->info.dict_tiles == 0)
        uniform = 2;
    }
    if (T->d_lean && T->staged_tiles == 0 && T->slots == 2 &&
        (T->lean_vd == 2 || (!getenv("LMPK_NO_LEAN_RUN") && lean_xs_runnable(T, y, ldy, cplx)))) {
      bool plain = !use_acc;
      for (int i = 0; i < P; ++i) plain = plain && C.kernel[i] == LMPK_KERNEL_SPMV;
      return launch_lean(ctx, T, Pm, C, cplx, exact, !plain, grid, st);
    }
    return launch_ring(ctx, Pm, C, cplx, exact, T->info.max_row_nnz > 8, uniform, grid, T->info.smem_bytes, st);
  }
  // co-residency of all CTAs is part of the deadlock-freedom argument.
  // LMPK_FLAG_NO_TMA: blocks are streamed from global memory by the
  // consumers, so no slot buffers -- the unified L1 is left to the gathers.
  const bool no_tma = (flags & LMPK_FLAG_NO_TMA) != 0;
  return launch_group(ctx, Pm, C, cplx, exact, true, grid, no_tma ? 0 : T->info.smem_bytes, st);
}

extern "C" int64_t lmpk_ctx_set_epoch(lmpk_ctx* ctx, int64_t epoch) {
  if (!ctx) return -1;
  const int64_t old = ctx->epoch;
  ctx->epoch = static_cast<uint32_t>(std::max<int64_t>(0, std::min<int64_t>(epoch, (1 << 24) - 1)));
  return old;
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

