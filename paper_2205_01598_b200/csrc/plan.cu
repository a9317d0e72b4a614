// plan.cu -- dependency analysis of flat execution plans on the GPU
// (lmpk_plan.h): the true dependencies of an item list (reference
// pkg/src/levelmpk/plan.py:103-129, a per-item np.unique over all read
// columns: 15-37 s on the BASELINE shapes) and the column maximum inside a
// target row range that decides BOUNDARY-granular checks (plan.py:356-365).
//
// Items of one power are disjoint row intervals, so "who owns column c at
// power p-1" is a binary search in that power's sorted interval starts.  Each
// item gets a bitmap row over the intervals of the previous power; chunks of
// <= kChunkRows rows of an item are processed by one CTA that strides its
// threads over the chunk's nonzeros, and a bit is set with atomicOr only when
// a thread meets an interval it has not just seen.
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <vector>

#include "lmpk_internal.cuh"
#include "lmpk_plan.h"

namespace lmpk {
namespace {

constexpr int kChunkRows = 512;
constexpr int kPlanThreads = 256;

struct ItemDesc {
  int64_t bm_off;   // first bitmap word of the item (-1: no previous power)
  int32_t iv_off;   // interval table of the previous power
  int32_t iv_cnt;
};

struct Chunk {
  int32_t item, r0, r1;
};

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  int alloc(size_t bytes) {
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) {
      set_error("plan scratch cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
      p = nullptr;
      return LMPK_ERR_NOMEM;
    }
    return LMPK_OK;
  }
  template <typename T>
  T* as() {
    return reinterpret_cast<T*>(p);
  }
};

// index of the interval of [ivs, ive) (sorted, disjoint) containing c, or -1
__device__ __forceinline__ int32_t find_interval(const int32_t* ivs, const int32_t* ive, int32_t cnt, int32_t c) {
  int32_t lo = 0, hi = cnt;  // last start <= c
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if (ivs[mid] <= c) lo = mid + 1;
    else hi = mid;
  }
  const int32_t i = lo - 1;
  return (i >= 0 && c < ive[i]) ? i : -1;
}

__global__ void __launch_bounds__(kPlanThreads)
k_item_deps(const int32_t* row_ptr, const int32_t* col, const Chunk* chunks, int64_t n_chunks,
            const ItemDesc* items, const int32_t* ivs, const int32_t* ive, uint32_t* bitmap) {
  for (int64_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const Chunk ch = chunks[ci];
    const ItemDesc it = items[ch.item];
    if (it.bm_off < 0) continue;
    const int32_t* s = ivs + it.iv_off;
    const int32_t* e = ive + it.iv_off;
    uint32_t* bm = bitmap + it.bm_off;
    int32_t last = -1, last_lo = 0, last_hi = 0;
    auto mark = [&](int32_t c) {
      if (last >= 0 && c >= last_lo && c < last_hi) return;
      const int32_t i = find_interval(s, e, it.iv_cnt, c);
      if (i < 0) return;
      last = i;
      last_lo = s[i];
      last_hi = e[i];
      const uint32_t bit = 1u << (i & 31);
      if (!(bm[i >> 5] & bit)) atomicOr(bm + (i >> 5), bit);
    };
    for (int32_t r = ch.r0 + threadIdx.x; r < ch.r1; r += blockDim.x) mark(r);  // own rows
    const int64_t k0 = row_ptr[ch.r0], k1 = row_ptr[ch.r1];
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) mark(col[k]);
  }
}

__global__ void __launch_bounds__(kPlanThreads)
k_item_col_max(const int32_t* row_ptr, const int32_t* col, const Chunk* chunks, int64_t n_chunks,
               const int32_t* col_lo, const int32_t* col_hi, int32_t* out_max) {
  __shared__ int32_t s_best;
  for (int64_t ci = blockIdx.x; ci < n_chunks; ci += gridDim.x) {
    const Chunk ch = chunks[ci];
    const int32_t lo = col_lo[ch.item], hi = col_hi[ch.item];
    if (threadIdx.x == 0) s_best = -1;
    __syncthreads();
    int32_t best = -1;
    if (lo < hi) {
      const int64_t k0 = row_ptr[ch.r0], k1 = row_ptr[ch.r1];
      for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        const int32_t c = col[k];
        if (c >= lo && c < hi) best = max(best, c);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best >= 0) atomicMax(&s_best, best);
    __syncthreads();
    if (threadIdx.x == 0 && s_best >= 0) atomicMax(out_max + ch.item, s_best);
    __syncthreads();
  }
}

static void make_chunks(int64_t n_items, const int64_t* rs, const int64_t* re, std::vector<Chunk>& out) {
  for (int64_t u = 0; u < n_items; ++u)
    for (int64_t r = rs[u]; r < re[u]; r += kChunkRows)
      out.push_back({int32_t(u), int32_t(r), int32_t(std::min<int64_t>(r + kChunkRows, re[u]))});
}

}  // namespace
}  // namespace lmpk

using namespace lmpk;

extern "C" void lmpk_host_free(void* p) { free(p); }

extern "C" int lmpk_item_deps(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col, int64_t n_items,
                              const int64_t* row_start, const int64_t* row_end, const int64_t* power,
                              int64_t* dep_ptr, int64_t** dep_out, void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && col && dep_ptr && dep_out, "lmpk_item_deps: NULL argument");
  LMPK_ARG_CHECK(n_items >= 0 && (n_items == 0 || (row_start && row_end && power)), "lmpk_item_deps: bad items");
  cudaStream_t st = as_stream(stream);
  *dep_out = nullptr;
  dep_ptr[0] = 0;
  if (n_items == 0) return LMPK_OK;
  // items of each power, sorted by first row
  std::map<int64_t, std::vector<int32_t>> by_power;
  for (int64_t u = 0; u < n_items; ++u) {
    LMPK_ARG_CHECK(0 <= row_start[u] && row_start[u] <= row_end[u] && row_end[u] <= n,
                   "item %lld: rows [%lld, %lld) out of range", (long long)u, (long long)row_start[u],
                   (long long)row_end[u]);
    if (row_end[u] > row_start[u]) by_power[power[u]].push_back(int32_t(u));
  }
  std::vector<int32_t> ivs, ive, iv_item;
  std::map<int64_t, std::pair<int32_t, int32_t>> table;  // power -> (offset, count)
  for (auto& kv : by_power) {
    auto& v = kv.second;
    std::sort(v.begin(), v.end(), [&](int32_t a, int32_t b) { return row_start[a] < row_start[b]; });
    table[kv.first] = {int32_t(ivs.size()), int32_t(v.size())};
    for (size_t i = 0; i < v.size(); ++i) {
      LMPK_ARG_CHECK(i == 0 || row_end[v[i - 1]] <= row_start[v[i]], "items of power %lld overlap",
                     (long long)kv.first);
      ivs.push_back(int32_t(row_start[v[i]]));
      ive.push_back(int32_t(row_end[v[i]]));
      iv_item.push_back(v[i]);
    }
  }
  std::vector<ItemDesc> desc(n_items);
  int64_t words = 0;
  for (int64_t u = 0; u < n_items; ++u) {
    auto f = table.find(power[u] - 1);
    if (f == table.end() || row_end[u] <= row_start[u]) {
      desc[u] = {-1, 0, 0};
    } else {
      desc[u] = {words, f->second.first, f->second.second};
      words += (f->second.second + 31) / 32;
    }
  }
  std::vector<uint32_t> h_bm(std::max<int64_t>(words, 1), 0);
  if (words > 0) {
    std::vector<Chunk> chunks;
    make_chunks(n_items, row_start, row_end, chunks);
    DevBuf d_chunks, d_desc, d_iv, d_bm;
    LMPK_TRY(d_chunks.alloc(chunks.size() * sizeof(Chunk)));
    LMPK_TRY(d_desc.alloc(desc.size() * sizeof(ItemDesc)));
    LMPK_TRY(d_iv.alloc(ivs.size() * 8));
    LMPK_TRY(d_bm.alloc(size_t(words) * 4));
    int32_t* d_ivs = d_iv.as<int32_t>();
    int32_t* d_ive = d_ivs + ivs.size();
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_chunks.p, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_desc.p, desc.data(), desc.size() * sizeof(ItemDesc), cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_ivs, ivs.data(), ivs.size() * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(d_ive, ive.data(), ive.size() * 4, cudaMemcpyHostToDevice, st));
    LMPK_CHECK_CUDA(cudaMemsetAsync(d_bm.p, 0, size_t(words) * 4, st));
    const int grid = int(std::min<int64_t>(int64_t(chunks.size()), int64_t(ctx->sm_count) * 16));
    k_item_deps<<<grid, kPlanThreads, 0, st>>>(row_ptr, col, d_chunks.as<Chunk>(), int64_t(chunks.size()),
                                               d_desc.as<ItemDesc>(), d_ivs, d_ive, d_bm.as<uint32_t>());
    launch_count_add(ctx, 1);
    LMPK_CHECK_CUDA(cudaGetLastError());
    LMPK_CHECK_CUDA(cudaMemcpyAsync(h_bm.data(), d_bm.p, size_t(words) * 4, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  // decode: interval ranks -> item indices, ascending per item
  std::vector<int64_t> deps;
  std::vector<int64_t> row;
  for (int64_t u = 0; u < n_items; ++u) {
    if (desc[u].bm_off >= 0) {
      row.clear();
      const uint32_t* bm = h_bm.data() + desc[u].bm_off;
      const int32_t nw = (desc[u].iv_cnt + 31) / 32;
      for (int32_t w = 0; w < nw; ++w) {
        uint32_t m = bm[w];
        while (m) {
          const int b = __builtin_ctz(m);
          m &= m - 1;
          row.push_back(iv_item[desc[u].iv_off + w * 32 + b]);
        }
      }
      std::sort(row.begin(), row.end());
      deps.insert(deps.end(), row.begin(), row.end());
    }
    dep_ptr[u + 1] = int64_t(deps.size());
  }
  int64_t* out = static_cast<int64_t*>(malloc(std::max<size_t>(deps.size(), 1) * 8));
  if (!out) {
    set_error("lmpk_item_deps: host allocation failed");
    return LMPK_ERR_NOMEM;
  }
  std::copy(deps.begin(), deps.end(), out);
  *dep_out = out;
  return LMPK_OK;
}

extern "C" int lmpk_item_col_max_in_range(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col,
                                          int64_t n_items, const int64_t* row_start, const int64_t* row_end,
                                          const int64_t* col_lo, const int64_t* col_hi, int32_t* out_max,
                                          void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && col && out_max, "lmpk_item_col_max_in_range: NULL argument");
  if (n_items <= 0) return LMPK_OK;
  LMPK_ARG_CHECK(row_start && row_end && col_lo && col_hi, "lmpk_item_col_max_in_range: NULL item arrays");
  cudaStream_t st = as_stream(stream);
  std::vector<Chunk> chunks;
  std::vector<int64_t> rs(n_items), re(n_items);
  std::vector<int32_t> lo(n_items), hi(n_items);
  for (int64_t u = 0; u < n_items; ++u) {
    lo[u] = int32_t(col_lo[u]);
    hi[u] = int32_t(col_hi[u]);
    rs[u] = row_start[u];
    re[u] = lo[u] < hi[u] ? row_end[u] : row_start[u];  // nothing to scan for empty ranges
    out_max[u] = -1;
  }
  make_chunks(n_items, rs.data(), re.data(), chunks);
  if (chunks.empty()) return LMPK_OK;
  DevBuf d_chunks, d_rng, d_out;
  LMPK_TRY(d_chunks.alloc(chunks.size() * sizeof(Chunk)));
  LMPK_TRY(d_rng.alloc(size_t(n_items) * 8));
  LMPK_TRY(d_out.alloc(size_t(n_items) * 4));
  int32_t* d_lo = d_rng.as<int32_t>();
  int32_t* d_hi = d_lo + n_items;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_chunks.p, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_lo, lo.data(), size_t(n_items) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(d_hi, hi.data(), size_t(n_items) * 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_out.p, 0xff, size_t(n_items) * 4, st));
  const int grid = int(std::min<int64_t>(int64_t(chunks.size()), int64_t(ctx->sm_count) * 16));
  k_item_col_max<<<grid, kPlanThreads, 0, st>>>(row_ptr, col, d_chunks.as<Chunk>(), int64_t(chunks.size()), d_lo,
                                                d_hi, d_out.as<int32_t>());
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  LMPK_CHECK_CUDA(cudaMemcpyAsync(out_max, d_out.p, size_t(n_items) * 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  return LMPK_OK;
}
