// radix_sort.cuh -- device-wide primitives written for liblmpk (no CUB):
//   * exclusive scan (int32/int64 inputs, int64 accumulation)
//   * stable LSD radix sort of (uint32 key, uint32 value) pairs, 8-bit digits
// Stability is what makes the BFS ordering bit-exact: sorting vertex ids by
// level id while they enter in id order reproduces "each level sorted
// ascending" of pkg/src/levelmpk/levels.py:94.
#pragma once
#include "lmpk_internal.cuh"

namespace lmpk {
namespace {  // internal linkage: included by several translation units

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// block-wide exclusive scan of one value per thread; returns exclusive prefix,
// *total receives the block sum.  blockDim.x must be a multiple of 32 (<=1024).
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* total) {
  __shared__ T s_warp[32];
  __shared__ T s_total;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? s_warp[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < nw) s_warp[lane] = wi - w;
    if (lane == 31) s_total = wi;  // lanes >= nw contribute 0
  }
  __syncthreads();
  T res = inc - v + s_warp[warp];
  if (total) *total = s_total;
  __syncthreads();
  return res;
}

template <typename TIn>
__global__ void k_scan_partials(const TIn* in, int64_t n, int64_t* partials) {
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  int64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + int64_t(i) * kScanThreads + threadIdx.x;
    if (idx < n) s += int64_t(in[idx]);
  }
  int64_t tot;
  block_excl_scan<int64_t>(s, &tot);
  if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// single block, loops over the partials
__global__ void k_scan_partials_scan(int64_t* partials, int64_t nb, int64_t init) {
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = init;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? partials[i] : 0;
    int64_t tot;
    int64_t ex = block_excl_scan<int64_t>(v, &tot);
    if (i < nb) partials[i] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// out[i] = init + sum_{j<i} in[j]; out may have n+1 entries (write_total)
template <typename TIn, typename TOut>
__global__ void k_scan_final(const TIn* in, int64_t n, const int64_t* partials, TOut* out,
                             int write_total) {
  __shared__ int64_t s_items[kScanTile];
  const int64_t base = int64_t(blockIdx.x) * kScanTile;
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + int64_t(i) * kScanThreads + threadIdx.x;
    s_items[i * kScanThreads + threadIdx.x] = idx < n ? int64_t(in[idx]) : 0;
  }
  __syncthreads();
  // each thread scans kScanItems consecutive elements
  int64_t loc[kScanItems];
  int64_t s = 0;
  for (int i = 0; i < kScanItems; ++i) {
    loc[i] = s;
    s += s_items[threadIdx.x * kScanItems + i];
  }
  int64_t tot;
  int64_t ex = block_excl_scan<int64_t>(s, &tot) + partials[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + int64_t(threadIdx.x) * kScanItems + i;
    if (idx < n) out[idx] = TOut(ex + loc[i]);
  }
  if (write_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == blockDim.x - 1)
    out[n] = TOut(ex + s);
}

// Exclusive scan with `init`; when write_total, out[n] = init + sum(in).
// tmp must hold ceil(n / kScanTile) int64.
template <typename TIn, typename TOut>
inline int device_excl_scan(lmpk_ctx* ctx, const TIn* in, int64_t n, TOut* out, int64_t init,
                            bool write_total, int64_t* tmp, cudaStream_t st) {
  const int64_t nb = n > 0 ? (n + kScanTile - 1) / kScanTile : 1;
  if (n > 0) k_scan_partials<TIn><<<int(nb), kScanThreads, 0, st>>>(in, n, tmp);
  else cudaMemsetAsync(tmp, 0, 8, st);
  k_scan_partials_scan<<<1, 1024, 0, st>>>(tmp, nb, init);
  k_scan_final<TIn, TOut><<<int(nb), kScanThreads, 0, st>>>(in, n, tmp, out, write_total ? 1 : 0);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 3);
  return LMPK_OK;
}

// ----------------------------------------------------------------- radix sort
constexpr int kSortThreads = 256;
constexpr int kSortRounds = 16;  // elements per block = 256 * 16
constexpr int kSortTile = kSortThreads * kSortRounds;

__global__ void k_radix_hist(const uint32_t* keys, int64_t n, int shift, uint32_t* counts,
                             int nblocks) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
  for (int r = 0; r < kSortRounds; ++r) {
    int64_t i = base + int64_t(r) * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  counts[int64_t(threadIdx.x) * nblocks + blockIdx.x] = h[threadIdx.x];  // digit-major
}

__global__ void k_radix_scatter(const uint32_t* kin, const uint32_t* vin, uint32_t* kout,
                                uint32_t* vout, int64_t n, int shift, const int64_t* offsets,
                                int nblocks) {
  __shared__ uint32_t s_run[256];      // running count per digit within this tile
  __shared__ uint32_t s_wc[8][256];    // per-warp digit counts of the current round
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  s_run[threadIdx.x] = 0;
  const int64_t gofs = offsets[int64_t(threadIdx.x) * nblocks + blockIdx.x];
  __shared__ int64_t s_gofs[256];
  s_gofs[threadIdx.x] = gofs;
  const int64_t base = int64_t(blockIdx.x) * kSortTile;
  for (int r = 0; r < kSortRounds; ++r) {
#pragma unroll
    for (int w = 0; w < 8; ++w) s_wc[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = base + int64_t(r) * kSortThreads + threadIdx.x;
    const bool valid = i < n;
    uint32_t k = 0, v = 0, d = 0xffffffffu;
    if (valid) {
      k = kin[i];
      v = vin[i];
      d = (k >> shift) & 255u;
    }
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t rank_w = __popc(peers & lt);
    if (valid && rank_w == 0) s_wc[warp][d] = __popc(peers);  // leader records group size
    __syncthreads();
    // exclusive prefix over warps for this lane's digit
    uint32_t before = 0;
    if (valid) {
      for (int w = 0; w < warp; ++w) before += s_wc[w][d];
    }
    const uint32_t pos_in_tile = valid ? s_run[d] + before + rank_w : 0;
    __syncthreads();
    // advance the running counts: thread t owns digit t
    {
      uint32_t add = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) add += s_wc[w][threadIdx.x];
      s_run[threadIdx.x] += add;
    }
    if (valid) {
      const int64_t dst = s_gofs[d] + pos_in_tile;
      kout[dst] = k;
      vout[dst] = v;
    }
    __syncthreads();
  }
}

// Stable sort of n (key, value) pairs by the low `bits` key bits.  Buffers
// k0/v0 hold the input; the result lands in (k0, v0) if the number of passes
// is even, else in (k1, v1): *out_in_first says which.
// counts must hold 256 * nblocks uint32, offsets 256 * nblocks int64 and
// scan_tmp ceil(256*nblocks / kScanTile) int64.
inline int device_radix_sort(lmpk_ctx* ctx, uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                             int64_t n, int bits, uint32_t* counts, int64_t* offsets,
                             int64_t* scan_tmp, bool* out_in_first, cudaStream_t st) {
  *out_in_first = true;
  if (n <= 1 || bits <= 0) return LMPK_OK;
  const int nblocks = int((n + kSortTile - 1) / kSortTile);
  uint32_t *ka = k0, *va = v0, *kb = k1, *vb = v1;
  for (int shift = 0; shift < bits; shift += 8) {
    k_radix_hist<<<nblocks, kSortThreads, 0, st>>>(ka, n, shift, counts, nblocks);
    launch_count_add(ctx, 1);
    LMPK_TRY(device_excl_scan<uint32_t, int64_t>(ctx, counts, int64_t(256) * nblocks, offsets, 0,
                                                 false, scan_tmp, st));
    k_radix_scatter<<<nblocks, kSortThreads, 0, st>>>(ka, va, kb, vb, n, shift, offsets, nblocks);
    launch_count_add(ctx, 1);
    LMPK_CHECK_CUDA(cudaGetLastError());
    uint32_t* t = ka;
    ka = kb;
    kb = t;
    t = va;
    va = vb;
    vb = t;
    *out_in_first = !*out_in_first;
  }
  return LMPK_OK;
}

inline int64_t radix_counts_len(int64_t n) { return int64_t(256) * ((n + kSortTile - 1) / kSortTile); }
inline int64_t scan_tmp_len(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

}  // namespace
}  // namespace lmpk
