// bfs.cu -- BFS level construction and level ordering on sm_100a.
//
// Reference semantics (pkg/src/levelmpk/levels.py:48-114):
//   * traverse the symmetrized pattern A|A^T (levels.py:48-61);
//   * level 0 = {root}; level i+1 = sorted unvisited neighbours of level i;
//   * when a component is exhausted, restart at the lowest unvisited vertex.
// Restated (bit-exact): perm = stable sort of vertex ids by
// the key (component rank, BFS distance), where the root's component ranks
// first and the remaining components follow in order of their minimum
// vertex, each traversed from that minimum vertex.  The lowest unvisited
// vertex after finishing a set of whole components is always the minimum of
// its own component, so this is exactly the reference's restart order.
//
// GPU pipeline:
//   1. symmetry check of the pattern (binary search of (c, r) for every
//      (r, c)); if asymmetric, A|A^T is built by a stable radix transpose and
//      a per-row sorted union.
//   2. frontier BFS from root in ONE cooperative persistent kernel (grid
//      barrier per level, warp-cooperative load-balanced edge expansion,
//      atomicCAS visit, warp-aggregated queue pushes).
//   3. if vertices remain: connected components of the rest by min-root
//      hooking (root = minimum vertex id), then a multi-source BFS from all
//      component roots (same kernel).
//   4. level ids: root component -> dist; other components -> L0 + offset
//      (exclusive scan over roots in id order) + dist.
//   5. perm = stable radix sort of ids by level id; level_ptr = exclusive
//      scan of the level histogram; inv_perm = scatter.
#include <algorithm>

#include "lmpk_internal.cuh"
#include "radix_sort.cuh"

namespace lmpk {

constexpr int kBfsThreads = 512;
constexpr int kBfsBatch = 8;  // edges per lane and round of the frontier expansion

// Grid barrier of the cooperative BFS kernel: one arrival counter that only
// grows (zeroed before the launch); a barrier completes when it reaches the
// running sum of the arrivals expected so far.  One atomic per arriving CTA
// and a spin on the same word -- no reset, no generation word, no sleep: ~598
// of these are cfg2's whole level loop.
struct GridBar {
  unsigned int count;
  unsigned int pad;
};

// Only the `active` CTAs of a level arrive (the others did no work and just
// wait): `target` accumulates the active counts, which every CTA derives from
// the same frontier size.  A narrow frontier (cfg2: ~30K vertices = 59 CTAs of
// 512 vertices) then costs 59 serialised atomics on the word instead of 296.
__device__ __forceinline__ void grid_barrier(GridBar* gb, unsigned int active, bool arrive, unsigned int& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += active;
    if (arrive) {
      __threadfence();
      atomicAdd(&gb->count, 1u);
    }
    volatile unsigned int* vc = &gb->count;
    while (*vc < target) {
    }
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------------- symmetry
template <typename RP>
__global__ void k_check_symmetric(int32_t n, const RP* row_ptr, const int32_t* col, int* asym) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t k = row_ptr[r]; k < int64_t(row_ptr[r + 1]); ++k) {
    const int32_t c = col[k];
    if (c == r) continue;
    int64_t lo = row_ptr[c], hi = int64_t(row_ptr[c + 1]) - 1;
    bool found = false;
    while (lo <= hi) {
      int64_t mid = (lo + hi) >> 1;
      int32_t v = col[mid];
      if (v == r) {
        found = true;
        break;
      }
      if (v < r)
        lo = mid + 1;
      else
        hi = mid - 1;
    }
    if (!found) {
      atomicExch(asym, 1);
      return;
    }
  }
}

__global__ void k_expand_rows(int32_t n, const int32_t* row_ptr, uint32_t* rows_out) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) rows_out[k] = uint32_t(r);
}

__global__ void k_iota_u32(uint32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = uint32_t(i);
}

// transpose row pointer: counts of each column
__global__ void k_col_counts(const int32_t* col, int64_t nnz, int64_t* cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz; i += int64_t(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + col[i]), 1ull);
}

// merge row r of A (sorted cols) with row r of A^T (sorted rows): union size / write
__global__ void k_union_rows(int32_t n, const int32_t* arp, const int32_t* acol, const int64_t* trp,
                             const uint32_t* tcol, int64_t* out_cnt, const int64_t* out_rp,
                             int32_t* out_col) {
  const int32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int64_t i = arp[r], ie = arp[r + 1], j = trp[r], je = trp[r + 1];
  int64_t w = out_rp ? out_rp[r] : 0, c = 0;
  while (i < ie || j < je) {
    int32_t a = i < ie ? acol[i] : INT32_MAX;
    int32_t b = j < je ? int32_t(tcol[j]) : INT32_MAX;
    int32_t v;
    if (a < b) {
      v = a;
      ++i;
    } else if (b < a) {
      v = b;
      ++j;
    } else {
      v = a;
      ++i;
      ++j;
    }
    if (out_col) out_col[w + c] = v;
    ++c;
  }
  if (out_cnt) out_cnt[r] = c;
}

// ------------------------------------------------------------- BFS kernel
struct BfsState {
  int32_t* dist;      // -1 = unvisited (in this phase: eligible)
  int32_t* qa;        // frontier queues
  int32_t* qb;
  uint32_t* sizes;    // [0] size of qa, [1] size of qb, [2] max level reached
  GridBar* bar;
  int32_t n;
};

// Expand the frontier q_in (size n_in) at level `lev` into q_out.
// Warp-cooperative: each warp takes 32 frontier vertices, computes the
// exclusive prefix of their degrees and strides the lanes over the combined
// edge list (load balance independent of the degree distribution).
template <typename RP>
__device__ void bfs_expand(const RP* row_ptr, const int32_t* col, const BfsState& S,
                           const int32_t* q_in, uint32_t n_in, int32_t* q_out, uint32_t* out_size,
                           int32_t lev, uint32_t n_ctas) {
  const int lane = threadIdx.x & 31;
  const int64_t warp_global = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (int64_t(n_ctas) * blockDim.x) >> 5;
  for (int64_t base = warp_global * 32; base < n_in; base += n_warps * 32) {
    const int64_t qi = base + lane;
    int64_t start = 0, deg = 0;
    if (qi < n_in) {
      const int32_t u = q_in[qi];
      start = row_ptr[u];
      deg = int64_t(row_ptr[u + 1]) - start;
    }
    // inclusive scan of deg across the warp
    int64_t inc = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    const int64_t total = __shfl_sync(0xffffffffu, inc, 31);
    const int64_t excl = inc - deg;
    // kBfsBatch edges per lane and round: the column loads, then the
    // dist reads, then the CAS of the unvisited ones are each issued together,
    // so a round costs one chain of dependent L2 round trips instead of kBfsBatch
    // (cfg2: 32 frontier vertices x 7 edges = one round per warp)
    for (int64_t e0 = 0; e0 < total; e0 += 32 * kBfsBatch) {
      int32_t v[kBfsBatch];
#pragma unroll
      for (int j = 0; j < kBfsBatch; ++j) {
        const int64_t e = e0 + 32 * j + lane;
        const bool act = e < total;
        const int64_t ee = act ? e : total - 1;
        // owner = largest lane whose exclusive degree prefix is <= ee
        int owner = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
          const int cand = owner + step;
          const int64_t ex_c = __shfl_sync(0xffffffffu, excl, cand & 31);
          if (cand < 32 && ex_c <= ee) owner = cand;
        }
        const int64_t st_o = __shfl_sync(0xffffffffu, start, owner);
        const int64_t ex_o = __shfl_sync(0xffffffffu, excl, owner);
        v[j] = act ? col[st_o + (ee - ex_o)] : -1;
      }
      bool push[kBfsBatch];
bool fresh[kBfsBatch];
#pragma unroll
      for (int j = 0; j < kBfsBatch; ++j) fresh[j] = v[j] >= 0 && S.dist[v[j]] == -1;
#pragma unroll
      for (int j = 0; j < kBfsBatch; ++j) push[j] = fresh[j] && atomicCAS(S.dist + v[j], -1, lev + 1) == -1;
      uint32_t m[kBfsBatch], cntj[kBfsBatch], tot = 0;
#pragma unroll
      for (int j = 0; j < kBfsBatch; ++j) {
        m[j] = __ballot_sync(0xffffffffu, push[j]);
        cntj[j] = tot;
        tot += uint32_t(__popc(m[j]));
      }
      if (tot) {
        uint32_t off = 0;
        if (lane == 0) off = atomicAdd(out_size, tot);
        off = __shfl_sync(0xffffffffu, off, 0);
#pragma unroll
        for (int j = 0; j < kBfsBatch; ++j)
          if (push[j]) q_out[off + cntj[j] + __popc(m[j] & ((1u << lane) - 1u))] = v[j];
      }
    }
  }
}

// Level loop: ONE grid barrier per level.  The frontier sizes rotate through
// three counters (sizes[4 + lev % 3]): level lev reads its own, pushes into the
// next one and resets the third, which nobody touches until the level after
// next.  sizes[0] is the seeded frontier, sizes[2] the last level reached.
template <typename RP>
__global__ void __launch_bounds__(kBfsThreads) k_bfs(const RP* row_ptr, const int32_t* col, BfsState S) {
  int32_t lev = 0;
  int32_t* qin = S.qa;
  int32_t* qout = S.qb;
  uint32_t* cnt = S.sizes + 4;
  unsigned int target = 0;
  while (true) {
    const uint32_t n_in = *((volatile uint32_t*)(lev == 0 ? S.sizes : cnt + lev % 3));
    if (n_in == 0) break;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (lev > 0) S.sizes[2] = uint32_t(lev);
      cnt[(lev + 2) % 3] = 0;
    }
    // one CTA per 512 frontier vertices (32 per warp), at most the grid
    const uint32_t active = min(gridDim.x, max(1u, (n_in + kBfsThreads - 1) / kBfsThreads));
    const bool mine = blockIdx.x < active;
    if (mine) bfs_expand(row_ptr, col, S, qin, n_in, qout, cnt + (lev + 1) % 3, lev, active);
    grid_barrier(S.bar, active, mine, target);
    int32_t* t = qin;
    qin = qout;
    qout = t;
    ++lev;
  }
}

// ------------------------------------------------------------- components
__device__ __forceinline__ int32_t cc_find(int32_t* parent, int32_t x) {
  int32_t p = *((volatile int32_t*)&parent[x]);
  while (p != x) {
    const int32_t gp = *((volatile int32_t*)&parent[p]);
    if (gp != p) atomicCAS(parent + x, p, gp);  // path halving
    x = p;
    p = gp;
  }
  return x;
}

__global__ void k_cc_init(int32_t n, const int32_t* dist, int32_t* parent) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    parent[v] = v;
}

template <typename RP>
__global__ void k_cc_hook(int32_t n, const RP* row_ptr, const int32_t* col, const int32_t* dist,
                          int32_t* parent) {
  for (int32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x) {
    if (dist[u] != -1) continue;  // belongs to the root component
    for (int64_t k = row_ptr[u]; k < int64_t(row_ptr[u + 1]); ++k) {
      const int32_t v = col[k];
      if (v <= u) continue;  // each undirected edge once (pattern is symmetric)
      int32_t ru = cc_find(parent, u), rv = cc_find(parent, v);
      while (ru != rv) {
        if (ru < rv) {
          const int32_t t = ru;
          ru = rv;
          rv = t;
        }
        // link the larger root under the smaller one: roots stay minimal
        const int32_t old = atomicCAS(parent + ru, ru, rv);
        if (old == ru) break;
        ru = cc_find(parent, ru);
        rv = cc_find(parent, rv);
      }
    }
  }
}

// finalize labels; seed the multi-source frontier with the component roots
__global__ void k_cc_finalize(int32_t n, int32_t* dist, int32_t* parent, int32_t* q, uint32_t* qsize) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (dist[v] != -1) continue;
    const int32_t r = cc_find(parent, v);
    parent[v] = r;
    if (r == v) {
      dist[v] = 0;
      q[atomicAdd(qsize, 1u)] = v;
    }
  }
}

__global__ void k_comp_maxdist(int32_t n, const int32_t* dist, const int32_t* label,
                               const uint8_t* is_tail, int32_t* cmax) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (is_tail[v]) atomicMax(cmax + label[v], dist[v]);
}

__global__ void k_comp_levels(int32_t n, const int32_t* label, const uint8_t* is_tail,
                              const int32_t* cmax, int32_t* nlev) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    nlev[v] = (is_tail[v] && label[v] == v) ? cmax[v] + 1 : 0;
}

__global__ void k_level_ids(int32_t n, const int32_t* dist, const int32_t* label, const uint8_t* is_tail,
                            const int64_t* cbase, uint32_t L0, uint32_t* keys, uint32_t* vals,
                            unsigned long long* hist) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    uint32_t lid;
    if (is_tail && is_tail[v])
      lid = L0 + uint32_t(cbase[label[v]]) + uint32_t(dist[v]);
    else
      lid = uint32_t(dist[v]);
    keys[v] = lid;
    vals[v] = uint32_t(v);
    atomicAdd(hist + lid, 1ull);
  }
}

__global__ void k_mark_tail(int32_t n, const int32_t* dist, uint8_t* is_tail) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    is_tail[v] = dist[v] == -1 ? 1 : 0;
}

__global__ void k_perm_out(int32_t n, const uint32_t* sorted_vals, int32_t* perm, int32_t* inv) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t v = int32_t(sorted_vals[i]);
    perm[i] = v;
    inv[v] = i;
  }
}

template <typename RP>
static int launch_bfs(lmpk_ctx* ctx, const RP* row_ptr, const int32_t* col, BfsState S, cudaStream_t st) {
  int occ = 0;
  LMPK_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bfs<RP>, kBfsThreads, 0));
  occ = std::max(1, std::min(occ, 2));
  const int grid = occ * ctx->sm_count;
  // rotating frontier counters and the barrier's arrival counter start at zero
  LMPK_CHECK_CUDA(cudaMemsetAsync(S.sizes + 4, 0, 16, st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(S.bar, 0, sizeof(GridBar), st));
  void* args[] = {(void*)&row_ptr, (void*)&col, (void*)&S};
  LMPK_CHECK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_bfs<RP>), dim3(grid),
                                              dim3(kBfsThreads), args, 0, st));
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

static inline int grid_for(lmpk_ctx* ctx, int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(ctx->sm_count) * 16)));
}

template <typename RP>
static int bfs_core(lmpk_ctx* ctx, int32_t n, const RP* row_ptr, const int32_t* col, int32_t root,
                    int32_t* perm, int32_t* inv, int64_t* level_ptr, int64_t* n_levels, cudaStream_t st) {
  // scratch layout (ctx->s_a .. s_e)
  const size_t N = size_t(n);
  LMPK_TRY(ctx->s_a.ensure(N * 4 * 4 + 4096));  // dist, qa, qb, parent
  int32_t* dist = reinterpret_cast<int32_t*>(ctx->s_a.ptr);
  int32_t* qa = dist + N;
  int32_t* qb = qa + N;
  int32_t* parent = qb + N;
  LMPK_TRY(ctx->s_small.ensure(4096));
  uint32_t* sizes = reinterpret_cast<uint32_t*>(ctx->s_small.ptr);
  GridBar* bar = reinterpret_cast<GridBar*>(sizes + 8);
  LMPK_CHECK_CUDA(cudaMemsetAsync(ctx->s_small.ptr, 0, 256, st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(dist, 0xff, N * 4, st));
  // seed: dist[root] = 0, qa = [root]
  const int32_t zero = 0;
  const uint32_t one = 1;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(dist + root, &zero, 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(qa, &root, 4, cudaMemcpyHostToDevice, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(sizes, &one, 4, cudaMemcpyHostToDevice, st));
  BfsState S{dist, qa, qb, sizes, bar, n};
  LMPK_TRY(launch_bfs<RP>(ctx, row_ptr, col, S, st));
  uint32_t h_sizes[4];
  LMPK_CHECK_CUDA(cudaMemcpyAsync(h_sizes, sizes, 16, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  const uint32_t L0 = h_sizes[2] + 1;  // levels of the root component

  // count unvisited via the tail mask
  LMPK_TRY(ctx->s_b.ensure(N + 64));
  uint8_t* is_tail = reinterpret_cast<uint8_t*>(ctx->s_b.ptr);
  k_mark_tail<<<grid_for(ctx, n), 256, 0, st>>>(n, dist, is_tail);
  launch_count_add(ctx, 1);

  // scratch for sort + scans
  const int64_t cnt_len = radix_counts_len(n);
  const int64_t tmp_len = std::max(scan_tmp_len(cnt_len), scan_tmp_len(int64_t(n) + 1)) + 8;
  LMPK_TRY(ctx->s_c.ensure(N * 4 * 4 + 64));  // keys0, vals0, keys1, vals1
  uint32_t* k0 = reinterpret_cast<uint32_t*>(ctx->s_c.ptr);
  uint32_t* v0 = k0 + N;
  uint32_t* k1 = v0 + N;
  uint32_t* v1 = k1 + N;
  LMPK_TRY(ctx->s_d.ensure(size_t(cnt_len) * 4 + size_t(cnt_len) * 8 + size_t(tmp_len) * 8 + 64));
  uint32_t* counts = reinterpret_cast<uint32_t*>(ctx->s_d.ptr);
  int64_t* offsets = reinterpret_cast<int64_t*>(counts + ((cnt_len + 1) & ~int64_t(1)));
  int64_t* stmp = offsets + cnt_len;
  LMPK_TRY(ctx->s_e.ensure((N + 2) * 8 * 2 + 64));
  unsigned long long* hist = reinterpret_cast<unsigned long long*>(ctx->s_e.ptr);
  int64_t* cbase = reinterpret_cast<int64_t*>(hist + N + 1);

  uint32_t total_levels = L0;
  // number of visited = 1 + all pushes; pushes are not counted separately, so
  // reduce the tail mask instead (cheap: one scan)
  int64_t tail_count = 0;
  LMPK_TRY(device_excl_scan<uint8_t, int64_t>(ctx, is_tail, n, cbase, 0, true, stmp, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&tail_count, cbase + n, 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));

  if (tail_count > 0) {
    // connected components of the remaining vertices, roots = minimum ids
    k_cc_init<<<grid_for(ctx, n), 256, 0, st>>>(n, dist, parent);
    k_cc_hook<RP><<<grid_for(ctx, n), 256, 0, st>>>(n, row_ptr, col, dist, parent);
    LMPK_CHECK_CUDA(cudaMemsetAsync(sizes, 0, 16, st));
    k_cc_finalize<<<grid_for(ctx, n), 256, 0, st>>>(n, dist, parent, qa, sizes);
    launch_count_add(ctx, 3);
    // multi-source BFS over the tail (main-component vertices have dist >= 0)
    LMPK_TRY(launch_bfs<RP>(ctx, row_ptr, col, S, st));
    // per-component level counts -> exclusive scan in root-id order
    int32_t* cmax = qb;  // reuse
    LMPK_CHECK_CUDA(cudaMemsetAsync(cmax, 0xff, N * 4, st));
    k_comp_maxdist<<<grid_for(ctx, n), 256, 0, st>>>(n, dist, parent, is_tail, cmax);
    int32_t* nlev = qa;  // reuse
    k_comp_levels<<<grid_for(ctx, n), 256, 0, st>>>(n, parent, is_tail, cmax, nlev);
    launch_count_add(ctx, 2);
    LMPK_TRY(device_excl_scan<int32_t, int64_t>(ctx, nlev, n, cbase, 0, true, stmp, st));
    int64_t tail_levels = 0;
    LMPK_CHECK_CUDA(cudaMemcpyAsync(&tail_levels, cbase + n, 8, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    total_levels = L0 + uint32_t(tail_levels);
  }
  LMPK_CHECK_CUDA(cudaMemsetAsync(hist, 0, (size_t(total_levels) + 1) * 8, st));
  k_level_ids<<<grid_for(ctx, n), 256, 0, st>>>(n, dist, parent, tail_count > 0 ? is_tail : nullptr, cbase,
                                                L0, k0, v0, hist);
  launch_count_add(ctx, 1);
  int bits = 0;
  while (bits < 32 && (uint64_t(1) << bits) < uint64_t(total_levels)) ++bits;
  bool in_first = true;
  LMPK_TRY(device_radix_sort(ctx, k0, v0, k1, v1, n, bits, counts, offsets, stmp, &in_first, st));
  k_perm_out<<<grid_for(ctx, n), 256, 0, st>>>(n, in_first ? v0 : v1, perm, inv);
  launch_count_add(ctx, 1);
  // level_ptr = exclusive scan of the histogram, L+1 entries
  LMPK_TRY(device_excl_scan<unsigned long long, int64_t>(ctx, hist, total_levels, level_ptr, 0, true,
                                                         stmp, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  *n_levels = total_levels;
  return LMPK_OK;
}

}  // namespace lmpk

using namespace lmpk;

// Returns 1 in *asym if the pattern is not symmetric.
static int check_symmetric(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                           int* asym, cudaStream_t st) {
  LMPK_TRY(ctx->s_small.ensure(4096));
  int* d = reinterpret_cast<int*>(ctx->s_small.ptr) + 64;
  LMPK_CHECK_CUDA(cudaMemsetAsync(d, 0, 4, st));
  k_check_symmetric<int32_t><<<div_up(n, 256), 256, 0, st>>>(n, row_ptr, col, d);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(asym, d, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  return LMPK_OK;
}

// Build A|A^T into (sym_rp int64 [n+1], sym_col) allocated in ctx->s_f/s_g.
static int build_union(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                       int64_t** out_rp, int32_t** out_col, int64_t* out_nnz, cudaStream_t st) {
  int32_t h_nnz = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&h_nnz, row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  const int64_t nnz = h_nnz;
  const size_t N = size_t(n);
  // transpose: stable sort of (col -> row) pairs, rows enter in ascending order
  LMPK_TRY(ctx->s_c.ensure(size_t(nnz) * 16 + 64));
  uint32_t* k0 = reinterpret_cast<uint32_t*>(ctx->s_c.ptr);
  uint32_t* v0 = k0 + nnz;
  uint32_t* k1 = v0 + nnz;
  uint32_t* v1 = k1 + nnz;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(k0, col, size_t(nnz) * 4, cudaMemcpyDeviceToDevice, st));
  k_expand_rows<<<div_up(n, 256), 256, 0, st>>>(n, row_ptr, v0);
  launch_count_add(ctx, 1);
  const int64_t cnt_len = radix_counts_len(nnz);
  const int64_t tmp_len = std::max(scan_tmp_len(cnt_len), scan_tmp_len(int64_t(n) + 1)) + 8;
  LMPK_TRY(ctx->s_d.ensure(size_t(cnt_len) * 12 + size_t(tmp_len) * 8 + 64));
  uint32_t* counts = reinterpret_cast<uint32_t*>(ctx->s_d.ptr);
  int64_t* offsets = reinterpret_cast<int64_t*>(counts + ((cnt_len + 1) & ~int64_t(1)));
  int64_t* stmp = offsets + cnt_len;
  int bits = 0;
  while (bits < 32 && (int64_t(1) << bits) < int64_t(n)) ++bits;
  bool in_first = true;
  LMPK_TRY(device_radix_sort(ctx, k0, v0, k1, v1, nnz, bits, counts, offsets, stmp, &in_first, st));
  uint32_t* trows = in_first ? v0 : v1;
  // transposed row pointer
  LMPK_TRY(ctx->s_e.ensure((N + 2) * 8 * 3 + 64));
  int64_t* cnt = reinterpret_cast<int64_t*>(ctx->s_e.ptr);
  int64_t* trp = cnt + N + 2;
  int64_t* urp = trp + N + 2;
  LMPK_CHECK_CUDA(cudaMemsetAsync(cnt, 0, N * 8, st));
  k_col_counts<<<grid_for(ctx, nnz), 256, 0, st>>>(col, nnz, cnt);
  launch_count_add(ctx, 1);
  LMPK_TRY(device_excl_scan<int64_t, int64_t>(ctx, cnt, n, trp, 0, true, stmp, st));
  // union sizes -> row pointer -> write
  k_union_rows<<<div_up(n, 256), 256, 0, st>>>(n, row_ptr, col, trp, trows, cnt, nullptr, nullptr);
  launch_count_add(ctx, 1);
  LMPK_TRY(device_excl_scan<int64_t, int64_t>(ctx, cnt, n, urp, 0, true, stmp, st));
  int64_t unnz = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&unnz, urp + n, 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  LMPK_TRY(ctx->s_f.ensure((N + 1) * 8 + 64));
  LMPK_TRY(ctx->s_g.ensure(size_t(unnz) * 4 + 64));
  int64_t* srp = reinterpret_cast<int64_t*>(ctx->s_f.ptr);
  int32_t* scol = reinterpret_cast<int32_t*>(ctx->s_g.ptr);
  LMPK_CHECK_CUDA(cudaMemcpyAsync(srp, urp, (N + 1) * 8, cudaMemcpyDeviceToDevice, st));
  k_union_rows<<<div_up(n, 256), 256, 0, st>>>(n, row_ptr, col, trp, trows, nullptr, srp, scol);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  *out_rp = srp;
  *out_col = scol;
  *out_nnz = unnz;
  return LMPK_OK;
}

extern "C" int lmpk_symmetrized_pattern(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr,
                                        const int32_t* col, int* is_symmetric, int64_t* sym_nnz,
                                        int64_t* out_row_ptr, int32_t* out_col, int64_t cap,
                                        void* stream) {
  LMPK_ARG_CHECK(ctx && is_symmetric && sym_nnz, "lmpk_symmetrized_pattern: NULL argument");
  cudaStream_t st = as_stream(stream);
  int asym = 0;
  if (n > 0) LMPK_TRY(check_symmetric(ctx, n, row_ptr, col, &asym, st));
  if (!asym) {
    int32_t h_nnz = 0;
    LMPK_CHECK_CUDA(cudaMemcpyAsync(&h_nnz, row_ptr + n, 4, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    *is_symmetric = 1;
    *sym_nnz = h_nnz;
    return LMPK_OK;
  }
  *is_symmetric = 0;
  int64_t* srp;
  int32_t* scol;
  int64_t unnz;
  LMPK_TRY(build_union(ctx, n, row_ptr, col, &srp, &scol, &unnz, st));
  *sym_nnz = unnz;
  if (out_col != nullptr) {
    LMPK_ARG_CHECK(cap >= unnz, "out_col capacity %lld < %lld", (long long)cap, (long long)unnz);
    LMPK_CHECK_CUDA(cudaMemcpyAsync(out_row_ptr, srp, (size_t(n) + 1) * 8, cudaMemcpyDeviceToDevice, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(out_col, scol, size_t(unnz) * 4, cudaMemcpyDeviceToDevice, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  return LMPK_OK;
}

extern "C" int lmpk_bfs_levels(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                               int32_t root, int32_t* perm, int32_t* inv_perm, int64_t* level_ptr,
                               int64_t* n_levels, void* stream) {
  LMPK_ARG_CHECK(ctx && perm && inv_perm && level_ptr && n_levels, "lmpk_bfs_levels: NULL argument");
  LMPK_ARG_CHECK(n >= 1, "matrix must have at least one row");
  LMPK_ARG_CHECK(0 <= root && root < n, "root %d out of range for n=%d", root, n);
  cudaStream_t st = as_stream(stream);
  int asym = 0;
  LMPK_TRY(check_symmetric(ctx, n, row_ptr, col, &asym, st));
  if (!asym) return bfs_core<int32_t>(ctx, n, row_ptr, col, root, perm, inv_perm, level_ptr, n_levels, st);
  int64_t* srp;
  int32_t* scol;
  int64_t unnz;
  LMPK_TRY(build_union(ctx, n, row_ptr, col, &srp, &scol, &unnz, st));
  return bfs_core<int64_t>(ctx, n, srp, scol, root, perm, inv_perm, level_ptr, n_levels, st);
}

__global__ void k_level_nnz(const int32_t* row_ptr, const int64_t* level_ptr, int64_t L, int64_t* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < L; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = int64_t(row_ptr[level_ptr[i + 1]]) - int64_t(row_ptr[level_ptr[i]]);
}

extern "C" int lmpk_level_nnz(lmpk_ctx* ctx, const int32_t* row_ptr, const int64_t* level_ptr,
                              int64_t n_levels, int64_t* out, void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && level_ptr && out, "lmpk_level_nnz: NULL argument");
  if (n_levels <= 0) return LMPK_OK;
  k_level_nnz<<<grid_for(ctx, n_levels), 256, 0, as_stream(stream)>>>(row_ptr, level_ptr, n_levels, out);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

// ===================================================================
// Recursive refinement (lmpk_plan.h): induced-subgraph BFS of a span and the
// diamond-halo key sort, pkg/src/levelmpk/groups.py:238-335.
#include "lmpk_plan.h"

namespace lmpk {

struct TmpBuf {  // cudaMalloc'ed scratch of one planning call
  void* p = nullptr;
  ~TmpBuf() {
    if (p) cudaFree(p);
  }
  int alloc(size_t bytes) {
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) {
      set_error("planning scratch cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
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

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

__global__ void k_level_nnz_perm(const int32_t* row_ptr, const int32_t* perm, const int64_t* level_ptr,
                                 int64_t L, int64_t* out) {
  // one warp per level
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= L) return;
  int64_t s = 0;
  for (int64_t r = level_ptr[w] + lane; r < level_ptr[w + 1]; r += 32) {
    const int32_t o = perm[r];
    s += int64_t(row_ptr[o + 1]) - int64_t(row_ptr[o]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[w] = s;
}

__global__ void k_local_of(const int32_t* perm, int32_t r0, int32_t m, int32_t* local_of) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    local_of[perm[r0 + i]] = i;
}

// induced pattern: count (out_col == nullptr) or fill the kept neighbours of
// local row i, in the order of the original row (groups.py:244-254)
template <typename RP>
__global__ void k_induced(const RP* sp, const int32_t* sc, const int32_t* perm, int32_t r0, int32_t m,
                          const int32_t* local_of, int64_t* cnt, const int64_t* ptr, int32_t* out_col) {
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const int32_t o = perm[r0 + w];
  const int64_t b = sp[o], e = sp[o + 1];
  int64_t base = ptr ? ptr[w] : 0, total = 0;
  for (int64_t k0 = b; k0 < e; k0 += 32) {
    const int64_t k = k0 + lane;
    const int32_t l = k < e ? local_of[sc[k]] : -1;
    const uint32_t mask = __ballot_sync(0xffffffffu, l >= 0);
    if (out_col && l >= 0) out_col[base + total + __popc(mask & ((1u << lane) - 1u))] = l;
    total += __popc(mask);
  }
  if (!out_col && lane == 0) cnt[w] = total;
}

__global__ void k_apply_order(const int32_t* src, const int32_t* order, int32_t m, int32_t* dst) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    dst[i] = src[order[i]];
}

template <typename RP>
static int refine_span(lmpk_ctx* ctx, int32_t n, const RP* sp, const int32_t* sc, int32_t* perm, int32_t r0,
                       int32_t r1, int64_t* level_ptr_out, int64_t* n_levels, cudaStream_t st) {
  const int32_t m = r1 - r0;
  const size_t M = size_t(m);
  TmpBuf b_local, b_cnt, b_col, b_perm;
  LMPK_TRY(b_local.alloc(size_t(n) * 4));
  LMPK_TRY(b_cnt.alloc((M + 2) * 8 * 2 + (scan_tmp_len(int64_t(m) + 1) + 8) * 8));
  LMPK_TRY(b_perm.alloc(M * 4 * 3));
  int32_t* local_of = b_local.as<int32_t>();
  int64_t* cnt = b_cnt.as<int64_t>();
  int64_t* ptr = cnt + M + 2;
  int64_t* stmp = ptr + M + 2;
  int32_t* perm_l = b_perm.as<int32_t>();
  int32_t* inv_l = perm_l + M;
  int32_t* old = inv_l + M;
  k_fill_i32<<<grid_for(ctx, n), 256, 0, st>>>(local_of, n, -1);
  k_local_of<<<grid_for(ctx, m), 256, 0, st>>>(perm, r0, m, local_of);
  const int wgrid = int((int64_t(m) * 32 + 255) / 256);
  k_induced<RP><<<wgrid, 256, 0, st>>>(sp, sc, perm, r0, m, local_of, cnt, nullptr, nullptr);
  launch_count_add(ctx, 3);
  LMPK_TRY(device_excl_scan<int64_t, int64_t>(ctx, cnt, m, ptr, 0, true, stmp, st));
  int64_t total = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&total, ptr + m, 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  LMPK_TRY(b_col.alloc(size_t(total) * 4));
  k_induced<RP><<<wgrid, 256, 0, st>>>(sp, sc, perm, r0, m, local_of, nullptr, ptr, b_col.as<int32_t>());
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  LMPK_TRY(bfs_core<int64_t>(ctx, m, ptr, b_col.as<int32_t>(), 0, perm_l, inv_l, level_ptr_out, n_levels, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(old, perm + r0, M * 4, cudaMemcpyDeviceToDevice, st));
  k_apply_order<<<grid_for(ctx, m), 256, 0, st>>>(old, perm_l, m, perm + r0);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  return LMPK_OK;
}

__global__ void k_halo_seed(const int32_t* perm, int64_t G, const int64_t* gp, int32_t* key_orig) {
  // one block per group
  for (int64_t g = blockIdx.x; g < G; g += gridDim.x)
    for (int64_t r = gp[g] + threadIdx.x; r < gp[g + 1]; r += blockDim.x) key_orig[perm[r]] = int32_t(g);
}

template <typename RP>
__global__ void k_halo_keys(const RP* sp, const int32_t* sc, const int32_t* perm, int32_t lo, int32_t m,
                            const int32_t* key_orig, uint32_t* keys, uint32_t* vals) {
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const int32_t o = perm[lo + w];
  int32_t best = -1;
  for (int64_t k = int64_t(sp[o]) + lane; k < int64_t(sp[o + 1]); k += 32) best = max(best, key_orig[sc[k]]);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, s));
  if (lane == 0) {
    keys[w] = uint32_t(best + 1);
    vals[w] = uint32_t(w);
  }
}

__global__ void k_halo_apply(const int32_t* old, const uint32_t* skeys, const uint32_t* svals, int32_t m,
                             int32_t* perm_lo, int32_t* key_orig, int32_t* keys_out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int32_t v = old[svals[i]];
    const int32_t k = int32_t(skeys[i]) - 1;
    perm_lo[i] = v;
    key_orig[v] = k;
    keys_out[i] = k;
  }
}

template <typename RP>
static int halo_level_sort(lmpk_ctx* ctx, const RP* sp, const int32_t* sc, int32_t* perm, int32_t* key_orig,
                           int32_t lo, int32_t hi, int32_t* keys_out, cudaStream_t st) {
  const int32_t m = hi - lo;
  if (m <= 0) return LMPK_OK;
  const size_t M = size_t(m);
  const int64_t cnt_len = radix_counts_len(m);
  const int64_t tmp_len = scan_tmp_len(cnt_len) + 8;
  TmpBuf b;
  LMPK_TRY(b.alloc(M * 4 * 5 + size_t(cnt_len) * 12 + size_t(tmp_len) * 8 + 256));
  uint32_t* k0 = b.as<uint32_t>();
  uint32_t* v0 = k0 + M;
  uint32_t* k1 = v0 + M;
  uint32_t* v1 = k1 + M;
  int32_t* old = reinterpret_cast<int32_t*>(v1 + M);
  uintptr_t q = (reinterpret_cast<uintptr_t>(old + M) + 15) & ~uintptr_t(15);
  int64_t* offsets = reinterpret_cast<int64_t*>(q);
  int64_t* stmp = offsets + cnt_len;
  uint32_t* counts = reinterpret_cast<uint32_t*>(stmp + tmp_len);
  const int wgrid = int((int64_t(m) * 32 + 255) / 256);
  k_halo_keys<RP><<<wgrid, 256, 0, st>>>(sp, sc, perm, lo, m, key_orig, k0, v0);
  launch_count_add(ctx, 1);
  bool in_first = true;
  // keys are child group indices + 1: the child tree never has more groups than the matrix has rows
  LMPK_TRY(device_radix_sort(ctx, k0, v0, k1, v1, m, 32, counts, offsets, stmp, &in_first, st));
  LMPK_CHECK_CUDA(cudaMemcpyAsync(old, perm + lo, M * 4, cudaMemcpyDeviceToDevice, st));
  k_halo_apply<<<grid_for(ctx, m), 256, 0, st>>>(old, in_first ? k0 : k1, in_first ? v0 : v1, m, perm + lo,
                                                 key_orig, keys_out);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  return LMPK_OK;
}

__global__ void k_invert_perm(int32_t n, const int32_t* perm, int32_t* inv) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) inv[perm[i]] = i;
}

}  // namespace lmpk

extern "C" int lmpk_level_nnz_perm(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* perm,
                                   const int64_t* level_ptr, int64_t n_levels, int64_t* out, void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && perm && level_ptr && out, "lmpk_level_nnz_perm: NULL argument");
  if (n_levels <= 0) return LMPK_OK;
  k_level_nnz_perm<<<int((n_levels * 32 + 255) / 256), 256, 0, as_stream(stream)>>>(row_ptr, perm, level_ptr,
                                                                                   n_levels, out);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

extern "C" int lmpk_refine_span(lmpk_ctx* ctx, int32_t n, const void* sym_ptr, int ptr64, const int32_t* sym_col,
                                int32_t* perm, int32_t r0, int32_t r1, int64_t* level_ptr_out, int64_t* n_levels,
                                void* stream) {
  LMPK_ARG_CHECK(ctx && sym_ptr && sym_col && perm && level_ptr_out && n_levels, "lmpk_refine_span: NULL argument");
  LMPK_ARG_CHECK(0 <= r0 && r0 < r1 && r1 <= n, "span [%d, %d) out of range for n=%d", r0, r1, n);
  cudaStream_t st = as_stream(stream);
  if (ptr64)
    return refine_span<int64_t>(ctx, n, static_cast<const int64_t*>(sym_ptr), sym_col, perm, r0, r1, level_ptr_out,
                                n_levels, st);
  return refine_span<int32_t>(ctx, n, static_cast<const int32_t*>(sym_ptr), sym_col, perm, r0, r1, level_ptr_out,
                              n_levels, st);
}

extern "C" int lmpk_halo_seed(lmpk_ctx* ctx, int32_t n, const int32_t* perm, int64_t n_groups,
                              const int64_t* group_ptr, int32_t* key_orig, void* stream) {
  LMPK_ARG_CHECK(ctx && perm && group_ptr && key_orig, "lmpk_halo_seed: NULL argument");
  cudaStream_t st = as_stream(stream);
  k_fill_i32<<<grid_for(ctx, n), 256, 0, st>>>(key_orig, n, -1);
  if (n_groups > 0)
    k_halo_seed<<<int(std::min<int64_t>(n_groups, 4096)), 256, 0, st>>>(perm, n_groups, group_ptr, key_orig);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 2);
  return LMPK_OK;
}

extern "C" int lmpk_halo_level_sort(lmpk_ctx* ctx, int32_t n, const void* sym_ptr, int ptr64,
                                    const int32_t* sym_col, int32_t* perm, int32_t* key_orig, int32_t lo,
                                    int32_t hi, int32_t* keys_out, void* stream) {
  LMPK_ARG_CHECK(ctx && sym_ptr && sym_col && perm && key_orig && keys_out, "lmpk_halo_level_sort: NULL argument");
  LMPK_ARG_CHECK(0 <= lo && lo <= hi && hi <= n, "level [%d, %d) out of range for n=%d", lo, hi, n);
  cudaStream_t st = as_stream(stream);
  if (ptr64)
    return halo_level_sort<int64_t>(ctx, static_cast<const int64_t*>(sym_ptr), sym_col, perm, key_orig, lo, hi,
                                    keys_out, st);
  return halo_level_sort<int32_t>(ctx, static_cast<const int32_t*>(sym_ptr), sym_col, perm, key_orig, lo, hi,
                                  keys_out, st);
}

extern "C" int lmpk_invert_perm(lmpk_ctx* ctx, int32_t n, const int32_t* perm, int32_t* inv, void* stream) {
  LMPK_ARG_CHECK(ctx && perm && inv, "lmpk_invert_perm: NULL argument");
  if (n <= 0) return LMPK_OK;
  k_invert_perm<<<grid_for(ctx, n), 256, 0, as_stream(stream)>>>(n, perm, inv);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}
