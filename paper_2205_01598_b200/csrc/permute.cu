// permute.cu -- symmetric permutation B[i,j] = A[perm[i], perm[j]] and vector
// gathers/scatters on sm_100a.
//
// Reference: permute_symmetric (pkg/src/levelmpk/csr.py:169-187): row gather,
// column map through inv_perm, then columns re-sorted ascending per row
// (lexsort).  Column indices are unique within a row, so any correct sort is
// bit-exact.  Rows of <= 32 entries are sorted by a sub-warp bitonic network
// in registers (width 8/16/32 chosen from the longest short row); longer rows
// go through the stable radix sort (by column, then by segment).
#include <algorithm>

#include "lmpk_internal.cuh"
#include "radix_sort.cuh"

namespace lmpk {

__global__ void k_perm_counts(int32_t n, const int32_t* row_ptr, const int32_t* perm, int32_t* cnt,
                              int32_t* is_long, int long_threshold) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t o = perm[i];
    const int32_t c = row_ptr[o + 1] - row_ptr[o];
    cnt[i] = c;
    is_long[i] = c > long_threshold ? 1 : 0;
  }
}

// one W-lane segment per row; rows longer than W are skipped (long path)
template <int W>
__global__ void k_perm_short_rows(int32_t n, const int32_t* row_ptr, const int32_t* col,
                                  const double* val, const int32_t* perm, const int32_t* inv,
                                  const int32_t* out_rp, int32_t* out_col, double* out_val) {
  const int64_t gt = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int sub = int(gt % W);
  const int64_t nseg = (int64_t(gridDim.x) * blockDim.x) / W;
  for (int64_t base = gt / W; base < n + 0 * nseg; base += nseg) {
    // all lanes of a segment iterate together (segments never straddle warps)
    const int32_t i = int32_t(base);
    const int32_t o = perm[i];
    const int32_t a = row_ptr[o], len = row_ptr[o + 1] - a;
    if (len > W) continue;  // uniform across the segment
    int32_t key = INT32_MAX;
    double v = 0.0;
    if (sub < len) {
      key = inv[col[a + sub]];
      v = val[a + sub];
    }
    const unsigned mask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << ((threadIdx.x & 31) & ~(W - 1)));
#pragma unroll
    for (int k = 2; k <= W; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const int32_t pk = __shfl_xor_sync(mask, key, j, W);
        const double pv = __shfl_xor_sync(mask, v, j, W);
        const bool up = (sub & k) == 0;
        const bool lower = (sub & j) == 0;
        const bool take_min = (lower == up);
        const bool swap = take_min ? (pk < key) : (pk > key);
        if (swap) {
          key = pk;
          v = pv;
        }
      }
    }
    if (sub < len) {
      const int32_t w = out_rp[i] + sub;
      out_col[w] = key;
      out_val[w] = v;
    }
  }
}

// long rows: build (key = new col, value = element id) with a segment id per element
__global__ void k_perm_long_fill(int32_t n_long, const int32_t* long_rows, const int64_t* seg_ofs,
                                 const int32_t* row_ptr, const int32_t* col, const int32_t* perm,
                                 const int32_t* inv, uint32_t* keys, uint32_t* vals, uint32_t* seg_of,
                                 int64_t* src_of) {
  for (int32_t s = blockIdx.x; s < n_long; s += gridDim.x) {
    const int32_t i = long_rows[s];
    const int32_t o = perm[i];
    const int32_t a = row_ptr[o], len = row_ptr[o + 1] - a;
    const int64_t base = seg_ofs[s];
    for (int32_t j = threadIdx.x; j < len; j += blockDim.x) {
      const int64_t e = base + j;
      keys[e] = uint32_t(inv[col[a + j]]);
      vals[e] = uint32_t(e);
      seg_of[e] = uint32_t(s);
      src_of[e] = int64_t(a) + j;
    }
  }
}

__global__ void k_gather_seg_keys(int64_t E, const uint32_t* sorted_ids, const uint32_t* seg_of,
                                  uint32_t* keys2) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < E; q += int64_t(gridDim.x) * blockDim.x)
    keys2[q] = seg_of[sorted_ids[q]];
}

__global__ void k_perm_long_write(int64_t E, const uint32_t* final_ids, const uint32_t* seg_of,
                                  const int64_t* seg_ofs, const int32_t* long_rows, const int32_t* out_rp,
                                  const int64_t* src_of, const int32_t* col, const double* val,
                                  const int32_t* inv, int32_t* out_col, double* out_val) {
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < E; q += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = final_ids[q];
    const uint32_t s = seg_of[e];
    const int64_t w = int64_t(out_rp[long_rows[s]]) + (q - seg_ofs[s]);
    const int64_t src = src_of[e];
    out_col[w] = inv[col[src]];
    out_val[w] = val[src];
  }
}

__global__ void k_compact_long(int32_t n, const int32_t* is_long, const int64_t* pos, int32_t* long_rows,
                               const int32_t* cnt, int64_t* long_len) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (is_long[i]) {
      long_rows[pos[i]] = i;
      long_len[pos[i]] = cnt[i];
    }
}

__global__ void k_max_i32(const int32_t* a, int32_t n, int* out) {
  int m = 0;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) m = max(m, a[i]);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

template <int W>
__global__ void k_permute_vec(int32_t n, const int32_t* perm, const double* in, int64_t ld_in, double* out,
                              int64_t ld_out, int32_t n_vec, int scatter) {
  const int64_t total = int64_t(n) * n_vec;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int32_t v = int32_t(q / n), i = int32_t(q % n);
    const int64_t src = scatter ? i : perm[i];
    const int64_t dst = scatter ? perm[i] : i;
#pragma unroll
    for (int w = 0; w < W; ++w) out[v * ld_out + dst * W + w] = in[v * ld_in + src * W + w];
  }
}

}  // namespace lmpk

using namespace lmpk;

static inline int grid_n(lmpk_ctx* ctx, int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(ctx->sm_count) * 16)));
}

extern "C" int lmpk_permute_symmetric(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                                      const double* val, const int32_t* perm, const int32_t* inv,
                                      int32_t* out_rp, int32_t* out_col, double* out_val, void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && perm && inv && out_rp, "lmpk_permute_symmetric: NULL argument");
  LMPK_ARG_CHECK(n >= 0, "n must be >= 0");
  cudaStream_t st = as_stream(stream);
  const size_t N = size_t(n);
  if (n == 0) {
    LMPK_CHECK_CUDA(cudaMemsetAsync(out_rp, 0, 4, st));
    return LMPK_OK;
  }
  LMPK_TRY(ctx->s_a.ensure(N * 4 * 2 + (N + 2) * 8 * 3 + 64));
  int32_t* cnt = reinterpret_cast<int32_t*>(ctx->s_a.ptr);
  int32_t* is_long = cnt + N;
  int64_t* pos = reinterpret_cast<int64_t*>(is_long + N + (N & 1));
  int64_t* long_len = pos + N + 1;
  int64_t* seg_ofs = long_len + N + 1;
  const int64_t tmp_len = scan_tmp_len(int64_t(n) + 1) + 8;
  LMPK_TRY(ctx->s_small.ensure(4096 + size_t(tmp_len) * 8));
  int* d_max = reinterpret_cast<int*>(ctx->s_small.ptr) + 128;
  int64_t* stmp = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(ctx->s_small.ptr) + 4096);
  k_perm_counts<<<grid_n(ctx, n), 256, 0, st>>>(n, row_ptr, perm, cnt, is_long, 32);
  launch_count_add(ctx, 1);
  LMPK_TRY(device_excl_scan<int32_t, int32_t>(ctx, cnt, n, out_rp, 0, true, stmp, st));
  // longest short row picks the bitonic width
  LMPK_CHECK_CUDA(cudaMemsetAsync(d_max, 0, 4, st));
  k_max_i32<<<grid_n(ctx, n), 256, 0, st>>>(cnt, n, d_max);
  launch_count_add(ctx, 1);
  int max_len = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&max_len, d_max, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  const int gs = int(std::min<int64_t>(int64_t(ctx->sm_count) * 32, (int64_t(n) * 32 + 255) / 256));
  if (max_len <= 8)
    k_perm_short_rows<8><<<gs, 256, 0, st>>>(n, row_ptr, col, val, perm, inv, out_rp, out_col, out_val);
  else if (max_len <= 16)
    k_perm_short_rows<16><<<gs, 256, 0, st>>>(n, row_ptr, col, val, perm, inv, out_rp, out_col, out_val);
  else
    k_perm_short_rows<32><<<gs, 256, 0, st>>>(n, row_ptr, col, val, perm, inv, out_rp, out_col, out_val);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  if (max_len > 32) {
    // long rows: compact them, then stable radix sort by column and by segment
    LMPK_TRY(device_excl_scan<int32_t, int64_t>(ctx, is_long, n, pos, 0, true, stmp, st));
    int64_t n_long = 0;
    LMPK_CHECK_CUDA(cudaMemcpyAsync(&n_long, pos + n, 8, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    LMPK_TRY(ctx->s_b.ensure(size_t(n_long) * 4 + 64));
    int32_t* long_rows = reinterpret_cast<int32_t*>(ctx->s_b.ptr);
    k_compact_long<<<grid_n(ctx, n), 256, 0, st>>>(n, is_long, pos, long_rows, cnt, long_len);
    launch_count_add(ctx, 1);
    LMPK_TRY(device_excl_scan<int64_t, int64_t>(ctx, long_len, n_long, seg_ofs, 0, true, stmp, st));
    int64_t E = 0;
    LMPK_CHECK_CUDA(cudaMemcpyAsync(&E, seg_ofs + n_long, 8, cudaMemcpyDeviceToHost, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    LMPK_ARG_CHECK(E < (int64_t(1) << 32), "long-row elements exceed 2^32");
    LMPK_TRY(ctx->s_c.ensure(size_t(E) * (4 * 5 + 8) + 64));
    uint32_t* k0 = reinterpret_cast<uint32_t*>(ctx->s_c.ptr);
    uint32_t* v0 = k0 + E;
    uint32_t* k1 = v0 + E;
    uint32_t* v1 = k1 + E;
    uint32_t* seg_of = v1 + E;
    int64_t* src_of = reinterpret_cast<int64_t*>(seg_of + E + (E & 1));
    const int64_t cnt_len = radix_counts_len(E);
    const int64_t tmp2 = scan_tmp_len(cnt_len) + 8;
    LMPK_TRY(ctx->s_d.ensure(size_t(cnt_len) * 12 + size_t(tmp2) * 8 + 64));
    uint32_t* counts = reinterpret_cast<uint32_t*>(ctx->s_d.ptr);
    int64_t* offsets = reinterpret_cast<int64_t*>(counts + ((cnt_len + 1) & ~int64_t(1)));
    int64_t* stmp2 = offsets + cnt_len;
    k_perm_long_fill<<<int(std::min<int64_t>(n_long, 65535)), 256, 0, st>>>(
        int32_t(n_long), long_rows, seg_ofs, row_ptr, col, perm, inv, k0, v0, seg_of, src_of);
    launch_count_add(ctx, 1);
    int bits = 0;
    while (bits < 32 && (int64_t(1) << bits) < int64_t(n)) ++bits;
    bool first = true;
    LMPK_TRY(device_radix_sort(ctx, k0, v0, k1, v1, E, bits, counts, offsets, stmp2, &first, st));
    uint32_t* ids = first ? v0 : v1;
    uint32_t* kk = first ? k0 : k1;
    uint32_t* ko = first ? k1 : k0;
    uint32_t* vo = first ? v1 : v0;
    k_gather_seg_keys<<<grid_n(ctx, E), 256, 0, st>>>(E, ids, seg_of, kk);
    launch_count_add(ctx, 1);
    int sbits = 0;
    while (sbits < 32 && (int64_t(1) << sbits) < n_long) ++sbits;
    bool first2 = true;
    LMPK_TRY(device_radix_sort(ctx, kk, ids, ko, vo, E, sbits, counts, offsets, stmp2, &first2, st));
    uint32_t* final_ids = first2 ? ids : vo;
    k_perm_long_write<<<grid_n(ctx, E), 256, 0, st>>>(E, final_ids, seg_of, seg_ofs, long_rows, out_rp,
                                                      src_of, col, val, inv, out_col, out_val);
    launch_count_add(ctx, 1);
  }
  LMPK_CHECK_CUDA(cudaGetLastError());
  return LMPK_OK;
}

extern "C" int lmpk_permute_vectors(lmpk_ctx* ctx, int32_t n, const int32_t* perm, const double* in,
                                    int64_t ld_in, double* out, int64_t ld_out, int32_t n_vec,
                                    int32_t width, int scatter, void* stream) {
  LMPK_ARG_CHECK(ctx && perm && in && out, "lmpk_permute_vectors: NULL argument");
  LMPK_ARG_CHECK(width == 1 || width == 2, "width must be 1 (real) or 2 (complex)");
  LMPK_ARG_CHECK(in != out, "in and out must not alias");
  if (n == 0 || n_vec == 0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  const int g = grid_n(ctx, int64_t(n) * n_vec);
  if (width == 1)
    k_permute_vec<1><<<g, 256, 0, st>>>(n, perm, in, ld_in, out, ld_out, n_vec, scatter);
  else
    k_permute_vec<2><<<g, 256, 0, st>>>(n, perm, in, ld_in, out, ld_out, n_vec, scatter);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

namespace lmpk {
// one CTA per row segment: min of first columns, max of last columns
__global__ void k_segment_col_range(const int32_t* row_ptr, const int32_t* col, int64_t n_seg,
                                    const int64_t* seg_ptr, int32_t* out_min, int32_t* out_max) {
  __shared__ int32_t s_mn[32], s_mx[32];
  for (int64_t g = blockIdx.x; g < n_seg; g += gridDim.x) {
    int32_t mn = INT32_MAX, mx = -1;
    for (int64_t r = seg_ptr[g] + threadIdx.x; r < seg_ptr[g + 1]; r += blockDim.x) {
      const int32_t a = row_ptr[r], b = row_ptr[r + 1];
      if (b > a) {
        mn = min(mn, col[a]);
        mx = max(mx, col[b - 1]);
      }
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if ((threadIdx.x & 31) == 0) {
      s_mn[threadIdx.x >> 5] = mn;
      s_mx[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int nw = blockDim.x >> 5;
      mn = threadIdx.x < nw ? s_mn[threadIdx.x] : INT32_MAX;
      mx = threadIdx.x < nw ? s_mx[threadIdx.x] : -1;
      mn = __reduce_min_sync(0xffffffffu, mn);
      mx = __reduce_max_sync(0xffffffffu, mx);
      if (threadIdx.x == 0) {
        out_min[g] = mn;
        out_max[g] = mx;
      }
    }
    __syncthreads();
  }
}
}  // namespace lmpk

extern "C" int lmpk_segment_col_range(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col,
                                      int64_t n_seg, const int64_t* seg_ptr, int32_t* out_min,
                                      int32_t* out_max, void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && col && seg_ptr && out_min && out_max,
                 "lmpk_segment_col_range: NULL argument");
  if (n_seg <= 0) return LMPK_OK;
  const int g = int(std::min<int64_t>(n_seg, int64_t(ctx->sm_count) * 8));
  k_segment_col_range<<<g, 256, 0, as_stream(stream)>>>(row_ptr, col, n_seg, seg_ptr, out_min, out_max);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}

// ------------------------------------------------------------------ windows
// Rows [lo, hi) of a CRS matrix with the columns outside [lo, hi) dropped and
// the rest shifted by -lo, entry order kept (dist.py window_csr): one rank's
// level-range window, cut in HBM.
namespace lmpk {
__global__ void k_win_count(const int32_t* row_ptr, const int32_t* col, int32_t lo, int32_t hi, int32_t* cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < int64_t(hi) - lo;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = lo + int32_t(i);
    int32_t c = 0;
    for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) c += (col[e] >= lo && col[e] < hi) ? 1 : 0;
    cnt[i] = c;
  }
}
__global__ void k_win_emit(const int32_t* row_ptr, const int32_t* col, const double* val, int32_t lo, int32_t hi,
                           const int32_t* out_rp, int32_t* out_col, double* out_val) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < int64_t(hi) - lo;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int32_t r = lo + int32_t(i);
    int32_t o = out_rp[i];
    for (int32_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
      const int32_t c = col[e];
      if (c >= lo && c < hi) {
        out_col[o] = c - lo;
        out_val[o] = val[e];
        ++o;
      }
    }
  }
}
// out = c * x in the reference's order (complex: re = cr xr - ci xi, im = cr xi + ci xr)
template <bool CPLX>
__global__ void k_vec_scale(int64_t n, const double* x, double cr, double ci, double* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if constexpr (CPLX) {
      const double xr = x[2 * i], xi = x[2 * i + 1];
      out[2 * i] = __dsub_rn(__dmul_rn(cr, xr), __dmul_rn(ci, xi));
      out[2 * i + 1] = __dadd_rn(__dmul_rn(cr, xi), __dmul_rn(ci, xr));
    } else {
      out[i] = __dmul_rn(cr, x[i]);
    }
  }
}
}  // namespace lmpk

extern "C" int lmpk_csr_window(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                               const double* val, int32_t lo, int32_t hi, int32_t* out_row_ptr, int32_t* out_col,
                               double* out_val, int64_t* out_nnz, void* stream) {
  LMPK_ARG_CHECK(ctx && row_ptr && out_row_ptr && out_nnz, "lmpk_csr_window: NULL argument");
  LMPK_ARG_CHECK(0 <= lo && lo <= hi && hi <= n, "window [%d, %d) out of bounds for n=%d", lo, hi, n);
  cudaStream_t st = as_stream(stream);
  const int32_t w = hi - lo;
  if (w == 0) {
    LMPK_CHECK_CUDA(cudaMemsetAsync(out_row_ptr, 0, 4, st));
    *out_nnz = 0;
    return LMPK_OK;
  }
  LMPK_TRY(ctx->s_a.ensure(size_t(w) * 4 + 64));
  int32_t* cnt = reinterpret_cast<int32_t*>(ctx->s_a.ptr);
  const int64_t tmp_len = scan_tmp_len(int64_t(w) + 1) + 8;
  LMPK_TRY(ctx->s_small.ensure(4096 + size_t(tmp_len) * 8));
  int64_t* stmp = reinterpret_cast<int64_t*>(reinterpret_cast<char*>(ctx->s_small.ptr) + 4096);
  k_win_count<<<grid_n(ctx, w), 256, 0, st>>>(row_ptr, col, lo, hi, cnt);
  launch_count_add(ctx, 1);
  LMPK_TRY(device_excl_scan<int32_t, int32_t>(ctx, cnt, w, out_row_ptr, 0, true, stmp, st));
  int32_t total = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&total, out_row_ptr + w, 4, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  *out_nnz = total;
  if (total > 0) {
    LMPK_ARG_CHECK(out_col && out_val, "lmpk_csr_window: NULL output arrays");
    k_win_emit<<<grid_n(ctx, w), 256, 0, st>>>(row_ptr, col, val, lo, hi, out_row_ptr, out_col, out_val);
    launch_count_add(ctx, 1);
  }
  LMPK_CHECK_CUDA(cudaGetLastError());
  return LMPK_OK;
}

extern "C" int lmpk_vec_scale(lmpk_ctx* ctx, int64_t n, const double* x, double c_re, double c_im, int complex_state,
                              double* out, void* stream) {
  LMPK_ARG_CHECK(ctx && x && out, "lmpk_vec_scale: NULL argument");
  if (n == 0) return LMPK_OK;
  cudaStream_t st = as_stream(stream);
  if (complex_state)
    k_vec_scale<true><<<grid_n(ctx, n), 256, 0, st>>>(n, x, c_re, c_im, out);
  else
    k_vec_scale<false><<<grid_n(ctx, n), 256, 0, st>>>(n, x, c_re, 0.0, out);
  LMPK_CHECK_CUDA(cudaGetLastError());
  launch_count_add(ctx, 1);
  return LMPK_OK;
}
