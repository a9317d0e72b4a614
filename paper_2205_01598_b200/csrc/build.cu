// build.cu -- device CRS build from COO triplets (CsrMatrix.from_triplets,
// pkg/src/levelmpk/csr.py:72-94): range checks, stable (row, col) order,
// duplicate sums, row_ptr.  Bit-exact with the reference's numpy build:
//   * order: np.lexsort((cols, rows)) is stable, so two stable LSD radix
//     passes (col, then row) over the triplet ids give the same permutation;
//   * sums: np.add.reduceat(vals, starts) (csr.py:88) adds, per segment
//     [a0, a1 .. am], a0 + pairwise(a1 .. am) -- numpy's float64 reduce loop
//     (IS_BINARY_REDUCE branch) with its 8-accumulator pairwise summation,
//     restated in pw_sum below and pinned against numpy by
//     tests/test_build.py (oracle/cpu_build.py is the same restatement);
//   * row_ptr: counts of the unique rows, cumsum (csr.py:91-93), here read
//     off the sorted rows of the output entries.
#include "radix_sort.cuh"

namespace lmpk {
namespace {

__global__ void k_trip_check(int64_t m, const int64_t* rows, const int64_t* cols, int64_t n, int* bad,
                             uint32_t* r32, uint32_t* c32, int32_t* row_cnt) {
  // also narrows the indices to u32: the later gathers by triplet id then
  // touch 4 B instead of 8 B per random access
  int local = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = rows[i], c = cols[i];
    if (r < 0 || r >= n) local |= 1;
    if (c < 0 || c >= n) local |= 2;
    r32[i] = uint32_t(r);
    c32[i] = uint32_t(c);
    if (r >= 0 && r < n) atomicAdd(row_cnt + r, 1);
  }
  if (local) atomicOr(bad, local);
}

// pass 1 input: key = col, value = triplet id
__global__ void k_trip_keys_col(int64_t m, const uint32_t* cols, uint32_t* k, uint32_t* v) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    k[i] = cols[i];
    v[i] = uint32_t(i);
  }
}

// pass 2 input: key = row of the id at position i (ids already col-sorted)
__global__ void k_trip_keys_row(int64_t m, const uint32_t* rows, const uint32_t* ids, uint32_t* k) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    k[i] = rows[ids[i]];
}

// sorted columns as u32 (the one random gather of cols), so the passes
// below read (row, col) of neighbouring positions sequentially
__global__ void k_trip_cols_sorted(int64_t m, const uint32_t* cols, const uint32_t* ids, uint32_t* cs) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    cs[i] = cols[ids[i]];
}

// head[i] = 1 where (row, col) of sorted position i starts a new entry
__global__ void k_trip_heads(int64_t m, const uint32_t* rk, const uint32_t* cs, int sum_dup, int32_t* head) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    int h = 1;
    if (sum_dup && i > 0) h = (rk[i] != rk[i - 1] || cs[i] != cs[i - 1]) ? 1 : 0;
    head[i] = h;
  }
}

// numpy's pairwise float64 sum (loops_utils.h: DOUBLE_pairwise_sum) over
// b[ids[0..n)], n >= 1: < 8 terms sequential (from -0.0, which is exact),
// <= 128 terms eight strided accumulators, larger halves split at a multiple of 8.
__device__ double pw_sum(const double* val, const uint32_t* ids, int64_t n) {
  // explicit stack of (offset, length) halves, evaluated in the recursive order
  struct Frame {
    const uint32_t* p;
    int64_t n;
    int state;
    double left;
  };
  Frame st[40];
  int sp = 0;
  st[0] = Frame{ids, n, 0, 0.0};
  double ret = 0.0;
  for (;;) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      double res;
      if (f.n < 8) {
        res = -0.0;
        for (int64_t i = 0; i < f.n; ++i) res += val[f.p[i]];
      } else {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = val[f.p[j]];
        int64_t i = 8;
        for (; i < f.n - (f.n % 8); i += 8) {
#pragma unroll
          for (int j = 0; j < 8; ++j) r[j] += val[f.p[i + j]];
        }
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < f.n; ++i) res += val[f.p[i]];
      }
      // return to the parent
      ret = res;
      for (;;) {
        if (sp == 0) return ret;
        Frame& par = st[--sp];
        if (par.state == 1) {  // left half done: evaluate the right half
          par.left = ret;
          par.state = 2;
          int64_t n2 = par.n / 2;
          n2 -= n2 % 8;
          st[++sp] = Frame{par.p + n2, par.n - n2, 0, 0.0};
          break;
        }
        ret = par.left + ret;  // right half done
      }
    } else {
      int64_t n2 = f.n / 2;
      n2 -= n2 % 8;
      f.state = 1;
      st[++sp] = Frame{f.p, n2, 0, 0.0};
    }
  }
}

// one thread per output entry: col, summed value, its row
__global__ void k_trip_emit(int64_t m, const uint32_t* rk, const uint32_t* cs, const double* vals,
                            const uint32_t* ids, const int32_t* head, const int64_t* pos, int32_t* out_col,
                            double* out_val, uint32_t* out_row) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    if (!head[i]) continue;
    const int64_t o = pos[i];
    int64_t e = i + 1;
    while (e < m && !head[e]) ++e;  // duplicates of one entry are rare and short
    double s = vals[ids[i]];
    if (e - i > 1) s = s + pw_sum(vals, ids + i + 1, e - i - 1);
    out_col[o] = int32_t(cs[i]);
    out_val[o] = s;
    out_row[o] = rk[i];
  }
}

// row_ptr from the (sorted) rows of the output entries: entry o opens rows
// (row[o-1], row[o]]; the last entry closes the rows after it
__global__ void k_trip_row_ptr(int64_t n_out, const uint32_t* orow, int32_t n, int32_t* row_ptr) {
  for (int64_t o = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; o < n_out; o += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = orow[o];
    const int64_t prev = o == 0 ? -1 : int64_t(orow[o - 1]);
    for (int64_t q = prev + 1; q <= r; ++q) row_ptr[q] = int32_t(o);
    if (o == n_out - 1)
      for (int64_t q = r + 1; q <= n; ++q) row_ptr[q] = int32_t(n_out);
  }
}

// ---- row-bucket path (every row holds <= kLongRow triplets): rows are
// bucketed by a counting sort, then each row's (col, id) pairs are sorted --
// by one thread for rows of <= kShortRow, by one CTA (bitonic, smem) for
// longer ones -- the same order as the two stable radix passes (lexsort by
// (row, col), ties by triplet id), without their 6 passes and id gathers.
constexpr int kShortRow = 32;

__global__ void k_trip_max(int32_t n, const int32_t* cnt, int* out) {
  int v = 0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v = max(v, cnt[i]);
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, v);
}

__global__ void k_trip_bucket(int64_t m, const uint32_t* r32, int32_t* cur, uint32_t* bucket) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    bucket[atomicAdd(cur + r32[i], 1)] = uint32_t(i);
}

__global__ void k_trip_row_sort(int32_t n, const int32_t* rstart, const uint32_t* c32, uint32_t* ids,
                                uint32_t* rk, uint32_t* cs) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < n; r += int64_t(gridDim.x) * blockDim.x) {
    const int32_t b = rstart[r], L = rstart[r + 1] - b;
    if (L > kShortRow) continue;  // k_trip_long_row_sort
    uint64_t key[kShortRow];
    for (int j = 0; j < L; ++j) {
      const uint32_t id = ids[b + j];
      uint64_t k = (uint64_t(c32[id]) << 32) | id;
      int q = j;
      for (; q > 0 && key[q - 1] > k; --q) key[q] = key[q - 1];  // insertion sort
      key[q] = k;
    }
    for (int j = 0; j < L; ++j) {
      ids[b + j] = uint32_t(key[j]);
      cs[b + j] = uint32_t(key[j] >> 32);
      rk[b + j] = uint32_t(r);
    }
  }
}

// rows of kShortRow < L <= kLongRow triplets: one CTA per row, bitonic sort
// of the (col, id) keys in shared memory (keys are unique: ids differ)
constexpr int kLongRow = 4096;

__global__ void __launch_bounds__(256) k_trip_long_row_sort(int32_t n, const int32_t* rstart, const uint32_t* c32,
                                                            uint32_t* ids, uint32_t* rk, uint32_t* cs) {
  __shared__ uint64_t key[kLongRow];
  for (int64_t r = blockIdx.x; r < n; r += gridDim.x) {
    const int32_t b = rstart[r], L = rstart[r + 1] - b;
    if (L <= kShortRow) continue;  // uniform per CTA
    int P = 1;
    while (P < L) P <<= 1;
    for (int j = threadIdx.x; j < P; j += blockDim.x) {
      if (j < L) {
        const uint32_t id = ids[b + j];
        key[j] = (uint64_t(c32[id]) << 32) | id;
      } else {
        key[j] = ~uint64_t(0);  // padding sorts last
      }
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1) {
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
          const int l = i ^ jj;
          if (l > i) {
            const uint64_t a = key[i], c = key[l];
            const bool up = (i & k) == 0;
            if ((a > c) == up) {
              key[i] = c;
              key[l] = a;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int j = threadIdx.x; j < L; j += blockDim.x) {
      ids[b + j] = uint32_t(key[j]);
      cs[b + j] = uint32_t(key[j] >> 32);
      rk[b + j] = uint32_t(r);
    }
    __syncthreads();
  }
}

inline int grid_trip(lmpk_ctx* ctx, int64_t m) {
  return int(std::max<int64_t>(1, std::min<int64_t>(int64_t(ctx->sm_count) * 8, (m + 255) / 256)));
}

}  // namespace
}  // namespace lmpk

using namespace lmpk;

extern "C" int lmpk_csr_from_triplets(lmpk_ctx* ctx, int32_t n, int64_t m, const int64_t* rows,
                                      const int64_t* cols, const double* vals, int sum_duplicates,
                                      int32_t* out_row_ptr, int32_t* out_col, double* out_val,
                                      int64_t* out_nnz, void* stream) {
  LMPK_ARG_CHECK(ctx && out_row_ptr && out_nnz, "lmpk_csr_from_triplets: NULL argument");
  LMPK_ARG_CHECK(n >= 0 && m >= 0, "n and m must be >= 0");
  LMPK_ARG_CHECK(m < (int64_t(1) << 31), "triplet count exceeds the 32-bit index range");
  LMPK_ARG_CHECK(m == 0 || (rows && cols && vals && out_col && out_val), "lmpk_csr_from_triplets: NULL argument");
  cudaStream_t st = as_stream(stream);
  *out_nnz = 0;
  if (m == 0) {
    LMPK_CHECK_CUDA(cudaMemsetAsync(out_row_ptr, 0, (size_t(n) + 1) * 4, st));
    LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
    return LMPK_OK;
  }
  const size_t M = size_t(m);
  // scratch: pos (i64, m+1) | k0 v0 k1 v1 head r32 c32 (u32/i32, m each) | cnt rstart cur (i32, n+1 each)
  const size_t N1 = size_t(n) + 1;
  LMPK_TRY(ctx->s_a.ensure((M + 1) * 8 + M * 4 * 7 + N1 * 4 * 3 + 64));
  int64_t* pos = reinterpret_cast<int64_t*>(ctx->s_a.ptr);
  uint32_t* k0 = reinterpret_cast<uint32_t*>(pos + M + 1);
  uint32_t* v0 = k0 + M;
  uint32_t* k1 = v0 + M;
  uint32_t* v1 = k1 + M;
  int32_t* head = reinterpret_cast<int32_t*>(v1 + M);
  uint32_t* r32 = reinterpret_cast<uint32_t*>(head + M);
  uint32_t* c32 = r32 + M;
  int32_t* cnt = reinterpret_cast<int32_t*>(c32 + M);
  int32_t* rstart = cnt + N1;
  int32_t* cur = rstart + N1;
  const int64_t cnt_len = radix_counts_len(m);
  const int64_t tmp_len = scan_tmp_len(std::max<int64_t>(std::max<int64_t>(cnt_len, m), int64_t(n) + 1)) + 8;
  LMPK_TRY(ctx->s_d.ensure(size_t(cnt_len) * 12 + size_t(tmp_len) * 8 + 4096));
  int* bad = reinterpret_cast<int*>(ctx->s_d.ptr);
  uint32_t* counts = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ctx->s_d.ptr) + 256);
  int64_t* offsets = reinterpret_cast<int64_t*>(counts + ((cnt_len + 1) & ~int64_t(1)));
  int64_t* stmp = offsets + cnt_len;
  const int g = grid_trip(ctx, m);
  LMPK_CHECK_CUDA(cudaMemsetAsync(bad, 0, 8, st));
  LMPK_CHECK_CUDA(cudaMemsetAsync(cnt, 0, N1 * 4, st));
  k_trip_check<<<g, 256, 0, st>>>(m, rows, cols, int64_t(n), bad, r32, c32, cnt);
  launch_count_add(ctx, 1);
  k_trip_max<<<grid_trip(ctx, n), 256, 0, st>>>(n, cnt, bad + 1);
  launch_count_add(ctx, 1);
  int h_bad2[2] = {0, 0};
  LMPK_CHECK_CUDA(cudaMemcpyAsync(h_bad2, bad, 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  const int h_bad = h_bad2[0], max_row = h_bad2[1];
  LMPK_ARG_CHECK(!(h_bad & 1), "row index out of range");
  LMPK_ARG_CHECK(!(h_bad & 2), "column index out of range");
  const uint32_t* sorted;
  const uint32_t* rk;
  uint32_t* cs;
  uint32_t* orow;
  bool have_cols = false;
  if (max_row <= kLongRow) {
    LMPK_TRY(device_excl_scan<int32_t, int32_t>(ctx, cnt, int64_t(n), rstart, 0, true, stmp, st));
    LMPK_CHECK_CUDA(cudaMemcpyAsync(cur, rstart, size_t(n) * 4, cudaMemcpyDeviceToDevice, st));
    k_trip_bucket<<<g, 256, 0, st>>>(m, r32, cur, v0);
    launch_count_add(ctx, 1);
    k_trip_row_sort<<<grid_trip(ctx, n), 256, 0, st>>>(n, rstart, c32, v0, k0, k1);
    launch_count_add(ctx, 1);
    if (max_row > kShortRow) {
      k_trip_long_row_sort<<<int(std::min<int64_t>(n, int64_t(ctx->sm_count) * 8)), 256, 0, st>>>(n, rstart, c32, v0,
                                                                                                   k0, k1);
      launch_count_add(ctx, 1);
    }
    sorted = v0;
    rk = k0;
    cs = k1;
    orow = v1;
    have_cols = true;
  } else {
    int bits = 0;
    while (bits < 32 && (int64_t(1) << bits) < int64_t(n)) ++bits;
    // pass 1: stable sort of the ids by col
    k_trip_keys_col<<<g, 256, 0, st>>>(m, c32, k0, v0);
    launch_count_add(ctx, 1);
    bool first = true;
    LMPK_TRY(device_radix_sort(ctx, k0, v0, k1, v1, m, bits, counts, offsets, stmp, &first, st));
    uint32_t* ids = first ? v0 : v1;
    uint32_t* kk = first ? k0 : k1;
    uint32_t* ko = first ? k1 : k0;
    uint32_t* vo = first ? v1 : v0;
    // pass 2: stable sort by row (lexsort's primary key)
    k_trip_keys_row<<<g, 256, 0, st>>>(m, r32, ids, kk);
    launch_count_add(ctx, 1);
    bool first2 = true;
    LMPK_TRY(device_radix_sort(ctx, kk, ids, ko, vo, m, bits, counts, offsets, stmp, &first2, st));
    sorted = first2 ? ids : vo;
    rk = first2 ? kk : ko;  // rows in sorted order
    cs = first2 ? ko : kk;  // the two free buffers of pass 2
    orow = first2 ? vo : ids;
  }
  if (!have_cols) {
    k_trip_cols_sorted<<<g, 256, 0, st>>>(m, c32, sorted, cs);
    launch_count_add(ctx, 1);
  }
  k_trip_heads<<<g, 256, 0, st>>>(m, rk, cs, sum_duplicates ? 1 : 0, head);
  launch_count_add(ctx, 1);
  LMPK_TRY(device_excl_scan<int32_t, int64_t>(ctx, head, m, pos, 0, true, stmp, st));
  int64_t n_out = 0;
  LMPK_CHECK_CUDA(cudaMemcpyAsync(&n_out, pos + m, 8, cudaMemcpyDeviceToHost, st));
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  LMPK_ARG_CHECK(n_out <= int64_t(INT32_MAX), "nnz exceeds the 32-bit index range");
  k_trip_emit<<<g, 256, 0, st>>>(m, rk, cs, vals, sorted, head, pos, out_col, out_val, orow);
  launch_count_add(ctx, 1);
  k_trip_row_ptr<<<grid_trip(ctx, n_out), 256, 0, st>>>(n_out, orow, n, out_row_ptr);
  launch_count_add(ctx, 1);
  LMPK_CHECK_CUDA(cudaGetLastError());
  LMPK_CHECK_CUDA(cudaStreamSynchronize(st));
  *out_nnz = n_out;
  return LMPK_OK;
}
