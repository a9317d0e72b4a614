/*
 * lmpk.h -- C ABI of the B200-native level-blocked matrix power kernel (MPK).
 *
 * This is the drop-in boundary that replaces the numba/numpy hot paths of the
 * reference package `levelmpk` (arXiv 2205.01598, /root/reference/pkg).  The
 * reference selects its kernels through LEVELMPK_BACKEND at import time
 * (pkg/src/levelmpk/backend.py:21-40); a `cuda` backend binds these entry
 * points with ctypes (see INTEGRATION.md for the binding a maintainer adds).
 *
 * Conventions
 *   - All array pointers are DEVICE pointers owned by the caller (torch
 *     tensors in the Python host layer).  The library never frees them.
 *   - CRS layout follows pkg/src/levelmpk/csr.py:16-20,35-37: row_ptr int32
 *     [n+1], col int32 [nnz] (strictly increasing per row), val f64 [nnz].
 *   - Power vectors follow PowerVectors (pkg/src/levelmpk/executor.py:33-53):
 *     slot s of a y block is y + s*ldy, each slot n contiguous doubles.
 *     Complex128 state (Chebyshev, LMPK_COMPLEX) stores interleaved (re, im)
 *     pairs, i.e. slot s occupies 2*n doubles starting at y + s*ldy.
 *   - `stream` is a cudaStream_t passed as void*; NULL is the legacy stream.
 *     Calls are stream-ordered and asynchronous unless stated otherwise.
 *   - Every entry point returns an int status: 0 (LMPK_OK) or a negative
 *     code; lmpk_last_error() returns a thread-local message.  The Python
 *     layer maps LMPK_ERR_ARG to ValueError and everything else to
 *     RuntimeError, mirroring the reference's exception contract
 *     (SURVEY.md section 8b "Errors").
 *   - Summation semantics.  Every output row is
 *       tmp = 0.0; for k in row order: tmp = tmp + val[k]*x[col[k]]
 *     (the numba kernel csr.py:195-201 / executor.py:127-135).  With
 *     LMPK_FLAG_EXACT the multiply and add are separately rounded (no FMA
 *     contraction): results are bitwise identical to the reference's numba
 *     backend on the same permuted matrix.  Without it the same ordered chain
 *     uses fused multiply-adds (one fp64 op per nonzero instead of two); the
 *     per-power relative L2 error stays far below the 1e-12 the MPK contract
 *     allows.  lmpk_spmv_rows / lmpk_mpk_baseline are always exact.
 */
#ifndef LMPK_H
#define LMPK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMPK_ABI_VERSION 1

/* status codes */
#define LMPK_OK 0
#define LMPK_ERR_ARG -1         /* invalid argument -> ValueError            */
#define LMPK_ERR_CUDA -2        /* CUDA runtime failure -> RuntimeError       */
#define LMPK_ERR_WATCHDOG -3    /* device spin watchdog fired -> RuntimeError */
#define LMPK_ERR_NOMEM -4       /* allocation failure -> RuntimeError         */
#define LMPK_ERR_UNSUPPORTED -5 /* configuration not supported                */

/* kernel ids per power (pkg/src/levelmpk/plan.py:34-35) */
#define LMPK_KERNEL_SPMV 0 /* y_out = A y_in                                */
#define LMPK_KERNEL_CHEB 1 /* y_out = 2 A y_in - y_prev (Chebyshev T_{n+1}) */

/* flags */
#define LMPK_FLAG_COMPLEX 0x1       /* vectors are complex128 (interleaved)      */
#define LMPK_FLAG_MODE_STREAM 0x10  /* force streaming (L2) wavefront mode       */
#define LMPK_FLAG_MODE_RESIDENT 0x20/* force SMEM-resident wavefront mode       */
#define LMPK_FLAG_NO_TMA 0x40       /* read tile blocks from global memory (no   */
                                    /* shared-memory staging)                   */
#define LMPK_FLAG_SWEEP 0x80        /* lmpk_mpk_run: n_powers dependency-free   */
                                    /* sweeps (k back-to-back SpMVs) on the     */
                                    /* same tiles -- the blocking-free baseline */
#define LMPK_FLAG_EXACT 0x400       /* bit-exact row sums (see Summation below) */
#define LMPK_FLAG_READY_QUEUE 0x1000 /* q = 1: dependency-driven ready-queue walk */
#define LMPK_FLAG_RING 0x4000       /* tiling: ring walk (small tiles streamed   */
                                    /* through a ring of smem pieces; items are */
                                    /* runs of tiles, tile_nnz_hint = run nnz,  */
                                    /* slots = ring depth <= 16)                */
#define LMPK_FLAG_PLAIN 0x8000      /* tiling: default plan on plain blocks      */
#define LMPK_FLAG_NO_HUB_ROWS 0x10000 /* lmpk_spmv_rows / lmpk_mpk_baseline: the    */
                                    /* caller knows that no row of the range    */
                                    /* holds more than 128 entries, so the call */
                                    /* skips the hub-row scan and its one       */
                                    /* host synchronisation (fully asynchronous)*/
#define LMPK_FLAG_COMPRESS 0x2000   /* tiling: compressed tile blocks (int16     */
                                    /* column offsets, per-tile dictionary of   */
                                    /* <= 256 values), bitwise-identical sums   */
                                     /* instead of the skewed-key item order      */
/* bits 8-9 (0x100, 0x200): L2 eviction policy of staged blocks that a later
 * power group re-reads: 0 evict_last, 1 evict_normal, 2/3 evict_first.      */

#define LMPK_MAX_POWERS 64

typedef struct lmpk_ctx lmpk_ctx;       /* per-device scratch + epoch counters */
typedef struct lmpk_tiling lmpk_tiling; /* tile geometry of one matrix for MPK */

/* ---------------------------------------------------------------- misc */
int lmpk_abi_version(void);
const char* lmpk_last_error(void);
/* Device properties used for planning. */
int lmpk_device_info(int device, int* sm_count, int* max_smem_per_block,
                     int* max_smem_per_sm, int* l2_bytes, int* cc_major, int* cc_minor);

int lmpk_ctx_create(lmpk_ctx** out, int device);
int lmpk_ctx_destroy(lmpk_ctx* ctx);
/* Number of kernel launches this ctx issued since creation (for gpu_launches). */
int64_t lmpk_ctx_launch_count(const lmpk_ctx* ctx);
/* Phase counters of the pipelined MPK kernels, collected only when the
 * environment variable LMPK_PROFILE is set at ctx creation (16 words). */
int lmpk_ctx_profile(lmpk_ctx* ctx, unsigned long long* out, int reset);
/* Debug: event trace of CTAs 0-1 of the last MPK launch (LMPK_PROFILE and
 * LMPK_TRACE set at ctx creation); 16-byte records, returns the count. */
int lmpk_ctx_trace(lmpk_ctx* ctx, void* out, int64_t max_records);

/* ---------------------------------------------------------------- SpMV
 * out[r] = sum_k val[k]*x[col[k]] for r in [r0, r1); other rows untouched.
 * Replaces spmv_rows / _spmv_rows_kernel (pkg/src/levelmpk/csr.py:192-233);
 * spmv_range's inclusive-bounds and alias checks live in the Python layer
 * (csr.py:235-249).  x and out must not alias. */
int lmpk_spmv_rows(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                   const double* val, const double* x, double* out, int32_t r0, int32_t r1,
                   int flags, void* stream);

/* Baseline MPK: p_m back-to-back full-range SpMV sweeps,
 *   y[p] = A y[p-1], p = 1..p_m, slot p at y + p*ldy.
 * Replaces run_baseline / build_baseline_plan (executor.py:233-266): one
 * kernel launch per power (the "k back-to-back SpMVs" roofline). */
int lmpk_mpk_baseline(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                      const double* val, double* y, int64_t ldy, int32_t p_m, int flags,
                      void* stream);

/* ---------------------------------------------------------------- level-blocked MPK
 * Tiling: contiguous row tiles of the (level-permuted) matrix sized to the
 * on-chip budget, plus each tile's dependency range [dep_lo, dep_hi] (tiles
 * owning its column indices).  The kernel walks the power/tile wavefront:
 * tile t at power p runs only after tiles dep_lo(t)..dep_hi(t) finished
 * power p-1 -- the GPU form of the Lp-diagram conditions (A)/(B)/(C)
 * (pkg/src/levelmpk/schedule.py:195-240, plan.py:322-370). */
typedef struct lmpk_tiling_info {
  int32_t n_tiles;
  int32_t p_m;
  int32_t mode;          /* 1 = SMEM-resident (q = p_m), 2 = grouped streaming  */
  int32_t grid;          /* CTAs launched                                       */
  int32_t block;         /* threads per CTA                                     */
  int32_t smem_bytes;    /* dynamic shared memory per CTA                       */
  int32_t tile_nnz_cap;  /* max nonzeros per tile                               */
  int32_t max_fwd_reach; /* max over tiles of (dep_hi - t)                      */
  int32_t chain_reach;   /* max (p_m-1)-step forward dependency chain, in tiles */
  int32_t max_row_nnz;
  int32_t queue_slack;   /* key spacing M - q*D between power groups           */
  int64_t nnz;
  int64_t block_bytes;   /* size of the tile-SELL-32 copy of the matrix         */
  int32_t powers_per_item; /* q: powers computed per staged tile block          */
  int32_t slots;         /* R: staged items held per CTA                        */
  int32_t x_staged_tiles; /* tiles whose gathers come from a staged x buffer    */
  int32_t compressed_tiles; /* tiles in the compressed block format (int16      */
                            /* column offsets; LMPK_FLAG_COMPRESS)              */
  int32_t dict_tiles;    /* compressed tiles with a value dictionary (<= 256)   */
  int32_t super_tiles;   /* ring walk (mode 3): work items per power = runs of  */
                         /* consecutive tiles streamed through the smem ring   */
  int64_t lean_bytes;    /* ring walk: width-sorted lean copy of the blocks    */
                         /* (0: the tiling runs the general ring kernel)      */
  int32_t lean_pattern_tiles; /* lean tiles storing each slice's distinct rows once */
  int32_t lean_xstaged;  /* 1: the lean walk stages the gathered runs of y_{p-1} */
                         /* in shared memory (a piece = lean block + x buffer)  */
  int32_t lean_ring;     /* staged lean walk: pieces in the shared-memory ring   */
  int32_t lean_piece;    /* staged lean walk: bytes of one piece                 */
  int32_t dp_tiles;      /* tiles in the diagonal-private dictionary format (DP  */
                         /* tiling: one global dictionary of off-diagonal values, */
                         /* a private diagonal value per row, 32-bit offsets)    */
} lmpk_tiling_info;

/* Tuning knobs of lmpk_tiling_create (0 = library default). */
typedef struct lmpk_tiling_params {
  int32_t tile_nnz_hint; /* cap a tile block near this many nonzeros            */
  int32_t ctas_per_sm;   /* reserved (one CTA per SM)                           */
  int32_t threads;       /* reserved (1 producer + LMPK_NC consumer warps)      */
  int32_t queue_slack;   /* streaming: key spacing M - D (tiles)                */
  int32_t mode_flags;    /* LMPK_FLAG_MODE_STREAM / LMPK_FLAG_MODE_RESIDENT;    */
                         /* LMPK_FLAG_COMPLEX: tiling for complex vectors (no */
                         /* x staging); LMPK_FLAG_NO_TMA: unstaged blocks     */
  int32_t slots;         /* staged items held per CTA (<= 4)                    */
  int32_t powers_per_item; /* q: powers per staged tile (0 = plan; MODE_RESIDENT */
                           /* forces q = p_m, MODE_STREAM defaults to q = 1)   */
} lmpk_tiling_params;

/* Build the tiling for an n-row matrix already resident on the device and
 * re-lay the matrix out as tile-SELL-32 blocks (a copy owned by the tiling).
 * Synchronizes `stream` (small D2H of tile geometry). */
int lmpk_tiling_create(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                       const double* val, int32_t p_m, const lmpk_tiling_params* params,
                       lmpk_tiling** out, lmpk_tiling_info* info, void* stream);
int lmpk_tiling_destroy(lmpk_tiling* t);
/* Copy tile geometry to host arrays: tile_row[n_tiles+1], dep_lo/dep_hi[n_tiles]. */
int lmpk_tiling_geometry(const lmpk_tiling* t, int32_t* tile_row, int32_t* dep_lo,
                         int32_t* dep_hi);

/* Per-power kernel configuration (plan.py:206-211 out_slot/in_slot/prev_slot/
 * kernel/acc_coef, which in the reference depend only on an item's power). */
typedef struct lmpk_power_cfg {
  int32_t n_powers;                    /* p = 1..n_powers                       */
  int32_t out_slot[LMPK_MAX_POWERS];   /* index by p-1                          */
  int32_t in_slot[LMPK_MAX_POWERS];
  int32_t prev_slot[LMPK_MAX_POWERS];
  int32_t kernel[LMPK_MAX_POWERS];     /* LMPK_KERNEL_SPMV | LMPK_KERNEL_CHEB   */
  double acc_coef_re[LMPK_MAX_POWERS]; /* acc += coef * y_out (if use_acc)      */
  double acc_coef_im[LMPK_MAX_POWERS]; /* imaginary part (LMPK_FLAG_COMPLEX)    */
} lmpk_power_cfg;

/* Run the level-blocked MPK over `tiling` (built for this matrix).
 * Replaces run_plan / _run_numba / _walk (executor.py:84-230).  y holds
 * n_slots slots of stride ldy (in doubles); acc (length n, or 2n complex)
 * is accumulated in place when use_acc != 0 (cheb.py:229,240). */
int lmpk_mpk_run(lmpk_ctx* ctx, const lmpk_tiling* tiling, double* y, int64_t ldy, int32_t n_slots,
                 const lmpk_power_cfg* cfg, double* acc, int use_acc, int flags, void* stream);

/* The same plan semantics as lmpk_mpk_run on the CRS arrays, one sweep per
 * power with the power's kernel (SpMV / Chebyshev step) and accumulation
 * fused into the row store -- run_plan's path (executor.py:213-230) for
 * matrices whose rows exceed the tile format (> 65535 entries, power-law
 * hubs): real or complex128 (LMPK_FLAG_COMPLEX) vectors, results bitwise those
 * of the level-blocked walk. */
int lmpk_mpk_crs_run(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                     const double* val, double* y, int64_t ldy, int32_t n_slots,
                     const lmpk_power_cfg* cfg, double* acc, int use_acc, int flags, void* stream);

/* Synchronize `stream` and report a device-side failure of the last MPK
 * launches (watchdog: a dependency spin exceeded its bound, the analogue of
 * the reference's join watchdog executor.py:173-179). */
int lmpk_ctx_check(lmpk_ctx* ctx, void* stream);
/* Test hook: set the ctx's epoch counter (the next MPK launch uses epoch + 1;
 * values >= 2^24 - 1 make it wrap).  Returns the previous value. */
int64_t lmpk_ctx_set_epoch(lmpk_ctx* ctx, int64_t epoch);

/* ---------------------------------------------------------------- BFS levels + permutation
 * Level construction of levels.py:48-114: BFS distance classes of the
 * symmetrized pattern A|A^T from `root`; each level sorted ascending by
 * vertex id; exhausted components restart at the lowest unvisited vertex.
 * Outputs perm (new->old), inv_perm (old->new) and level_ptr (int64, up to
 * n+1 entries; *n_levels receives L so that level_ptr[0..L] is valid).
 * Bit-exact with the reference.  Synchronizes `stream`. */
int lmpk_bfs_levels(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                    int32_t root, int32_t* perm, int32_t* inv_perm, int64_t* level_ptr,
                    int64_t* n_levels, void* stream);

/* Symmetrized pattern A|A^T (levels.py:48-61).  Returns via *sym_nnz the
 * pattern size; if the pattern of A is already symmetric *is_symmetric = 1
 * and nothing is written.  Otherwise out_row_ptr (int64[n+1]) and out_col
 * (capacity cap) receive the canonical pattern; call with out_col == NULL
 * to query the size first.  Synchronizes `stream`. */
int lmpk_symmetrized_pattern(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr,
                             const int32_t* col, int* is_symmetric, int64_t* sym_nnz,
                             int64_t* out_row_ptr, int32_t* out_col, int64_t cap, void* stream);

/* CRS build from COO triplets (replaces CsrMatrix.from_triplets,
 * csr.py:72-94): rows/cols int64[m], vals f64[m] (device).  Range errors
 * ("row index out of range" / "column index out of range") return
 * LMPK_ERR_ARG.  Entries are ordered by (row, col) stably; with
 * sum_duplicates, repeated (row, col) entries are summed in numpy's
 * np.add.reduceat order (bit-exact).  out_row_ptr holds n+1 entries,
 * out_col/out_val m (capacity); *out_nnz (host) receives the entry count.
 * Synchronises the stream. */
int lmpk_csr_from_triplets(lmpk_ctx* ctx, int32_t n, int64_t m, const int64_t* rows,
                           const int64_t* cols, const double* vals, int sum_duplicates,
                           int32_t* out_row_ptr, int32_t* out_col, double* out_val,
                           int64_t* out_nnz, void* stream);

/* B[i,j] = A[perm[i], perm[j]], canonical (csr.py:169-187).  out arrays are
 * n+1 / nnz long.  Bit-exact with the reference. */
int lmpk_permute_symmetric(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                           const double* val, const int32_t* perm, const int32_t* inv_perm,
                           int32_t* out_row_ptr, int32_t* out_col, double* out_val, void* stream);

/* Vector permutations (csr.py:158-166, executor.py:69-76) on `n_vec`
 * vectors of `width` doubles per entry (1 real, 2 complex), stride ldv.
 * gather:  out[v][i] = in[v][perm[i]]   (apply_to_vector)
 * scatter: out[v][perm[i]] = in[v][i]   (undo_on_vector / undo_permutation) */
int lmpk_permute_vectors(lmpk_ctx* ctx, int32_t n, const int32_t* perm, const double* in,
                         int64_t ld_in, double* out, int64_t ld_out, int32_t n_vec, int32_t width,
                         int scatter, void* stream);

/* One rank's window of a level-permuted matrix (multi-GPU, dist.py
 * window_csr; no reference counterpart -- the reference has no multi-process
 * code): rows [lo, hi), columns outside [lo, hi) dropped, the
 * rest shifted by -lo, entry order kept.  out_row_ptr[hi-lo+1]; out_col /
 * out_val need room for row_ptr[hi] - row_ptr[lo] entries (may be NULL when
 * that is 0).  *out_nnz = kept entries.  Synchronizes the stream. */
int lmpk_csr_window(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col,
                    const double* val, int32_t lo, int32_t hi, int32_t* out_row_ptr, int32_t* out_col,
                    double* out_val, int64_t* out_nnz, void* stream);

/* out = c * x over n entries (complex_state: interleaved (re, im) pairs and
 * re = c_re x_re - c_im x_im, im = c_re x_im + c_im x_re) -- the accumulator
 * start acc = c_0 T_0 of ChebPropagator.step (cheb.py:229). */
int lmpk_vec_scale(lmpk_ctx* ctx, int64_t n, const double* x, double c_re, double c_im, int complex_state,
                   double* out, void* stream);

/* Per-level nonzero counts: out[i] = row_ptr[level_ptr[i+1]] - row_ptr[level_ptr[i]]
 * (groups.py:257-262 _level_nnz on the permuted matrix). */
int lmpk_level_nnz(lmpk_ctx* ctx, const int32_t* row_ptr, const int64_t* level_ptr,
                   int64_t n_levels, int64_t* out, void* stream);

/* Column range of row segments [seg_ptr[g], seg_ptr[g+1]): out_min[g] / out_max[g]
 * = smallest / largest column index (INT32_MAX / -1 for empty segments).
 * Feeds the point-to-point checks of plan.py:322-370 for whole level groups. */
int lmpk_segment_col_range(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col,
                           int64_t n_seg, const int64_t* seg_ptr, int32_t* out_min,
                           int32_t* out_max, void* stream);

/* The item queue of a tiling as int32 triples (tile, first power (1-based),
 * number of powers) in the order the kernel's producers take them; out may be
 * NULL to query the count.  Host arrays.  Feeds the traffic oracle below with
 * the schedule the GPU really walks. */
int lmpk_tiling_items(const lmpk_tiling* t, int32_t* out, int64_t cap, int64_t* n_out);

/* Software cache oracle (HOST pointers, no GPU work): replays the per-row
 * accesses of a plan's items (row_start/row_end/power/in_slot/out_slot, int64
 * [n_items]) in list order through a fully associative LRU of cap_lines lines
 * of line_bytes; by_power int64[n_powers][4] receives the bytes missed per
 * power and stream (val, col, row_ptr, y).  bypass != 0: no cache, every
 * access counts its own size.  Replaces _sim_numba / _sim_python
 * (pkg/src/levelmpk/traffic.py:78-189). */
int lmpk_simulate_traffic(int64_t n_rows, const int32_t* row_ptr, const int32_t* col,
                          int64_t n_items, const int64_t* row_start, const int64_t* row_end,
                          const int64_t* power, const int64_t* in_slot, const int64_t* out_slot,
                          int64_t n_powers, int64_t cap_lines, int64_t line_bytes, int bypass,
                          int64_t* by_power);

#ifdef __cplusplus
}
#endif
#endif /* LMPK_H */
