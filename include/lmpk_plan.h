/*
 * lmpk_plan.h -- C ABI of the planning side of liblmpk: recursive level
 * refinement and the dependency analysis behind execution plans.
 *
 * Companion of lmpk.h (same conventions: device pointers owned by the caller
 * unless stated, int status, lmpk_last_error()).  These entry points replace
 * the numpy planning code of the reference package:
 *   - pkg/src/levelmpk/groups.py:192-366  (_Builder: induced-subgraph BFS of a
 *     refined span, diamond-halo key sort)
 *   - pkg/src/levelmpk/plan.py:103-129    (_item_deps: the true dependencies of
 *     a flat item list)
 *   - pkg/src/levelmpk/plan.py:322-370    (_runtime_checks: boundary-granular
 *     second check)
 * so that preprocessing of a 10^8-nonzero matrix stays on the GPU.
 */
#ifndef LMPK_PLAN_H
#define LMPK_PLAN_H

#include "lmpk.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Per-level nonzero counts under a permutation that has not been applied yet:
 * out[i] = sum over rows r in [level_ptr[i], level_ptr[i+1]) of the length of
 * row perm[r] of the ORIGINAL matrix (groups.py:260-262 _level_nnz).
 * level_ptr: device int64[n_levels+1]; out: device int64[n_levels]. */
int lmpk_level_nnz_perm(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* perm,
                        const int64_t* level_ptr, int64_t n_levels, int64_t* out, void* stream);

/* Refine one span (groups.py:238-258, :354-357): the subgraph induced by the
 * permuted rows [r0, r1) of the symmetric pattern (sym_ptr / sym_col in
 * ORIGINAL numbering; sym_ptr is int64 when ptr64 != 0, else int32) is
 * traversed by BFS from its first row with the reference's restart rule, and
 * perm[r0:r1] is reordered in place by that traversal.  level_ptr_out (device
 * int64, capacity r1 - r0 + 1) receives the child level pointer relative to
 * r0; *n_levels the level count.  Synchronises the stream. */
int lmpk_refine_span(lmpk_ctx* ctx, int32_t n, const void* sym_ptr, int ptr64, const int32_t* sym_col,
                     int32_t* perm, int32_t r0, int32_t r1, int64_t* level_ptr_out, int64_t* n_levels,
                     void* stream);

/* Diamond-halo keys (groups.py:305-307): key_orig[v] = -1 for every vertex,
 * then key_orig[perm[r]] = g for rows r of child group g
 * (group_ptr device int64[n_groups+1], permuted row numbers). */
int lmpk_halo_seed(lmpk_ctx* ctx, int32_t n, const int32_t* perm, int64_t n_groups,
                   const int64_t* group_ptr, int32_t* key_orig, void* stream);

/* One halo level (groups.py:264-280, :318-324): keys[i] = max of key_orig over
 * the neighbourhood of row perm[lo + i] (-1 without neighbours); the rows
 * [lo, hi) of perm are stably reordered by key, key_orig of those vertices is
 * set to their key, and keys_out (device int32[hi - lo]) receives the sorted
 * keys. */
int lmpk_halo_level_sort(lmpk_ctx* ctx, int32_t n, const void* sym_ptr, int ptr64, const int32_t* sym_col,
                         int32_t* perm, int32_t* key_orig, int32_t lo, int32_t hi, int32_t* keys_out,
                         void* stream);

/* inv[perm[i]] = i. */
int lmpk_invert_perm(lmpk_ctx* ctx, int32_t n, const int32_t* perm, int32_t* inv, void* stream);

/* True dependencies of a flat item list (plan.py:103-129).  Items are row
 * ranges [row_start[u], row_end[u]) at power[u] (HOST int64 arrays); items of
 * one power must not overlap.  Item u depends on the items of power[u] - 1
 * that own one of u's rows or one of the columns u's rows read (device CRS).
 * Output (HOST): dep_ptr int64[n_items + 1] and, through *dep_out, a
 * malloc'ed int64 array of dependency item indices, ascending per item, which
 * the caller releases with lmpk_host_free. */
int lmpk_item_deps(lmpk_ctx* ctx, int32_t n, const int32_t* row_ptr, const int32_t* col, int64_t n_items,
                   const int64_t* row_start, const int64_t* row_end, const int64_t* power,
                   int64_t* dep_ptr, int64_t** dep_out, void* stream);
void lmpk_host_free(void* p);

/* For every item u (HOST int64 row ranges): the largest column of its rows
 * that lies in [col_lo[u], col_hi[u]) -- -1 if none (plan.py:360-362: the
 * columns "inside" the second check's target).  out_max: HOST int32[n_items]. */
int lmpk_item_col_max_in_range(lmpk_ctx* ctx, const int32_t* row_ptr, const int32_t* col, int64_t n_items,
                               const int64_t* row_start, const int64_t* row_end, const int64_t* col_lo,
                               const int64_t* col_hi, int32_t* out_max, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LMPK_PLAN_H */
