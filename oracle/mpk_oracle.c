/*
 * mpk_oracle.c -- C restatement of the reference's CPU hot path.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/ as a checker and by bench.py's
 * cpu_baseline / --impl reference legs as the CPU implementation of the
 * reference (the reference is Python+numba and does not travel to the GPU
 * box).  The product (paper_2205_01598_b200) never links or calls it.
 *
 * Every routine restates /root/reference/pkg/src/levelmpk with the same
 * floating-point operation order (compiled with -ffp-contract=off, no
 * -ffast-math), so results are bitwise equal to the numba backend:
 *   spmv_rows      csr.py:195-201     tmp = 0.0; tmp += val*x[col] in order
 *   mpk_baseline   executor.py:261    p_m full sweeps (rows split over threads)
 *   mpk_walk       executor.py:84-179 the point-to-point walker: W threads
 *                  walk the same item list; per-(item, worker) done/bnd_done
 *                  flags; checks FULL/BOUNDARY wait on all W flags
 *   bfs_levels     levels.py:64-103   key-sort form: BFS distances from root,
 *                  remaining components rooted at their minimum vertex, stable
 *                  counting sort by (component rank, distance)
 *   permute_symm   csr.py:169-187     row gather, inv_perm map, per-row sort
 * Parity pin: tests/test_oracle_golden.py (fixtures from the reference itself).
 */
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <sched.h>
#include <omp.h>

/* ------------------------------------------------------------------ SpMV */
static inline double row_sum(const int32_t* rp, const int32_t* col, const double* val,
                             const double* x, int64_t r) {
  double tmp = 0.0;
  for (int64_t k = rp[r]; k < rp[r + 1]; ++k) tmp += val[k] * x[col[k]];
  return tmp;
}

void oracle_spmv_rows(const int32_t* rp, const int32_t* col, const double* val, const double* x,
                      double* out, int64_t r0, int64_t r1) {
  for (int64_t r = r0; r < r1; ++r) out[r] = row_sum(rp, col, val, x, r);
}

/* y[p] = A y[p-1], p = 1..p_m, rows split statically over `threads` */
void oracle_mpk_baseline(int64_t n, const int32_t* rp, const int32_t* col, const double* val,
                         double* y, int64_t ldy, int32_t p_m, int32_t threads) {
  for (int32_t p = 1; p <= p_m; ++p) {
    const double* x = y + (int64_t)(p - 1) * ldy;
    double* out = y + (int64_t)p * ldy;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t r = 0; r < n; ++r) out[r] = row_sum(rp, col, val, x, r);
  }
}

/* ------------------------------------------------------------------ p2p walker */
static inline void wait_all(_Atomic uint8_t* flags, int64_t m, int32_t workers) {
  for (int32_t w = 0; w < workers; ++w) {
    int spins = 0;
    while (atomic_load_explicit(&flags[m * workers + w], memory_order_acquire) == 0) {
      if ((++spins & 63) == 0) sched_yield();
    }
  }
}

/* Restatement of _walk (executor.py:101-150) executed by `workers` threads.
 * chunks: (n_items, workers+1); bnd_point: (n_items, workers);
 * per-item kernel slots as in plan.py:206-211. */
void oracle_mpk_walk(const int32_t* rp, const int32_t* col, const double* val, double* y,
                     int64_t ldy, double* acc, int32_t use_acc, int64_t n_items,
                     const int64_t* out_slot, const int64_t* in_slot, const int64_t* prev_slot,
                     const int64_t* kern, const double* acoef, const int64_t* chunks,
                     const int64_t* bnd_point, int32_t barrier, const int64_t* check_ptr,
                     const int64_t* check_item, const int64_t* check_kind, int32_t workers) {
  _Atomic uint8_t* done = calloc((size_t)(n_items > 0 ? n_items : 1) * workers, 1);
  _Atomic uint8_t* bnd = calloc((size_t)(n_items > 0 ? n_items : 1) * workers, 1);
#pragma omp parallel num_threads(workers)
  {
    const int32_t wid = omp_get_thread_num();
    for (int64_t it = 0; it < n_items; ++it) {
      if (barrier) {
        if (it > 0) wait_all(done, it - 1, workers);
      } else {
        for (int64_t c = check_ptr[it]; c < check_ptr[it + 1]; ++c)
          wait_all(check_kind[c] == 1 ? bnd : done, check_item[c], workers);
      }
      const int64_t cs = chunks[it * (workers + 1) + wid];
      const int64_t ce = chunks[it * (workers + 1) + wid + 1];
      const int64_t bp = bnd_point[it * workers + wid];
      const double* yin = y + in_slot[it] * ldy;
      const double* ypv = y + prev_slot[it] * ldy;
      double* yout = y + out_slot[it] * ldy;
      const int cheb = kern[it] == 1;
      const double cf = acoef[it];
      for (int64_t r = cs; r < ce; ++r) {
        if (r == bp) atomic_store_explicit(&bnd[it * workers + wid], 1, memory_order_release);
        double tmp = row_sum(rp, col, val, yin, r);
        if (cheb) tmp = 2.0 * tmp - ypv[r];
        yout[r] = tmp;
        if (use_acc) acc[r] += cf * tmp;
      }
      atomic_store_explicit(&bnd[it * workers + wid], 1, memory_order_release);
      atomic_store_explicit(&done[it * workers + wid], 1, memory_order_release);
    }
  }
  free((void*)done);
  free((void*)bnd);
}

/* ------------------------------------------------------------------ BFS levels */
/* Symmetric pattern (rp, col) of n vertices.  perm[n], level_ptr[n+1] out.
 * Returns the number of levels. */
int64_t oracle_bfs_levels(int64_t n, const int64_t* rp, const int32_t* col, int64_t root,
                          int32_t* perm, int64_t* level_ptr) {
  int32_t* dist = malloc(sizeof(int32_t) * n);
  int32_t* comp = malloc(sizeof(int32_t) * n); /* component rank */
  int32_t* queue = malloc(sizeof(int32_t) * n);
  for (int64_t v = 0; v < n; ++v) dist[v] = -1;
  int32_t rank = 0;
  int64_t next_root = 0;
  int64_t total_levels = 0;
  int64_t* comp_levels = malloc(sizeof(int64_t) * (n + 1));
  int64_t start_vertex = root;
  while (1) {
    /* BFS of one component from start_vertex */
    int64_t qh = 0, qt = 0;
    queue[qt++] = (int32_t)start_vertex;
    dist[start_vertex] = 0;
    comp[start_vertex] = rank;
    int32_t maxd = 0;
    while (qh < qt) {
      const int32_t u = queue[qh++];
      for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
        const int32_t v = col[k];
        if (dist[v] < 0) {
          dist[v] = dist[u] + 1;
          comp[v] = rank;
          if (dist[v] > maxd) maxd = dist[v];
          queue[qt++] = v;
        }
      }
    }
    comp_levels[rank] = maxd + 1;
    total_levels += maxd + 1;
    ++rank;
    /* restart at the lowest unvisited vertex = minimum of its component */
    while (next_root < n && dist[next_root] >= 0) ++next_root;
    if (next_root >= n) break;
    start_vertex = next_root;
  }
  /* level id = base[comp] + dist; stable counting sort of ids 0..n-1 */
  int64_t* base = malloc(sizeof(int64_t) * (rank + 1));
  base[0] = 0;
  for (int32_t c = 0; c < rank; ++c) base[c + 1] = base[c] + comp_levels[c];
  int64_t* cnt = calloc((size_t)total_levels + 1, sizeof(int64_t));
  for (int64_t v = 0; v < n; ++v) cnt[base[comp[v]] + dist[v] + 1]++;
  for (int64_t l = 0; l < total_levels; ++l) cnt[l + 1] += cnt[l];
  for (int64_t l = 0; l <= total_levels; ++l) level_ptr[l] = cnt[l];
  for (int64_t v = 0; v < n; ++v) perm[cnt[base[comp[v]] + dist[v]]++] = (int32_t)v;
  free(cnt);
  free(base);
  free(comp_levels);
  free(queue);
  free(comp);
  free(dist);
  return total_levels;
}

/* ------------------------------------------------------------------ permutation */
typedef struct {
  int32_t key;
  double val;
} kv_t;

static int kv_cmp(const void* a, const void* b) {
  const int32_t x = ((const kv_t*)a)->key, y = ((const kv_t*)b)->key;
  return (x > y) - (x < y);
}

void oracle_permute_symmetric(int64_t n, const int32_t* rp, const int32_t* col, const double* val,
                              const int32_t* perm, const int32_t* inv, int32_t* out_rp,
                              int32_t* out_col, double* out_val, int32_t threads) {
  out_rp[0] = 0;
  for (int64_t i = 0; i < n; ++i) out_rp[i + 1] = out_rp[i] + (rp[perm[i] + 1] - rp[perm[i]]);
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const int32_t o = perm[i];
    const int32_t a = rp[o], len = rp[o + 1] - a;
    int32_t* c = out_col + out_rp[i];
    double* v = out_val + out_rp[i];
    if (len > 64) { /* long rows: qsort (keys are unique, so order is exact) */
      kv_t* buf = malloc(sizeof(kv_t) * (size_t)len);
      for (int32_t j = 0; j < len; ++j) {
        buf[j].key = inv[col[a + j]];
        buf[j].val = val[a + j];
      }
      qsort(buf, (size_t)len, sizeof(kv_t), kv_cmp);
      for (int32_t j = 0; j < len; ++j) {
        c[j] = buf[j].key;
        v[j] = buf[j].val;
      }
      free(buf);
      continue;
    }
    for (int32_t j = 0; j < len; ++j) {
      /* insertion sort by new column (unique keys) */
      const int32_t key = inv[col[a + j]];
      const double vv = val[a + j];
      int32_t q = j;
      while (q > 0 && c[q - 1] > key) {
        c[q] = c[q - 1];
        v[q] = v[q - 1];
        --q;
      }
      c[q] = key;
      v[q] = vv;
    }
  }
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
