// traffic.cu -- software cache oracle (host code): replay of an execution
// plan's row order through a single-level, fully associative, line-granular
// LRU cache.  Replaces the numba replay of pkg/src/levelmpk/traffic.py:118-189
// (_sim_numba; the Python twin is traffic.py:78-111) behind the same
// simulate_traffic() front end.  This is an analysis model, not a compute
// path: it takes HOST pointers and never touches the GPU.
//
// Every array lives in its own address space (traffic.py:10-13), so a line is
// identified by (stream, line index); all keys are dense, and the LRU is a
// direct table key -> cache slot plus a doubly linked list over the slots
// (no hashing).  A capacity of zero bypasses the cache: every access counts
// its own bytes (traffic.py:15-17, :164-166).
#include <stdint.h>

#include <vector>

#include "lmpk_internal.cuh"

using namespace lmpk;

namespace {

enum { S_VAL = 0, S_COL = 1, S_ROWPTR = 2, S_Y = 3 };  // traffic.py:27
const int64_t kStreamBytes[4] = {8, 4, 4, 8};          // traffic.py:28

struct Lru {
  int64_t cap, n_used = 0, head, tail;
  std::vector<int64_t> key_of, nxt, prv;
  std::vector<int32_t> slot_of;  // dense key -> slot, -1 = not cached

  Lru(int64_t cap_lines, int64_t n_keys)
      : cap(cap_lines > 0 ? cap_lines : 1), key_of(cap), nxt(cap + 2, -1), prv(cap + 2, -1),
        slot_of(n_keys, -1) {
    head = cap;
    tail = cap + 1;
    nxt[head] = tail;
    prv[tail] = head;
  }
  // true on a miss (the line is fetched and becomes most recently used)
  inline bool touch(int64_t key) {
    int64_t s = slot_of[key];
    bool miss = s < 0;
    if (!miss) {
      prv[nxt[s]] = prv[s];
      nxt[prv[s]] = nxt[s];
    } else {
      if (n_used < cap) {
        s = n_used++;
      } else {
        s = prv[tail];
        prv[nxt[s]] = prv[s];
        nxt[prv[s]] = nxt[s];
        slot_of[key_of[s]] = -1;
      }
      key_of[s] = key;
      slot_of[key] = (int32_t)s;
    }
    nxt[s] = nxt[head];
    prv[s] = head;
    prv[nxt[head]] = s;
    nxt[head] = s;
    return miss;
  }
};

}  // namespace

extern "C" int lmpk_simulate_traffic(int64_t n_rows, const int32_t* row_ptr, const int32_t* col,
                                     int64_t n_items, const int64_t* row_start, const int64_t* row_end,
                                     const int64_t* power, const int64_t* in_slot, const int64_t* out_slot,
                                     int64_t n_powers, int64_t cap_lines, int64_t line_bytes, int bypass,
                                     int64_t* by_power) {
  if (n_rows < 0 || n_items < 0 || n_powers < 1 || line_bytes <= 0 || line_bytes % 4 || !by_power ||
      (n_items > 0 && (!row_ptr || !row_start || !row_end || !power || !in_slot || !out_slot))) {
    set_error("simulate_traffic: bad arguments");
    return LMPK_ERR_ARG;
  }
  const int64_t lv = line_bytes / 8, li = line_bytes / 4;
  for (int64_t i = 0; i < n_powers * 4; ++i) by_power[i] = 0;
  int64_t max_slot = 0;
  for (int64_t it = 0; it < n_items; ++it) {
    if (power[it] < 0 || power[it] >= n_powers || row_start[it] < 0 || row_end[it] > n_rows ||
        in_slot[it] < 0 || out_slot[it] < 0) {
      set_error("simulate_traffic: item %lld out of range", (long long)it);
      return LMPK_ERR_ARG;
    }
    max_slot = std::max(max_slot, std::max(in_slot[it], out_slot[it]));
  }
  if (bypass) {
    for (int64_t it = 0; it < n_items; ++it) {
      int64_t* bp = by_power + power[it] * 4;
      for (int64_t r = row_start[it]; r < row_end[it]; ++r) {
        int64_t w = (int64_t)row_ptr[r + 1] - row_ptr[r];
        bp[S_ROWPTR] += kStreamBytes[S_ROWPTR];
        bp[S_VAL] += w * kStreamBytes[S_VAL];
        bp[S_COL] += w * kStreamBytes[S_COL];
        bp[S_Y] += (w + 1) * kStreamBytes[S_Y];
      }
    }
    return LMPK_OK;
  }
  const int64_t nnz = n_rows > 0 ? row_ptr[n_rows] : 0;
  // dense key spaces per stream
  const int64_t base_val = 0;
  const int64_t base_col = base_val + nnz / lv + 1;
  const int64_t base_rp = base_col + nnz / li + 1;
  const int64_t base_y = base_rp + n_rows / li + 1;
  const int64_t n_keys = base_y + ((max_slot + 1) * n_rows) / lv + 1;
  if (cap_lines > 0x7fffffffLL) cap_lines = 0x7fffffffLL;
  if (cap_lines > n_keys) cap_lines = n_keys;  // never more resident lines than exist
  Lru lru(cap_lines, n_keys);
  for (int64_t it = 0; it < n_items; ++it) {
    int64_t* bp = by_power + power[it] * 4;
    const int64_t s_in = in_slot[it] * n_rows, s_out = out_slot[it] * n_rows;
    for (int64_t r = row_start[it]; r < row_end[it]; ++r) {
      if (lru.touch(base_rp + r / li)) bp[S_ROWPTR] += line_bytes;
      for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
        if (lru.touch(base_val + k / lv)) bp[S_VAL] += line_bytes;
        if (lru.touch(base_col + k / li)) bp[S_COL] += line_bytes;
        if (lru.touch(base_y + (s_in + col[k]) / lv)) bp[S_Y] += line_bytes;
      }
      if (lru.touch(base_y + (s_out + r) / lv)) bp[S_Y] += line_bytes;
    }
  }
  return LMPK_OK;
}
