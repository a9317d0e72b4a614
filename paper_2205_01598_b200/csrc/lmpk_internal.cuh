// lmpk_internal.cuh -- shared device/host helpers of liblmpk (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <chrono>
#include <vector>

#include "lmpk.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "liblmpk is written for sm_100a (B200) only"
#endif

namespace lmpk {

constexpr int kTraceCtas = 2;        // CTAs traced with LMPK_TRACE
constexpr int kTraceEvents = 16384;  // records per traced CTA

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);

#define LMPK_CHECK_CUDA(call)                                                              \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      cudaGetLastError();                                                                  \
      ::lmpk::set_error("%s:%d: %s failed: %s", __FILE__, __LINE__, #call,                 \
                        cudaGetErrorString(e_));                                           \
      return LMPK_ERR_CUDA;                                                                \
    }                                                                                      \
  } while (0)

#define LMPK_ARG_CHECK(cond, ...)                                                          \
  do {                                                                                     \
    if (!(cond)) {                                                                         \
      ::lmpk::set_error(__VA_ARGS__);                                                      \
      return LMPK_ERR_ARG;                                                                 \
    }                                                                                      \
  } while (0)

#define LMPK_TRY(...)                                                                      \
  do {                                                                                     \
    int rc_ = (__VA_ARGS__);                                                               \
    if (rc_ != LMPK_OK) return rc_;                                                        \
  } while (0)

// ------------------------------------------------------------------ ctx
// Grow-only device scratch buffer owned by a ctx.
struct Scratch {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t want);
  void release();
};

struct DeviceFlags {  // host-mapped pinned words the device writes on failure
  volatile int* host = nullptr;
  int* dev = nullptr;
};

}  // namespace lmpk

struct lmpk_ctx {
  int device = 0;
  int sm_count = 0;
  int max_smem_block = 0;  // opt-in max per block
  int max_smem_sm = 0;
  int l2_bytes = 0;
  int64_t launches = 0;
  lmpk::DeviceFlags err;   // watchdog / device error word
  // MPK synchronisation state (epoch-tagged counters, never memset per call)
  uint32_t epoch = 0;
  uint32_t wrap_gen = 0;   // bumped when the epoch counter wraps
  // scratch pools
  lmpk::Scratch s_small, s_a, s_b, s_c, s_d, s_e, s_f, s_g;
  lmpk::Scratch s_heavy;  // CRS kernel: list of heavy rows (count, entries, (row, product offset) pairs)
  lmpk::Scratch s_prod;   // CRS kernel: products of the heavy rows' entries (compact)
  cudaEvent_t heavy_ev = nullptr;  // recorded after the last kernel reading s_heavy
  uint64_t* queue_ctr = nullptr;  // monotone work-queue counter (device)
  uint64_t queue_base = 0;        // host mirror of the counter value
  unsigned long long* prof = nullptr;  // phase counters when LMPK_PROFILE is set
  size_t prof_words = 0;
};

// Tile geometry + the matrix re-laid out as tile-SELL-32 blocks (see mpk.cu).
struct lmpk_tiling {
  lmpk_ctx* ctx = nullptr;
  lmpk_tiling_info info{};
  int32_t n = 0;
  int32_t* d_tile_row = nullptr;   // [n_tiles+1] first row of each tile (multiples of 32)
  int64_t* d_tile_ofs = nullptr;   // [n_tiles+1] byte offset of each tile block
  int32_t* d_tile_E = nullptr;     // [n_tiles] padded entries (multiple of 32) per tile
  int32_t* d_dep_lo = nullptr;     // [n_tiles]
  int32_t* d_dep_hi = nullptr;     // [n_tiles]
  int32_t* d_tile_nseg = nullptr;  // [n_tiles] x-segments (0: global columns)
  int32_t* d_tile_xent = nullptr;  // [n_tiles] x-buffer entries
  int32_t* d_tile_mode = nullptr;  // [n_tiles] compressed block format (NULL: all plain)
  bool ring = false;               // ring walk (mpk_ring_kernel): items are super-tiles
  int32_t piece = 0;               // ring: bytes of one smem piece (= tile cap)
  int32_t* d_st_first = nullptr;   // ring: [n_super+1] first tile of each super-tile
  int32_t* d_st_lo = nullptr;      // ring: [n_super] dependency range (tiles)
  int32_t* d_st_hi = nullptr;
  int32_t staged_tiles = 0, max_xent = 0;
  int64_t xoff = 0;                // byte offset of the x buffer in a slot (0: no staging)
  int32_t* d_rdep_ptr = nullptr;   // [n_tiles+1] reverse dependencies (ready-queue walk)
  int32_t* d_rdep = nullptr;
  uint32_t* d_rcnt = nullptr;      // [p_m][n_tiles] readiness counters
  int32_t* d_rqueue = nullptr;     // [p_m * n_tiles] ready queue
  uint32_t* d_rctrl = nullptr;     // head / tail / next power-1 tile
  int32_t* d_items = nullptr;      // item queue order, packed (t << 8) | power group
  int32_t n_items = 0;
  uint32_t* d_progress = nullptr;  // [n_tiles] epoch-tagged power counters
  unsigned char* d_blocks = nullptr;  // tile-SELL-32 matrix blocks
  int64_t block_bytes = 0;
  int32_t max_block = 0;           // largest tile block (bytes)
  int32_t slots = 1;               // staged items held per CTA
  std::vector<int32_t> h_tile_row, h_dep_lo, h_dep_hi;
  std::vector<int32_t> h_items, h_st_first;  // host copies of the item queue (lmpk_tiling_items)
  // lean blocks (lean_kernel.cuh): width-sorted units, built when every tile
  // is a compressed tile of width <= 8 with one value format
  unsigned char* d_lean = nullptr;
  int64_t* d_lean_ofs = nullptr;   // [n_tiles + 1]
  uint8_t* d_rowlen = nullptr;     // [n] row lengths (slow path of padded rows)
  int32_t lean_vd = -1;            // -1 none, 0 raw values, 1 dictionary
  int64_t lean_bytes = 0;
  int32_t lean_piece = 0;          // bytes of the largest lean block (the lean ring's piece)
  // lean x staging (mpk_xlean_kernel): a piece is [lean block | x buffer]
  int32_t lean_xs = 0;             // 1: column fields are x-buffer entries, gathers come from shared memory
  int32_t lean_xp = 0;             // 1: XP blocks (row records, units of up to 4 slices; lean_kernel.cuh)
  int32_t lean_xoff = 0;           // byte offset of the x buffer in a piece (= largest lean block)
  int32_t lean_np = 0;             // ring depth of the staged kernel
  int32_t lean_ctas = 1;           // CTAs per SM the staged kernel runs with (2: 12 consumer warps each)
  int32_t lean_cplx = 0;           // vectors the x buffer was sized for (16-byte entries)
  int4* d_lean_runs = nullptr;     // [n_tiles * 32] {first entry, entries, buffer entry, 0}
  int2* d_lean_xinfo = nullptr;    // [n_tiles] {runs, staged entries}
  int4* d_lean_wl = nullptr;       // staged kernel: per-CTA work lists (2 x int4 per piece, mpk_lean.cu)
  int32_t* d_lean_wl_ptr = nullptr;  // [grid + 1] first piece record of each CTA's list
  int32_t lean_wl_grid = 0;        // grid the work lists were cut for
  std::vector<int64_t> h_lean_ofs;
  std::vector<int2> h_lean_xinfo;
  uint32_t wrap_gen = 0;           // ctx wrap generation its progress words belong to
};

namespace lmpk {

int ctx_check_device_error(lmpk_ctx* ctx, const char* what);
static inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// LMPK_TILING_PROF=1: host wall-clock marks of lmpk_tiling_create's phases
struct PhaseTimer {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTimer(cudaStream_t s) : on(getenv("LMPK_TILING_PROF") != nullptr), st(s) {
    if (on) t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t1 = std::chrono::steady_clock::now();
    fprintf(stderr, "[tiling] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};



// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acqrel_cta_smem(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old)
               : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// try_wait with a suspend-time hint: the warp sleeps in the barrier unit until
// the phase completes (or ~hint ns pass) instead of re-issuing the poll, so
// idle warps leave the issue slots to the warps that compute.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity, 1000000u)) {
  }
}

// 1-D TMA bulk copy global -> shared (cp.async.bulk), completion on mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// L2 prefetch of a global range (bytes a multiple of 16, 16-byte aligned).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}
// Same with a 32-bit shared-memory destination address.
__device__ __forceinline__ void bulk_g2s_a(uint32_t dst_smem, const void* src_gmem, uint32_t bytes,
                                           uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(dst_smem),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Coherent (weak, L1-allocating) global load -- never the .nc path, since the
// MPK kernel reads vectors other CTAs write during the same launch.
__device__ __forceinline__ double ld_weak(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_weak2(const double2* p) {
  double2 v;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_cg(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Coherent global load of a gathered operand (non-volatile so the scheduler
// may batch it; its address depends on data read after the acquire points).
__device__ __forceinline__ double ldg_f64(const char* p) {
  double v;
  asm("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t lds_s32(uint32_t a) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// Readers of one staged tile block, by byte offset.  SmemBlk reads a block
// staged in shared memory (volatile so nothing is hoisted above the mbarrier
// wait that publishes the TMA bytes); GlbBlk reads the block straight from
// global memory (immutable for the whole launch, so the .nc path is safe).
struct SmemBlk {
  uint32_t a;
  __device__ __forceinline__ int32_t i1(uint32_t o) const {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a + o));
    return v;
  }
  __device__ __forceinline__ int2 i2(uint32_t o) const {
    int2 v;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a + o));
    return v;
  }
  __device__ __forceinline__ int4 i4(uint32_t o) const {
    int4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a + o));
    return v;
  }
  __device__ __forceinline__ double d1(uint32_t o) const {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a + o));
    return v;
  }
  __device__ __forceinline__ double2 d2(uint32_t o) const {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a + o));
    return v;
  }
  __device__ __forceinline__ uint32_t u16(uint32_t o) const {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a + o));
    return v;
  }
  __device__ __forceinline__ uint32_t u8(uint32_t o) const {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a + o));
    return v;
  }
};
struct GlbBlk {
  const unsigned char* a;
  // streamed once per power: keep it out of L1 (the gathers own the L1)
  __device__ __forceinline__ int32_t i1(uint32_t o) const {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(a + o));
    return v;
  }
  __device__ __forceinline__ int2 i2(uint32_t o) const {
    int2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a + o));
    return v;
  }
  __device__ __forceinline__ int4 i4(uint32_t o) const {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(a + o));
    return v;
  }
  __device__ __forceinline__ double d1(uint32_t o) const {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(a + o));
    return v;
  }
  __device__ __forceinline__ double2 d2(uint32_t o) const {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a + o));
    return v;
  }
  __device__ __forceinline__ uint32_t u16(uint32_t o) const {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(a + o));
    return v;
  }
};
__device__ __forceinline__ double2 ldg_f64x2(const char* p) {
  double2 v;
  asm("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_acquire_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s32(int32_t* p, int32_t v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acqrel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Bit-exact CRS row sum: tmp = 0.0; tmp = tmp + v[k]*x[c[k]] in storage order,
// each multiply and add separately rounded (csr.py:196-201, executor.py:127-130).
// The gathers of a chunk of 8 are issued before the dependent add chain.
template <typename LoadX>
__device__ __forceinline__ double row_sum_exact(const int32_t* c, const double* v, int len,
                                                LoadX ldx) {
  double tmp = 0.0;
  int k = 0;
  for (; k + 8 <= len; k += 8) {
    int cc[8];
    double vv[8], xx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      cc[j] = c[k + j];
      vv[j] = v[k + j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) xx[j] = ldx(cc[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) tmp = __dadd_rn(tmp, __dmul_rn(vv[j], xx[j]));
  }
  const int rem = len - k;
  if (rem > 0) {
    int cc[8];
    double vv[8], xx[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < rem) {
        cc[j] = c[k + j];
        vv[j] = v[k + j];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < rem) xx[j] = ldx(cc[j]);
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < rem) tmp = __dadd_rn(tmp, __dmul_rn(vv[j], xx[j]));
  }
  return tmp;
}

// Same for complex128 vectors with a real matrix: real and imaginary parts
// are two independent storage-order sums.
template <typename LoadX2>
__device__ __forceinline__ double2 row_sum_exact_c(const int32_t* c, const double* v, int len,
                                                   LoadX2 ldx) {
  double tr = 0.0, ti = 0.0;
  int k = 0;
  for (; k + 4 <= len; k += 4) {
    int cc[4];
    double vv[4];
    double2 xx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cc[j] = c[k + j];
      vv[j] = v[k + j];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) xx[j] = ldx(cc[j]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      tr = __dadd_rn(tr, __dmul_rn(vv[j], xx[j].x));
      ti = __dadd_rn(ti, __dmul_rn(vv[j], xx[j].y));
    }
  }
  for (; k < len; ++k) {
    const double vv = v[k];
    const double2 xx = ldx(c[k]);
    tr = __dadd_rn(tr, __dmul_rn(vv, xx.x));
    ti = __dadd_rn(ti, __dmul_rn(vv, xx.y));
  }
  return make_double2(tr, ti);
}

// ------------------------------------------------------------------ planning temporaries
// Stream-ordered scratch of the tiling / planning code (cudaMallocAsync on
// the call's stream; the ctx raises the default pool's release threshold so
// the blocks are reused): a cudaFree synchronises the device, and a tiling
// used to pay ~25 of them.
template <typename T>
static inline int tmp_alloc(T** p, size_t count, cudaStream_t st) {
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(p), (count > 0 ? count : 1) * sizeof(T), st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ::lmpk::set_error("cudaMallocAsync(%zu) failed: %s", count * sizeof(T), cudaGetErrorString(e));
    *p = nullptr;
    return LMPK_ERR_NOMEM;
  }
  return LMPK_OK;
}
static inline void tmp_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

// ------------------------------------------------------------------ host helpers
int launch_count_add(lmpk_ctx* ctx, int n);
static inline int div_up(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace lmpk
