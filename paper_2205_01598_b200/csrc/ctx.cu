// ctx.cu -- error reporting, per-device context, scratch pools.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>

#include "lmpk_internal.cuh"

namespace lmpk {

static thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int Scratch::ensure(size_t want) {
  if (want <= bytes && ptr) return LMPK_OK;
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
  size_t grow = want + want / 4 + 256;
  cudaError_t e = cudaMalloc(&ptr, grow);
  if (e != cudaSuccess) {
    set_error("scratch cudaMalloc(%zu) failed: %s", grow, cudaGetErrorString(e));
    ptr = nullptr;
    return LMPK_ERR_NOMEM;
  }
  bytes = grow;
  return LMPK_OK;
}

void Scratch::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

int launch_count_add(lmpk_ctx* ctx, int n) {
  if (ctx) ctx->launches += n;
  return LMPK_OK;
}

int ctx_check_device_error(lmpk_ctx* ctx, const char* what) {
  if (ctx && ctx->err.host && *ctx->err.host != 0) {
    int code = *ctx->err.host;
    *ctx->err.host = 0;
    set_error("%s: device watchdog fired (code %d): a dependency spin exceeded its bound",
              what, code);
    return LMPK_ERR_WATCHDOG;
  }
  return LMPK_OK;
}

}  // namespace lmpk

using namespace lmpk;

extern "C" int lmpk_abi_version(void) { return LMPK_ABI_VERSION; }

extern "C" const char* lmpk_last_error(void) { return g_last_error.c_str(); }

extern "C" int lmpk_device_info(int device, int* sm_count, int* max_smem_per_block,
                                int* max_smem_per_sm, int* l2_bytes, int* cc_major,
                                int* cc_minor) {
  int v;
  LMPK_CHECK_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  if (sm_count) *sm_count = v;
  LMPK_CHECK_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  if (max_smem_per_block) *max_smem_per_block = v;
  LMPK_CHECK_CUDA(
      cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device));
  if (max_smem_per_sm) *max_smem_per_sm = v;
  LMPK_CHECK_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, device));
  if (l2_bytes) *l2_bytes = v;
  LMPK_CHECK_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, device));
  if (cc_major) *cc_major = v;
  LMPK_CHECK_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, device));
  if (cc_minor) *cc_minor = v;
  return LMPK_OK;
}

extern "C" int lmpk_ctx_create(lmpk_ctx** out, int device) {
  LMPK_ARG_CHECK(out != nullptr, "lmpk_ctx_create: out is NULL");
  *out = nullptr;
  int major = 0, minor = 0;
  lmpk_ctx* c = new lmpk_ctx();
  c->device = device;
  int rc = lmpk_device_info(device, &c->sm_count, &c->max_smem_block, &c->max_smem_sm,
                            &c->l2_bytes, &major, &minor);
  if (rc != LMPK_OK) {
    delete c;
    return rc;
  }
  if (major < 10) {
    delete c;
    set_error("liblmpk requires an sm_100a (Blackwell) device, found sm_%d%d", major, minor);
    return LMPK_ERR_UNSUPPORTED;
  }
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) {
    void* hp = nullptr;
    e = cudaHostAlloc(&hp, 64, cudaHostAllocMapped);
    if (e == cudaSuccess) {
      memset(hp, 0, 64);
      c->err.host = reinterpret_cast<volatile int*>(hp);
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->err.dev), hp, 0);
    }
  }
  if (e == cudaSuccess) e = cudaMalloc(&c->queue_ctr, 64);
  if (e == cudaSuccess) {
    // planning temporaries come from the device's default stream-ordered pool
    // (tmp_alloc): keep freed blocks cached instead of returning them at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  if (e == cudaSuccess && getenv("LMPK_PROFILE") != nullptr) {
    // 16 phase counters + (LMPK_TRACE) an event trace of CTAs 0 and 1
    const size_t words = 16 + (getenv("LMPK_TRACE") ? size_t(kTraceCtas) * kTraceEvents * 2 : 0);
    c->prof_words = words;
    e = cudaMalloc(&c->prof, words * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->prof, 0, words * sizeof(unsigned long long));
  }
  if (e == cudaSuccess) e = cudaMemset(c->queue_ctr, 0, 64);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    set_error("lmpk_ctx_create: %s", cudaGetErrorString(e));
    lmpk_ctx_destroy(c);
    return LMPK_ERR_CUDA;
  }
  *out = c;
  return LMPK_OK;
}

extern "C" int lmpk_ctx_destroy(lmpk_ctx* c) {
  if (!c) return LMPK_OK;
  cudaDeviceSynchronize();
  Scratch* pools[] = {&c->s_small, &c->s_a, &c->s_b, &c->s_c,
                      &c->s_d,     &c->s_e, &c->s_f, &c->s_g, &c->s_heavy, &c->s_prod};
  for (Scratch* s : pools) s->release();
  if (c->queue_ctr) cudaFree(c->queue_ctr);
  if (c->heavy_ev) cudaEventDestroy(c->heavy_ev);
  if (c->prof) cudaFree(c->prof);
  if (c->err.host) cudaFreeHost(const_cast<int*>(c->err.host));
  delete c;
  return LMPK_OK;
}

extern "C" int64_t lmpk_ctx_launch_count(const lmpk_ctx* c) { return c ? c->launches : 0; }

// Event trace of the last MPK launch (LMPK_PROFILE + LMPK_TRACE at ctx
// creation): per traced CTA kTraceEvents records {time_ns, kind | slot << 8 |
// warp << 16, item}; returns the number of 16-byte records copied.
extern "C" int lmpk_ctx_trace(lmpk_ctx* c, void* out, int64_t max_records) {
  LMPK_ARG_CHECK(c && out, "lmpk_ctx_trace: NULL argument");
  if (!c->prof || c->prof_words <= 16) return 0;
  const int64_t n = std::min<int64_t>(max_records, int64_t(kTraceCtas) * kTraceEvents);
  LMPK_CHECK_CUDA(cudaDeviceSynchronize());
  LMPK_CHECK_CUDA(cudaMemcpy(out, c->prof + 16, size_t(n) * 16, cudaMemcpyDeviceToHost));
  LMPK_CHECK_CUDA(cudaMemset(c->prof + 16, 0, (c->prof_words - 16) * sizeof(unsigned long long)));
  return static_cast<int>(n);
}

// Phase counters of the pipelined kernels (LMPK_PROFILE=1 at ctx creation):
// [0] consumer ns waiting for work, [1] consumer ns computing, [2] items
// consumed (per warp), [3] producer dependency poll rounds, [4] rounds with
// nothing ready, [5] producer ns alive, [6] items grabbed, [7] ns TMA issue ->
// staged observed, [8] ns staged -> pushed (dependency wait), [9] ns last push
// -> slot free observed (compute + publish), [10] producer loop iterations,
// [12] item slot cycles.  reset != 0 zeroes them.
extern "C" int lmpk_ctx_profile(lmpk_ctx* c, unsigned long long* out, int reset) {
  LMPK_ARG_CHECK(c && out, "lmpk_ctx_profile: NULL argument");
  if (!c->prof) {
    memset(out, 0, 16 * sizeof(unsigned long long));
    return LMPK_OK;
  }
  LMPK_CHECK_CUDA(cudaDeviceSynchronize());
  LMPK_CHECK_CUDA(cudaMemcpy(out, c->prof, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  if (reset) LMPK_CHECK_CUDA(cudaMemset(c->prof, 0, 16 * sizeof(unsigned long long)));
  return LMPK_OK;
}
