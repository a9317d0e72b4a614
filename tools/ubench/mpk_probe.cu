// mpk_probe.cu -- compute probe of the row kernel (tools only, not the walk).
#include "mpk_kernel.cuh"

namespace lmpk {
// ---------------------------------------------------------------- compute probe
// Each CTA stages tile blockIdx.x once and runs the row kernel `iters` times
// (power 1 into slot 1) with no cross-CTA synchronisation: the attainable
// per-SM rate of the tile kernel itself.
template <bool EXACT, int MODE>
__global__ void k_probe_compute(MpkParams P, PowerCfgDev C, int iters, int n_tiles) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ uint64_t bar;
  __shared__ PowTab s_pow[1];
  build_powtab(s_pow, P, C);
  const int32_t t = blockIdx.x % n_tiles;
  const int64_t ofs = P.tile_ofs[t], bytes = P.tile_ofs[t + 1] - ofs;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const bool staged = bytes <= P.smem_cap;
  if (threadIdx.x == 0) {
    if (staged) {
      mbar_arrive_expect_tx(&bar, uint32_t(bytes));
      bulk_g2s(smem_raw, P.blocks + ofs, uint32_t(bytes), &bar, policy_evict_normal());
    } else {
      mbar_arrive_expect_tx(&bar, 0);
    }
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  const int32_t r0 = P.tile_row[t], rows = P.tile_row[t + 1] - r0;
  const uint32_t E = uint32_t(P.tile_E[t]);
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  const int32_t tmode = P.tile_mode ? P.tile_mode[t] : 0;
  __shared__ uint32_t probe_ctr;
  for (int it = 0; it < iters; ++it) {
    if (tmode != 0) {
      __syncthreads();
      if (threadIdx.x == 0) probe_ctr = 0;
      __syncthreads();
      // compressed tile: MODE 0 = the production row kernel, 1..3 = W=7 full
      // slices with the probe gather variants
      if (!staged) return;
      const SmemBlk B{smem_u32(smem_raw)};
      const GatherGlobal G{s_pow[0].yin};
      const int32_t nd = tmode >> 8;
      const bool vd = (tmode & kModeDict) != 0;
      if constexpr (MODE == 0) {
        if (vd)
          tile_power_c<false, EXACT, false, true>(s_pow[0], P.acc, false, B, G, r0, rows, E, nd, 0, wid, nw, smem_u32(&probe_ctr));
        else
          tile_power_c<false, EXACT, false, false>(s_pow[0], P.acc, false, B, G, r0, rows, E, nd, 0, wid, nw, smem_u32(&probe_ctr));
      } else {
        const int32_t ns = (rows + 31) >> 5;
        const uint32_t dict = B.a + uint32_t(cblk_dict_off(ns, 0));
        const uint32_t col_o = uint32_t(cblk_col_off(ns, nd, 0)), val_o = uint32_t(cblk_val_off(ns, nd, E, 0));
        double* yout = s_pow[0].yout + r0;
        for (int32_t s = wid; s < ns; s += nw) {
          const int2 rec = B.i2(uint32_t(s) * 8);
          if ((rec.y & 0xffff) != 7 || (int(uint32_t(rec.y) >> 16) != 7) || !vd) continue;
          const double v = cslice_real_w<7, EXACT, true, true, GatherGlobal, MODE>(
              B, cslice<true>(col_o, val_o, uint32_t(rec.x)), uint32_t(lane), r0 + s * 32 + lane, dict, G, 7);
          stg_f64(yout + s * 32 + lane, v);
        }
      }
      continue;
    }
    if constexpr (MODE == 0) {
      if (staged)
        tile_power<false, EXACT, false>(s_pow[0], P.acc, false, SmemBlk{smem_u32(smem_raw)},
                                        GatherGlobal{s_pow[0].yin}, r0, rows, E, 0, wid, nw);
      else
        tile_power<false, EXACT, true>(s_pow[0], P.acc, false, GlbBlk{P.blocks + ofs}, GatherGlobal{s_pow[0].yin},
                                       r0, rows, E, 0, wid, nw);
    } else {
      // MODE 1..3: width-7 full slices only, single-slice path with the
      // gather variant of slice_real_w<..., PROBE = MODE>
      if (!staged) return;
      const SmemBlk B{smem_u32(smem_raw)};
      const int32_t ns = (rows + 31) >> 5;
      const uint32_t col_o = uint32_t(blk_col_off(ns, 0));
      const uint32_t vdelta = col_o + E * 4 - 2 * col_o;
      double* yout = s_pow[0].yout + r0;
      for (int32_t s = wid; s < ns; s += nw) {
        const int2 rec = B.i2(uint32_t(s) * 8);
        if ((rec.y & 0xffff) != 7 || (int(uint32_t(rec.y) >> 16) != 7)) continue;
        const uint32_t cb = uint32_t(rec.x);
        const double v = slice_real_w<7, EXACT, true, SmemBlk, GatherGlobal, MODE>(
            B, cb, 2 * cb + vdelta, uint32_t(lane) * 4, GatherGlobal{s_pow[0].yin}, 7);
        stg_f64(yout + s * 32 + lane, v);
      }
    }
  }
}

}  // namespace lmpk

using namespace lmpk;

// ns per 1000 nonzeros per SM of the tile kernel alone (see k_probe_compute).
// flags: LMPK_FLAG_EXACT selects the separately rounded chain.
extern "C" int lmpk_probe_tile_compute(lmpk_ctx* ctx, const lmpk_tiling* T, double* y, int64_t ldy,
                                       int iters, int threads, int ctas_per_sm, double* ns_per_knnz) {
  LMPK_ARG_CHECK(ctx && T && y && ns_per_knnz, "probe: NULL argument");
  const bool exact = (ctas_per_sm & 0x100) != 0;
  const int mode = (ctas_per_sm >> 12) & 7;
  ctas_per_sm &= 0xff;
  MpkParams Pm;
  memset(&Pm, 0, sizeof(Pm));
  Pm.blocks = T->d_blocks;
  Pm.tile_ofs = T->d_tile_ofs;
  Pm.tile_E = T->d_tile_E;
  Pm.tile_row = T->d_tile_row;
  Pm.y = y;
  Pm.acc = y;
  Pm.ldy = ldy;
  Pm.smem_cap = T->max_block;
  Pm.tile_mode = T->d_tile_mode;
  Pm.n_powers = 1;
  PowerCfgDev C;
  memset(&C, 0, sizeof(C));
  C.out_slot[0] = 1;
  C.in_slot[0] = 0;
  const int smem = T->max_block;
  void (*fn)(MpkParams, PowerCfgDev, int, int) = nullptr;
  switch (mode) {
    case 1: fn = exact ? k_probe_compute<true, 1> : k_probe_compute<false, 1>; break;
    case 2: fn = exact ? k_probe_compute<true, 2> : k_probe_compute<false, 2>; break;
    case 3: fn = exact ? k_probe_compute<true, 3> : k_probe_compute<false, 3>; break;
    default: fn = exact ? k_probe_compute<true, 0> : k_probe_compute<false, 0>; break;
  }
  LMPK_CHECK_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ctx->max_smem_block - 1024));
  const int grid = ctx->sm_count * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fn<<<grid, threads, smem>>>(Pm, C, 1, T->info.n_tiles);
  cudaEventRecord(a);
  fn<<<grid, threads, smem>>>(Pm, C, iters, T->info.n_tiles);
  cudaEventRecord(b);
  LMPK_CHECK_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  LMPK_CHECK_CUDA(cudaGetLastError());
  // nnz processed: each CTA one tile per iteration
  const double avg_nnz = double(T->info.nnz) / std::max(1, T->info.n_tiles);
  const double nnz = avg_nnz * grid * iters;
  *ns_per_knnz = (ms * 1e6) * ctx->sm_count / (nnz / 1000.0);
  return LMPK_OK;
}
