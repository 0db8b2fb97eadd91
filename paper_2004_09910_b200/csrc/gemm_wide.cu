// Persistent tcgen05 GEMM for the WIDE per-micro-batch GEMMs (N >= 256 rows, e.g. C5's
// 1024-token micro-batches), with the fused epilogues of the skinny GEMM (epilogue.cuh):
//
//   D[m][n] = sum_k A(m, k) * B[n][k]      m = output feature (weight row), n = micro-batch row
//
// Why a second kernel: gemm_tc is one output tile per CTA with the epilogue after the mainloop --
// right for the weight-streaming M = 16 tiles of C2, but at N = 1024 the per-element epilogue (bias,
// GELU, fp32 pre-activation and bf16 operand stores) is as long as the mainloop and nothing overlaps
// it (ncu: tensor pipe ~2 % active, profiles/r4b_c5_gemm_*).  Here one CTA per SM loops over 128 x 128
// tiles (static round-robin, n fastest so the CTAs working on one weight tile run together and share
// it through L2) with the accumulator double-buffered in TMEM: tile t+1's TMA loads and MMAs run
// while the sixteen epilogue warps finish tile t straight from TMEM (thread = feature, 32 rows per
// tcgen05.ld chunk; every global operand of a chunk is requested before any is used).
// Deterministic: each output element comes from one CTA with a fixed k order (no split-K), so F'
// reproduces F bit-exactly (reading Z21).
#include "common.cuh"
#include "epilogue.cuh"
#include "host.h"
#include "kernels.h"

#include <algorithm>

namespace tgp {

namespace {
constexpr int WG_BM = 128, WG_BN = 128, WG_BK = 64;
constexpr int WG_STAGE = (WG_BM + WG_BN) * WG_BK * 2;  // 32 KB
#ifndef TGP_WG_STAGES
#define TGP_WG_STAGES 7
#endif
constexpr int WG_STAGES = TGP_WG_STAGES;
constexpr int WG_OFF_BAR = WG_STAGES * WG_STAGE;
constexpr int WG_SMEM = WG_OFF_BAR + 256 + 1024;
// The epilogue, not the MMA, bounds these tiles (~40 instructions per element vs 5.5 us of tensor
// work per 128 x 128 x 1600 tile), so 16 epilogue warps: four per TMEM lane quadrant, each taking
// one of the tile's four 32-row chunks (measured C5 8-layer step: 4 warps 83 ms, 8 warps 69 ms,
// 16 warps 62 ms).
#ifndef TGP_WG_EPI_WARPS
#define TGP_WG_EPI_WARPS 16
#endif
constexpr int WG_EPI_WARPS = TGP_WG_EPI_WARPS;
constexpr int WG_THREADS = 64 + 32 * WG_EPI_WARPS;

struct WideParams {
  int M, N, K;  // K multiple of 64
  int n0;       // row offset of the micro-batch inside B's tensor
  int tiles_n, tiles;
  EpiParams epi;
};
}  // namespace

template <bool A_MN, int MODE>
__global__ void __launch_bounds__(WG_THREADS, 1)
    gemm_wide_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const WideParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + WG_OFF_BAR);
  uint64_t* empty = full + WG_STAGES;
  uint64_t* tfull = empty + WG_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2] (one arrival per epilogue thread)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.K / WG_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < WG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 32 * WG_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------- TMA producer
      const uint64_t pol = policy_evict_last();  // A tiles are shared by the tiles_n CTAs of a row
      int it = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int m0 = (tile / p.tiles_n) * WG_BM, n0 = (tile % p.tiles_n) * WG_BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % WG_STAGES, r = it / WG_STAGES;
          mbar_wait(&empty[s], (uint32_t)((r & 1) ^ 1));
          uint8_t* st = smem + s * WG_STAGE;
          mbar_arrive_expect_tx(&full[s], WG_STAGE);
          const int k = kb * WG_BK;
          if (A_MN) {
            tma_load_2d(&tmA, &full[s], st, m0, k, pol);
            tma_load_2d(&tmA, &full[s], st + 8192, m0 + 64, k, pol);
          } else {
            tma_load_2d(&tmA, &full[s], st, k, m0, pol);
          }
          tma_load_2d(&tmB, &full[s], st + 16384, k, p.n0 + n0, pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16(WG_BM, WG_BN, A_MN, false);
      int it = 0, n = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++n) {
        const int buf = n & 1, u = n >> 1;
        mbar_wait(&tempty[buf], (uint32_t)((u & 1) ^ 1));
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(buf * WG_BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % WG_STAGES, r = it / WG_STAGES;
          mbar_wait(&full[s], (uint32_t)(r & 1));
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * WG_STAGE), b = a + 16384;
#pragma unroll
          for (int kk = 0; kk < WG_BK / 16; ++kk) {
            const uint64_t ad = A_MN ? make_sdesc_sw128(a + kk * 2048, 8192, 1024) : make_sdesc_sw128(a + kk * 32, 16, 1024);
            tc_mma_bf16(dacc, ad, make_sdesc_sw128(b + kk * 32, 16, 1024), idesc, (kb | kk) ? 1u : 0u);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps: thread = output feature f (TMEM lane), 32 rows per chunk
    const int lg = warp & 3, fl = lg * 32 + lane;
    constexpr int CPW = (WG_BN / 32) / (WG_EPI_WARPS / 4);  // chunks per warp
    const int c0 = ((warp - 2) / 4) * CPW;
    int n = 0;
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++n) {
      const int m0 = (tile / p.tiles_n) * WG_BM, nb = (tile % p.tiles_n) * WG_BN;
      const int buf = n & 1, u = n >> 1;
      const int f = m0 + fl;
      const bool fok = f < p.M;
      mbar_wait(&tfull[buf], (uint32_t)(u & 1));
      tc_fence_after();
      const uint32_t taddr = tmem + (uint32_t)(buf * WG_BN) + ((uint32_t)(lg * 32) << 16);
      // 8-column groups (tcgen05.ld 32x32b.x8): 8 operand gathers in flight per thread, and a loop
      // body small enough for the instruction cache (the fully unrolled 32-column body stalled on
      // instruction fetch, ncu "no_instructions")
      float part = 0.0f;
      // shared dropout draws (needs the 4-feature groups aligned: width % 4 == 0; the ACT_BWD
      // epilogue keeps the per-element draw)
      const bool wide_drop = (MODE == EPI_LINEAR_FWD || MODE == EPI_RESID_FWD) && p.epi.drop_thresh &&
                             (p.epi.drop_width & 3) == 0;
      const uint32_t dstep = wide_drop ? *p.epi.step : 0u;
#pragma unroll 1
      for (int cg = c0 * 4; cg < (c0 + CPW) * 4; ++cg) {
        const int r0 = nb + cg * 8;
        float v[8];
        tmem_ld8(taddr + cg * 8, v);
        if (cg == (c0 + CPW) * 4 - 1) {  // this warp's part of the accumulator is in registers
          tc_fence_before();
          mbar_arrive(&tempty[buf]);
        }
        if (r0 >= p.N) continue;
        // dropout bits of rows r0..r0+7 at this thread's feature: the flat index (row * width + f)
        // of 4 consecutive features is one Philox call (width % 4 == 0), so lane (lane & ~3) + k
        // draws row r0 + 4h + k for the 4 features of its group and 4 shuffles per half hand every
        // lane its own bit -- 2 calls per thread per 8 rows instead of 8 (same decisions, O8)
        uint32_t kbits = 0xFFu;
        if (wide_drop) {
          kbits = 0u;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const uint64_t rg = (uint64_t)(p.epi.row_global0 + r0 + hh * 4 + (lane & 3));
            const uint64_t qi = (rg * (uint64_t)p.epi.drop_width + (uint64_t)(f & ~3)) >> 2;
            const uint4 o = philox4x32_10(make_uint4((uint32_t)qi, (uint32_t)(qi >> 32), p.epi.site, dstep),
                                          make_uint2((uint32_t)p.epi.seed, (uint32_t)(p.epi.seed >> 32)));
            const uint32_t wbits = ((o.x >> 8) >= p.epi.drop_thresh ? 1u : 0u) | ((o.y >> 8) >= p.epi.drop_thresh ? 2u : 0u) |
                                   ((o.z >> 8) >= p.epi.drop_thresh ? 4u : 0u) | ((o.w >> 8) >= p.epi.drop_thresh ? 8u : 0u);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t b = __shfl_sync(0xffffffffu, wbits, (lane & ~3) | k);
              kbits |= ((b >> (lane & 3)) & 1u) << (hh * 4 + k);
            }
          }
        }
        if (!fok) continue;
        EpiPre pre[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (r0 + j < p.N) {
            if (wide_drop) {
              pre[j] = epi_load<MODE, false>(p.epi, f, r0 + j);
              pre[j].keep = (kbits >> j) & 1u;
            } else {
              pre[j] = epi_load<MODE>(p.epi, f, r0 + j);
            }
          }
        if (!nkb) {
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = 0.0f;
        }
        part = epi_finish_rows<MODE, 8>(p.epi, f, r0, min(8, p.N - r0), v, pre, part);
        if (MODE == EPI_ACT_BWD && ((cg & 1) || r0 + 8 >= p.N)) {  // per-16-row column partials
          if (p.epi.colsum) p.epi.colsum[(int64_t)(r0 / 16) * p.M + f] = part;
          part = 0.0f;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

int gemm_wide(cudaStream_t st, const TcMat& A, bool a_mn, const TcMat& B, const GemmParams& gp) {
  const EpiParams& e = gp.epi;
  if (gp.M % 64 || gp.K % 64 || gp.N < 1) {
    set_error("gemm_wide: unsupported shape M=%d N=%d K=%d", gp.M, gp.N, gp.K);
    return -5;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, 64, a_mn ? 64 : 128) || !make_map(&mb, B, 64, 128)) return -3;
  WideParams p{};
  p.M = gp.M;
  p.N = gp.N;
  p.K = gp.K;
  p.n0 = gp.n0;
  p.tiles_n = (gp.N + WG_BN - 1) / WG_BN;
  p.tiles = ((gp.M + WG_BM - 1) / WG_BM) * p.tiles_n;
  p.epi = e;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = std::min(p.tiles, sms > 0 ? sms : 148);
#define WG_LAUNCH(AM, MD)                                                                                    \
  if (a_mn == AM && e.mode == MD) {                                                                          \
    static bool attr = false;                                                                                \
    if (!attr) {                                                                                             \
      cudaError_t err = cudaFuncSetAttribute(gemm_wide_kernel<AM, MD>,                                       \
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, WG_SMEM);          \
      if (err != cudaSuccess) {                                                                              \
        set_error("gemm_wide smem attribute: %s", cudaGetErrorString(err));                                  \
        return -3;                                                                                           \
      }                                                                                                      \
      attr = true;                                                                                           \
    }                                                                                                        \
    gemm_wide_kernel<AM, MD><<<grid, WG_THREADS, WG_SMEM, st>>>(ma, mb, p);                                         \
    const cudaError_t err = cudaGetLastError();                                                              \
    if (err != cudaSuccess) {                                                                                \
      set_error("gemm_wide launch: %s", cudaGetErrorString(err));                                            \
      return -3;                                                                                             \
    }                                                                                                        \
    return 0;                                                                                                \
  }
  WG_LAUNCH(false, EPI_LINEAR_FWD)
  WG_LAUNCH(false, EPI_RESID_FWD)
  WG_LAUNCH(false, EPI_STORE)
  WG_LAUNCH(true, EPI_ACT_BWD)
  WG_LAUNCH(true, EPI_STORE)
#undef WG_LAUNCH
  set_error("gemm_wide: no instantiation for a_mn=%d mode=%d", (int)a_mn, e.mode);
  return -5;
}

}  // namespace tgp
