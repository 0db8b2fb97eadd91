// Deferred weight-gradient task W_j fused with the plain SGD update ("SGD fused into
// the W_j epilogue"):
//
//   g[m][n]  = sum_k A[k][m] B[k][n]            (g^j = sum_i g_i^j; reading Z12)
//   W[m][n] -= lr g[m][n],  shadow[m][n] = bf16(W[m][n])   (plain SGD; fp32 master, Z14)
//
// for every GEMM of a partition's W_j task in ONE persistent launch (all weight matrices of the
// partition: 64 GEMMs of 4096 x 4096 x 512 at C2 n = 1).  The gradient never goes to HBM: unfused,
// W_j writes g (4 B/param) and SGD reads it back with the master (18 B/param in all); fused, only the
// master read-modify-write and the bf16 shadow write remain (10 B/param), so the task is bound by
// that traffic, with the tensor work (AI 228) hidden under it.
//
// One CTA per SM loops over 128 x 128 output tiles of all GEMMs in order (GEMM-major, n fastest: the
// 8 MB of operands of the GEMM in flight stay in L2).  Warp roles:
//   warp 0  TMA producer of the bf16 operands (MN-major SW128, 3-stage ring of 64-row k-blocks)
//   warp 1  TMEM allocator + single-thread tcgen05.mma issuer, accumulator double-buffered in TMEM
//   warp 6  TMA producer of the fp32 master chunks (128 rows x 32 columns, 5-deep ring), running
//           ahead of the epilogue by up to 4 chunks
//   warps 2-5  epilogue: thread = tile row (TMEM lane); per 32-column chunk: tcgen05.ld the gradient,
//           W = fma(-lr, g, W) in the shared master chunk, bf16 into a 64-column shadow chunk, TMA
//           stores of both.
// Each output element is produced by one CTA with a fixed k order and the same fma as sgd_kernel, so
// the result is bitwise identical to gemm_dw + sgd_step (tested).
#include "common.cuh"
#include "host.h"
#include "kernels.h"

#include <algorithm>

namespace tgp {

namespace {
constexpr int WS_BM = 128, WS_BN = 128, WS_BK = 64;
constexpr int WS_STAGE = (WS_BM + WS_BN) * WS_BK * 2;  // 32 KB of operands per k-block
#ifndef TGP_WS_STAGES
#define TGP_WS_STAGES 3
#endif
#ifndef TGP_WS_NM
#define TGP_WS_NM 5
#endif
constexpr int WS_STAGES = TGP_WS_STAGES;
constexpr int WS_MCHUNK = 128 * 32 * 4;                // 16 KB master chunk (128 rows x 32 fp32)
constexpr int WS_NM = TGP_WS_NM;                       // master chunk ring
constexpr int WS_SCHUNK = 128 * 64 * 2;                // 16 KB shadow chunk (128 rows x 64 bf16)
constexpr int WS_OFF_M = WS_STAGES * WS_STAGE;
constexpr int WS_OFF_S = WS_OFF_M + WS_NM * WS_MCHUNK;
constexpr int WS_OFF_BAR = WS_OFF_S + 2 * WS_SCHUNK;
constexpr int WS_SMEM = WS_OFF_BAR + 512 + 1024;
constexpr int WS_THREADS = 224;
}  // namespace

struct WsParams {
  const WsGemm* g;  // [ngemm] device descriptors
  int ngemm, tiles;
  const float* lr;  // device scalar (a graph replay reads the current value)
};

TGP_DEV void tma_store_2d(const void* desc, const void* smem, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(desc),
               "r"(c0), "r"(c1), "r"(smem_u32(smem))
               : "memory");
}

// GEMM of global tile `tile` (tiles are numbered GEMM after GEMM; `g` is the caller's cursor)
TGP_DEV const WsGemm& ws_find(const WsParams& p, int tile, int& g) {
  while (g + 1 < p.ngemm && tile >= p.g[g + 1].tile0) ++g;
  return p.g[g];
}

__global__ void __launch_bounds__(WS_THREADS, 1) wgrad_sgd_kernel(const __grid_constant__ WsParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + WS_OFF_BAR);
  uint64_t* empty = full + WS_STAGES;
  uint64_t* mfull = empty + WS_STAGES;  // [WS_NM] master chunk landed
  uint64_t* mempty = mfull + WS_NM;     // [WS_NM] master chunk stored back (its buffer is free)
  uint64_t* tfull = mempty + WS_NM;     // [2]
  uint64_t* tempty = tfull + 2;         // [2] (128 epilogue arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < WS_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < WS_NM; ++s) {
      mbar_init(&mfull[s], 1);
      mbar_init(&mempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * WS_BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------- operand producer
      const uint64_t pol = policy_evict_last();  // a GEMM's operands are re-read by all its tiles
      int it = 0, g = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const WsGemm& G = ws_find(p, tile, g);
        const int lt = tile - G.tile0;
        const int m0 = (lt / G.tiles_n) * WS_BM, n0 = (lt % G.tiles_n) * WS_BN;
        const int nkb = (G.K + WS_BK - 1) / WS_BK;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % WS_STAGES, r = it / WS_STAGES;
          mbar_wait(&empty[s], (uint32_t)((r & 1) ^ 1));
          uint8_t* st = smem + s * WS_STAGE;
          mbar_arrive_expect_tx(&full[s], WS_STAGE);
          const int k = kb * WS_BK;
          tma_load_2d(&G.a, &full[s], st, m0, k, pol);
          tma_load_2d(&G.a, &full[s], st + 8192, m0 + 64, k, pol);
          tma_load_2d(&G.b, &full[s], st + 16384, n0, k, pol);
          tma_load_2d(&G.b, &full[s], st + 24576, n0 + 64, k, pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16(WS_BM, WS_BN, true, true);
      int it = 0, n = 0, g = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++n) {
        const WsGemm& G = ws_find(p, tile, g);
        const int nkb = (G.K + WS_BK - 1) / WS_BK;
        const int buf = n & 1, u = n >> 1;
        mbar_wait(&tempty[buf], (uint32_t)((u & 1) ^ 1));
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(buf * WS_BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % WS_STAGES, r = it / WS_STAGES;
          mbar_wait(&full[s], (uint32_t)(r & 1));
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * WS_STAGE), b = a + 16384;
#pragma unroll
          for (int kk = 0; kk < WS_BK / 16; ++kk)
            tc_mma_bf16(dacc, make_sdesc_sw128(a + kk * 2048, 8192, 1024), make_sdesc_sw128(b + kk * 2048, 8192, 1024),
                        idesc, (kb | kk) ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else if (warp == 6) {
    if (elect_one()) {
      // ---------------- master chunk producer (fp32, streamed once)
      const uint64_t pol = policy_evict_first();
      int ck = 0, g = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const WsGemm& G = ws_find(p, tile, g);
        const int lt = tile - G.tile0;
        const int m0 = (lt / G.tiles_n) * WS_BM, n0 = (lt % G.tiles_n) * WS_BN;
        for (int c = 0; c < WS_BN / 32; ++c, ++ck) {
          const int b = ck % WS_NM, r = ck / WS_NM;
          mbar_wait(&mempty[b], (uint32_t)((r & 1) ^ 1));
          mbar_arrive_expect_tx(&mfull[b], WS_MCHUNK);
          tma_load_2d(&G.w, &mfull[b], smem + WS_OFF_M + b * WS_MCHUNK, n0 + 32 * c, m0, pol);
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5: TMEM lanes 32*(warp&3).. = rows of the tile
    const int lg = warp & 3, fl = lg * 32 + lane;
    const bool leader = threadIdx.x == 64;
    const float lr = *p.lr;
    int n = 0, ck = 0, g = 0;
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++n) {
      const WsGemm& G = ws_find(p, tile, g);
      const int lt = tile - G.tile0;
      const int m0 = (lt / G.tiles_n) * WS_BM, n0 = (lt % G.tiles_n) * WS_BN;
      const int buf = n & 1, u = n >> 1;
      mbar_wait(&tfull[buf], (uint32_t)(u & 1));
      tc_fence_after();
      const uint32_t taddr = tmem + (uint32_t)(buf * WS_BN) + ((uint32_t)(lg * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < WS_BN / 32; ++c, ++ck) {
        const int b = ck % WS_NM;
        uint8_t* sb = smem + WS_OFF_S + ((ck >> 1) & 1) * WS_SCHUNK;
        if (ck >= 2) {
          // the stores of chunk ck - 2 have read their shared buffers: its master buffer goes back to
          // the producer; the barrier also frees the shadow buffer used two chunk pairs ago
          if (leader) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            mbar_arrive(&mempty[(ck - 2) % WS_NM]);
          }
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        float v[32];
        tmem_ld16(taddr + c * 32, v);
        tmem_ld16(taddr + c * 32 + 16, v + 16);
        if (c == WS_BN / 32 - 1) {  // the tile's accumulator is read: the MMA may reuse it
          tc_fence_before();
          mbar_arrive(&tempty[buf]);
        }
        mbar_wait(&mfull[b], (uint32_t)((ck / WS_NM) & 1));
        uint8_t* mrow = smem + WS_OFF_M + b * WS_MCHUNK + fl * 128;
        uint8_t* srow = sb + fl * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4* wp = reinterpret_cast<float4*>(mrow + ((q ^ (fl & 7)) << 4));
          float4 w = *wp;
          w.x = __fmaf_rn(-lr, v[4 * q], w.x);
          w.y = __fmaf_rn(-lr, v[4 * q + 1], w.y);
          w.z = __fmaf_rn(-lr, v[4 * q + 2], w.z);
          w.w = __fmaf_rn(-lr, v[4 * q + 3], w.w);
          *wp = w;
          v[4 * q] = w.x;
          v[4 * q + 1] = w.y;
          v[4 * q + 2] = w.z;
          v[4 * q + 3] = w.w;
        }
        // shadow: 32 bf16 = 4 chunks of 16 B at chunk positions 4 (c & 1) + j of the 64-column row
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          __nv_bfloat162 h[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) h[e] = __floats2bfloat162_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
          const int qs = 4 * (c & 1) + j;
          *reinterpret_cast<uint4*>(srow + ((qs ^ (fl & 7)) << 4)) = *reinterpret_cast<const uint4*>(h);
        }
        fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (leader) {
          tma_store_2d(&G.w, smem + WS_OFF_M + b * WS_MCHUNK, n0 + 32 * c, m0);
          if (c & 1) tma_store_2d(&G.sh, sb, n0 + 64 * (c >> 1), m0);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * WS_BN);
}

bool wgrad_sgd_desc(WsGemm* d, const void* A, int64_t lda, const void* B, int64_t ldb, float* W, __nv_bfloat16* shadow,
                    int64_t ldw, int M, int N, int K) {
  if (M % WS_BM || N % WS_BN || K <= 0 || ldw % 8) {
    set_error("wgrad_sgd: unsupported shape M=%d N=%d K=%d ldw=%lld (need M, N %% 128)", M, N, K, (long long)ldw);
    return false;
  }
  const Driver* drv = driver();
  if (!drv) return false;
  if (!make_map(&d->a, TcMat{A, K, M, lda}, 64, 64) || !make_map(&d->b, TcMat{B, K, N, ldb}, 64, 64)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
  cuuint32_t es[2] = {1, 1};
  {
    cuuint64_t strides[1] = {(cuuint64_t)ldw * 4};
    cuuint32_t box[2] = {32, 128};
    CUresult r = drv->tensorMapEncodeTiled(&d->w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, W, dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("wgrad_sgd master tensor map failed (%d)", (int)r);
      return false;
    }
  }
  {
    cuuint64_t strides[1] = {(cuuint64_t)ldw * 2};
    cuuint32_t box[2] = {64, 128};
    CUresult r = drv->tensorMapEncodeTiled(&d->sh, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, shadow, dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("wgrad_sgd shadow tensor map failed (%d)", (int)r);
      return false;
    }
  }
  d->M = M;
  d->N = N;
  d->K = K;
  d->tiles_n = N / WS_BN;
  d->tiles = (M / WS_BM) * d->tiles_n;
  return true;
}

int wgrad_sgd(cudaStream_t st, const WsGemm* dev_descs, const WsGemm* host_descs, int ngemm, const float* lr) {
  if (ngemm <= 0) return 0;
  const int tiles = host_descs[ngemm - 1].tile0 + host_descs[ngemm - 1].tiles;
  static int sms = 0;
  static bool attr = false;
  if (!attr) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(wgrad_sgd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, WS_SMEM);
    if (e != cudaSuccess) {
      set_error("wgrad_sgd smem attribute: %s", cudaGetErrorString(e));
      return -3;
    }
    attr = true;
  }
  WsParams p{dev_descs, ngemm, tiles, lr};
  const int grid = std::min(tiles, sms > 0 ? sms : 148);
  wgrad_sgd_kernel<<<grid, WS_THREADS, WS_SMEM, st>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("wgrad_sgd launch: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

}  // namespace tgp
