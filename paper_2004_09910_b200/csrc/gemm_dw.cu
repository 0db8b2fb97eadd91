// Persistent deferred weight-gradient GEMM (task W_j, g^j = sum_i g_i^j; reading Z12):
//
//   dW[m][n] (=|+=) sum_k A[k][m] * B[k][n]      A = dY^T-operand [K rows][M], B = X [K rows][N] (bf16)
//
// K = the mini-batch rows (512 at C2), M = N = 4096.  One CTA per SM loops over 128 x 128 output
// tiles (static round-robin: 1024 tiles on 148 SMs, <= 7 each), TMA -> 5-stage shared-memory ring ->
// (128 x 256 tiles, TGP_DW_BN=256, measured 1 % faster on C5 but hit intermittent illegal-address
// faults with two partitions on one device, profiles/r7/r8d_summary.txt -- not used)
// tcgen05.mma (both operands MN-major SW128, fp32 in TMEM) with TMEM double-buffered across tiles,
// so tile t+1's loads and MMAs overlap tile t's epilogue.  Epilogue: TMEM -> 128-byte-swizzled
// shared-memory chunk -> TMA tensor store (first backward after a step) or TMA reduce-add
// (accumulation, the read-modify-write happens in L2).  Each output element is produced by one CTA
// with a fixed k order: deterministic.
#include "common.cuh"
#include "host.h"
#include "kernels.h"

#include <algorithm>

namespace tgp {

namespace {
#ifndef TGP_DW_BN
#define TGP_DW_BN 128
#endif
constexpr int DW_BM = 128, DW_BN = TGP_DW_BN, DW_BK = 64;
constexpr int DW_STAGE = (DW_BM + DW_BN) * DW_BK * 2;  // 32 KB
constexpr int DW_STAGES = DW_BN == 256 ? 4 : 5;
constexpr int DW_CHUNK = 128 * 32 * 4;                 // 16 KB epilogue chunk (128 rows x 32 fp32)
constexpr int DW_OFF_C = DW_STAGES * DW_STAGE;
constexpr int DW_OFF_BAR = DW_OFF_C + 2 * DW_CHUNK;
constexpr int DW_SMEM = DW_OFF_BAR + 256 + 1024;
}  // namespace

struct DwParams {
  int M, N, K;
  int tiles_n, tiles;
  int accumulate;
};

TGP_DEV void dw_store(const void* desc, const void* smem, int32_t c0, int32_t c1, bool add) {
  if (add)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(desc),
                 "r"(c0), "r"(c1), "r"(smem_u32(smem))
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(desc), "r"(c0),
                 "r"(c1), "r"(smem_u32(smem))
                 : "memory");
}

__global__ void __launch_bounds__(192, 1)
    gemm_dw_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmD, const DwParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + DW_OFF_BAR);
  uint64_t* empty = full + DW_STAGES;
  uint64_t* tfull = empty + DW_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2] (128 epilogue arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = p.K / DW_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmD);
    for (int s = 0; s < DW_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 2 * DW_BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------- TMA producer
      const uint64_t pol = policy_evict_last();  // operands (8 MB) are re-read by every tile row / column
      int it = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
        const int m0 = (tile / p.tiles_n) * DW_BM, n0 = (tile % p.tiles_n) * DW_BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % DW_STAGES, r = it / DW_STAGES;
          mbar_wait(&empty[s], (uint32_t)((r & 1) ^ 1));
          uint8_t* st = smem + s * DW_STAGE;
          mbar_arrive_expect_tx(&full[s], DW_STAGE);
          const int k = kb * DW_BK;
          tma_load_2d(&tmA, &full[s], st, m0, k, pol);
          tma_load_2d(&tmA, &full[s], st + 8192, m0 + 64, k, pol);
#pragma unroll
          for (int c = 0; c < DW_BN / 64; ++c) tma_load_2d(&tmB, &full[s], st + 16384 + c * 8192, n0 + c * 64, k, pol);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16(DW_BM, DW_BN, true, true);
      int it = 0, n = 0;
      for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++n) {
        const int buf = n & 1, u = n >> 1;
        mbar_wait(&tempty[buf], (uint32_t)((u & 1) ^ 1));
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(buf * DW_BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % DW_STAGES, r = it / DW_STAGES;
          mbar_wait(&full[s], (uint32_t)(r & 1));
          tc_fence_after();
          const uint32_t a = smem_u32(smem + s * DW_STAGE), b = a + 16384;
#pragma unroll
          for (int kk = 0; kk < DW_BK / 16; ++kk)
            tc_mma_bf16(dacc, make_sdesc_sw128(a + kk * 2048, 8192, 1024), make_sdesc_sw128(b + kk * 2048, 8192, 1024),
                        idesc, (kb | kk) ? 1u : 0u);
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue warps 2..5: TMEM lanes 32*(warp&3).. = output rows of the tile
    const int lg = warp & 3, fl = lg * 32 + lane;
    const bool leader = threadIdx.x == 64;
    const bool add = p.accumulate != 0;
    int n = 0, chunk = 0;
    for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x, ++n) {
      const int m0 = (tile / p.tiles_n) * DW_BM, n0 = (tile % p.tiles_n) * DW_BN;
      const int buf = n & 1, u = n >> 1;
      mbar_wait(&tfull[buf], (uint32_t)(u & 1));
      tc_fence_after();
      const uint32_t taddr = tmem + (uint32_t)(buf * DW_BN) + ((uint32_t)(lg * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < DW_BN / 32; ++c, ++chunk) {
        uint8_t* cb = smem + DW_OFF_C + (chunk & 1) * DW_CHUNK;
        if (chunk >= 2) {
          if (leader) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        float v[32];
        tmem_ld16(taddr + c * 32, v);
        tmem_ld16(taddr + c * 32 + 16, v + 16);
        if (c == DW_BN / 32 - 1) {  // all of this tile's TMEM read: the MMA may reuse the buffer
          tc_fence_before();
          mbar_arrive(&tempty[buf]);
        }
        uint8_t* row = cb + fl * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(row + ((q ^ (fl & 7)) << 4)) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (leader) {
          dw_store(&tmD, cb, n0 + c * 32, m0, add);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    }
    if (leader) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 2 * DW_BN);
}

// A: [K][M] bf16 (row stride lda elements), B: [K][N] bf16 (ldb), D: [M][N] fp32 (ldd).
int gemm_dw(cudaStream_t st, const void* A, int64_t lda, const void* B, int64_t ldb, float* D, int64_t ldd, int M,
            int N, int K, bool accumulate) {
  if (M % 64 || N % 64 || K <= 0) {
    // M, N % 64 (GPT-2's d = 1600): the last tile row / column is half empty -- TMA zero-fills the
    // operand loads past M / N and clips the output stores
    set_error("gemm_dw: unsupported shape M=%d N=%d K=%d (need M, N %% 64)", M, N, K);
    return -5;
  }
  const int Kp = (K + DW_BK - 1) / DW_BK * DW_BK;  // rows past K read as zeros (TMA bounds)
  const Driver* drv = driver();
  if (!drv) return -3;
  CUtensorMap ma, mb, md;
  if (!make_map(&ma, TcMat{A, K, M, lda}, 64, 64) || !make_map(&mb, TcMat{B, K, N, ldb}, 64, 64)) return -3;
  {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)ldd * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = drv->tensorMapEncodeTiled(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("gemm_dw output tensor map failed (%d)", (int)r);
      return -3;
    }
  }
  static int sms = 0;
  static bool attr = false;
  if (!attr) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(gemm_dw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DW_SMEM);
    if (e != cudaSuccess) {
      set_error("gemm_dw smem attribute: %s", cudaGetErrorString(e));
      return -3;
    }
    attr = true;
  }
  const int tn = (N + DW_BN - 1) / DW_BN, tm = (M + DW_BM - 1) / DW_BM;
  DwParams p{M, N, Kp, tn, tm * tn, accumulate ? 1 : 0};
  const int grid = std::min(p.tiles, sms > 0 ? sms : 148);
  gemm_dw_kernel<<<grid, 192, DW_SMEM, st>>>(ma, mb, md, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("gemm_dw launch: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

}  // namespace tgp
