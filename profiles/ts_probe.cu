// Probe (diagnostics, not product code): does tcgen05.cp (smem -> TMEM, 128x256b) from a K-major
// 128-byte-swizzled bf16 tile produce the A-operand layout tcgen05.mma ... [a_tmem] expects?
// D_ss = A(smem) x B(smem)^T and D_ts = A(tmem, copied) x B(smem)^T for a 128 x 64 A tile and a
// 16 x 64 B tile; both compared with a host reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2004_09910_b200/csrc -o ts_probe ts_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace tgp;

__device__ void cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                                                float* dss, float* dts, int mode) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a = sm;
  uint8_t* b = sm + 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 2048);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    mbar_init(&bar[3], 1);
    for (int q = 4; q < 8; ++q) mbar_init(&bar[q], 1000);
    for (int q = 8; q < 16; ++q) mbar_init(&bar[q], 1);
    fence_barrier_init();
  }
  if (threadIdx.x == 0) slot[2] = 1;
  if (warp == 0) tmem_alloc(slot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;  // cols [0,16) D_ss, [16,32) D_ts, [64, 96) A copy
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar[0], 16384 + 2048);
    tma_load_2d(&tA, &bar[0], a, 0, 0, policy_evict_first());
    tma_load_2d(&tB, &bar[0], b, 0, 0, policy_evict_first());
    mbar_wait(&bar[0], 0);
    tc_fence_after();
    const uint32_t idesc = make_idesc_bf16(128, 16, false, false);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    for (int kk = 0; kk < 4; ++kk)
      tc_mma_bf16(tmem, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, kk);
    // copy A into TMEM columns 64.. : each K=16 slice (256 bits per row) -> 8 columns
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t sd = (mode == 0) ? make_sdesc_sw128(sa + kk * 32, 16, 1024) : make_sdesc_sw128(sa + kk * 32, 16, 1024);
      cp_128x256b(tmem + 64 + kk * 8, sd);
    }
    for (int kk = 0; kk < 4; ++kk)
      mma_ts(tmem + 16, tmem + 64 + kk * 8, make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, kk);
    tc_commit(&bar[1]);
    mbar_wait(&bar[1], 0);
    // timing: 64 back-to-back MMAs (N=16, K=16) SS and TS, each completion-waited
    for (int rep = 0; rep < 2; ++rep) {
      long long t0 = clock64();
      for (int i = 0; i < 64; ++i) {
        const int kk = i & 3;
        if (rep == 0)
          tc_mma_bf16(tmem + 32, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
        else
          mma_ts(tmem + 32, tmem + 64 + kk * 8, make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
      }
      tc_commit(&bar[2 + rep]);
      mbar_wait(&bar[2 + rep], 0);
      long long t1 = clock64();
      dss[16 * 128 + rep] = (float)(t1 - t0);
    }
    // 64 SS MMAs round-robin over 4 independent accumulators (cols 32, 48, 96+32.. ) ; and N=32 / N=64 chains
    {
      long long t0 = clock64();
      for (int i = 0; i < 64; ++i) {
        const int kk = i & 3;
        tc_mma_bf16(tmem + 32 + (uint32_t)((i & 3) * 16), make_sdesc_sw128(sa + kk * 32, 16, 1024),
                    make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
      }
      tc_commit(&bar[2]);
      mbar_wait(&bar[2], 1);
      long long t1 = clock64();
      dss[16 * 128 + 3] = (float)(t1 - t0);
    }
    for (int variant = 0; variant < 2; ++variant) {
      const int every = variant ? 16 : 4;
      long long t0 = clock64();
      for (int i = 0; i < 64; ++i) {
        const int kk = i & 3;
        tc_mma_bf16(tmem + 32, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
        if ((i + 1) % every == 0) tc_commit(&bar[4 + ((i / every) & 3)]);
      }
      tc_commit(&bar[8 + variant]);
      mbar_wait(&bar[8 + variant], 0);
      long long t1 = clock64();
      dss[16 * 128 + 5 + variant] = (float)(t1 - t0);
    }
    {
      const uint32_t idesc64 = make_idesc_bf16(128, 64, false, false);
      long long t0 = clock64();
      for (int i = 0; i < 64; ++i) {
        const int kk = i & 3;
        tc_mma_bf16(tmem + 32, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc64, 1);
      }
      tc_commit(&bar[3]);
      mbar_wait(&bar[3], 1);
      long long t1 = clock64();
      dss[16 * 128 + 4] = (float)(t1 - t0);
    }
    // 16 x 4 cp of 128x256b
    {
      long long t0 = clock64();
      for (int i = 0; i < 16; ++i)
        for (int kk = 0; kk < 4; ++kk) cp_128x256b(tmem + 96 + kk * 8, make_sdesc_sw128(sa + kk * 32, 16, 1024));
      tc_commit(&bar[0]);
      mbar_wait(&bar[0], 1);
      long long t1 = clock64();
      dss[16 * 128 + 2] = (float)(t1 - t0);
    }
  }
  __syncwarp();
  __syncthreads();
  // two issuing warps, 32 MMAs each into different accumulators, concurrently
  {
    const uint32_t idesc = make_idesc_bf16(128, 16, false, false);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    if ((threadIdx.x == 0 || threadIdx.x == 32)) {
      const int w = threadIdx.x >> 5;
      long long t0 = clock64();
      for (int i = 0; i < 32; ++i) {
        const int kk = i & 3;
        tc_mma_bf16(tmem + 32 + w * 16, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024),
                    idesc, 1);
      }
      tc_commit(&bar[8 + w]);
      mbar_wait(&bar[8 + w], 1);
      long long t1 = clock64();
      dss[16 * 128 + 7 + w] = (float)(t1 - t0);
    }
  }
  __syncthreads();
  // "tile loop" as in the stream kernel: per tile test_wait(complete barrier) + fence + 4 MMAs + commit
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(128, 16, false, false);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    for (int variant = 0; variant < 6; ++variant) {
      long long t0 = clock64();
      if (variant >= 4) {  // batched: per group of 4 tiles, the waits first, then 16 MMAs, then 4 commits
        for (int gi = 0; gi < 4; ++gi) {
          for (int q = 0; q < (variant == 4 ? 4 : 1); ++q)
            while (!mbar_test_wait(smem_u32(&bar[1]), 0)) {
            }
          tc_fence_after();
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc_mma_bf16(tmem + 32, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
          for (int q = 0; q < 4; ++q) tc_commit(&bar[4 + q]);
        }
      }
      for (int i = 0; i < (variant >= 4 ? 0 : 16); ++i) {
        if (variant == 1) {
          while (!mbar_test_wait(smem_u32(&bar[1]), 0)) {
          }
        }
        if (variant >= 2) {  // smem flag read (ld.acquire.cta) instead of an mbarrier probe
          uint32_t v;
          do {
            asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(slot + 2)) : "memory");
          } while (v == 0);
        }
        if (variant >= 2) tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_bf16(tmem + 32, make_sdesc_sw128(sa + kk * 32, 16, 1024), make_sdesc_sw128(sb + kk * 32, 16, 1024), idesc, 1);
        if (variant >= 3) tc_commit(&bar[4 + (i & 3)]);
      }
      tc_commit(&bar[10 + variant]);
      mbar_wait(&bar[10 + variant], 0);
      long long t1 = clock64();
      dss[16 * 128 + 9 + variant] = (float)(t1 - t0);
    }
  }
  __syncthreads();
  mbar_wait(&bar[1], 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 16; ++n) dss[n * 128 + warp * 32 + lane] = v[n];
  tmem_ld16(tmem + 16 + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 16; ++n) dts[n * 128 + warp * 32 + lane] = v[n];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
}

static void mk(CUtensorMap* m, void* p, int rows, int cols, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("map failed %d\n", (int)r);
}

int main() {
  std::vector<__nv_bfloat16> A(128 * 64), B(16 * 64);
  std::vector<float> Af(128 * 64), Bf(16 * 64);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xFFFF) / 32768.0f - 1.0f; };
  for (int i = 0; i < 128 * 64; ++i) { A[i] = __float2bfloat16(rnd()); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < 16 * 64; ++i) { B[i] = __float2bfloat16(rnd()); Bf[i] = __bfloat162float(B[i]); }
  void *dA, *dB;
  float *dss, *dts;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dss, 16 * 128 * 4 + 128);
  cudaMalloc(&dts, 16 * 128 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  mk(&tA, dA, 128, 64, 128);
  mk(&tB, dB, 16, 64, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<<<1, 128, 64 * 1024>>>(tA, tB, dss, dts, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> hss(16 * 128), hts(16 * 128);
  cudaMemcpy(hss.data(), dss, hss.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hts.data(), dts, hts.size() * 4, cudaMemcpyDeviceToHost);
  double ess = 0, ets = 0, mx = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 16; ++n) {
      double r = 0;
      for (int k = 0; k < 64; ++k) r += (double)Af[m * 64 + k] * Bf[n * 64 + k];
      ess = fmax(ess, fabs(hss[n * 128 + m] - r));
      ets = fmax(ets, fabs(hts[n * 128 + m] - r));
      mx = fmax(mx, fabs(r));
    }
  printf("max |ref| %.4f  max err SS %.3e  TS %.3e  (SS==TS bitwise: %d)\n", mx, ess, ets,
         (int)(memcmp(hss.data(), hts.data(), hss.size() * 4) == 0));
  float tm[15];
  cudaMemcpy(tm, dss + 16 * 128, 60, cudaMemcpyDeviceToHost);
  printf("batched per 4 tiles: 4 waits %.0f, 1 wait %.0f clk\n", tm[13], tm[14]);
  printf("16 tiles x 4 MMAs: plain %.0f, +mbar test_wait %.0f, smem flag + fence %.0f, + commit %.0f clk\n", tm[9], tm[10], tm[11], tm[12]);
  printf("2 warps x 32 MMAs concurrently: %.0f / %.0f clk\n", tm[7], tm[8]);
  printf("64 SS MMAs with a commit after every 4: %.0f clk; with a commit after every 16: %.0f clk\n", tm[5], tm[6]);
  printf("64 SS MMAs over 4 accumulators: %.0f clk; 64 SS MMAs N=64 (B rows beyond 16 = garbage smem): %.0f clk\n", tm[3], tm[4]);
  printf("64 MMAs SS: %.0f clk (%.1f clk/MMA), TS: %.0f clk (%.1f clk/MMA); 64 cp 128x256b: %.0f clk\n", tm[0], tm[0] / 64,
         tm[1], tm[1] / 64, tm[2]);
  return 0;
}
