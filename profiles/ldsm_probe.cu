// Probe (diagnostics, not product code): does ldmatrix.x4.trans + tcgen05.st.16x256b.x4 move an MN-major
// 128-byte-swizzled bf16 tile ([64 k][64 f] halves) into the K-major A-in-TMEM layout (lane = feature,
// column c = k pair (2c, 2c+1))?  Fills the tile with code(f, k), copies it with the product's address
// arithmetic, reads TMEM back with tcgen05.ld.32x32b.x32 and compares on the host.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2004_09910_b200/csrc -o ldsm_probe ldsm_probe.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "common.cuh"

using namespace tgp;

__device__ void st16x256x4(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ void ldsm4t(uint32_t a, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a)
               : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(uint32_t* out) {
  __shared__ __align__(1024) uint16_t tile[16384 / 2];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // element (k, f): half f/64, row k, chunk ((f%64)/8) ^ (k&7), position f%8; value = f * 64 + k
  for (int i = threadIdx.x; i < 64 * 128; i += 128) {
    const int k = i / 128, f = i % 128;
    const int off = (f >> 6) * 4096 + k * 64 + ((((f & 63) >> 3) ^ (k & 7)) << 3) + (f & 7);
    tile[off] = (uint16_t)(f * 64 + k);
  }
  if (warp == 0) tmem_alloc(&slot, 32);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const int q = warp;
  const uint32_t base = smem_u32(tile);
  uint32_t v[32];
  const int mi = lane >> 3, ri = lane & 7;
  const int kr = ((ri >> 1) << 2) + (ri & 1) + 2 * (mi & 1);
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) {
    const int jj = 4 * q + 2 * h2 + (mi >> 1);
    const uint32_t hb = base + (uint32_t)((jj >> 3) * 8192);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int k = 16 * cc + kr;
      ldsm4t(hb + (uint32_t)(k * 128 + (((jj & 7) ^ (k & 7)) << 4)), v + 4 * (4 * h2 + cc));
    }
  }
  const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
#pragma unroll
  for (int h2 = 0; h2 < 2; ++h2) st16x256x4(trow + ((uint32_t)(16 * h2) << 16), v + 16 * h2);
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  float w[32];
  tmem_ld16(trow, w);
  tmem_ld16(trow + 16, w + 16);
  for (int c = 0; c < 32; ++c) out[(32 * q + lane) * 32 + c] = __float_as_uint(w[c]);
  // also the raw register fragments of warp 0 (first chunk) for diagnosis
  if (q == 0)
    for (int i = 0; i < 4; ++i) out[128 * 32 + lane * 4 + i] = v[i];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 32);
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, (128 * 32 + 128) * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<uint32_t> h(128 * 32 + 128);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int f = 0; f < 128; ++f)
    for (int c = 0; c < 32; ++c) {
      const uint32_t want = (uint32_t)(f * 64 + 2 * c) | ((uint32_t)(f * 64 + 2 * c + 1) << 16);
      const uint32_t got = h[f * 32 + c];
      if (got != want) {
        if (bad < 12)
          printf("lane %3d col %2d: got f=%d k=%d | f=%d k=%d, want f=%d k=%d,%d\n", f, c, (got & 0xffff) / 64,
                 (got & 0xffff) % 64, (got >> 16) / 64, (got >> 16) % 64, f, 2 * c, 2 * c + 1);
        ++bad;
      }
    }
  printf("mismatches: %d of %d\n", bad, 128 * 32);
  for (int t = 0; t < 8; ++t) {
    printf("warp0 thread %d regs:", t);
    for (int i = 0; i < 4; ++i) {
      const uint32_t g = h[128 * 32 + t * 4 + i];
      printf(" (f%d k%d|f%d k%d)", (g & 0xffff) / 64, (g & 0xffff) % 64, (g >> 16) / 64, (g >> 16) % 64);
    }
    printf("\n");
  }
  return bad != 0;
}
