// Read-bandwidth probe (diagnostics, not product code): N CTAs stream a 1 GiB buffer into a
// shared-memory ring with 1-D bulk copies (cp.async.bulk) and discard it -- the ceiling a
// weight-streaming kernel with this many SMs / this ring depth / chunk size / access pattern can
// reach.  Also a 2-D TMA variant reading 128 x 128 B boxes of a row-major [rows][4096] bf16 matrix
// (the layout of the stream kernel's K-major weight tiles).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(ph)
                 : "memory");
}

// mode 0: CTA c reads a contiguous range; mode 1: chunk q of CTA c is chunk c + q*N (interleaved);
// mode 2: 2-D TMA boxes {64 cols, 128 rows} of a row-major [rows][4096] bf16 matrix, CTA c owns a
// 128-row slab x K-quarter like the stream kernel (grid must be 4 * rows / 128).
__global__ void probe(const char* buf, size_t total, int chunk, int nst, int mode, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* ring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nst * chunk);
  uint64_t* empty = full + nst;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t N = gridDim.x, c = blockIdx.x;
  const size_t nch = total / chunk / N;
  if (threadIdx.x == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (size_t q = 0; q < nch; ++q) {
      const int s = q % nst;
      const uint32_t r = q / nst;
      mb_wait(&empty[s], (r & 1) ^ 1);
      mb_expect(&full[s], chunk);
      if (mode == 2) {
        // slab = c / 4, quarter = c % 4; 16 k-blocks per quarter of 4096 columns; rows of 8 KB
        const int slab = c / 4, quarter = c % 4;
        const int kb = (int)(q % 16), rep = (int)(q / 16);
        const int row0 = (slab * 128 + rep * (int)(N / 4) * 128) % 32768;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(su32(ring + (size_t)s * chunk)),
            "l"(&tm), "r"(su32(&full[s])), "r"((quarter * 16 + kb) * 64), "r"(row0), "l"(pol)
            : "memory");
      } else {
        const size_t idx = mode == 0 ? c * nch + q : q * N + c;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                su32(ring + (size_t)s * chunk)),
            "l"(buf + idx * chunk), "r"(chunk), "r"(su32(&full[s])), "l"(pol)
            : "memory");
      }
    }
  } else if (threadIdx.x == 32) {
    for (size_t q = 0; q < nch; ++q) {
      const int s = q % nst;
      const uint32_t r = q / nst;
      mb_wait(&full[s], r & 1);
      mb_arrive(&empty[s]);
    }
  }
}

int main() {
  const size_t total = (size_t)1 << 30;
  char* buf;
  cudaMalloc(&buf, total + (1 << 20));
  cudaMemset(buf, 1, total);
  CUtensorMap tm;
  {
    cuuint64_t dims[2] = {4096, 32768};  // bf16 [32768][4096] = 256 MiB view
    cuuint64_t strides[1] = {8192};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("tensor map failed %d\n", (int)r);
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg {
    int grid, chunk, nst, mode, cluster;
  } cfgs[] = {{128, 16384, 10, 2, 4}, {128, 16384, 11, 2, 4}, {128, 16384, 10, 0, 4}, {128, 16384, 10, 1, 4},
              {148, 16384, 10, 1, 4}, {128, 32768, 6, 1, 4}, {128, 32768, 6, 1, 2},{128, 16384, 10, 0}, {148, 16384, 10, 0}, {128, 16384, 10, 1}, {148, 16384, 10, 1},
              {296, 16384, 5, 1},  {128, 32768, 6, 1},  {148, 32768, 6, 1},  {128, 8192, 20, 1},
              {128, 16384, 4, 1},  {128, 16384, 13, 1}, {148, 16384, 13, 1}, {128, 16384, 10, 2},
              {128, 16384, 13, 2}, {256, 16384, 6, 2}, {128, 16384, 10, 2, 2}};
  for (const Cfg& k : cfgs) {
    const size_t smem = (size_t)k.chunk * k.nst + 1024 + 512;
    float best = 1e9;
    const size_t bytes = (k.mode == 2) ? (total / 4) : total;  // mode 2 reads a 256 MiB matrix view
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(a);
      if (k.cluster > 1) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(k.grid);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = k.cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, probe, (const char*)buf, bytes, k.chunk, k.nst, k.mode, tm);
      } else {
        probe<<<k.grid, 64, smem>>>(buf, bytes, k.chunk, k.nst, k.mode, tm);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("grid %3d cluster %d chunk %5d stages %2d mode %d: %.1f GB/s %s\n", k.grid, k.cluster, k.chunk, k.nst, k.mode,
           bytes / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
