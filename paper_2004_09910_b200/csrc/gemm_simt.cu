// fp32 SIMT GEMM (FFMA, no TF32; reading Z16) for the fp32 parity mode, with the same
// D[m][n] = sum_k A[m][k] B[n][k] semantics and epilogues as the tcgen05 kernel.  Each thread owns
// one output feature m and walks the rows n in chunks of 16, so the EPI_ACT_BWD column sum is a
// per-thread sum (deterministic, sequential k order).
#include "epilogue.cuh"
#include "host.h"
#include "kernels.h"

namespace tgp {

__global__ void __launch_bounds__(128) gemm_simt_kernel(SimtOperand A, SimtOperand B0, SimtOperand B1, GemmParams p) {
  griddep_wait();
  griddep_launch();
  __shared__ float Bs[16][65];
  const int m = blockIdx.x * 128 + threadIdx.x;
  float csum = 0.0f;
  for (int n0 = 0; n0 < p.N; n0 += 16) {
    float acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0.0f;
    for (int k0 = 0; k0 < p.K; k0 += 64) {
      for (int e = threadIdx.x; e < 16 * 64; e += 128) {
        const int j = e / 64, kk = e % 64;
        const int n = n0 + j, k = k0 + kk;
        float v = 0.0f;
        if (n < p.N && k < p.K) {
          const int64_t nn = (int64_t)(p.n0 + n);
          v = k < p.k_seg ? B0.ptr[nn * B0.s_i + (int64_t)k * B0.s_k]
                          : B1.ptr[nn * B1.s_i + (int64_t)(k - p.k_seg) * B1.s_k];
        }
        Bs[j][kk] = v;
      }
      __syncthreads();
      if (m < p.M) {
        const int kend = min(64, p.K - k0);
        for (int kk = 0; kk < kend; ++kk) {
          const float a = A.ptr[(int64_t)m * A.s_i + (int64_t)(k0 + kk) * A.s_k];
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = fmaf(a, Bs[j][kk], acc[j]);
        }
      }
      __syncthreads();
    }
    if (m < p.M) {
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + j;
        if (n >= p.N) break;
        if (p.epi.mode == EPI_DW) {
          float* d = p.epi.dw + (int64_t)m * p.epi.ldw + n;
          *d = p.epi.accumulate ? *d + acc[j] : acc[j];
        } else {
          csum += epi_apply(p.epi, m, n, acc[j]);
        }
      }
    }
  }
  if (m < p.M && p.epi.mode == EPI_ACT_BWD && p.epi.colsum) p.epi.colsum[m] = csum;
}

int gemm_simt(cudaStream_t st, bool pdl, SimtOperand A, SimtOperand B0, SimtOperand B1, GemmParams p) {
  if (!B1.ptr) {
    B1 = B0;
    p.k_seg = p.K;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.M + 127) / 128, 1, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_simt_kernel, A, B0, B1, p);
  if (e != cudaSuccess) {
    set_error("gemm_simt launch: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

}  // namespace tgp
