// Cluster LayerNorm kernels for the skinny micro-batch rows (16 rows x 4096 at C2): a row is split
// over a thread-block cluster along the features (<= 512 features per CTA), each CTA keeps its tile
// in registers, and the per-row partial sums are exchanged through DSMEM and added in FIXED rank
// order (every CTA of the cluster computes bit-identical statistics; F' == F bitwise).  This puts
// cluster-size x row-blocks CTAs on a 256 KB problem instead of one CTA per row.
//
// Also: the column-partial kernels (bias-gradient partial sums per 16-row block) used by the
// backward, with a wide grid.
#include <cuda_bf16.h>

#include "common.cuh"
#include "host.h"
#include "kernels.h"

namespace tgp {

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum of `v` over the NQ threads of a row set (NQ / 32 warps), fixed order; result valid in all
// threads of the set.  sh: [16][4] scratch, row = row index within the CTA's 16-row block.
template <int NQ>
__device__ __forceinline__ void rowset_partial(float v, int row, float (*sh)[4]) {
  v = warp_sum(v);
  const int w = (threadIdx.x % NQ) >> 5;
  if ((threadIdx.x & 31) == 0) sh[row][w] = v;
}

template <int NQ>
__device__ __forceinline__ float rowset_total(int row, float (*sh)[4]) {
  float s = 0.0f;
#pragma unroll
  for (int w = 0; w < NQ / 32; ++w) s += sh[row][w];
  return s;
}

// Cluster exchange of per-row partials: every CTA publishes xp[nv][16]; one parallel gather pulls
// the CL ranks' values into local smem (one remote load per thread), then each row total is a
// local sum over the ranks in FIXED rank order (bit-identical on every CTA of the cluster).
__device__ __forceinline__ void cluster_gather(const float* xp, int nv, float* gath, int CL) {
  for (int t = threadIdx.x; t < nv * 16 * CL; t += blockDim.x) {
    const int v = t / (16 * CL), q = (t / 16) % CL, row = t % 16;
    gath[(v * 16 + q) * 16 + row] = ld_dsmem_f32(mapa_shared(smem_u32(xp + v * 16 + row), (uint32_t)q));
  }
  __syncthreads();
}
__device__ __forceinline__ float gathered_total(const float* gath, int v, int row, int CL) {
  float s = 0.0f;
  for (int q = 0; q < CL; ++q) s += gath[(v * 16 + q) * 16 + row];
  return s;
}

// ------------------------------------------------------------------------------ forward
template <int NQ>
__global__ void __launch_bounds__(256) ln_fwd_cl_kernel(const float* __restrict__ x, int64_t ldx, int rows, int d,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta, void* h, int64_t ldh,
                                                        int h_bf16, float* mean, float* rstd) {
  constexpr int RS = 256 / NQ, RPT = 16 / RS;
  __shared__ float sh[16][4];
  __shared__ float xp[2][16];
  __shared__ float gath[2 * 16 * 16];
  griddep_wait();
  griddep_launch();
  const int CL = gridDim.x;
  const int cq = threadIdx.x % NQ, rs = threadIdx.x / NQ;
  const int c0 = (blockIdx.x * NQ + cq) * 4;
  const int rb0 = blockIdx.y * 16;
  float4 v[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = rb0 + rs + k * RS;
    v[k] = r < rows ? *reinterpret_cast<const float4*>(x + (int64_t)r * ldx + c0) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // pass 1: mean
#pragma unroll
  for (int k = 0; k < RPT; ++k) rowset_partial<NQ>((v[k].x + v[k].y) + (v[k].z + v[k].w), rs + k * RS, sh);
  __syncthreads();
  if (threadIdx.x < 16) xp[0][threadIdx.x] = rowset_total<NQ>(threadIdx.x, sh);
  cluster_sync();
  cluster_gather(&xp[0][0], 1, gath, CL);
  float mu[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) mu[k] = gathered_total(gath, 0, rs + k * RS, CL) / (float)d;
  // pass 2: centred second moment
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const float a = v[k].x - mu[k], b = v[k].y - mu[k], e = v[k].z - mu[k], f = v[k].w - mu[k];
    rowset_partial<NQ>((a * a + b * b) + (e * e + f * f), rs + k * RS, sh);
  }
  __syncthreads();
  if (threadIdx.x < 16) xp[1][threadIdx.x] = rowset_total<NQ>(threadIdx.x, sh);
  cluster_sync();
  cluster_gather(&xp[1][0], 1, gath + 256, CL);
  const float4 g = *reinterpret_cast<const float4*>(gamma + c0);
  const float4 bb = *reinterpret_cast<const float4*>(beta + c0);
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int rl = rs + k * RS, r = rb0 + rl;
    const float var = gathered_total(gath + 256, 0, rl, CL) / (float)d;
    const float rsd = 1.0f / sqrtf(var + 1e-5f);
    if (r < rows) {
      const float o0 = g.x * ((v[k].x - mu[k]) * rsd) + bb.x, o1 = g.y * ((v[k].y - mu[k]) * rsd) + bb.y;
      const float o2 = g.z * ((v[k].z - mu[k]) * rsd) + bb.z, o3 = g.w * ((v[k].w - mu[k]) * rsd) + bb.w;
      if (h_bf16) {
        __nv_bfloat162* hp =
            reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(h) + (int64_t)r * ldh + c0);
        hp[0] = __floats2bfloat162_rn(o0, o1);
        hp[1] = __floats2bfloat162_rn(o2, o3);
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(h) + (int64_t)r * ldh + c0) = make_float4(o0, o1, o2, o3);
      }
      if (blockIdx.x == 0 && cq == 0) {
        mean[r] = mu[k];
        rstd[r] = rsd;
      }
    }
  }
  cluster_sync();  // keep xp alive until every CTA of the cluster has read it
}

// ------------------------------------------------------------------------------ backward
// dx = dy + r (dn - mean_row(dn) - n mean_row(dn n)), dn = dh gamma, n = (x - mu) r.
// Column partials over the CTA's 16 rows -> row-block `blockIdx.y` of dgp / dbp.  Optionally the
// NEXT layer's operand copy of dx (op dtype) and its column partial (the bias grad b2 of the
// residual block below), fused here instead of a separate convert kernel.
template <int NQ>
__global__ void __launch_bounds__(256) ln_bwd_cl_kernel(const float* __restrict__ dh, const float* __restrict__ x,
                                                        const float* __restrict__ mean,
                                                        const float* __restrict__ rstd,
                                                        const float* __restrict__ gamma, const float* dy, float* dx,
                                                        int rows, int d, float* dgp, float* dbp, void* op,
                                                        int op_bf16, float* opsum) {
  constexpr int RS = 256 / NQ, RPT = 16 / RS;
  __shared__ float sh[16][4];
  __shared__ float xp[2][16];
  __shared__ float4 cp[3][RS][NQ];
  __shared__ float gath[2 * 16 * 16];
  griddep_wait();
  griddep_launch();
  const int CL = gridDim.x;
  const int cq = threadIdx.x % NQ, rs = threadIdx.x / NQ;
  const int c0 = (blockIdx.x * NQ + cq) * 4;
  const int rb0 = blockIdx.y * 16;
  const float4 g = *reinterpret_cast<const float4*>(gamma + c0);
  float4 vdh[RPT], vn[RPT];
  float rr[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int r = rb0 + rs + k * RS;
    if (r < rows) {
      vdh[k] = *reinterpret_cast<const float4*>(dh + (int64_t)r * d + c0);
      const float4 xv = *reinterpret_cast<const float4*>(x + (int64_t)r * d + c0);
      const float m = mean[r];
      rr[k] = rstd[r];
      vn[k] = make_float4((xv.x - m) * rr[k], (xv.y - m) * rr[k], (xv.z - m) * rr[k], (xv.w - m) * rr[k]);
    } else {
      vdh[k] = vn[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      rr[k] = 0.0f;
    }
  }
  // row sums of dn and dn*n
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const float d0 = vdh[k].x * g.x, d1 = vdh[k].y * g.y, d2 = vdh[k].z * g.z, d3 = vdh[k].w * g.w;
    rowset_partial<NQ>((d0 + d1) + (d2 + d3), rs + k * RS, sh);
  }
  __syncthreads();
  if (threadIdx.x < 16) xp[0][threadIdx.x] = rowset_total<NQ>(threadIdx.x, sh);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const float d0 = vdh[k].x * g.x * vn[k].x, d1 = vdh[k].y * g.y * vn[k].y;
    const float d2 = vdh[k].z * g.z * vn[k].z, d3 = vdh[k].w * g.w * vn[k].w;
    rowset_partial<NQ>((d0 + d1) + (d2 + d3), rs + k * RS, sh);
  }
  __syncthreads();
  if (threadIdx.x < 16) xp[1][threadIdx.x] = rowset_total<NQ>(threadIdx.x, sh);
  cluster_sync();
  cluster_gather(&xp[0][0], 2, gath, CL);
  float4 sg = make_float4(0.f, 0.f, 0.f, 0.f), sb = sg, so = sg;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int rl = rs + k * RS, r = rb0 + rl;
    const float m1 = gathered_total(gath, 0, rl, CL) / (float)d;
    const float m2 = gathered_total(gath, 1, rl, CL) / (float)d;
    if (r < rows) {
      const float4 dyv = dy ? *reinterpret_cast<const float4*>(dy + (int64_t)r * d + c0) : make_float4(0.f, 0.f, 0.f, 0.f);  // dy nullable: no residual
      const float4 n = vn[k], a = vdh[k];
      float4 o;
      o.x = dyv.x + rr[k] * (a.x * g.x - m1 - n.x * m2);
      o.y = dyv.y + rr[k] * (a.y * g.y - m1 - n.y * m2);
      o.z = dyv.z + rr[k] * (a.z * g.z - m1 - n.z * m2);
      o.w = dyv.w + rr[k] * (a.w * g.w - m1 - n.w * m2);
      *reinterpret_cast<float4*>(dx + (int64_t)r * d + c0) = o;
      if (op) {
        if (op_bf16) {
          __nv_bfloat162* p2 =
              reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(op) + (int64_t)r * d + c0);
          p2[0] = __floats2bfloat162_rn(o.x, o.y);
          p2[1] = __floats2bfloat162_rn(o.z, o.w);
        } else {
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(op) + (int64_t)r * d + c0) = o;
        }
      }
      sg.x += a.x * n.x;
      sg.y += a.y * n.y;
      sg.z += a.z * n.z;
      sg.w += a.w * n.w;
      sb.x += a.x;
      sb.y += a.y;
      sb.z += a.z;
      sb.w += a.w;
      so.x += o.x;
      so.y += o.y;
      so.z += o.z;
      so.w += o.w;
    }
  }
  cp[0][rs][cq] = sg;
  cp[1][rs][cq] = sb;
  cp[2][rs][cq] = so;
  __syncthreads();
  if (rs == 0) {
    float4 a = cp[0][0][cq], b = cp[1][0][cq], o = cp[2][0][cq];
#pragma unroll
    for (int q = 1; q < RS; ++q) {
      const float4 a2 = cp[0][q][cq], b2 = cp[1][q][cq], o2 = cp[2][q][cq];
      a.x += a2.x; a.y += a2.y; a.z += a2.z; a.w += a2.w;
      b.x += b2.x; b.y += b2.y; b.z += b2.z; b.w += b2.w;
      o.x += o2.x; o.y += o2.y; o.z += o2.z; o.w += o2.w;
    }
    const int64_t pr = (int64_t)blockIdx.y * d + c0;
    *reinterpret_cast<float4*>(dgp + pr) = a;
    *reinterpret_cast<float4*>(dbp + pr) = b;
    if (opsum) *reinterpret_cast<float4*>(opsum + pr) = o;
  }
  cluster_sync();
}

// ------------------------------------------------------------------------------ host launchers
static int ln_cluster_shape(int d, int* NQ, int* CL) {
  if (d % 128) return -1;
  const int nq4 = d / 4;
  int cl = (nq4 + 127) / 128;
  while (cl <= 16 && (nq4 % cl || (nq4 / cl) > 128)) ++cl;
  if (cl > 16) return -1;
  const int nq = nq4 / cl;
  if (nq != 32 && nq != 64 && nq != 128) return -1;
  *NQ = nq;
  *CL = cl;
  return 0;
}

template <typename K, typename... Args>
static int launch_cluster(const char* name, K kern, int CL, int rowblocks, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL, rowblocks, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  if (CL > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess) {
    set_error("%s launch (cluster %d): %s", name, CL, cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

int ln_fwd_cl(cudaStream_t st, bool pdl, const float* x, int64_t ldx, int rows, int d, const float* gamma,
              const float* beta, void* h, int64_t ldh, bool h_bf16, float* mean, float* rstd) {
  int NQ, CL;
  // the cluster split exists to give a 16-row micro-batch enough CTAs; from 64 rows one CTA per row
  // is enough parallelism and skips the three cluster exchanges (C3 m = 4: 9 -> ~3 us per launch)
  if (rows >= 64 || ln_cluster_shape(d, &NQ, &CL))
    return ln_fwd(st, pdl, x, ldx, rows, d, gamma, beta, h, ldh, h_bf16, mean, rstd);
  const int rb = (rows + 15) / 16;
#define L_(N)                                                                                                 \
  if (NQ == N)                                                                                                \
    return launch_cluster("ln_fwd_cl", ln_fwd_cl_kernel<N>, CL, rb, st, pdl, x, ldx, rows, d, gamma, beta, h, \
                          ldh, (int)h_bf16, mean, rstd);
  L_(32) L_(64) L_(128)
#undef L_
  set_error("ln_fwd_cl: no cluster shape for d=%d", d);
  return -5;
}

int ln_bwd_cl(cudaStream_t st, bool pdl, const float* dh, const float* x, const float* mean, const float* rstd,
              const float* gamma, const float* dy, float* dx, int rows, int d, int rowblocks, float* dgp, float* dbp,
              void* op, bool op_bf16, float* opsum) {
  int NQ, CL;
  if (ln_cluster_shape(d, &NQ, &CL)) {
    set_error("ln_bwd_cl: no cluster shape for d=%d", d);
    return -5;
  }
  // from 64 rows: clusters of 16 (non-portable size), twice the CTAs of the 8-wide split (C3 m = 4: B
  // task 1376 -> 1244 us, profiles/r6/)
  static int cl16 = -1;  // can this device co-schedule a cluster of 16 of these CTAs?
  if (cl16 < 0) {
    cudaFuncSetAttribute(ln_bwd_cl_kernel<64>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 16;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    int n = 0;
    cl16 = (cudaOccupancyMaxActiveClusters(&n, ln_bwd_cl_kernel<64>, &cfg) == cudaSuccess && n > 0) ? 1 : 0;
    cudaGetLastError();
  }
  if (cl16 && rowblocks >= 4 && CL == 8 && NQ == 128) {
    CL = 16;
    NQ = 64;
  }
#define L_(N)                                                                                                   \
  if (NQ == N)                                                                                                  \
    return launch_cluster("ln_bwd_cl", ln_bwd_cl_kernel<N>, CL, rowblocks, st, pdl, dh, x, mean, rstd, gamma, dy, \
                          dx, rows, d, dgp, dbp, op, (int)op_bf16, opsum);
  L_(32) L_(64) L_(128)
#undef L_
  set_error("ln_bwd_cl: no cluster shape for d=%d", d);
  return -5;
}

bool ln_cluster_ok(int d) {
  int a, b;
  return ln_cluster_shape(d, &a, &b) == 0;
}

// ------------------------------------------------------------------------------ column kernels
// out = op(dy [* dropout] * act'(z)) with column partial sums per 16-row block:
// CTA = 32 float4 columns x 16 rows (4 row sets of 4), 128 threads.
__global__ void __launch_bounds__(128) colwise_kernel(const float* __restrict__ src, int64_t lds, const float* z,
                                                      int rows, int d, int act, uint32_t thresh, float scale,
                                                      uint64_t seed, const uint32_t* step, uint32_t site,
                                                      int64_t row0, void* out, int64_t ldo, int out_bf16,
                                                      float* colsum) {
  __shared__ float4 cp[4][32];
  griddep_wait();
  griddep_launch();
  const int cq = threadIdx.x & 31, rs = threadIdx.x >> 5;
  const int c0 = (blockIdx.x * 32 + cq) * 4;
  const int rb0 = blockIdx.y * 16;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c0 < d) {
    const uint32_t st = (thresh && step) ? *step : 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = rb0 + rs + 4 * k;
      if (r >= rows) break;
      float4 v = *reinterpret_cast<const float4*>(src + (int64_t)r * lds + c0);
      float vv[4] = {v.x, v.y, v.z, v.w};
      uint32_t kw[4] = {0u, 0u, 0u, 0u};
      if (thresh) {
        // the 4 elements of this float4 share one Philox call: their flat index (row * d + c0 + e,
        // d % 4 == 0, c0 % 4 == 0) has the same counter q = idx >> 2 and picks word e (O8)
        const uint64_t q = ((uint64_t)(row0 + r) * (uint64_t)d + (uint64_t)c0) >> 2;
        const uint4 o = philox4x32_10(make_uint4((uint32_t)q, (uint32_t)(q >> 32), site, st),
                                      make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
        kw[0] = o.x;
        kw[1] = o.y;
        kw[2] = o.z;
        kw[3] = o.w;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (thresh) vv[e] = (kw[e] >> 8) >= thresh ? vv[e] * scale : 0.0f;
        if (act) vv[e] *= act_df(act, z[(int64_t)r * d + c0 + e]);
      }
      v = make_float4(vv[0], vv[1], vv[2], vv[3]);
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
      if (out_bf16) {
        __nv_bfloat162* p2 =
            reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(out) + (int64_t)r * ldo + c0);
        p2[0] = __floats2bfloat162_rn(v.x, v.y);
        p2[1] = __floats2bfloat162_rn(v.z, v.w);
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + (int64_t)r * ldo + c0) = v;
      }
    }
  }
  cp[rs][cq] = s;
  __syncthreads();
  if (rs == 0 && colsum && c0 < d) {
    float4 a = cp[0][cq];
#pragma unroll
    for (int q = 1; q < 4; ++q) {
      a.x += cp[q][cq].x;
      a.y += cp[q][cq].y;
      a.z += cp[q][cq].z;
      a.w += cp[q][cq].w;
    }
    *reinterpret_cast<float4*>(colsum + (int64_t)blockIdx.y * d + c0) = a;
  }
}

int colwise(cudaStream_t st, bool pdl, const float* src, int64_t lds, const float* z, int rows, int d, int act,
            uint32_t drop_thresh, float drop_scale, uint64_t seed, const uint32_t* step, uint32_t site,
            int64_t row_global0, void* out, int64_t ldo, bool out_bf16, float* colsum) {
  if (d % 4 || lds % 4 || ldo % 4) {
    set_error("colwise: d=%d, lds=%lld, ldo=%lld must be multiples of 4", d, (long long)lds, (long long)ldo);
    return -5;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((d / 4 + 31) / 32, (rows + 15) / 16, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, colwise_kernel, src, lds, z, rows, d, act, drop_thresh, drop_scale, seed,
                                     step, site, row_global0, out, ldo, (int)out_bf16, colsum);
  if (e != cudaSuccess) {
    set_error("colwise launch: %s", cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

}  // namespace tgp
