// Vectorised / coalesced element-wise, normalisation, loss, optimizer and transport kernels.
// All reductions use fixed trees / fixed orders (deterministic: F' == F bitwise, reading Z21).
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "host.h"
#include "kernels.h"

namespace tgp {

template <typename Kern, typename... Args>
static int launch(const char* name, Kern k, dim3 grid, dim3 block, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
  if (e != cudaSuccess) {
    set_error("%s launch: %s", name, cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

// block-wide sum (fixed tree), blockDim.x multiple of 32, <= 1024
template <typename T>
__device__ T block_sum(T v, T* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  T t = 0;
  if (w == 0) {
    t = l < nw ? sh[l] : T(0);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (l == 0) sh[0] = t;
  }
  __syncthreads();
  return sh[0];
}

// ------------------------------------------------------------------------------- LayerNorm
// one CTA per row; two-pass statistics (mean, then centred second moment)
__global__ void ln_fwd_kernel(const float* __restrict__ x, int64_t ldx, int d, const float* __restrict__ gamma,
                              const float* __restrict__ beta, void* h, int64_t ldh, int h_bf16, float* mean,
                              float* rstd) {
  griddep_wait();
  griddep_launch();
  __shared__ float sh[32];
  const int r = blockIdx.x;
  const float* xr = x + (int64_t)r * ldx;
  float s = 0.0f;
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    s += (v.x + v.y) + (v.z + v.w);
  }
  const float mu = block_sum(s, sh) / (float)d;
  float q = 0.0f;
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    const float a = v.x - mu, b = v.y - mu, e = v.z - mu, f = v.w - mu;
    q += (a * a + b * b) + (e * e + f * f);
  }
  const float var = block_sum(q, sh) / (float)d;
  const float rs = 1.0f / sqrtf(var + 1e-5f);
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(xr + c);
    const float4 g = *reinterpret_cast<const float4*>(gamma + c);
    const float4 b = *reinterpret_cast<const float4*>(beta + c);
    const float o0 = g.x * ((v.x - mu) * rs) + b.x, o1 = g.y * ((v.y - mu) * rs) + b.y;
    const float o2 = g.z * ((v.z - mu) * rs) + b.z, o3 = g.w * ((v.w - mu) * rs) + b.w;
    if (h_bf16) {
      __nv_bfloat162* hp = reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<__nv_bfloat16*>(h) + (int64_t)r * ldh + c);
      hp[0] = __floats2bfloat162_rn(o0, o1);
      hp[1] = __floats2bfloat162_rn(o2, o3);
    } else {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(h) + (int64_t)r * ldh + c) = make_float4(o0, o1, o2, o3);
    }
  }
  if (threadIdx.x == 0) {
    mean[r] = mu;
    rstd[r] = rs;
  }
}

int ln_fwd(cudaStream_t st, bool pdl, const float* x, int64_t ldx, int rows, int d, const float* gamma,
           const float* beta, void* h, int64_t ldh, bool h_bf16, float* mean, float* rstd) {
  if (d % 4) {
    set_error("ln_fwd: d=%d must be a multiple of 4", d);
    return -5;
  }
  const int threads = d >= 1024 ? 256 : 128;
  return launch("ln_fwd", ln_fwd_kernel, dim3(rows), dim3(threads), st, pdl, x, ldx, d, gamma, beta, h, ldh,
                (int)h_bf16, mean, rstd);
}

__global__ void ln_bwd_rows_kernel(const float* __restrict__ dh, const float* __restrict__ x,
                                   const float* __restrict__ mean, const float* __restrict__ rstd,
                                   const float* __restrict__ gamma, const float* __restrict__ dy, float* dx, int d) {
  griddep_wait();
  griddep_launch();
  __shared__ float sh[32];
  const int r = blockIdx.x;
  const float mu = mean[r], rs = rstd[r];
  const float* dhr = dh + (int64_t)r * d;
  const float* xr = x + (int64_t)r * d;
  float s1 = 0.0f, s2 = 0.0f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float dn = dhr[c] * gamma[c];
    const float nn = (xr[c] - mu) * rs;
    s1 += dn;
    s2 += dn * nn;
  }
  const float m1 = block_sum(s1, sh) / (float)d;
  const float m2 = block_sum(s2, sh) / (float)d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float dn = dhr[c] * gamma[c];
    const float nn = (xr[c] - mu) * rs;
    dx[(int64_t)r * d + c] = (dy ? dy[(int64_t)r * d + c] : 0.0f) + rs * (dn - m1 - nn * m2);
  }
}

// column partials per 16-row block (same layout as the cluster LayerNorm and the GEMM colsum:
// block y of the micro-batch writes dgp/dbp + y*d): dgamma = sum dh * n, dbeta = sum dh
__global__ void ln_bwd_cols_kernel(const float* __restrict__ dh, const float* __restrict__ x,
                                   const float* __restrict__ mean, const float* __restrict__ rstd, int rows, int d,
                                   float* dgp, float* dbp) {
  griddep_wait();
  griddep_launch();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const int r0 = blockIdx.y * 16, r1 = min(rows, r0 + 16);
  float sg = 0.0f, sb = 0.0f;
  for (int r = r0; r < r1; ++r) {
    const float v = dh[(int64_t)r * d + c];
    sg += v * ((x[(int64_t)r * d + c] - mean[r]) * rstd[r]);
    sb += v;
  }
  dgp[(int64_t)blockIdx.y * d + c] = sg;
  dbp[(int64_t)blockIdx.y * d + c] = sb;
}

int ln_bwd(cudaStream_t st, bool pdl, const float* dh, const float* x, const float* mean, const float* rstd,
           const float* gamma, const float* dy, float* dx, int rows, int d, float* dgp, float* dbp) {
  int e = launch("ln_bwd_cols", ln_bwd_cols_kernel, dim3((d + 127) / 128, (rows + 15) / 16), dim3(128), st, pdl, dh,
                 x, mean, rstd, rows, d, dgp, dbp);
  if (e) return e;
  return launch("ln_bwd_rows", ln_bwd_rows_kernel, dim3(rows), dim3(d >= 1024 ? 256 : 128), st, pdl, dh, x, mean,
                rstd, gamma, dy, dx, d);
}

// ------------------------------------------------------------------------------- conversions
__global__ void convert_rows_kernel(const float* __restrict__ x, int64_t ldx, int rows, int d, void* out, int64_t ldo,
                                    int out_bf16, float* colsum) {
  griddep_wait();
  griddep_launch();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float s = 0.0f;
  for (int r = 0; r < rows; ++r) {
    const float v = x[(int64_t)r * ldx + c];
    s += v;
    if (out_bf16)
      reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)r * ldo + c] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float*>(out)[(int64_t)r * ldo + c] = v;
  }
  if (colsum) colsum[c] = s;
}

int convert_rows(cudaStream_t st, bool pdl, const float* x, int64_t ldx, int rows, int d, void* out, int64_t ldo,
                 bool out_bf16, float* colsum) {
  return launch("convert_rows", convert_rows_kernel, dim3((d + 127) / 128), dim3(128), st, pdl, x, ldx, rows, d, out,
                ldo, (int)out_bf16, colsum);
}

__global__ void act_bwd_rows_kernel(const float* __restrict__ dy, const float* __restrict__ z, int rows, int d,
                                    int act, uint32_t thresh, float scale, uint64_t seed, const uint32_t* step,
                                    uint32_t site, int64_t row0, void* out, int64_t ldo, int out_bf16,
                                    float* colsum) {
  griddep_wait();
  griddep_launch();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float s = 0.0f;
  for (int r = 0; r < rows; ++r) {
    float v = dy[(int64_t)r * d + c];
    if (thresh) {
      const uint64_t idx = (uint64_t)(row0 + r) * (uint64_t)d + (uint64_t)c;
      v = dropout_keep(seed, *step, site, idx, thresh) ? v * scale : 0.0f;
    }
    if (act) v *= act_df(act, z[(int64_t)r * d + c]);
    s += v;
    if (out_bf16)
      reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)r * ldo + c] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float*>(out)[(int64_t)r * ldo + c] = v;
  }
  if (colsum) colsum[c] = s;
}

int act_bwd_rows(cudaStream_t st, bool pdl, const float* dy, const float* z, int rows, int d, int act,
                 uint32_t drop_thresh, float drop_scale, uint64_t seed, const uint32_t* step, uint32_t site,
                 int64_t row_global0, void* out, int64_t ldo, bool out_bf16, float* colsum) {
  return launch("act_bwd_rows", act_bwd_rows_kernel, dim3((d + 127) / 128), dim3(128), st, pdl, dy, z, rows, d, act,
                drop_thresh, drop_scale, seed, step, site, row_global0, out, ldo, (int)out_bf16, colsum);
}

__global__ void add_rows_kernel(float* y, const float* __restrict__ a, int64_t n) {
  griddep_wait();
  griddep_launch();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a[i];
}
int add_rows(cudaStream_t st, bool pdl, float* y, const float* a, int64_t n) {
  const int blocks = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  return launch("add_rows", add_rows_kernel, dim3(blocks), dim3(256), st, pdl, y, a, n);
}

__global__ void reduce_partials_kernel(const float* __restrict__ part, int m, int d, float* out, int acc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float s = 0.0f;
  for (int i = 0; i < m; ++i) s += part[(int64_t)i * d + c];
  out[c] = acc ? out[c] + s : s;
}
// all column-partial reductions of a partition in one launch: item blockIdx.y reduces its [m][d]
// partial rows into out (fixed row order per column, as reduce_partials_kernel)
__global__ void reduce_partials_multi_kernel(const RedItem* __restrict__ items, int m, int acc) {
  const RedItem it = items[blockIdx.y];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= it.d) return;
  float s = 0.0f;
#pragma unroll 8
  for (int i = 0; i < m; ++i) s += it.part[(int64_t)i * it.d + c];
  it.out[c] = acc ? it.out[c] + s : s;
}
int reduce_partials_multi(cudaStream_t st, const RedItem* items, int n_items, int max_d, int m, bool accumulate) {
  return launch("reduce_partials_multi", reduce_partials_multi_kernel, dim3((max_d + 255) / 256, n_items), dim3(256),
                st, false, items, m, (int)accumulate);
}
int reduce_partials(cudaStream_t st, const float* part, int m, int d, float* out, bool accumulate) {
  return launch("reduce_partials", reduce_partials_kernel, dim3((d + 255) / 256), dim3(256), st, false, part, m, d,
                out, (int)accumulate);
}

// ------------------------------------------------------------------------------- loss
constexpr int kLossBlocks = 296;
__global__ void mse_partial_kernel(const float* __restrict__ y, const float* __restrict__ t, int64_t n, float* dy,
                                   double* part) {
  __shared__ double sh[32];
  const double scale = 2.0 / (double)n;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)y[i] - (double)t[i];
    s += d * d;
    dy[i] = (float)(scale * d);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void mse_final_kernel(const double* part, int np, int64_t n, double* loss) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < np; ++i) s += part[i];
    loss[0] = s / (double)n;
  }
}
int mse_loss_grad(cudaStream_t st, const float* y, const float* t, int64_t n, float* dy, double* loss_dev) {
  // loss_dev must hold kLossBlocks + 1 doubles: [0] = loss, [1..] = partials
  int e = launch("mse_partial", mse_partial_kernel, dim3(kLossBlocks), dim3(256), st, false, y, t, n, dy,
                 loss_dev + 1);
  if (e) return e;
  return launch("mse_final", mse_final_kernel, dim3(1), dim3(32), st, false, (const double*)(loss_dev + 1),
                kLossBlocks, n, loss_dev);
}

// ------------------------------------------------------------------------------- optimizer
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, __nv_bfloat16* __restrict__ sh,
                           int64_t n4, float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<float4*>(w)[i];
    const float4 b = reinterpret_cast<const float4*>(g)[i];
    a.x = __fmaf_rn(-lr, b.x, a.x);  // the same fma as the fused W_j + SGD epilogue (gemm_dw_sgd.cu)
    a.y = __fmaf_rn(-lr, b.y, a.y);
    a.z = __fmaf_rn(-lr, b.z, a.z);
    a.w = __fmaf_rn(-lr, b.w, a.w);
    reinterpret_cast<float4*>(w)[i] = a;
    if (sh) {
      __nv_bfloat162* s2 = reinterpret_cast<__nv_bfloat162*>(sh) + 2 * i;
      s2[0] = __floats2bfloat162_rn(a.x, a.y);
      s2[1] = __floats2bfloat162_rn(a.z, a.w);
    }
  }
}
int sgd_step(cudaStream_t st, float* master, const float* grad, __nv_bfloat16* shadow, int64_t n, float lr) {
  if (n % 4) {
    set_error("sgd_step: arena size %lld not a multiple of 4", (long long)n);
    return -5;
  }
  const int64_t n4 = n / 4;
  const int blocks = (int)(n4 / 256 + 1 < 148 * 8 ? n4 / 256 + 1 : 148 * 8);
  return launch("sgd", sgd_kernel, dim3(blocks), dim3(256), st, false, master, grad, shadow, n4, lr);
}

__global__ void sgd_segments_kernel(float* __restrict__ w, const float* __restrict__ g, __nv_bfloat16* __restrict__ sh,
                                    const int64_t* __restrict__ seg, const float* __restrict__ lrp) {
  const int64_t off = seg[2 * blockIdx.y], len = seg[2 * blockIdx.y + 1];
  const float lr = *lrp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const float a = __fmaf_rn(-lr, g[off + i], w[off + i]);
    w[off + i] = a;
    if (sh) sh[off + i] = __float2bfloat16_rn(a);
  }
}
int sgd_segments(cudaStream_t st, float* master, const float* grad, __nv_bfloat16* shadow, const int64_t* seg, int nseg,
                 int64_t max_len, const float* lr) {
  if (nseg <= 0) return 0;
  if (nseg > 65535) {
    set_error("sgd_segments: %d segments (max 65535)", nseg);
    return -5;
  }
  const int bx = (int)std::min<int64_t>((max_len + 255) / 256, 64);
  return launch("sgd_segments", sgd_segments_kernel, dim3(bx, nseg), dim3(256), st, false, master, grad, shadow, seg, lr);
}

__global__ void cast_bf16_kernel(const float* __restrict__ s, __nv_bfloat16* __restrict__ d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = __float2bfloat16_rn(s[i]);
}
int cast_bf16(cudaStream_t st, const float* src, __nv_bfloat16* dst, int64_t n) {
  return launch("cast_bf16", cast_bf16_kernel, dim3(148 * 8), dim3(256), st, false, src, dst, n);
}

__global__ void init_uniform_kernel(float* d, int64_t n, float lo, float hi, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 o = philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), 0x1417u, 0u),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const float u = (float)(o.x >> 8) * 5.9604644775390625e-08f;
    d[i] = lo + (hi - lo) * u;
  }
}
int init_uniform(cudaStream_t st, float* dst, int64_t n, float lo, float hi, uint64_t seed) {
  return launch("init_uniform", init_uniform_kernel, dim3(148 * 8), dim3(256), st, false, dst, n, lo, hi, seed);
}

// ------------------------------------------------------------------------------- BatchNorm
__global__ void bn_fwd_kernel(const float* __restrict__ x, int rows, int d, const float* gamma, const float* beta,
                              int act, float* y, float* z, float* mu_o, float* rstd_o, float* var_o) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float s = 0.0f;
  for (int r = 0; r < rows; ++r) s += x[(int64_t)r * d + c];
  const float mu = s / (float)rows;
  float q = 0.0f;
  for (int r = 0; r < rows; ++r) {
    const float a = x[(int64_t)r * d + c] - mu;
    q += a * a;
  }
  const float var = q / (float)rows;
  const float rs = 1.0f / sqrtf(var + 1e-5f);
  for (int r = 0; r < rows; ++r) {
    const float zz = gamma[c] * ((x[(int64_t)r * d + c] - mu) * rs) + beta[c];
    z[(int64_t)r * d + c] = zz;
    y[(int64_t)r * d + c] = act_f(act, zz);
  }
  mu_o[c] = mu;
  rstd_o[c] = rs;
  var_o[c] = var;
}
int bn_fwd(cudaStream_t st, const float* x, int rows, int d, const float* gamma, const float* beta, int act, float* y,
           float* z, float* mu, float* rstd, float* var_out) {
  return launch("bn_fwd", bn_fwd_kernel, dim3((d + 127) / 128), dim3(128), st, false, x, rows, d, gamma, beta, act, y,
                z, mu, rstd, var_out);
}

__global__ void bn_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ z,
                              const float* mu, const float* rstd, const float* gamma, int rows, int d, int act,
                              float* dx, float* dgp, float* dbp) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  const float m = mu[c], rs = rstd[c], g = gamma[c];
  float sg = 0.0f, sb = 0.0f, s1 = 0.0f, s2 = 0.0f;
  for (int r = 0; r < rows; ++r) {
    const int64_t i = (int64_t)r * d + c;
    const float dz = dy[i] * act_df(act, z[i]);
    const float nn = (x[i] - m) * rs;
    sg += dz * nn;
    sb += dz;
    s1 += dz * g;
    s2 += dz * g * nn;
  }
  const float m1 = s1 / (float)rows, m2 = s2 / (float)rows;
  for (int r = 0; r < rows; ++r) {
    const int64_t i = (int64_t)r * d + c;
    const float dn = dy[i] * act_df(act, z[i]) * g;
    const float nn = (x[i] - m) * rs;
    dx[i] = rs * (dn - m1 - nn * m2);
  }
  dgp[c] = sg;
  dbp[c] = sb;
}
int bn_bwd(cudaStream_t st, const float* dy, const float* x, const float* z, const float* mu, const float* rstd,
           const float* gamma, int rows, int d, int act, float* dx, float* dgp, float* dbp) {
  return launch("bn_bwd", bn_bwd_kernel, dim3((d + 127) / 128), dim3(128), st, false, dy, x, z, mu, rstd, gamma, rows,
                d, act, dx, dgp, dbp);
}

__global__ void bn_commit_kernel(const float* mu_p, const float* var_p, const int* rows, int m, int d, float mom,
                                 float* rm, float* rv) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  double nt = 0.0, s = 0.0;
  for (int i = 0; i < m; ++i) {
    nt += rows[i];
    s += (double)rows[i] * mu_p[(int64_t)i * d + c];
  }
  const double mean = s / nt;
  double q = 0.0;
  for (int i = 0; i < m; ++i) {
    const double dm = (double)mu_p[(int64_t)i * d + c] - mean;
    q += (double)rows[i] * ((double)var_p[(int64_t)i * d + c] + dm * dm);
  }
  const double var = q / nt;
  rm[c] = (float)((1.0 - mom) * rm[c] + mom * mean);
  rv[c] = (float)((1.0 - mom) * rv[c] + mom * var * nt / (nt - 1.0));
}
int bn_commit(cudaStream_t st, const float* mu_parts, const float* var_parts, const int* rows, int m, int d,
              float momentum, float* run_mean, float* run_var) {
  return launch("bn_commit", bn_commit_kernel, dim3((d + 127) / 128), dim3(128), st, false, mu_parts, var_parts, rows,
                m, d, momentum, run_mean, run_var);
}

// ------------------------------------------------------------------------------- transport
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t atom_add_acq_rel_sys(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.sys.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// The CTA's stores are ordered before thread 0's release-add by the barrier (release is cumulative);
// the last CTA's acquire-add reads the chain of every CTA's release, so its release store of the flag
// publishes the whole message at system scope (peer GPUs, CUDA-IPC mappings).  Single CTA: no counter.
__device__ __forceinline__ void finish_push(uint32_t* counter, uint32_t* flag, uint32_t seq) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (gridDim.x == 1) {
      st_release_sys(flag, seq);
    } else if (atom_add_acq_rel_sys(counter, 1u) == gridDim.x - 1) {
      *counter = 0u;  // reset for the next push on this stream (ordered before it by the stream)
      st_release_sys(flag, seq);
    }
  }
}

__global__ void push_rows_kernel(const float* __restrict__ src, void* dst, int dst_bf16, int64_t n, uint32_t* counter,
                                 uint32_t* flag, uint32_t seq) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    if (dst_bf16) {
      __nv_bfloat162* d2 = reinterpret_cast<__nv_bfloat162*>(dst) + 2 * i;
      d2[0] = __floats2bfloat162_rn(v.x, v.y);
      d2[1] = __floats2bfloat162_rn(v.z, v.w);
    } else {
      reinterpret_cast<float4*>(dst)[i] = v;
    }
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (dst_bf16)
      reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(src[i]);
    else
      reinterpret_cast<float*>(dst)[i] = src[i];
  }
  finish_push(counter, flag, seq);
}

__global__ void push_bytes_kernel(const int4* __restrict__ src, int4* dst, int64_t n16, uint32_t* counter,
                                  uint32_t* flag, uint32_t seq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
  finish_push(counter, flag, seq);
}

static int push_grid(int64_t n16) {
  int64_t b = (n16 + 255) / 256;
  if (b > 64) b = 64;
  return b < 1 ? 1 : (int)b;
}

int push_rows(cudaStream_t st, const float* src, void* dst, bool dst_bf16, int64_t n, uint32_t* counter,
              uint32_t* flag, uint32_t seq) {
  return launch("push_rows", push_rows_kernel, dim3(push_grid(n / 4)), dim3(256), st, false, src, dst, (int)dst_bf16,
                n, counter, flag, seq);
}

int push_bytes(cudaStream_t st, const void* src, void* dst, int64_t nbytes, uint32_t* counter, uint32_t* flag,
               uint32_t seq) {
  if (nbytes % 16) {
    set_error("push_bytes: %lld bytes not a multiple of 16", (long long)nbytes);
    return -5;
  }
  return launch("push_bytes", push_bytes_kernel, dim3(push_grid(nbytes / 16)), dim3(256), st, false,
                (const int4*)src, (int4*)dst, nbytes / 16, counter, flag, seq);
}

// test-only: occupy a stream for `ns` nanoseconds (negative-control tests delay a push with it)
__global__ void spin_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}
int spin(cudaStream_t st, uint64_t ns) { return launch("spin", spin_kernel, dim3(1), dim3(1), st, false, ns); }

__global__ void signal_kernel(uint32_t* flag, uint32_t v) { st_release_sys(flag, v); }

// watchdog release: every flag a stream may wait on is set far ahead of any sequence number
__global__ void fill_u32_kernel(uint32_t* p, int64_t n, uint32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    st_release_sys(p + i, v);
}
int fill_flags(cudaStream_t st, uint32_t* p, int64_t n, uint32_t v) {
  return launch("fill_flags", fill_u32_kernel, dim3(1), dim3(256), st, false, p, n, v);
}
int signal_flag(cudaStream_t st, uint32_t* flag, uint32_t value) {
  return launch("signal", signal_kernel, dim3(1), dim3(1), st, false, flag, value);
}

}  // namespace tgp
