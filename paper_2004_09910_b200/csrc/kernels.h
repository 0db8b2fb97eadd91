// Internal launcher declarations for the tgp CUDA kernels (host-callable; no torch types).
// All launchers return 0 on success, a negative tgp_status on failure (message in tgp_last_error).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "gemm_tc.cuh"

namespace tgp {

// A row-major bf16 matrix in device memory: [rows][cols] with leading dimension ld (elements).
struct TcMat {
  const void* ptr;
  int64_t rows, cols, ld;
};

// tcgen05 GEMM: D[m][n] = sum_k A[m][k] B[n][k].
//   A: a_mn == false -> memory [M][K] (K-major);  a_mn == true -> memory [K][M] (MN-major)
//   B: b_mn == false -> memory [rows][K] (K-major, n = row, offset p.n0);  b_mn == true -> [K][N]
//   B1: optional second K-segment (k >= p.k_seg), same majorness.
// splits <= 0: automatic split-K (cluster size) heuristic.
// Persistent deferred weight-gradient GEMM (gemm_dw.cu): D[M][N] (=|+=) sum_k A[k][m] B[k][n], bf16
// operands stored [K][M] / [K][N], fp32 D; M, N multiples of 128.
int gemm_dw(cudaStream_t st, const void* A, int64_t lda, const void* B, int64_t ldb, float* D, int64_t ldd, int M,
            int N, int K, bool accumulate);
// Deferred dW GEMMs fused with plain SGD (gemm_dw_sgd.cu): for each GEMM,
//   W[m][n] -= lr * sum_k A[k][m] B[k][n];  shadow[m][n] = bf16(W[m][n])
// A [K][M], B [K][N] bf16 (MN-major operands, TMA zero-fills rows past K), W fp32 / shadow bf16
// [M][N] with leading dimension ldw; M, N multiples of 128.  All GEMMs of the array run in one
// persistent launch, tiles numbered GEMM after GEMM (tile0 = running sum of the tile counts, set by
// the caller).  The gradient is not stored.
struct alignas(64) WsGemm {
  CUtensorMap a, b, w, sh;
  int M, N, K, tiles_n, tiles, tile0;
};
bool wgrad_sgd_desc(WsGemm* d, const void* A, int64_t lda, const void* B, int64_t ldb, float* W, __nv_bfloat16* shadow,
                    int64_t ldw, int M, int N, int K);
// dev_descs: device copy of host_descs[ngemm]; lr: device scalar.
int wgrad_sgd(cudaStream_t st, const WsGemm* dev_descs, const WsGemm* host_descs, int ngemm, const float* lr);
// Plain SGD over parameter segments {offset, length} (device array seg[2 * nseg], elements) of the
// arena: w -= lr g (fma, as sgd_kernel), shadow = bf16(w) when shadow != nullptr; lr: device scalar.
int sgd_segments(cudaStream_t st, float* master, const float* grad, __nv_bfloat16* shadow, const int64_t* seg, int nseg,
                 int64_t max_len, const float* lr);
// Persistent tcgen05 GEMM for wide per-micro-batch GEMMs (gemm_wide.cu): same D = A B^T semantics and
// epilogues as gemm_tc (B K-major, no second K-segment, no dW mode), one CTA per SM over 128 x 128 tiles.
int gemm_wide(cudaStream_t st, const TcMat& A, bool a_mn, const TcMat& B, const GemmParams& p);
int gemm_tc(cudaStream_t st, bool pdl, const TcMat& A, bool a_mn, const TcMat& B0, const TcMat* B1, bool b_mn,
            GemmParams p, int splits);
// 2-D bf16 TMA descriptor over a row-major matrix, 128-byte swizzle, box {box_inner, box_outer}.
bool make_map(CUtensorMap* map, const TcMat& t, int box_inner, int box_outer, bool l2_promote = true);

// fp32 SIMT GEMM with the same D = A * B^T semantics and epilogues, for fp32 mode (no TF32).
// Operand element (i, k) of A is at A[i * a_si + k * a_sk]; of B at B[n * b_sn + k * b_sk]
// (k < k_seg) or B1[n * b1_sn + (k - k_seg) * b1_sk].
struct SimtOperand {
  const float* ptr;
  int64_t s_i, s_k;
};
int gemm_simt(cudaStream_t st, bool pdl, SimtOperand A, SimtOperand B0, SimtOperand B1, GemmParams p);

// ----------------------------------------------------------------------------- element-wise
// LayerNorm forward over rows x d (fp32 in), writing h (op dtype) and per-row mean / rstd.
int ln_fwd(cudaStream_t st, bool pdl, const float* x, int64_t ldx, int rows, int d, const float* gamma,
           const float* beta, void* h, int64_t ldh, bool h_bf16, float* mean, float* rstd);
// LayerNorm backward: dx = dy + r (dn - mean(dn) - n mean(dn n)), dn = dh * gamma; writes the
// column partials per 16-row block y (dgamma_part + y*d = sum_rows dh n, dbeta_part + y*d = sum_rows dh).
int ln_bwd(cudaStream_t st, bool pdl, const float* dh, const float* x, const float* mean, const float* rstd,
           const float* gamma, const float* dy, float* dx, int rows, int d, float* dgamma_part, float* dbeta_part);
// Cluster LayerNorm (features split over a cluster, row statistics exchanged through DSMEM in fixed
// rank order).  ln_fwd_cl falls back to ln_fwd for widths it cannot tile.  ln_bwd_cl writes the
// column partials of 16-row block y to dgp/dbp + y*d (rowblocks >= ceil(rows/16); blocks past the
// rows write zeros) and optionally `op` = dx in op dtype and `opsum` = its column partials.
int ln_fwd_cl(cudaStream_t st, bool pdl, const float* x, int64_t ldx, int rows, int d, const float* gamma,
              const float* beta, void* h, int64_t ldh, bool h_bf16, float* mean, float* rstd);
int ln_bwd_cl(cudaStream_t st, bool pdl, const float* dh, const float* x, const float* mean, const float* rstd,
              const float* gamma, const float* dy, float* dx, int rows, int d, int rowblocks, float* dgp, float* dbp,
              void* op, bool op_bf16, float* opsum);
bool ln_cluster_ok(int d);
// out = op-dtype(src [* dropout(site, step)] * act'(z)), column partial sums per 16-row block into
// colsum + y*d (nullable).  act = 0 and no dropout: a plain cast (+ partials).
int colwise(cudaStream_t st, bool pdl, const float* src, int64_t lds, const float* z, int rows, int d, int act,
            uint32_t drop_thresh, float drop_scale, uint64_t seed, const uint32_t* step, uint32_t site,
            int64_t row_global0, void* out, int64_t ldo, bool out_bf16, float* colsum);
// Convert rows x d fp32 to op dtype (optionally also column partial sums of the fp32 values).
int convert_rows(cudaStream_t st, bool pdl, const float* x, int64_t ldx, int rows, int d, void* out, int64_t ldo,
                 bool out_bf16, float* colsum);
// dz = dy [* dropout] * act'(z) -> op dtype + column partial sum (fp32 path of EPI_ACT_BWD when no GEMM
// precedes it, i.e. the backward of a Linear layer).
int act_bwd_rows(cudaStream_t st, bool pdl, const float* dy, const float* z, int rows, int d, int act,
                 uint32_t drop_thresh, float drop_scale, uint64_t seed, const uint32_t* step, uint32_t site,
                 int64_t row_global0, void* out, int64_t ldo, bool out_bf16, float* colsum);
// y += a (rows x d fp32, same leading dimension d)
int add_rows(cudaStream_t st, bool pdl, float* y, const float* a, int64_t n);
// sum over m partial rows [m][d] in fixed order -> out[d] (=|+=)
int reduce_partials(cudaStream_t st, const float* part, int m, int d, float* out, bool accumulate);
struct RedItem {
  const float* part;  // [m][d] per-micro-batch column partials
  float* out;         // [d] gradient
  int d;
  int pad;
};
int reduce_partials_multi(cudaStream_t st, const RedItem* items, int n_items, int max_d, int m, bool accumulate);
// MSE loss + gradient: loss = sum (y-t)^2 / n_total; dy = 2 (y-t) / n_total. Deterministic.
int mse_loss_grad(cudaStream_t st, const float* y, const float* t, int64_t n, float* dy, double* loss_dev);
// SGD: master -= lr * grad; shadow (bf16, nullable) = bf16(master)
int sgd_step(cudaStream_t st, float* master, const float* grad, __nv_bfloat16* shadow, int64_t n, float lr);
// cast fp32 -> bf16
int cast_bf16(cudaStream_t st, const float* src, __nv_bfloat16* dst, int64_t n);
// deterministic on-device init: U(-bound, bound) or c + s N(0,1)-like (uniform-sum) from a hash
int init_uniform(cudaStream_t st, float* dst, int64_t n, float lo, float hi, uint64_t seed);
// BatchNorm (micro-batch statistics): forward y = act(gamma (x - mu) r + beta), stores mu, r and
// the pre-activation z; backward with the same statistics + column partials.
int bn_fwd(cudaStream_t st, const float* x, int rows, int d, const float* gamma, const float* beta, int act,
           float* y, float* z, float* mu, float* rstd, float* var_out);
int bn_bwd(cudaStream_t st, const float* dy, const float* x, const float* z, const float* mu, const float* rstd,
           const float* gamma, int rows, int d, int act, float* dx, float* dgamma_part, float* dbeta_part);
// commit BN running stats from per-micro-batch (rows_i, mean_i, var_i), fixed order (Chan et al.)
int bn_commit(cudaStream_t st, const float* mu_parts, const float* var_parts, const int* rows, int m, int d,
              float momentum, float* run_mean, float* run_var);

// ----------------------------------------------------------------------------- transport
// Copy n_rows x d elements from src (fp32) to a (possibly peer / IPC-mapped) dst in op dtype,
// then release-store `seq` into *flag (system scope) once every CTA has finished.
int push_rows(cudaStream_t st, const float* src, void* dst, bool dst_bf16, int64_t n, uint32_t* counter,
              uint32_t* flag, uint32_t seq);
int push_bytes(cudaStream_t st, const void* src, void* dst, int64_t nbytes, uint32_t* counter, uint32_t* flag,
               uint32_t seq);
// Release-store value into *flag (system scope) from a 1-thread kernel.
int signal_flag(cudaStream_t st, uint32_t* flag, uint32_t value);
int fill_flags(cudaStream_t st, uint32_t* p, int64_t n, uint32_t v);
// Test-only: busy a stream for ns nanoseconds.
int spin(cudaStream_t st, uint64_t ns);

}  // namespace tgp
