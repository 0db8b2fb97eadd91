// tcgen05 / TMA bf16 GEMM for sm_100a with fused epilogues (the dense layers of F_{i,j}, F'_{i,j},
// B_{i,j} and the deferred weight-gradient task W_j; PAPER.md Eq. F_{i,j} P:52-55, Eq. B_{i,j}
// P:58-68, g^j = sum_i g_i^j P:70).
//
//   D[m][n] = sum_k A[m][k] * B[n][k]      (fp32 accumulate in TMEM)
//
// "Swap-AB": for the per-micro-batch GEMMs the MMA M side (128 TMEM lanes) is the output-feature
// dimension (the weight rows) and the MMA N side is the micro-batch rows (16 at C2), because
// tcgen05 needs M >= 64 while a micro-batch has only 16 rows.  A therefore streams the weight
// matrix (the HBM-bound operand) and B the small activation tile.  Split-K over a thread-block
// cluster keeps >= 128 SMs streaming weights; the partial tiles are reduced through DSMEM in a
// FIXED rank order (deterministic: F' reproduces F bit-exactly, reading Z21).
//
// Operand majors (smem 128-byte swizzle, TMA box inner extent 64 bf16 = 128 B):
//   A K-major  (forward: W [out][in])         box {64 k, 128 m}
//   A MN-major (dX: W^T; dW: dY^T)            two boxes {64 m, 64 k}
//   B K-major  (activations [rows][in])       box {64 k, BN n}
//   B MN-major (dW: X [rows][in])             BN/64 boxes {64 n, 64 k}
#pragma once
#include "common.cuh"

namespace tgp {

enum EpiMode : int {
  EPI_LINEAR_FWD = 0,  // z = acc + bias; [zbuf = z]; y = act(z) [* dropout]; [out0 = y (f32)]; [op = y]
  EPI_RESID_FWD = 1,   // y = acc + bias + res; out0 = y (f32); [op = y]
  EPI_ACT_BWD = 2,     // d = acc [* dropout] * act'(zbuf); op = d; colsum[f] = sum_rows d
  EPI_STORE = 3,       // out0[r][f] = acc (f < split_f) else out1[r][f - split_f] = acc
  EPI_DW = 4,          // dw[m][n] (=|+=) acc      (deferred weight gradient, row-major [M][N])
};

struct EpiParams {
  int mode;
  int act;              // 0 none, 1 relu, 2 gelu
  int op_bf16;          // operand-dtype output is bf16 (1) or f32 (0)
  float* out0;
  int64_t ld0;
  float* out1;
  int64_t ld1;
  int split_f;
  void* op;
  int64_t ld_op;
  const float* bias;
  const float* res;
  int64_t ld_res;
  float* zbuf;
  int64_t ldz;
  float* colsum;
  // dropout (Philox, global element index = (row_global0 + r) * drop_width + f)
  uint32_t drop_thresh;  // 0 = no dropout
  float drop_scale;      // 1 / (1 - p)
  uint32_t site;
  const uint32_t* step;  // device pointer to the optimizer step counter (dropout key)
  uint64_t seed;
  int64_t row_global0;
  int64_t drop_width;
  // dW
  float* dw;
  int64_t ldw;
  int accumulate;
};

struct GemmParams {
  int M, N, K;        // D is M x N; K multiple of 64
  int n0;             // coordinate offset of B's n index inside its tensor (micro-batch row start)
  int k_seg;          // k >= k_seg reads B from the second tensor map (concat-merge), else K
  int kb_per_split;   // k-blocks handled by each cluster rank (split-K)
  int a_is_weight;    // A does not depend on the previous kernel (prefetch before griddep wait)
  // weight tiles beyond the smem pipeline depth are prefetched into L2 before the griddep wait
  // (HBM keeps streaming this kernel's weights while the previous kernel drains its epilogue)
  int a_l2pf;
  // L2 prefetch of the NEXT GEMM's weight matrix (the task's GEMM sequence is static): every CTA
  // prefetches its 1/grid share after issuing its own loads, so HBM keeps streaming across the
  // kernel boundary (epilogue / launch / prologue of the next GEMM).  pf_bytes = 0: none.
  const void* pf_ptr;
  int64_t pf_bytes;
  EpiParams epi;
};

}  // namespace tgp
