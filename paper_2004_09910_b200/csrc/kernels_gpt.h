// Launchers of the GPT-2-shaped stage kernels (kernels_attn.cu).  Return 0 or a negative tgp_status.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/tgp.h"

namespace tgp {

// Causal multi-head attention forward over whole sequences (head dim 64, seq % 64 == 0).
//   qkv [rows][3d] bf16 (q | k | v, head h = columns h*64 .. h*64+63 of each third), rows % seq == 0,
//   row_global0 = global token row of row 0 (dropout counters: flat index in [n_seq, nh, seq, seq]).
//   ctx [rows][d] bf16 = softmax(q k^T / 8, causal) [dropout] v;  lse [rows][nh] fp32 (log2 domain).
//   part_buf: rows * nh * 4 * 66 floats of scratch for the split-row partials (nullable: no split).
int attn_fwd(cudaStream_t st, const void* qkv, int rows, int d, int nh, int seq, int64_t row_global0,
             uint32_t thresh, float dscale, uint64_t seed, const uint32_t* step, uint32_t site, void* ctx, float* lse,
             float* part_buf);
constexpr int ATTN_PART_FLOATS = 4 * 66;  // per (row, head)
// Backward: dO [rows][d] fp32 -> dqkv [rows][3d] fp32.  Dbuf: rows*nh floats of scratch.
int attn_bwd(cudaStream_t st, const void* qkv, const void* ctx, const float* dO, const float* lse, float* Dbuf,
             int rows, int d, int nh, int seq, int64_t row_global0, uint32_t thresh, float dscale, uint64_t seed,
             const uint32_t* step, uint32_t site, float* dqkv);
bool attn_shape_ok(int rows, int d, int nh, int seq);
// Select the tcgen05 forward for seq % 128 == 0 (1), the mma.sync one (0), or the TGP_ATTN_TC
// environment default (-1).  Process-wide (option "attn_tc").
void attn_set_tc(int on);
// y[r] = wte[id_r] + wpe[(row_global0 + r) % seq] [dropout]; ids = token ids stored as fp32 (stride ldi)
int embed_fwd(cudaStream_t st, const float* ids, int64_t ldi, int rows, const float* wte, const float* wpe, int d,
              int seq, int64_t row_global0, uint32_t thresh, float dscale, uint64_t seed, const uint32_t* step,
              uint32_t site, float* y);
// Deterministic deferred embedding gradients over all `rows` tokens: dwte[v] (=|+=) sum of dE rows
// with id v (ascending row order), dwpe[p] (=|+=) sum of dE rows at position p.  scratch: 3V + rows ints.
int embed_wgrad(cudaStream_t st, const float* ids, int64_t ldi, int rows, const float* dE, int d, int V, int seq,
                int* scratch, float* dwte, float* dwpe, bool accumulate);
// Token cross-entropy: loss = mean_r (lse(y_r) - y_r[t_r]); dy = (softmax(y_r) - onehot(t_r)) / T.
// part: T doubles of scratch; loss_dev: 1 double.
int ce_loss_grad(cudaStream_t st, const float* y, int64_t ldy, const int* tgt, int T, int V, float* dy,
                 double* part, double* loss_dev);

}  // namespace tgp
