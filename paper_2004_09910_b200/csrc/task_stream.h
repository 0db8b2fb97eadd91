// Persistent weight-streaming task kernel (task_stream.cu): device descriptors and host entry points.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tgp {

// One pre-LN residual MLP block of a partition (micro-batch independent).
struct alignas(64) SLayer {
  CUtensorMap w1k;   // W1 [H][d] bf16, K-major box {64, 128}  (forward GEMM1: out H, K d)
  CUtensorMap w2k;   // W2 [d][H] bf16, K-major box {64, 128}  (forward GEMM2: out d, K H)
  CUtensorMap w2m;   // W2 [d][H] bf16, MN-major box {64, 64}  (backward dG = dY W2: out H, K d)
  CUtensorMap w1m;   // W1 [H][d] bf16, MN-major box {64, 64}  (backward dH = dA W1: out d, K H)
  CUtensorMap gop;   // Gop  [max_batch][H] bf16, box {64, 16}  (activation = GEMM2 operand, dW2 stash)
  CUtensorMap daop;  // dAop [max_batch][H] bf16, box {64, 16}  (pre-act grad = dH operand, dW1 stash)
  CUtensorMap ygm;   // yg [16][d] bf16, box {64, 16}: forward GEMM1 operand gamma (y - mu~) (task scratch)
  CUtensorMap ucm;   // uc [32][d] bf16, box {64, 32}: backward dG operand [u | n] (task scratch)
  const float* gamma;
  const float* beta;
  const float* b1;
  const float* b2;
  const float* cfold;  // [H] c_h = sum_k gamma_k W1[h][k]  (fp32 over the bf16 weights)
  const float* efold;  // [H] e_h = sum_k beta_k W1[h][k] + b1[h]
  const float* c2fold; // [H] c2_h = sum_k W2[k][h]  (column sums of W2 [d][H])
  float* c2part;       // [d/256][H] stage-1 partial column sums
  __nv_bfloat16* yg;   // [16][d] GEMM1 operand scratch (the memory behind ygm)
  __nv_bfloat16* uc;   // [32][d] backward dG operand scratch (the memory behind ucm)
  const __nv_bfloat16* w1;  // W1 [H][d] (for the fold kernel)
  const __nv_bfloat16* w2;  // W2 [d][H]
  uint32_t drop_thresh;  // dropout after GELU: keep iff (philox word >> 8) >= thresh (0 = none)
  float drop_scale;
  uint32_t site;         // global layer index (Philox counter word 2)
  uint32_t pad;
};

// Per (micro-batch, block) pointers, pre-offset to the micro-batch's first row.
struct SMicro {
  const float* x;  // block input rows [M][d] fp32
  float* y;        // block output rows [M][d] fp32
  float* a;        // pre-activation [M][H] fp32 (written by F, read by B)
  float* mean;     // LN statistics [M] (written by F, read by B)
  float* rstd;
  __nv_bfloat16 *hop, *gop, *dyop, *daop;  // operand stash rows (row r0)
  float *pb, *pb2, *pg, *pbt;              // column-partial rows of this micro-batch: db1 [H], db2 [d], dgamma, dbeta [d]
};

struct STask {
  const SLayer* layers;  // [L]
  const SMicro* micro;   // [L], this micro-batch
  int L, d, H, M, r0, bwd;
  int nv;                // output slabs per cluster: 1 = full grid, 2 = half grid (a paired task, runtime.cu)
  const float* gy_top;   // backward: incoming output gradient rows [M][d]
  float* dx_bottom;      // backward: input gradient rows [M][d] (message source)
  float* gbuf0;          // backward: inter-block gradient ping-pong [16][d]
  float* gbuf1;
  float* stats;          // [L + 1][d / 32][16][2] LN row statistics per 32-feature chunk
  unsigned* cnt;         // dependency counters, one per 128-byte line: [(3L + 3) * 5 + 1 (done)], zero
                         // before the launch; the last CTA of the task zeroes them again
  uint64_t seed;
  const uint32_t* step;  // device optimizer step (dropout counter word 3)
  // diagnostics only (nullptr on the product path): per CTA and phase, %globaltimer stamps
  // [grid][2L][ST_DBG_SLOTS] (TGP_ST_DEBUG); they do not change any result
  unsigned long long* dbg;
  // compute fused with send: the task's boundary tensor --
  // forward: the last block's output rows, y_send; backward: the input-gradient rows, dx_bottom -- is
  // stored straight into the consuming partition's receive slab (same device, peer or CUDA-IPC
  // mapping), and the last CTA to finish release-stores *send_seq into send_flag at system scope
  // (every CTA first makes its stores visible with a system-scope acq_rel atomic).  nullptr: no send.
  float* y_send;
  uint32_t* send_flag;
  const uint32_t* send_seq;  // device copy of the call sequence number (graph replays read it)
  int keep;           // forward: 1 = store the block intermediates (pre-activation a, LN-output stash, block
                      // outputs, LN statistics); 0 = a checkpointed F, whose intermediates F' recomputes
                      // before B reads them (a checkpointed F keeps only the stage input) -- only
                      // the stage output is stored
  unsigned sleep_ns;  // back-off between dependency polls
  unsigned inflight;  // max weight tiles issued but not landed per CTA (0 = limited by the ring only)
};
constexpr int ST_DBG_SLOTS = 13;

int task_stream_smem();
int task_stream_counter_bytes(int L);
// Clusters of 4 the device can co-schedule (0 if the kernel cannot run there).  A task launched on
// `clusters` clusters with t.nv = 2 covers 2 x clusters output slabs (half grid: two such tasks run
// side by side).
int task_stream_max_clusters(int dev);
int task_stream_launch(cudaStream_t st, const STask& t, int clusters);
// c[h] = sum_k gamma[k] W1[h][k], e[h] = sum_k beta[k] W1[h][k] + b1[h] (fixed-order fp32 sums over
// the bf16 weights; one warp per row)
// for all L blocks of `layers` (device array) in one launch
int task_stream_fold(cudaStream_t st, const SLayer* layers, int L, int d, int H);

}  // namespace tgp
