// Persistent forward-task kernel (task_fwd.cu) -- device descriptors and host entry points.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tgp {

// One RESMLP block of the task, micro-batch-specific pointers pre-offset to the micro-batch rows.
struct alignas(64) PLayer {
  CUtensorMap tmW1;  // W1 [H][d] bf16, K-major, box {64, 128}
  CUtensorMap tmW2;  // W2 [d][H] bf16, K-major, box {64, 128}
  CUtensorMap tmH;   // Hop [max_batch][d] bf16, box {64, 16}
  CUtensorMap tmG;   // Gop [max_batch][H] bf16, box {64, 16}
  const float* gamma;
  const float* beta;
  const float* b1;
  const float* b2;
  const float* x;       // block input rows [M][d] fp32
  float* y;             // block output rows [M][d] fp32
  float* a;             // pre-activation [M][H] fp32 (kept for the backward)
  __nv_bfloat16* hop;   // LN output rows (dW operand stash) [M][d]
  __nv_bfloat16* gop;   // activation rows (dW operand stash) [M][H]
  float* mean;          // LN statistics [M]
  float* rstd;
  uint32_t drop_thresh;
  float drop_scale;
  uint32_t site;
  uint32_t pad;
};

struct PTask {
  const PLayer* layers;  // device array [L]
  int L, d, H, M, r0;
  float* ws;             // split-K partial tiles: 2 x [max(d,H)/128][segmax][4][128] float4
  int64_t ws_stride;     // floats per parity half
  int segmax;
  float* stats;          // LN chunk statistics [4 d/128][4][2]
  unsigned* bar;         // grid barrier counter (reset before each launch)
  unsigned long long* dbg;  // diagnostics only (nullptr): [G][256][2] arrive / release %globaltimer
  uint64_t seed;
  const uint32_t* step;
};

int task_fwd_smem();
int task_fwd_max_phase_tiles();  // max k-blocks per CTA per GEMM phase (activation buffer size)
int task_fwd_launch(cudaStream_t st, const PTask& t, int grid);
int task_fwd_max_grid(int dev);

}  // namespace tgp
