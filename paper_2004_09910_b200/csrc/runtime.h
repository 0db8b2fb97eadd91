// Runtime data structures of a tgp context (host side).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tgp.h"
#include "kernels.h"
#include "plan.h"

namespace tgp {

// Device bump allocator (zero-initialised chunks).
struct Pool {
  int dev = 0;
  std::vector<void*> chunks;
  char* cur = nullptr;
  size_t left = 0;
  size_t used = 0, reserved = 0;  // bytes handed out / bytes cudaMalloc'ed (memory accounting)
  void* get(size_t bytes);
  void release();
};

struct Route {
  int id = -1;
  int stash_layer = -1, pop_layer = -1;
  int src = -1, dst = -1;  // 0-based partitions
  int width = 0;
};

// Pointers into a partition's peer-visible receive arena, valid in THIS process.
struct ArenaView {
  float* fwd_in = nullptr;            // [max_batch][d_in]  fp32: stage input (= checkpoint slot)
  float* grad_in = nullptr;           // [max_batch][d_out] fp32: incoming output gradient
  std::vector<void*> skip_in;         // per route with dst == part: [max_batch][w] op dtype
  std::vector<float*> dskip_in;       // per route with src == part (src != dst): [max_batch][w] fp32
  uint32_t* flags = nullptr;          // see flag_* helpers
};

struct ArenaLayout {
  size_t off_fwd = 0, off_grad = 0, off_flags = 0, bytes = 0;
  std::vector<size_t> off_skip, off_dskip;  // indexed by route id, SIZE_MAX when absent
};

struct LayerRT {
  tgp_layer L{};
  int idx = 0, part = 0, d_skip = 0;
  int nparam = 0, pidx0 = 0;
  int64_t poff[12] = {0}, pnum[12] = {0};
  // deferred-dW operand stash (global rows, op dtype, max_batch rows)
  void *Xop = nullptr, *Zop = nullptr, *Hop = nullptr, *Gop = nullptr, *dAop = nullptr, *dYop = nullptr;
  // per-micro-batch column partials [m][w] fp32
  float *pb = nullptr, *pb2 = nullptr, *pg = nullptr, *pbt = nullptr;
  // per activation slot (checkpoint-managed): layer output, pre-activation, LN stats
  std::vector<float*> out, z, mean, rstd;
  // GPT-2-shaped layers: block operand stash (global rows, bf16) -- QKV = [q|k|v] (attention input),
  // CTX = attention output (Wo operand), H2 = LN2 output, dQKV / dX1 = gradients at the QKV / Wo GEMMs
  void *QKVop = nullptr, *CTXop = nullptr, *H2op = nullptr, *dQKVop = nullptr, *dX1op = nullptr;
  float *pq = nullptr, *po = nullptr, *pg2 = nullptr, *pbt2 = nullptr;  // column partials (bqkv, bo, LN2)
  std::vector<float*> x1, mean2, rstd2, lse;  // per slot: attention-residual output, LN2 stats, log-sum-exp
  float* dE = nullptr;        // embedding: [max_batch][d] fp32 output gradient (after the dropout mask)
  int* emb_scratch = nullptr; // embedding: counting-sort scratch (3 vocab + max_batch ints)
  // BatchNorm per micro-batch statistics [m][d] and running stats [d]
  float *bn_mu = nullptr, *bn_var = nullptr, *bn_rstd = nullptr, *bn_rm = nullptr, *bn_rv = nullptr;
};

struct TaskGraph {
  cudaGraphExec_t exec = nullptr;
  int B = -1;
  int mode = 0;  // what else the captured kernels bake in (fused send on / off)
  int64_t kernels = 0;
};

struct Stage {
  int j = 0, dev = 0, l0 = 0, l1 = 0, d_in = 0, d_out = 0, maxw = 0;
  cudaStream_t comp = nullptr, cact = nullptr, cskip = nullptr;
  std::vector<cudaEvent_t> fdone, bdone;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_epoch = nullptr;  // timeline origin: the start of the last tgp_forward on this partition
  std::vector<cudaEvent_t> tr_ev;  // timeline events (pairs)
  Pool pool;
  void* arena = nullptr;
  size_t extra_bytes = 0;  // device allocations outside the pool (arena, descriptors, tables)
  size_t stash_bytes = 0;  // of pool.used: bf16 dW operand + skip stash (whole mini-batch, every mode)
  size_t slot_bytes = 0;   // of pool.used: per-activation-slot fp32 buffers (count set by the checkpoint mode)
  ArenaView self;
  float* out = nullptr;     // [max_batch][d_out] stage output (message source)
  float* dx_out = nullptr;  // [max_batch][d_in] input gradient (message source)
  std::vector<void*> skip_send;     // route id -> [max_batch][w] op dtype (src side, cross routes)
  std::vector<float*> dskip_send;   // route id -> [max_batch][w] fp32 (dst side, cross routes)
  std::vector<float*> dskip_local;  // route id -> [mb_cap][w] fp32 (src == dst)
  // Table 1 "no portals" ablation (option "ablate_portals"): tuple-threaded skip tensors held by
  // the partitions strictly between a route's stash and pop partitions
  std::vector<void*> relay_skip;    // route id -> [max_batch][w] op dtype (forward relay slot)
  std::vector<float*> relay_dskip;  // route id -> [max_batch][w] fp32 (backward relay slot)
  size_t relay_bytes = 0;
  std::vector<cudaEvent_t> abl_events;  // "ablate_copy_streams": events recorded on this stage's streams
  size_t abl_next = 0;
  float *master = nullptr, *grad = nullptr;
  __nv_bfloat16* shadow = nullptr;
  int64_t n_elems = 0;
  float* dh = nullptr;
  float* partials = nullptr;  // all column-partial buffers of the partition (contiguous)
  size_t partial_floats = 0;
  float* gbuf[2] = {nullptr, nullptr};
  float* tbuf = nullptr;   // [mb_cap][maxw] fp32 scratch (attention backward dqkv)
  float* attnD = nullptr;  // [mb_cap][max heads] fp32 scratch (attention backward rowsum(dO o O))
  float* attn_part = nullptr;  // [mb_cap][max heads][4][66] fp32: split-row forward partials
  double* ce_part = nullptr;  // [max_batch + 1] cross-entropy row losses (last partition)
  uint32_t* counters = nullptr;  // [8]
  double* loss_buf = nullptr;
  int* bn_rows = nullptr;
  uint32_t* dstep = nullptr;  // device copy of the optimizer step (dropout counter)
  // persistent weight-streaming task kernel (task_stream.cu): F / F' / B of all-RESMLP partitions
  bool st_ok = false;
  int st_clusters = 0;
  void* st_layers = nullptr;  // device SLayer[L]
  void* st_micro = nullptr;   // device SMicro[m][L]
  int st_micro_B = -1;
  float* st_stats = nullptr;
  unsigned* st_cnt = nullptr;
  float* st_fold = nullptr;   // per block [3][H]: c = W1 gamma, e = W1 beta + b1 (R3), c2 = 1^T W2 (R4)
  void* st_yg = nullptr;      // [16][d] bf16: GEMM1 operand gamma (y - mu~) of the current block
  void* st_uc = nullptr;      // [32][d] bf16: backward dG operand [u | n]
  float* st_c2part = nullptr; // [L][d/256][H] partial column sums of W2
  bool fold_dirty = true;     // weights / LN parameters changed since st_fold was computed
  // F' / B pairing (option "pair_recompute"): F'_{i-1,j} runs on lane 1 (comp2) beside B_{i,j} on
  // lane 0, both on a half grid (st_half clusters, two output slabs each); lane 1 has its own
  // counters / statistics scratch.  Checkpointed micro-batches alternate two scratch slots.
  bool pair_ok = false;
  bool pair_layer = false;  // pairing with per-layer kernels (no stream kernel): F' on comp2, full-size grids
  int st_half = 0;
  cudaStream_t comp2 = nullptr;
  unsigned* st_cnt2 = nullptr;
  float* st_stats2 = nullptr;
  cudaEvent_t ev_pair = nullptr;      // recorded on comp before a paired B: lane 1 waits for it
  cudaEvent_t ev_join[3] = {nullptr, nullptr, nullptr};  // async calls: comp2 / cact / cskip joined into comp
  cudaEvent_t ev_done = nullptr;
  int bn_rows_B = -1;                 // mini-batch size bn_rows was last written for      // async calls: the partition's share of the call is done (on comp)
  std::vector<cudaEvent_t> rdone;     // per micro-batch: its hoisted F' finished (recorded on comp2)
  std::vector<char> hoisted;          // per micro-batch: F' already issued on lane 1 in this call
  std::vector<TaskGraph> gR2, gB2;    // paired-task graphs (half grid)
  std::vector<TaskGraph> gR;          // F' graphs when F sends fused (F and F' differ then)
  uint32_t* dseq = nullptr;           // device copy of the call sequence number (fused-send flags)
  unsigned long long* st_dbg = nullptr;  // diagnostics (TGP_ST_DEBUG): [grid][2L][ST_DBG_SLOTS]
  cudaEvent_t* prof_ev = nullptr;  // tgp_profile_layers: per-layer boundary events (forward, then backward)
  void* red_items = nullptr;  // device RedItem[n_red]: column-partial -> gradient reductions of W_j
  int n_red = 0, red_maxd = 0;
  std::vector<TaskGraph> gF, gB;
  TaskGraph gW;
  bool grads_fresh = true;
  // W_j fused with SGD (tgp_backward_step; gemm_dw_sgd.cu): the bf16 RESMLP weight matrices go through
  // wgrad_sgd, every other parameter through sgd_segments
  std::vector<int> ws_layers;       // RESMLP layers whose W1 / W2 are fused
  std::vector<WsGemm> ws_host;      // descriptors for batch ws_B (operand maps have K = B rows)
  WsGemm* ws_dev = nullptr;         // device copy
  int ws_B = -1;
  int64_t* seg_dev = nullptr;       // non-fused parameter segments {offset, length}
  int n_seg = 0;
  int64_t seg_maxlen = 0;
  float* dlr = nullptr;             // device learning rate of the fused step
  TaskGraph gWs;
};

struct TraceRec {
  int part, stream, kind, i;
  cudaEvent_t a, b;
};

}  // namespace tgp

struct tgp_ctx {
  std::vector<tgp::LayerRT> layers;
  std::vector<tgp::Route> routes;
  std::vector<int> balance, devices, part_l0;
  int n = 0, m = 0, ckpt = 1, max_batch = 0, mb_cap = 0, nslots = 1;
  int unit = 1;  // rows per sample (seq for the GPT-2-shaped kinds): micro-batches split samples
  int pb = 1;  // 16-row blocks per micro-batch: column-partial buffers are [m * pb][width]
  bool bf16 = false;
  uint64_t seed = 0;
  uint32_t step = 0;
  uint32_t seq = 0;
  int state = 0;  // 0 created, 1 forwarded, 2 backwarded
  bool fuse_sgd = false;  // inside tgp_backward_step: W_j applies SGD with lr_host (no gradient stored)
  float lr_host = 0.0f;
  int cur_B = 0;
  std::vector<tgp::Stage*> local;       // by partition (nullptr if remote)
  std::vector<tgp::ArenaView> view;     // by partition
  std::vector<tgp::ArenaLayout> layout; // by partition
  std::vector<void*> imported;          // IPC mappings to close
  std::vector<tgp::Rec> fwd_recs, bwd_recs, w_recs;
  std::vector<tgp::Rec> issue_log;
  std::vector<int> slot_of;  // 1-based micro-batch -> slot
  int64_t kernels = 0;
  // options
  bool use_graphs = true, use_pdl = true, trace = false, poison = false, prefetch = false;
  bool l2pf = false;
  bool stream = true;
  bool pair = true;           // F'_{i-1,j} beside B_{i,j} on half grids (option "pair_recompute")
  bool fused_send = true;     // stream-kernel tasks store their boundary tensor into the consumer's slab (option "fused_send")
  bool pair_slots = false;    // checkpointed micro-batches alternate two scratch slots (set at create)
  bool gemm_wide = true;      // per-micro-batch GEMMs with >= 256 rows through the persistent gemm_wide kernel (option "gemm_wide")
  bool dw_persistent = true;  // deferred dW through the persistent gemm_dw kernel (option "dw_persistent")
  unsigned st_inflight = 0;  // stream kernel: max weight tiles in flight per CTA (0 = ring-limited; "stream_inflight")
  unsigned st_sleep_ns = 32;  // stream kernel: back-off between dependency polls (option "stream_poll_ns")
  // Table 1 ablation toggles: 0 / false = the torchgpipe design
  uint64_t order_seed = 0;   // "ablate_order": backward tasks in a seeded random topological order
  bool relay = false;        // "ablate_portals": skip tensors tuple-threaded through every partition
  bool abl_streams = false;  // "ablate_copy_streams": copies on the compute streams, two-way synchronised
  int64_t copy_bytes = 0, copy_msgs = 0;  // messages this process pushed since creation
  int splitk = 0, skip_wait_part = -1;
  uint64_t delay_push_ns = 0;
  int drop_push_part = -1;    // test only: partition whose forward messages are never sent (watchdog test)
  int transport = 2;          // 0 = SM push kernel + release flag, 1 = copy engine + stream write, 2 = auto by size (option "transport")
  int64_t watchdog_ms = 60000;  // bound on a call's device wait (option "watchdog_ms"); 0 = wait forever
  bool failed = false;        // a watchdog timeout left the context unusable (every call: TGP_E_STATE)
  bool wedged = false;        // ... and the device did not drain: destroy must not block (leaks)
  bool can_flush = false;
  std::vector<tgp::TraceRec> trace_recs;
  std::vector<int64_t> timeline;
  std::vector<std::pair<int, int>> route_parts_1b;
  bool connected = true;
  // asynchronous stream-ordered calls (tgp_*_async): the caller's stream while such a
  // call is being issued, and the event its work is ordered after (created on the stream's device)
  bool dead_stash = true;  // stream-kernel F of a checkpointed micro-batch skips its dead intermediates (option "dead_stash")
  bool nvtx = true;  // NVTX ranges per call and per issued task (option "nvtx")
  bool async_call = false;
  cudaStream_t ustream = nullptr;
  cudaEvent_t ev_user = nullptr;
  int ev_user_dev = -1;
  int n_params = 0;
  std::vector<int> param_layer, param_local;
};
