/* tgp.h -- C ABI of the B200-native GPipe training library (arXiv 2004.09910, torchgpipe).
 *
 * The hot path (BASELINE.json north_star): synchronous GPipe pipeline-parallel training of a
 * sequence of layers cut into n partitions, one partition per GPU; each mini-batch is cut into
 * m micro-batches run on the deterministic clock-cycle schedule (§3.2.1 Alg. 1,
 * m+n-1 forward clocks) and the mirrored backward, with checkpointed micro-batches
 * recomputed (F'_{i,j}) right before B_{i,j} under the restored counter-based
 * RNG, stage-to-stage activations / gradients / skip tensors moved by copy kernels on dedicated
 * copy streams, weight gradients g^j = sum_i g_i^j computed by one
 * deferred GEMM per weight, and a fused plain-SGD step.
 *
 * Conventions
 *  - Every call returns tgp_status (0 = TGP_OK).  On failure the reason is available from
 *    tgp_last_error() (thread-local, valid until the next failing call on the thread).
 *  - Partitions are numbered j = 0..n_parts-1 in this ABI (the paper's j = 1..n).
 *  - Matrices are row-major [rows][features], fp32, device memory unless stated "host".
 *  - Calls are blocking: they return after all device work THIS PROCESS issued for the call has
 *    completed (host timing around a call is valid; no hidden asynchronous state) -- except the
 *    *_async variants below, which are stream-ordered and return without a host wait.
 *  - A context is not thread-safe: one host thread drives it.
 *  - No CPU fallback: a process without a usable sm_100 GPU gets TGP_E_CUDA / TGP_E_UNSUPPORTED
 *    from tgp_create.  Pure host entry points (tgp_balance, tgp_split, tgp_schedule) need no GPU.
 */
#ifndef TGP_H
#define TGP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TGP_OK = 0,
  TGP_E_INVALID = -1,     /* bad argument, shape mismatch, bad balance / route        */
  TGP_E_STATE = -2,       /* call out of order (backward before forward, ...)         */
  TGP_E_CUDA = -3,        /* a CUDA runtime / driver call failed                      */
  TGP_E_NOMEM = -4,       /* device allocation failed                                 */
  TGP_E_UNSUPPORTED = -5, /* shape / device / feature not supported by this build     */
  TGP_E_TIMEOUT = -6      /* a cross-partition handshake did not complete in time (the
                             watchdog, option "watchdog_ms"): the call returns instead of
                             hanging; the context is failed (results garbage; every later
                             call except tgp_destroy / introspection -> TGP_E_STATE).  The
                             local receive flags are released to drain the device; if it
                             does not drain within 2 s, tgp_destroy leaks the device memory
                             to process exit rather than block                           */
} tgp_status;

/* Checkpoint policy (P:105, P:108, P:305 footnote; SURVEY reading Z4):
 * ALWAYS every micro-batch recomputed; EXCEPT_LAST all but i = m (the paper's default);
 * NEVER no recomputation (all activations kept). */
typedef enum { TGP_CKPT_ALWAYS = 0, TGP_CKPT_EXCEPT_LAST = 1, TGP_CKPT_NEVER = 2 } tgp_checkpoint;

/* Compute mode: FP32 = fp32 everything, SIMT FFMA GEMMs, no TF32 (reading Z16);
 * BF16 = bf16 GEMM operands on tcgen05 tensor cores with fp32 accumulation; fp32 residual stream,
 * LN statistics, messages, gradients and master weights (reading Z14). */
typedef enum { TGP_FP32 = 0, TGP_BF16 = 1 } tgp_dtype;

/* Layer kinds.  Parameters of layer l, in this order (canonical parameter index order):
 *  TGP_LINEAR    y = act(x W^T + b) [dropout]          W [d_out][d_in], b [d_out]
 *  TGP_RESMLP    y = x + W2 drop(act(W1 LN(x) + b1)) + b2, pre-LayerNorm (eps 1e-5), d_out == d_in
 *                gamma [d_in], beta [d_in], W1 [d_hidden][d_in], b1 [d_hidden], W2 [d_out][d_hidden], b2 [d_out]
 *  TGP_MERGE     y = act([x || s] W^T + b) [dropout], s = skip tensor popped from route pop_route
 *                (concat-merge of a long skip connection)   W [d_out][d_in + d_skip], b [d_out]
 *  TGP_BATCHNORM y = act(gamma (x - mu_i) / sqrt(var_i + 1e-5) + beta), statistics of micro-batch i
 *                (P:56 footnote); running stats committed once per forward call from the whole
 *                mini-batch (momentum 0.1, unbiased variance).   gamma [d], beta [d]   (FP32 mode only)
 *  TGP_LAYERNORM y = gamma (x - mu) / sqrt(var + 1e-5) + beta over the features of each row (biased
 *                variance), d_out == d_in, act none, no dropout.   gamma [d], beta [d]
 *  TGP_DROPOUT   y = x * keep / (1 - p), p = `dropout`, keep from Philox at site = layer index (the
 *                same counters as every other dropout site), d_out == d_in, act none; no parameters.
 *                (a partition is any sequence of layers; P:105 / P:212: the recompute
 *                regenerates the same mask from the restored RNG state.)
 *
 * GPT-2-shaped kinds (C5; BASELINE.json configs[4]; bf16 mode only).  Rows are TOKENS:
 * a sample is a sequence of `seq` tokens, B counts tokens and must be a multiple of seq, and the
 * micro-batches split the SEQUENCES (reading Z7 applied to samples), so attention never crosses one.
 *  TGP_EMBED       y = wte[id] + wpe[row % seq] [dropout, site = layer]; d_in = 1: column 0 of the
 *                  input holds the token id as an exactly representable fp32 integer.  Must be layer 0.
 *                  wte [vocab][d_out], wpe [seq][d_out]
 *  TGP_TRANSFORMER pre-LN GPT-2 block, d = 64 n_heads, MLP d_hidden with GELU, causal attention:
 *                  x1 = x + drop(Attn(LN1(x)) Wo^T + bo), y = x1 + drop(GELU(LN2(x1) W1^T + b1) W2^T + b2),
 *                  dropout (p = `dropout`) on the attention probabilities (site layer + 1<<16) and on
 *                  both residual branches (sites layer + 2<<16, + 3<<16).
 *                  gamma1 [d], beta1 [d], Wqkv [3d][d], bqkv [3d], Wo [d][d], bo [d], gamma2 [d], beta2 [d],
 *                  W1 [d_hidden][d], b1 [d_hidden], W2 [d][d_hidden], b2 [d]
 *  TGP_LMHEAD      logits y = LN(x) W^T (no bias), d_out = vocab.   gamma [d], beta [d], W [vocab][d]
 * (oracle/model.py states the same formulas; PAPER.md P:25 names GPT-2 as a GPipe workload.)
 */
typedef enum {
  TGP_LINEAR = 0,
  TGP_RESMLP = 1,
  TGP_MERGE = 2,
  TGP_BATCHNORM = 3,
  TGP_EMBED = 4,
  TGP_TRANSFORMER = 5,
  TGP_LMHEAD = 6,
  TGP_LAYERNORM = 7,
  TGP_DROPOUT = 8
} tgp_kind;
typedef enum { TGP_ACT_NONE = 0, TGP_ACT_RELU = 1, TGP_ACT_GELU = 2 } tgp_act;

typedef struct {
  int32_t kind;        /* tgp_kind */
  int32_t d_in, d_out; /* feature widths (TGP_MERGE: d_in = width of x; d_skip comes from the route) */
  int32_t d_hidden;    /* TGP_RESMLP hidden width, else 0 */
  int32_t act;         /* tgp_act */
  float dropout;       /* dropout probability after the activation (0 = none); Philox4x32-10 keyed by
                          (seed, step), counter = (global element index >> 2, layer index, step) */
  int32_t stash_route; /* route id whose skip tensor is this layer's OUTPUT, or -1 (@skippable stash) */
  int32_t pop_route;   /* route id consumed at this layer's INPUT (TGP_MERGE), or -1 (pop) */
  int32_t n_heads;     /* TGP_TRANSFORMER: attention heads (head dim 64), else 0 */
  int32_t seq;         /* TGP_EMBED / TGP_TRANSFORMER: tokens per sample (multiple of 64), else 0 */
  int32_t vocab;       /* TGP_EMBED / TGP_LMHEAD: vocabulary size (multiple of 128 for the LM head), else 0 */
} tgp_layer;

typedef struct tgp_ctx tgp_ctx;

/* ------------------------------------------------------------------ pure host entry points */

/* Partition balancer ("partition whose pairwise resource discrepancy is small"; reading Z8):
 * contiguous split of n_layers costs into n_parts non-empty blocks minimising the maximum block
 * sum, ties broken by the lexicographically smallest boundary vector.  balance_out[n_parts]. */
tgp_status tgp_balance(const double* layer_cost, int32_t n_layers, int32_t n_parts, int32_t* balance_out);

/* Size-based per-layer cost for tgp_balance (§4.2.2 P:312-317 "parameters consume 8 bytes
 * each for itself and its gradients"; SPEC profile_size): bytes_out[l] = 8 x (parameter count of
 * layer l) + rows x d_out x 4 (the fp32 activation output of a `rows`-row sample).  A MERGE layer's
 * skip width is taken from the layer that stashes its route.  Pure host; rows >= 1. */
tgp_status tgp_profile_size(const tgp_layer* layers, int32_t n_layers, int32_t rows, double* bytes_out);

/* Micro-batch split (reading Z7): sizes_out[m] = ceil(B/m) for the first B mod m
 * micro-batches, floor(B/m) after.  TGP_E_INVALID unless 1 <= m <= B. */
tgp_status tgp_split(int32_t B, int32_t m, int32_t* sizes_out);

/* The clock-cycle schedule the runtime issues (Alg. 1 + mirrored backward + deferred dW), as
 * 8-int32 records (phase, clock, kind, i, j, src, dst, route) with i, j 1-based:
 * phase 0 forward / 1 backward / 2 weight-gradient; kind 0 F, 1 F' (recompute), 2 B, 3 COPY_F,
 * 4 COPY_B, 5 SKIP_F, 6 SKIP_B, 7 W.  routes = n_routes (src, dst) partition pairs, 1-based.
 * rec may be NULL to query the count; *n_rec receives the record count. */
tgp_status tgp_schedule(int32_t m, int32_t n, tgp_checkpoint ckpt, const int32_t* routes, int32_t n_routes,
                        int32_t* rec, int64_t cap, int64_t* n_rec);

/* The same records under the Table 1 ablation toggles that
 * tgp_set_option's "ablate_portals" / "ablate_order" select: relay != 0 tuple-threads every skip
 * tensor through each partition between stash and pop (SKIP_F hop j-1 -> j issued with F_{i,j},
 * SKIP_B hop j+1 -> j with B_{i,j}, for every j the route spans) instead of one portal copy;
 * order_seed != 0 replaces the mirrored backward clocks by a seeded random topological order of
 * the backward tasks (each B_{i,j} with its COPY_B / SKIP_B messages and F'_{i,j} before it; the
 * clock field is then the issue step), emulating an autograd engine without Fork/Join edges.
 * relay = 0 and order_seed = 0 give exactly tgp_schedule's records. */
tgp_status tgp_schedule_ablation(int32_t m, int32_t n, tgp_checkpoint ckpt, const int32_t* routes, int32_t n_routes,
                                 int32_t relay, uint64_t order_seed, int32_t* rec, int64_t cap, int64_t* n_rec);

/* ------------------------------------------------------------------ context */

/* Create a pipeline.  layers[n_layers] as above; balance[n_parts] layers per partition (NULL:
 * tgp_balance on analytic per-layer costs); chunks = m; devices[n_parts]: CUDA ordinal hosting
 * partition j in THIS process (repeats allowed: several partitions may share a GPU), or -1 when
 * partition j is hosted by another process (multi-process pipeline: exchange tgp_ipc_export /
 * tgp_ipc_import blobs, then tgp_connect).  max_batch bounds B of later calls; seed keys the
 * dropout RNG.  All device memory (parameters, gradients, activation slots, receive buffers,
 * stash) is allocated here; nothing is allocated on the step path.
 * Errors: TGP_E_INVALID (chunks < 1, chunks > max_batch, sum(balance) != n_layers, a partition
 * with 0 layers, n_parts > n_layers, shape mismatch between consecutive layers or along a route,
 * pop before stash), TGP_E_UNSUPPORTED (bf16 widths not multiples of 128, BATCHNORM in bf16
 * mode, no peer access between two local devices), TGP_E_NOMEM, TGP_E_CUDA. */
tgp_status tgp_create(const tgp_layer* layers, int32_t n_layers, const int32_t* balance, int32_t n_parts,
                      int32_t chunks, tgp_checkpoint ckpt, const int32_t* devices, int32_t max_batch,
                      tgp_dtype dtype, uint64_t seed, tgp_ctx** out);
void tgp_destroy(tgp_ctx* ctx);

/* Multi-process pipelines: each local partition exports one opaque blob (its peer-visible
 * receive arena as a CUDA IPC handle).  Every process imports the blobs of the remote partitions
 * it exchanges data with (neighbours and skip-route peers; importing all is fine), then calls
 * tgp_connect.  tgp_ipc_export: buf may be NULL to query *len. */
tgp_status tgp_ipc_export(tgp_ctx* ctx, int32_t part, void* buf, int64_t cap, int64_t* len);
tgp_status tgp_ipc_import(tgp_ctx* ctx, int32_t part, const void* buf, int64_t len);
tgp_status tgp_connect(tgp_ctx* ctx);

/* ------------------------------------------------------------------ training step */

/* Forward pass F_{i,j} for all micro-batches on the clock-cycle schedule.
 * x: [B][d_in] fp32 on devices[0] (required iff partition 0 is local, else NULL);
 * y: [B][d_out] fp32 on devices[n-1] (required iff partition n-1 is local, else NULL).
 * A forward discards the state of a previous forward that was not followed by backward. */
tgp_status tgp_forward(tgp_ctx* ctx, const float* x, int32_t B, float* y);

/* Loss on the gathered output -- library helper on the last partition's device:
 * loss = sum (y - t)^2 / (B d_out), dy = 2 (y - t) / (B d_out).  loss_out: host, may be NULL. */
tgp_status tgp_mse_loss_grad(tgp_ctx* ctx, const float* y, const float* target, int32_t B, float* dy,
                             double* loss_out);

/* Token cross-entropy on the gathered logits (C5; loss "on the gathered output"):
 * loss = mean_r (logsumexp(y_r) - y_r[target_r]), dy = (softmax(y_r) - onehot(target_r)) / B.
 * y, dy: [B][vocab] fp32, target: [B] int32 token ids, all device memory on devices[n-1];
 * loss_out: host, may be NULL.  Deterministic (fixed-order reductions). */
tgp_status tgp_ce_loss_grad(tgp_ctx* ctx, const float* y, const int32_t* target, int32_t B, float* dy,
                            double* loss_out);

/* Backward pass: mirrored clock-cycle, F'_{i,j} before B_{i,j} for checkpointed micro-batches,
 * then the deferred weight-gradient task W_j.  dy: [B][d_out] fp32 on devices[n-1] (iff local);
 * dx: [B][d_in] fp32 on devices[0] or NULL.  Gradients accumulate over forward/backward pairs
 * until tgp_step.  TGP_E_STATE if no forward preceded it. */
tgp_status tgp_backward(tgp_ctx* ctx, const float* dy, float* dx);

/* Plain SGD on every local partition: theta <- theta - lr g (fp32 master; bf16 shadow refreshed),
 * then gradients are logically reset.  Advances the dropout step counter. */
tgp_status tgp_step(tgp_ctx* ctx, float lr);

/* tgp_backward followed by tgp_step(lr), with the SGD update fused into the deferred weight-gradient
 * task W_j (g^j = sum_i g_i^j; plain SGD).  In bf16 mode the W1 / W2
 * matrices of RESMLP blocks (d, H multiples of 128) are updated straight from the dW accumulator
 * (theta <- theta - lr g with the same fp32 fma as tgp_step, so results are bitwise identical to
 * tgp_backward + tgp_step); their gradients are NOT stored (tgp_get_grad returns stale values for
 * them).  Every other parameter, and fp32 mode, takes the unfused path.  Arguments as tgp_backward.
 * TGP_E_STATE if gradients of an earlier tgp_backward are still pending (call tgp_step first). */
tgp_status tgp_backward_step(tgp_ctx* ctx, const float* dy, float* dx, float lr);

/* ------------------------------------------------------------------ asynchronous, stream-ordered calls
 * (PAPER.md P:133 and Alg. 1: the host only issues tasks, the devices wait on
 * one another).  Each call below issues exactly the device work of its blocking twin (same arguments,
 * same results bit for bit) and returns as soon as it is issued:
 *  - ordering: the work starts after everything queued on `stream` before the call (so inputs may
 *    still be in production on `stream`), and `stream` waits for the call's work on every local
 *    partition (so work queued on `stream` afterwards sees the results).  `stream` is a cudaStream_t
 *    (NULL = the legacy default stream of the current device), cast to void* so this header needs no
 *    CUDA include; it may live on any device;
 *  - buffers: x, y, dy, dx, target, loss_dev must stay allocated and unmodified (outputs: unread)
 *    until `stream` reaches the call's completion;
 *  - errors: argument and state errors are reported at issue time exactly as by the blocking twin;
 *    device-side failures and a lost cross-partition message surface at the next tgp_sync (or the next
 *    blocking call) -- TGP_E_CUDA / TGP_E_TIMEOUT with the watchdog semantics above;
 *  - tracing (tgp_set_trace): timeline records of async calls become readable after tgp_sync. */
tgp_status tgp_forward_async(tgp_ctx* ctx, const float* x, int32_t B, float* y, void* stream);
/* loss_dev: DEVICE pointer to one double (the MSE loss), on the last partition's device, may be NULL */
tgp_status tgp_mse_loss_grad_async(tgp_ctx* ctx, const float* y, const float* target, int32_t B, float* dy,
                                   double* loss_dev, void* stream);
tgp_status tgp_backward_async(tgp_ctx* ctx, const float* dy, float* dx, void* stream);
tgp_status tgp_backward_step_async(tgp_ctx* ctx, const float* dy, float* dx, float lr, void* stream);
tgp_status tgp_step_async(tgp_ctx* ctx, float lr, void* stream);
/* Bounded host wait for every call issued so far on this context (TGP_E_TIMEOUT past "watchdog_ms"). */
tgp_status tgp_sync(tgp_ctx* ctx);

/* ------------------------------------------------------------------ parameters / introspection */

/* Parameters in canonical order over ALL layers (see tgp_kind).  Only parameters of local
 * partitions can be read / written (TGP_E_INVALID otherwise).  host buffers, fp32. */
tgp_status tgp_num_params(tgp_ctx* ctx, int32_t* n);
tgp_status tgp_param_info(tgp_ctx* ctx, int32_t idx, int32_t* layer, int32_t* part, int64_t* numel);
tgp_status tgp_set_param(tgp_ctx* ctx, int32_t idx, const float* host);
tgp_status tgp_get_param(tgp_ctx* ctx, int32_t idx, float* host);
tgp_status tgp_get_grad(tgp_ctx* ctx, int32_t idx, float* host);
/* Deterministic on-device initialisation of every local parameter (bench helper; W, b ~
 * U(+-1/sqrt(fan_in)), gamma = 1, beta = 0). */
tgp_status tgp_init_params(tgp_ctx* ctx, uint64_t seed);
/* BatchNorm running statistics of layer `layer` (host [d] each). */
tgp_status tgp_get_bn_running(tgp_ctx* ctx, int32_t layer, float* mean, float* var);

/* The records this process actually issued in its last forward+backward, in issue order (same
 * encoding as tgp_schedule; a multi-process context logs only records whose actor is local). */
tgp_status tgp_get_issue_log(tgp_ctx* ctx, int32_t* rec, int64_t cap, int64_t* n_rec);

/* Task timeline (enabled by tgp_set_trace(ctx, 1)): per executed compute task and copy, 6 int64
 * (part, stream, kind, i, t0_ns, t1_ns), times from CUDA events relative to the start of the last
 * tgp_forward on that partition's device, so a forward and the backward after it share one time axis
 * (not comparable across devices).  stream: 0 compute, 1 activation copies, 2 skip copies, 3 the
 * second compute lane (F' paired beside B). */
tgp_status tgp_set_trace(tgp_ctx* ctx, int32_t on);
tgp_status tgp_get_timeline(tgp_ctx* ctx, int64_t* rec, int64_t cap, int64_t* n_rec);

/* Number of kernels this process launched (or replayed through CUDA graphs) since creation. */
tgp_status tgp_kernel_count(tgp_ctx* ctx, int64_t* n);

/* Runtime options (TGP_E_INVALID for an unknown name):
 *  "graphs"   1 = capture each task's kernels into a CUDA graph and replay it (default 1)
 *  "pdl"      programmatic dependent launch between the kernels of a task (default 1)
 *  "splitk"   split-K cluster size of the weight-streaming GEMMs, 0 = automatic (default 0)
 *  "prefetch" L2 prefetch of the next GEMM's weights by the previous GEMM (default 0)
 *  "l2pf"     each weight-streaming GEMM prefetches its weight tiles beyond the shared-memory
 *             pipeline depth into L2 before its grid-dependency wait (default 0)
 *  "stream"   run F / F' / B of all-RESMLP partitions with <= 16-row micro-batches as ONE persistent
 *             weight-streaming kernel per task (task_stream.cu; default 1 where eligible)
 *  "dw_persistent" deferred weight gradients through the persistent 128x128-tile dW kernel (default 1)
 *  "stream_poll_ns" back-off of the stream kernel's dependency polling loops, ns (default 32)
 *  "stream_inflight" max weight tiles (16 KB) a stream-kernel CTA keeps in flight from HBM
 *                   (0 = as many as its ring has free stages; values >= the ring depth are ignored)
 *  "gemm_wide" per-micro-batch GEMMs with >= 256 rows through the persistent gemm_wide kernel
 *             (default 1; 0 = the one-tile-per-CTA GEMM)
 *  "attn_tc"  PROCESS-WIDE: 1 = tcgen05 attention forward where seq % 128 == 0, 0 = mma.sync,
 *             -1 = the TGP_ATTN_TC environment default (off)
 *  "dead_stash"  1 (default): the stream-kernel F task of a checkpointed micro-batch stores only its
 *                 output (F' recomputes the intermediates before B reads them); 0: it stores them too
 *  "nvtx"        1 (default): NVTX ranges per tgp_forward / tgp_backward call and per issued task
 *                 (named after its schedule record, e.g. "F i=3 j=2"); 0: none
 *  "watchdog_ms" bound on the host wait for a call's device work (forward / backward), ms
 *             (default 60000; 0 = unbounded): past it the call returns TGP_E_TIMEOUT (PAPER.md P:133,
 *             host issue with device-side waits: a lost message would otherwise hang the caller)
 *  "transport" stage-boundary messages (COPY_F / COPY_B): 0 = SM push kernel
 *             writing the consumer's receive slab + system-scope release store of the flag,
 *             1 = copy engine (cudaMemcpyAsync peer/D2D) + cuStreamWriteValue32 of the flag,
 *             2 = by message size: copy engine from 16 KiB up (the B200 crossover of
 *             tgp_bench_transport; default).  Skip tensors always use the push kernel (bf16
 *             conversion).  Same bytes either way: results are bitwise identical.
 *  "fused_send" 1 (default) = with transport 2, a persistent stream-kernel task stores its boundary
 *             tensor (F: the last block's output, B: the input gradient) straight into the
 *             neighbour partition's receive slab and release-stores the flag itself at system
 *             scope: compute fused with send, no copy kernel.  Off
 *             under the ablations and the transport negative controls.  Bitwise identical results.
 *  "pair_recompute" 1 (default) = F'_{i-1,j} runs on a second lane beside B_{i,j} (F' depends only
 *             on the stage input): both stream-kernel tasks on half grids, or -- partitions on
 *             the per-layer kernels -- full-size kernels sharing the SMs (bf16, not under the
 *             ablate_portals / ablate_copy_streams toggles); 0 = in place.  Results are bitwise equal.
 * Table 1 ablation toggles (results are bitwise those of the default -- only the
 * issue order and the copy path change).  Need every partition in this process, and not between
 * forward and backward (TGP_E_UNSUPPORTED / TGP_E_STATE):
 *  "ablate_order"        value = seed != 0: backward tasks in tgp_schedule_ablation's random
 *                        topological order instead of the Fork/Join order (0 = off)
 *  "ablate_copy_streams" 1 = copies on the producer's compute stream, waiting for all work issued
 *                        on the consumer's compute stream and waited on by it (default-stream copies)
 *  "ablate_portals"      1 = skip tensors relayed through every partition in between (extra relay
 *                        slots, allocated here and counted by tgp_memory; 0 frees them)
 * Test-only negative controls (never used on the product path):
 *  "test_poison"        fill the forward receive slabs with NaN before each forward call
 *  "test_skip_wait"     drop the receive waits of partition `value` (-1 = none)
 *  "test_delay_push_us" delay every push on its copy stream by `value` microseconds
 *  "test_drop_push"     partition `value` never sends its forward messages (watchdog test; -1 = off) */
tgp_status tgp_set_option(tgp_ctx* ctx, const char* name, int64_t value);

const char* tgp_last_error(void);

/* Measurement helper (bench.py's roofline line): times the dominant kernel of the step -- the
 * forward weight-streaming GEMM of every RESMLP/LINEAR layer of local partition `part`, launched
 * exactly as F_{i,j} launches it for micro-batch 1 of a batch of B rows -- cycling through the
 * partition's layers (cold weights) `reps` rounds, with CUDA events on the partition's compute
 * stream.  *ms: average ms per launch; *bytes: average algorithmic bytes per launch (weights +
 * activation operand + epilogue reads/writes); *launches: launches timed. */
tgp_status tgp_bench_dominant_gemm(tgp_ctx* ctx, int32_t part, int32_t B, int32_t reps, double* ms, double* bytes,
                                   int64_t* launches);

/* Static memory plan of local partition `part`: *used = bytes the plan uses (parameters, gradients,
 * operand stash, activation slots, receive arena, workspaces), *reserved = bytes allocated from the
 * device for it, *params = fp32 master + fp32 gradient (+ bf16 shadow) bytes.  Any pointer may be
 * NULL.  All of it is allocated in tgp_create; nothing on the step path. */
/* Messages (activation, gradient and skip copies) this process pushed since creation: *bytes
 * payload bytes, *messages count.  Either pointer may be NULL. */
tgp_status tgp_copy_stats(tgp_ctx* ctx, int64_t* bytes, int64_t* messages);

tgp_status tgp_memory(tgp_ctx* ctx, int32_t part, int64_t* used, int64_t* reserved, int64_t* params);

/* What the checkpoint mode changes in that plan (R1).  *stash =
 * bytes of the bf16 dW-operand and skip stash: rows of the WHOLE mini-batch, kept from F until W_j,
 * allocated in every checkpoint mode (deferred dW) -- checkpointing does NOT shrink it.
 * *slots = bytes of the per-activation-slot fp32 buffers (layer outputs, pre-activations, LayerNorm
 * statistics); *n_slots = slot count: the shared scratch slot(s) + one per non-checkpointed
 * micro-batch, i.e. m + 1 (never), 2 (except_last), 1 (always) -- one scratch slot more when F' / B
 * pairing is possible (stream-kernel shapes, >= 2 checkpointed micro-batches: alternating scratch
 * slots).  Only the slots are what checkpointing saves here.  Both
 * byte counts are included in tgp_memory's *used.  Any pointer may be NULL. */
tgp_status tgp_memory_breakdown(tgp_ctx* ctx, int32_t part, int64_t* stash, int64_t* slots, int32_t* n_slots);

/* Profile-based balancing input: per-layer device time in ms of a
 * forward + backward of one micro-batch (B / chunks rows) of local partition `part`, median of
 * `reps`, measured with CUDA events between the layers on the per-layer kernel path.
 * ms_per_layer: host array of the partition's layer count.  Feed it to tgp_balance. */
tgp_status tgp_profile_layers(tgp_ctx* ctx, int32_t part, int32_t B, int32_t reps, double* ms_per_layer);

/* Transport micro-benchmark (PAPER.md P:198-203 copy streams): messages of
 * `bytes` (multiple of 16) fp32 from a device buffer on dev_src to a receive buffer on dev_dst
 * (dev_src == dev_dst allowed; peer access is enabled for different devices) through the pipeline's
 * transports: mode 0 = SM push kernel + release flag, mode 1 = copy engine + stream-written flag.
 * *us_stream: device µs per message of `reps` back-to-back messages, each waited for by a consumer
 * stream; *us_pingpong: µs per message + acknowledgement round trip.  Buffers are allocated and freed
 * here.  TGP_E_UNSUPPORTED without peer access, TGP_E_INVALID for bad sizes. */
tgp_status tgp_bench_transport(int32_t dev_src, int32_t dev_dst, int64_t bytes, int32_t mode, int32_t reps,
                               double* us_stream, double* us_pingpong);

/* *on = 1 iff local partition `part` runs its F / F' / B tasks as the persistent weight-streaming
 * task kernel (eligible shape and option "stream" on); then tgp_bench_dominant_gemm times that
 * kernel (F_{1,j} launches: *bytes = its algorithmic bytes per SURVEY 8(d) -- the bf16 weights of
 * every block once plus the fp32 stage input read and stage output written; intermediates are not
 * counted) instead of the per-layer forward GEMM. */
tgp_status tgp_stream_enabled(tgp_ctx* ctx, int32_t part, int32_t* on);

/* Diagnostics of the persistent weight-streaming task kernel (only when the process runs with
 * TGP_ST_DEBUG set): per CTA and GEMM phase of the last task launched on partition `part`, 10
 * %globaltimer stamps (B operand issued, first / last weight tile issued, B landed, last MMA, TMEM
 * ready, partials received, outputs signalled, row statistics ready), as [grid][2L][10] uint64.
 * out may be NULL to query *n. */
tgp_status tgp_debug_stream_read(tgp_ctx* ctx, int32_t part, uint64_t* out, int64_t cap, int64_t* n);

/* ------------------------------------------------------------------ kernel-level test entry */

/* D[m][n] = sum_k A[m][k] B[n][k] on the tcgen05 path (bf16 in, fp32 out).
 * a_mn: A stored [K][M] (else [M][K]); b_mn: B stored [K][N] (else [N][K]).
 * D layout: b_mn == 1 -> row-major [M][N] (the weight-gradient orientation); b_mn == 0 -> [N][M]
 * (activation orientation: row n, feature m -- the swap-AB skinny path).  a_mn = b_mn = 1 with
 * splits = -1 (-2) runs the persistent deferred-dW kernel storing (accumulating) into D instead
 * (M, N multiples of 128).  splits: split-K
 * cluster size (0 = auto).  Device pointers; stream = cudaStream_t or NULL; synchronous.  Used by
 * the kernel unit tests and micro-benchmarks. */
tgp_status tgp_test_gemm_bf16(const void* A, const void* B, float* D, int32_t M, int32_t N, int32_t K,
                              int32_t a_mn, int32_t b_mn, int32_t splits, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TGP_H */
