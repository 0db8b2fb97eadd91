// tgp runtime: context creation, buffers, peer arenas (CUDA IPC), clock-cycle issue of tasks,
// copy-stream transport with flag handshakes, task executors (F / F' / B / W), SGD, ABI entry
// points.  PAPER.md references: Alg. 1 P:148-167 (clock cycle), P:103-108 (device order,
// checkpointing), P:198-203 (copy streams), P:212 (checkpoint slot shared with the receive
// buffer), P:242-245 (portals: one direct copy per skip tensor), P:70 (g = sum_i g_i), P:307 (SGD).
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>

#include "host.h"
#include "runtime.h"
#include "kernels_gpt.h"
#include "task_stream.h"

using namespace tgp;

// ============================================================================ errors / driver
namespace tgp {
static thread_local std::string g_err;
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}
const char* get_error() { return g_err.c_str(); }

const Driver* driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess && fn)
      d.tensorMapEncodeTiled = (decltype(d.tensorMapEncodeTiled))fn;
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess && fn)
      d.streamWaitValue32 = (decltype(d.streamWaitValue32))fn;
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) == cudaSuccess && fn)
      d.streamWriteValue32 = (decltype(d.streamWriteValue32))fn;
    d.ok = d.tensorMapEncodeTiled && d.streamWaitValue32 && d.streamWriteValue32;
  });
  if (!d.ok) {
    set_error("CUDA driver entry points unavailable (no GPU driver?)");
    return nullptr;
  }
  return &d;
}

void* Pool::get(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes == 0) bytes = 256;
  if (bytes > left) {
    const size_t cs = std::max(bytes, size_t(256) << 20);
    void* p = nullptr;
    if (cudaMalloc(&p, cs) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, cs) != cudaSuccess) return nullptr;
    chunks.push_back(p);
    reserved += cs;
    cur = (char*)p;
    left = cs;
  }
  void* r = cur;
  cur += bytes;
  left -= bytes;
  used += bytes;
  return r;
}
void Pool::release() {
  for (void* p : chunks) cudaFree(p);
  chunks.clear();
  cur = nullptr;
  left = 0;
}
}  // namespace tgp

// ============================================================================ helpers
static int op_size(const tgp_ctx* c) { return c->bf16 ? 2 : 4; }
static inline uint32_t* flag_fwd(const ArenaView& v, int i) { return v.flags + (i - 1); }
static inline uint32_t* flag_grad(const tgp_ctx* c, const ArenaView& v, int i) { return v.flags + c->m + (i - 1); }
static inline uint32_t* flag_skip(const tgp_ctx* c, const ArenaView& v, int r, int i) {
  return v.flags + 2 * c->m + r * c->m + (i - 1);
}
static inline uint32_t* flag_dskip(const tgp_ctx* c, const ArenaView& v, int r, int i) {
  return v.flags + 2 * c->m + (int)c->routes.size() * c->m + r * c->m + (i - 1);
}
static inline uint32_t* flag_done(const tgp_ctx* c, const ArenaView& v, int from_part) {
  return v.flags + 2 * c->m + 2 * (int)c->routes.size() * c->m + from_part;
}
static int n_flags(const tgp_ctx* c) { return 2 * c->m + 2 * (int)c->routes.size() * c->m + c->n; }

static int part_d_in(const tgp_ctx* c, int j) { return c->layers[c->part_l0[j]].L.d_in; }
static int part_d_out(const tgp_ctx* c, int j) { return c->layers[c->part_l0[j + 1] - 1].L.d_out; }

static ArenaLayout make_layout(const tgp_ctx* c, int j) {
  ArenaLayout a;
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t r = off;
    off += (b + 255) & ~size_t(255);
    return r;
  };
  a.off_fwd = take((size_t)c->max_batch * part_d_in(c, j) * 4);
  a.off_grad = take((size_t)c->max_batch * part_d_out(c, j) * 4);
  a.off_skip.assign(c->routes.size(), SIZE_MAX);
  a.off_dskip.assign(c->routes.size(), SIZE_MAX);
  for (const Route& r : c->routes) {
    if (r.dst == j) a.off_skip[r.id] = take((size_t)c->max_batch * r.width * op_size(c));
    if (r.src == j && r.dst != j) a.off_dskip[r.id] = take((size_t)c->max_batch * r.width * 4);
  }
  a.off_flags = take((size_t)n_flags(c) * 4);
  a.bytes = off;
  return a;
}

static ArenaView make_view(const tgp_ctx* c, int j, char* base) {
  const ArenaLayout& a = c->layout[j];
  ArenaView v;
  v.fwd_in = (float*)(base + a.off_fwd);
  v.grad_in = (float*)(base + a.off_grad);
  v.skip_in.assign(c->routes.size(), nullptr);
  v.dskip_in.assign(c->routes.size(), nullptr);
  for (size_t r = 0; r < c->routes.size(); ++r) {
    if (a.off_skip[r] != SIZE_MAX) v.skip_in[r] = base + a.off_skip[r];
    if (a.off_dskip[r] != SIZE_MAX) v.dskip_in[r] = (float*)(base + a.off_dskip[r]);
  }
  v.flags = (uint32_t*)(base + a.off_flags);
  return v;
}

// dropout threshold: keep iff (word >> 8) >= ceil(p * 2^24)  <=>  (word >> 8) * 2^-24 >= p
static uint32_t drop_thresh(float p) {
  if (p <= 0.0f) return 0u;
  const double t = std::ceil((double)p * 16777216.0);
  return (uint32_t)std::max(1.0, std::min(t, 16777216.0));
}

// ============================================================================ GEMM dispatch
namespace {
struct Opnd {
  const void* p;
  int64_t rows, cols, ld;
};
}  // namespace

// D[m][n] = sum_k A(m,k) B(n,k);  a_mn: A memory [K][M], else [M][K];  b_mn: B memory [K][N] else [rows][K]
struct Prefetch {
  const void* p = nullptr;
  int64_t bytes = 0;
};

static int run_gemm(tgp_ctx* c, Stage& s, bool pdl, Opnd A, bool a_mn, Opnd B0, const Opnd* B1, bool b_mn, int M,
                    int N, int K, int n0, int k_seg, bool a_weight, const EpiParams& e, Prefetch pf = Prefetch{}) {
  GemmParams p{};
  p.pf_ptr = c->prefetch ? pf.p : nullptr;
  p.pf_bytes = c->prefetch ? (pf.bytes & ~int64_t(15)) : 0;
  p.M = M;
  p.N = N;
  p.K = K;
  p.n0 = n0;
  p.k_seg = B1 ? k_seg : K;
  p.a_is_weight = a_weight ? 1 : 0;
  p.a_l2pf = a_weight && c->l2pf ? 1 : 0;
  p.epi = e;
  c->kernels += 1;
  if (c->bf16) {
    TcMat a{A.p, A.rows, A.cols, A.ld}, b0{B0.p, B0.rows, B0.cols, B0.ld};
    TcMat b1 = B1 ? TcMat{B1->p, B1->rows, B1->cols, B1->ld} : b0;
    const int Kp = (K + 63) / 64 * 64;
    p.K = Kp;
    if (B1 && k_seg % 64) {
      set_error("merge: d_in=%d must be a multiple of 64 in bf16 mode", k_seg);
      return TGP_E_UNSUPPORTED;
    }
    if (e.mode == EPI_DW && a_mn && b_mn && !B1 && M % 64 == 0 && N % 64 == 0 && c->dw_persistent)
      return gemm_dw(s.comp, A.p, A.ld, B0.p, B0.ld, e.dw, e.ldw, M, N, K, e.accumulate != 0);
    if (e.mode != EPI_DW && !B1 && !b_mn && N >= 256 && c->gemm_wide) return gemm_wide(s.comp, a, a_mn, b0, p);
    return gemm_tc(s.comp, pdl && c->use_pdl, a, a_mn, b0, B1 ? &b1 : nullptr, b_mn, p, c->splitk);
  }
  SimtOperand sa = a_mn ? SimtOperand{(const float*)A.p, 1, A.ld} : SimtOperand{(const float*)A.p, A.ld, 1};
  SimtOperand sb0 = b_mn ? SimtOperand{(const float*)B0.p, 1, B0.ld} : SimtOperand{(const float*)B0.p, B0.ld, 1};
  SimtOperand sb1{nullptr, 0, 0};
  if (B1) sb1 = b_mn ? SimtOperand{(const float*)B1->p, 1, B1->ld} : SimtOperand{(const float*)B1->p, B1->ld, 1};
  return gemm_simt(s.comp, pdl && c->use_pdl, sa, sb0, sb1, p);
}

static const void* wparam(tgp_ctx* c, Stage& s, const LayerRT& L, int k) {
  if (c->bf16) return s.shadow + L.poff[k];
  return s.master + L.poff[k];
}
static float* mparam(Stage& s, const LayerRT& L, int k) { return s.master + L.poff[k]; }
static float* gparam(Stage& s, const LayerRT& L, int k) { return s.grad + L.poff[k]; }

static char* opptr(tgp_ctx* c, void* base, int64_t row, int64_t w) {
  return (char*)base + (size_t)row * w * op_size(c);
}

// skip operand destination for route r at the stash side (global row r0)
static void* stash_dst(tgp_ctx* c, Stage& s, int r, int64_t r0) {
  const Route& R = c->routes[r];
  void* base = (R.dst == s.j) ? s.self.skip_in[r] : s.skip_send[r];
  return opptr(c, base, r0, R.width);
}

// The first weight matrix a layer's forward / backward GEMM sequence streams (for the L2 prefetch
// issued by the GEMM before it; the sequence of GEMMs inside a task is static).
static Prefetch first_fwd_weight(tgp_ctx* c, Stage& s, const LayerRT& L) {
  if (!c->bf16) return Prefetch{};
  if (L.L.kind == TGP_RESMLP) return Prefetch{wparam(c, s, L, 2), L.pnum[2] * 2};
  if (L.L.kind == TGP_LINEAR || L.L.kind == TGP_MERGE) return Prefetch{wparam(c, s, L, 0), L.pnum[0] * 2};
  return Prefetch{};
}
static Prefetch first_bwd_weight(tgp_ctx* c, Stage& s, const LayerRT& L) {
  if (!c->bf16) return Prefetch{};
  if (L.L.kind == TGP_RESMLP) return Prefetch{wparam(c, s, L, 4), L.pnum[4] * 2};
  if (L.L.kind == TGP_LINEAR || L.L.kind == TGP_MERGE) return Prefetch{wparam(c, s, L, 0), L.pnum[0] * 2};
  return Prefetch{};
}
static Prefetch next_fwd(tgp_ctx* c, Stage& s, int l) {  // after the last GEMM of layer l (forward order)
  return first_fwd_weight(c, s, c->layers[l + 1 < s.l1 ? l + 1 : s.l0]);
}
static Prefetch next_bwd(tgp_ctx* c, Stage& s, int l) {  // after the last GEMM of layer l (backward order)
  return first_bwd_weight(c, s, c->layers[l - 1 >= s.l0 ? l - 1 : s.l1 - 1]);
}

// ============================================================================ task executors
static void micro_rows(const tgp_ctx* c, int B, int i, int* r0, int* M);

// Persistent weight-streaming task kernel (task_stream.cu): layer descriptors (tensor maps of the
// weights and operand stashes) and per-(micro-batch, block) pointers, (re)built when B changes.
static int st_build_desc(tgp_ctx* c, Stage& s, int B) {
  const int L = s.l1 - s.l0;
  std::vector<SLayer> hl((size_t)L);
  for (int l = s.l0; l < s.l1; ++l) {
    LayerRT& Ly = c->layers[l];
    const int d = Ly.L.d_in, H = Ly.L.d_hidden;
    SLayer& P = hl[(size_t)(l - s.l0)];
    memset(&P, 0, sizeof(P));
    const void* w1 = wparam(c, s, Ly, 2);
    const void* w2 = wparam(c, s, Ly, 4);
    if (!make_map(&P.w1k, TcMat{w1, H, d, d}, 64, 128) || !make_map(&P.w2k, TcMat{w2, d, H, H}, 64, 128) ||
        !make_map(&P.w2m, TcMat{w2, d, H, H}, 64, 64) || !make_map(&P.w1m, TcMat{w1, H, d, d}, 64, 64) ||
        !make_map(&P.gop, TcMat{Ly.Gop, c->max_batch, H, H}, 64, 16) ||
        !make_map(&P.daop, TcMat{Ly.dAop, c->max_batch, H, H}, 64, 16) ||
        !make_map(&P.ygm, TcMat{s.st_yg, 16, d, d}, 64, 16) || !make_map(&P.ucm, TcMat{s.st_uc, 32, d, d}, 64, 32))
      return TGP_E_CUDA;
    P.yg = (__nv_bfloat16*)s.st_yg;
    P.uc = (__nv_bfloat16*)s.st_uc;
    P.gamma = mparam(s, Ly, 0);
    P.beta = mparam(s, Ly, 1);
    P.b1 = mparam(s, Ly, 3);
    P.b2 = mparam(s, Ly, 5);
    P.cfold = s.st_fold + (size_t)(l - s.l0) * 3 * H;
    P.efold = P.cfold + H;
    P.c2fold = P.cfold + 2 * H;
    P.c2part = s.st_c2part + (size_t)(l - s.l0) * (d / 256) * H;
    P.w2 = (const __nv_bfloat16*)w2;
    P.w1 = (const __nv_bfloat16*)w1;
    P.drop_thresh = drop_thresh(Ly.L.dropout);
    P.drop_scale = Ly.L.dropout > 0 ? 1.0f / (1.0f - Ly.L.dropout) : 1.0f;
    P.site = (uint32_t)l;
  }
  std::vector<SMicro> hm((size_t)c->m * L);
  for (int i = 1; i <= c->m; ++i) {
    int r0 = 0, M = 0;
    micro_rows(c, B, i, &r0, &M);
    const int slot = c->slot_of[i];
    for (int l = s.l0; l < s.l1; ++l) {
      LayerRT& Ly = c->layers[l];
      const int d = Ly.L.d_in, H = Ly.L.d_hidden;
      SMicro& P = hm[(size_t)(i - 1) * L + (l - s.l0)];
      P.x = (l == s.l0) ? s.self.fwd_in + (size_t)r0 * d : c->layers[l - 1].out[slot];
      P.y = (l == s.l1 - 1) ? s.out + (size_t)r0 * d : Ly.out[slot];
      P.a = Ly.z[slot];
      P.mean = Ly.mean[slot];
      P.rstd = Ly.rstd[slot];
      P.hop = (__nv_bfloat16*)opptr(c, Ly.Hop, r0, d);
      P.gop = (__nv_bfloat16*)opptr(c, Ly.Gop, r0, H);
      P.dyop = (__nv_bfloat16*)opptr(c, Ly.dYop, r0, d);
      P.daop = (__nv_bfloat16*)opptr(c, Ly.dAop, r0, H);
      const size_t po = (size_t)(i - 1) * c->pb;
      P.pb = Ly.pb + po * H;
      P.pb2 = Ly.pb2 + po * d;
      P.pg = Ly.pg + po * d;
      P.pbt = Ly.pbt + po * d;
    }
  }
  if (s.comp2) TGP_CUDA_TRY(cudaStreamSynchronize(s.comp2));  // a lane-1 task may read the old descriptors
  TGP_CUDA_TRY(cudaMemcpyAsync(s.st_layers, hl.data(), hl.size() * sizeof(SLayer), cudaMemcpyHostToDevice, s.comp));
  TGP_CUDA_TRY(cudaMemcpyAsync(s.st_micro, hm.data(), hm.size() * sizeof(SMicro), cudaMemcpyHostToDevice, s.comp));
  TGP_CUDA_TRY(cudaStreamSynchronize(s.comp));
  s.st_micro_B = B;
  return 0;
}

static bool use_stream(const tgp_ctx* c, const Stage& s, int M) { return s.st_ok && c->stream && M <= 16; }

// Compute fused with send: a stream-kernel task writes its boundary tensor straight
// into the neighbour's receive slab and release-stores the flag itself, so the copy record has no
// kernel.  Off under the Table 1 ablations and the transport negative controls (they act on the copy).
static bool send_ok(const tgp_ctx* c) {
  return c->fused_send && !c->abl_streams && !c->relay && c->order_seed == 0 && c->drop_push_part < 0 &&
         c->delay_push_ns == 0 && c->skip_wait_part < 0 && c->transport == 2;
}
static bool fuse_fwd(const tgp_ctx* c, const Stage& s, int M) {
  return send_ok(c) && s.j + 1 < c->n && use_stream(c, s, M) && c->view[s.j + 1].fwd_in;
}
static bool fuse_bwd(const tgp_ctx* c, const Stage& s, int M) {
  return send_ok(c) && s.j > 0 && use_stream(c, s, M) && c->view[s.j - 1].grad_in;
}

// LayerNorm folded into GEMM1 of the stream kernel: recompute c = W1 gamma, e = W1 beta + b1 of
// every block after the weights or LN parameters changed (SGD step, set / init).
static int st_refold(tgp_ctx* c, Stage& s, int B) {
  if (!s.st_ok || !s.fold_dirty) return 0;
  if (s.st_micro_B != B) TGP_TRY(st_build_desc(c, s, B));
  const LayerRT& L0 = c->layers[s.l0];
  TGP_TRY(task_stream_fold(s.comp, (const SLayer*)s.st_layers, s.l1 - s.l0, L0.L.d_in, L0.L.d_hidden));
  c->kernels++;
  s.fold_dirty = false;
  return 0;
}

// lane: 0 = full grid on comp; 1 = half grid on comp (a paired B); 2 = half grid on comp2 with the
// lane-1 counters / statistics (a paired F', beside the lane-1 B)
static int exec_task_stream(tgp_ctx* c, Stage& s, int i, int r0, int M, bool bwd, int lane = 0, float* send_to = nullptr,
                            uint32_t* send_flag = nullptr, bool keep = true) {
  const LayerRT& L0 = c->layers[s.l0];
  STask t{};
  t.L = s.l1 - s.l0;
  t.layers = (const SLayer*)s.st_layers;
  t.micro = (const SMicro*)s.st_micro + (size_t)(i - 1) * t.L;
  t.d = L0.L.d_in;
  t.H = L0.L.d_hidden;
  t.M = M;
  t.r0 = r0;
  t.bwd = bwd ? 1 : 0;
  t.nv = lane ? 2 : 1;
  t.gy_top = s.self.grad_in + (size_t)r0 * s.d_out;
  t.dx_bottom = s.dx_out + (size_t)r0 * s.d_in;
  // fused send (f3): forward -> the last block writes the consumer's receive slab; backward -> the
  // input gradient goes to the producer partition's gradient slab
  if (send_to && bwd) t.dx_bottom = send_to;
  t.y_send = (send_to && !bwd) ? send_to : nullptr;
  t.send_flag = send_to ? send_flag : nullptr;
  t.send_seq = s.dseq;
  t.gbuf0 = s.gbuf[0];
  t.gbuf1 = s.gbuf[1];
  t.stats = lane == 2 ? s.st_stats2 : s.st_stats;
  t.cnt = lane == 2 ? s.st_cnt2 : s.st_cnt;
  t.seed = c->seed;
  t.step = s.dstep;
  t.keep = keep ? 1 : 0;
  t.sleep_ns = c->st_sleep_ns;
  t.inflight = c->st_inflight;
  // diagnostics: per-CTA, per-phase %globaltimer stamps of the full-grid tasks (TGP_ST_DEBUG=1) or of the
  // paired backward task on lane 1 (TGP_ST_DEBUG=2; half grid, the two units of a phase share a record)
  const char* dbg_env = getenv("TGP_ST_DEBUG");
  if (dbg_env && ((lane == 0 && atoi(dbg_env) != 2) || (lane == 1 && atoi(dbg_env) == 2))) {
    const size_t nd = (size_t)s.st_clusters * 4 * 2 * t.L * ST_DBG_SLOTS;
    if (!s.st_dbg) {
      TGP_CUDA_TRY(cudaMalloc(&s.st_dbg, nd * 8));
      TGP_CUDA_TRY(cudaMemset(s.st_dbg, 0, nd * 8));
    }
    t.dbg = s.st_dbg;
  }
  c->kernels += 1;  // the task kernel (it resets its dependency counters itself)
  return task_stream_launch(lane == 2 ? s.comp2 : s.comp, t, lane ? s.st_half : s.st_clusters);
}

// F_{i,j} (and F'_{i,j}: identical kernels and launch configuration -> bitwise identical output).
// keep = false: a checkpointed F, whose backward-only intermediates (pre-activations) F' recomputes
// LayerNorm backward dx = dy + LN_bwd(dh) (dy nullable) with the per-16-row column partials.
static int ln_bwd_any(tgp_ctx* c, Stage& s, bool pdl, const float* dh, const float* x, const float* mean,
                      const float* rstd, const float* gamma, const float* dy, float* dx, int M, int d, float* pg,
                      float* pbt) {
  if (ln_cluster_ok(d)) {
    TGP_TRY(ln_bwd_cl(s.comp, pdl, dh, x, mean, rstd, gamma, dy, dx, M, d, c->pb, pg, pbt, nullptr, c->bf16, nullptr));
    c->kernels++;
  } else {
    TGP_TRY(ln_bwd(s.comp, pdl, dh, x, mean, rstd, gamma, dy, dx, M, d, pg, pbt));
    c->kernels += 2;
  }
  return 0;
}

static int exec_forward(tgp_ctx* c, Stage& s, int i, int r0, int M, bool keep = true) {
  if (use_stream(c, s, M)) return exec_task_stream(c, s, i, r0, M, false, 0, nullptr, nullptr, keep);
  const int slot = c->slot_of[i];
  float* x = s.self.fwd_in + (size_t)r0 * s.d_in;
  bool first_kernel = true;
  auto pdl = [&]() {
    bool r = !first_kernel;
    first_kernel = false;
    return r;
  };
  for (int l = s.l0; l < s.l1; ++l) {
    LayerRT& L = c->layers[l];
    const int din = L.L.d_in, dout = L.L.d_out;
    float* y = (l == s.l1 - 1) ? s.out + (size_t)r0 * dout : L.out[slot];
    EpiParams e{};
    e.op_bf16 = c->bf16 ? 1 : 0;
    e.seed = c->seed;
    e.step = s.dstep;
    e.site = (uint32_t)l;
    e.row_global0 = r0;
    switch (L.L.kind) {
      case TGP_LINEAR:
      case TGP_MERGE: {
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, x, din, nullptr, M, din, 0, 0u, 1.0f, c->seed, s.dstep,
                        (uint32_t)l, r0, opptr(c, L.Xop, r0, din), din, c->bf16, nullptr));
        c->kernels++;
        e.mode = EPI_LINEAR_FWD;
        e.act = L.L.act;
        e.bias = mparam(s, L, 1);
        e.zbuf = (L.L.act != TGP_ACT_NONE && keep) ? L.z[slot] : nullptr;  // pre-activation: backward only
        e.ldz = dout;
        e.out0 = y;
        e.ld0 = dout;
        e.drop_thresh = drop_thresh(L.L.dropout);
        e.drop_scale = L.L.dropout > 0 ? 1.0f / (1.0f - L.L.dropout) : 1.0f;
        e.drop_width = dout;
        if (L.L.stash_route >= 0) {
          e.op = stash_dst(c, s, L.L.stash_route, r0);
          e.ld_op = dout;
        }
        const int K = din + L.d_skip;
        Opnd A{wparam(c, s, L, 0), dout, K, K};
        Opnd B0{L.Xop, c->max_batch, din, din};
        if (L.L.kind == TGP_MERGE) {
          const Route& R = c->routes[L.L.pop_route];
          Opnd B1{s.self.skip_in[R.id], c->max_batch, R.width, R.width};
          TGP_TRY(run_gemm(c, s, pdl(), A, false, B0, &B1, false, dout, M, K, r0, din, true, e, next_fwd(c, s, l)));
        } else {
          TGP_TRY(run_gemm(c, s, pdl(), A, false, B0, nullptr, false, dout, M, K, r0, K, true, e, next_fwd(c, s, l)));
        }
        break;
      }
      case TGP_RESMLP: {
        const int H = L.L.d_hidden;
        TGP_TRY(ln_fwd_cl(s.comp, pdl() && c->use_pdl, x, din, M, din, mparam(s, L, 0), mparam(s, L, 1),
                       opptr(c, L.Hop, r0, din), din, c->bf16, L.mean[slot], L.rstd[slot]));
        c->kernels++;
        EpiParams e1 = e;
        e1.mode = EPI_LINEAR_FWD;
        e1.act = L.L.act;
        e1.bias = mparam(s, L, 3);
        e1.zbuf = keep ? L.z[slot] : nullptr;
        e1.ldz = H;
        e1.op = opptr(c, L.Gop, r0, H);
        e1.ld_op = H;
        e1.drop_thresh = drop_thresh(L.L.dropout);
        e1.drop_scale = L.L.dropout > 0 ? 1.0f / (1.0f - L.L.dropout) : 1.0f;
        e1.drop_width = H;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 2), H, din, din}, false,
                         Opnd{L.Hop, c->max_batch, din, din}, nullptr, false, H, M, din, r0, din, true, e1,
                         Prefetch{wparam(c, s, L, 4), L.pnum[4] * 2}));
        EpiParams e2 = e;
        e2.mode = EPI_RESID_FWD;
        e2.bias = mparam(s, L, 5);
        e2.res = x;
        e2.ld_res = din;
        e2.out0 = y;
        e2.ld0 = dout;
        if (L.L.stash_route >= 0) {
          e2.op = stash_dst(c, s, L.L.stash_route, r0);
          e2.ld_op = dout;
        }
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 4), dout, H, H}, false, Opnd{L.Gop, c->max_batch, H, H},
                         nullptr, false, dout, M, H, r0, H, true, e2, next_fwd(c, s, l)));
        break;
      }
      case TGP_EMBED: {
        const float p = L.L.dropout;
        TGP_TRY(embed_fwd(s.comp, x, s.d_in, M, mparam(s, L, 0), mparam(s, L, 1), dout, L.L.seq, r0, drop_thresh(p),
                          p > 0 ? 1.0f / (1.0f - p) : 1.0f, c->seed, s.dstep, (uint32_t)l, y));
        c->kernels++;
        first_kernel = false;
        break;
      }
      case TGP_LMHEAD: {
        TGP_TRY(ln_fwd_cl(s.comp, pdl() && c->use_pdl, x, din, M, din, mparam(s, L, 0), mparam(s, L, 1),
                          opptr(c, L.Hop, r0, din), din, true, L.mean[slot], L.rstd[slot]));
        c->kernels++;
        EpiParams e1 = e;
        e1.mode = EPI_LINEAR_FWD;
        e1.act = TGP_ACT_NONE;
        e1.bias = nullptr;
        e1.out0 = y;
        e1.ld0 = dout;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 2), dout, din, din}, false, Opnd{L.Hop, c->max_batch, din, din},
                         nullptr, false, dout, M, din, r0, din, true, e1));
        break;
      }
      case TGP_TRANSFORMER: {
        // x1 = x + drop(Attn(LN1(x)) Wo^T + bo); y = x1 + drop(GELU(LN2(x1) W1^T + b1) W2^T + b2)
        const int d = din, H = L.L.d_hidden, d3 = 3 * din;
        const float p = L.L.dropout;
        const uint32_t th = drop_thresh(p);
        const float dsc = p > 0 ? 1.0f / (1.0f - p) : 1.0f;
        TGP_TRY(ln_fwd_cl(s.comp, pdl() && c->use_pdl, x, d, M, d, mparam(s, L, 0), mparam(s, L, 1),
                          opptr(c, L.Hop, r0, d), d, true, L.mean[slot], L.rstd[slot]));
        c->kernels++;
        EpiParams e1 = e;
        e1.mode = EPI_LINEAR_FWD;
        e1.act = TGP_ACT_NONE;
        e1.bias = mparam(s, L, 3);
        e1.op = opptr(c, L.QKVop, r0, d3);
        e1.ld_op = d3;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 2), d3, d, d}, false, Opnd{L.Hop, c->max_batch, d, d},
                         nullptr, false, d3, M, d, r0, d, true, e1));
        TGP_TRY(attn_fwd(s.comp, opptr(c, L.QKVop, r0, d3), M, d, L.L.n_heads, L.L.seq, r0, th, dsc, c->seed, s.dstep,
                         (uint32_t)l + (1u << 16), opptr(c, L.CTXop, r0, d), L.lse[slot], s.attn_part));
        c->kernels++;
        first_kernel = true;  // the attention kernel does not trigger dependents early
        EpiParams e2 = e;
        e2.mode = EPI_RESID_FWD;
        e2.bias = mparam(s, L, 5);
        e2.res = x;
        e2.ld_res = d;
        e2.out0 = L.x1[slot];
        e2.ld0 = d;
        e2.drop_thresh = th;
        e2.drop_scale = dsc;
        e2.drop_width = d;
        e2.site = (uint32_t)l + (2u << 16);
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 4), d, d, d}, false, Opnd{L.CTXop, c->max_batch, d, d},
                         nullptr, false, d, M, d, r0, d, true, e2));
        TGP_TRY(ln_fwd_cl(s.comp, pdl() && c->use_pdl, L.x1[slot], d, M, d, mparam(s, L, 6), mparam(s, L, 7),
                          opptr(c, L.H2op, r0, d), d, true, L.mean2[slot], L.rstd2[slot]));
        c->kernels++;
        EpiParams e3 = e;
        e3.mode = EPI_LINEAR_FWD;
        e3.act = TGP_ACT_GELU;
        e3.bias = mparam(s, L, 9);
        e3.zbuf = keep ? L.z[slot] : nullptr;
        e3.ldz = H;
        e3.op = opptr(c, L.Gop, r0, H);
        e3.ld_op = H;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 8), H, d, d}, false, Opnd{L.H2op, c->max_batch, d, d},
                         nullptr, false, H, M, d, r0, d, true, e3));
        EpiParams e4 = e;
        e4.mode = EPI_RESID_FWD;
        e4.bias = mparam(s, L, 11);
        e4.res = L.x1[slot];
        e4.ld_res = d;
        e4.out0 = y;
        e4.ld0 = d;
        e4.drop_thresh = th;
        e4.drop_scale = dsc;
        e4.drop_width = d;
        e4.site = (uint32_t)l + (3u << 16);
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 10), d, H, H}, false, Opnd{L.Gop, c->max_batch, H, H},
                         nullptr, false, d, M, H, r0, H, true, e4));
        break;
      }
      case TGP_LAYERNORM:
      case TGP_DROPOUT: {
        if (L.L.kind == TGP_LAYERNORM) {
          TGP_TRY(ln_fwd(s.comp, pdl() && c->use_pdl, x, din, M, din, mparam(s, L, 0), mparam(s, L, 1), y, dout, false,
                         L.mean[slot], L.rstd[slot]));
        } else {  // y = x * keep / (1 - p): the Philox mask of site l (colwise, no activation)
          const float p = L.L.dropout;
          TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, x, din, nullptr, M, din, 0, drop_thresh(p),
                          p > 0 ? 1.0f / (1.0f - p) : 1.0f, c->seed, s.dstep, (uint32_t)l, r0, y, dout, false, nullptr));
        }
        c->kernels++;
        if (L.L.stash_route >= 0) {
          TGP_TRY(convert_rows(s.comp, false, y, dout, M, dout, stash_dst(c, s, L.L.stash_route, r0), dout, c->bf16,
                               nullptr));
          c->kernels++;
        }
        break;
      }
      case TGP_BATCHNORM: {
        const size_t so = (size_t)(i - 1) * din;
        TGP_TRY(bn_fwd(s.comp, x, M, din, mparam(s, L, 0), mparam(s, L, 1), L.L.act, y, L.z[slot], L.bn_mu + so,
                       L.bn_rstd + so, L.bn_var + so));
        c->kernels++;
        first_kernel = false;
        if (L.L.stash_route >= 0) {
          TGP_TRY(convert_rows(s.comp, false, y, dout, M, dout, stash_dst(c, s, L.L.stash_route, r0), dout, c->bf16,
                               nullptr));
          c->kernels++;
        }
        break;
      }
    }
    if (s.prof_ev) TGP_CUDA_TRY(cudaEventRecord(s.prof_ev[l - s.l0], s.comp));  // tgp_profile_layers
    x = y;
  }
  return 0;
}

// B_{i,j}: VJPs through the partition's layers in reverse; stashes dW operands, per-micro-batch
// column partials (bias / LN / BN grads), writes dx rows (message source) and skip gradients.
static int exec_backward(tgp_ctx* c, Stage& s, int i, int r0, int M) {
  if (use_stream(c, s, M)) return exec_task_stream(c, s, i, r0, M, true);
  const int slot = c->slot_of[i];
  float* g = s.self.grad_in + (size_t)r0 * s.d_out;
  int pp = 0;
  bool first_kernel = true;
  auto pdl = [&]() {
    bool r = !first_kernel;
    first_kernel = false;
    return r;
  };
  bool dyop_ready = false;  // the next RESMLP's bf16 dY operand was already written by the LN backward above it
  for (int l = s.l1 - 1; l >= s.l0; --l) {
    LayerRT& L = c->layers[l];
    const int din = L.L.d_in, dout = L.L.d_out;
    const float* xin = (l == s.l0) ? s.self.fwd_in + (size_t)r0 * s.d_in : c->layers[l - 1].out[slot];
    float* dx = (l == s.l0) ? s.dx_out + (size_t)r0 * s.d_in : s.gbuf[pp];
    pp ^= 1;
    if (L.L.stash_route >= 0) {  // add the skip gradient of the portal (reverse direction)
      const Route& R = c->routes[L.L.stash_route];
      const float* ds = (R.dst == s.j) ? s.dskip_local[R.id] : s.self.dskip_in[R.id] + (size_t)r0 * R.width;
      TGP_TRY(add_rows(s.comp, pdl() && c->use_pdl, g, ds, (int64_t)M * dout));
      c->kernels++;
      dyop_ready = false;
    }
    const size_t po = (size_t)(i - 1) * c->pb;  // first 16-row partial block of micro-batch i
    const size_t pbn = (size_t)(i - 1);          // BN per-micro-batch statistics
    EpiParams e{};
    e.op_bf16 = c->bf16 ? 1 : 0;
    e.seed = c->seed;
    e.step = s.dstep;
    e.site = (uint32_t)l;
    e.row_global0 = r0;
    switch (L.L.kind) {
      case TGP_LINEAR:
      case TGP_MERGE: {
        const float th_p = L.L.dropout;
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, g, dout, L.z[slot], M, dout, L.L.act, drop_thresh(th_p),
                        th_p > 0 ? 1.0f / (1.0f - th_p) : 1.0f, c->seed, s.dstep, (uint32_t)l, r0,
                        opptr(c, L.Zop, r0, dout), dout, c->bf16, L.pb + po * dout));
        c->kernels++;
        const int K = din + L.d_skip;
        e.mode = EPI_STORE;
        e.out0 = dx;
        e.ld0 = din;
        e.split_f = din;
        if (L.L.kind == TGP_MERGE) {
          const Route& R = c->routes[L.L.pop_route];
          e.out1 = (R.src == s.j) ? s.dskip_local[R.id] : s.dskip_send[R.id] + (size_t)r0 * R.width;
          e.ld1 = R.width;
        }
        // dx^T[m = in][n] = sum_k W[k = out][m] dZ[n][k]
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 0), dout, K, K}, true, Opnd{L.Zop, c->max_batch, dout, dout},
                         nullptr, false, K, M, dout, r0, dout, true, e, next_bwd(c, s, l)));
        dyop_ready = false;
        break;
      }
      case TGP_RESMLP: {
        const int H = L.L.d_hidden;
        if (!dyop_ready) {
          TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, g, dout, nullptr, M, dout, 0, 0u, 1.0f, c->seed, s.dstep,
                          (uint32_t)l, r0, opptr(c, L.dYop, r0, dout), dout, c->bf16, L.pb2 + po * dout));
          c->kernels++;
        }
        EpiParams e1 = e;
        e1.mode = EPI_ACT_BWD;
        e1.act = L.L.act;
        e1.zbuf = L.z[slot];
        e1.ldz = H;
        e1.op = opptr(c, L.dAop, r0, H);
        e1.ld_op = H;
        e1.colsum = L.pb + po * H;
        e1.drop_thresh = drop_thresh(L.L.dropout);
        e1.drop_scale = L.L.dropout > 0 ? 1.0f / (1.0f - L.L.dropout) : 1.0f;
        e1.drop_width = H;
        // dg^T[m = hidden][n] = sum_k W2[k = out][m] dY[n][k]
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 4), dout, H, H}, true, Opnd{L.dYop, c->max_batch, dout, dout},
                         nullptr, false, H, M, dout, r0, dout, true, e1, Prefetch{wparam(c, s, L, 2), L.pnum[2] * 2}));
        EpiParams e2 = e;
        e2.mode = EPI_STORE;
        e2.out0 = s.dh;
        e2.ld0 = din;
        e2.split_f = din;
        // dh^T[m = in][n] = sum_k W1[k = hidden][m] dA[n][k]
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 2), H, din, din}, true, Opnd{L.dAop, c->max_batch, H, H},
                         nullptr, false, din, M, H, r0, H, true, e2, next_bwd(c, s, l)));
        // the layer below consumes dx as its incoming gradient: if it is a RESMLP without a portal
        // stash, emit its bf16 dY operand and b2 partial here (fused; no separate cast kernel)
        LayerRT* below = (l > s.l0) ? &c->layers[l - 1] : nullptr;
        const bool fuse = below && below->L.kind == TGP_RESMLP && below->L.stash_route < 0 && ln_cluster_ok(din);
        if (ln_cluster_ok(din)) {
          TGP_TRY(ln_bwd_cl(s.comp, pdl() && c->use_pdl, s.dh, xin, L.mean[slot], L.rstd[slot], mparam(s, L, 0), g, dx,
                            M, din, c->pb, L.pg + po * din, L.pbt + po * din,
                            fuse ? opptr(c, below->dYop, r0, din) : nullptr, c->bf16,
                            fuse ? below->pb2 + po * din : nullptr));
          c->kernels++;
          dyop_ready = fuse;
        } else {
          TGP_TRY(ln_bwd(s.comp, pdl() && c->use_pdl, s.dh, xin, L.mean[slot], L.rstd[slot], mparam(s, L, 0), g, dx, M,
                         din, L.pg + po * din, L.pbt + po * din));
          c->kernels += 2;
          dyop_ready = false;
        }
        break;
      }
      case TGP_EMBED: {
        // stash the output gradient (dropout mask applied) for the deferred embedding gradient in W_j
        const float p = L.L.dropout;
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, g, dout, nullptr, M, dout, 0, drop_thresh(p),
                        p > 0 ? 1.0f / (1.0f - p) : 1.0f, c->seed, s.dstep, (uint32_t)l, r0,
                        L.dE + (size_t)r0 * dout, dout, false, nullptr));
        c->kernels++;
        dyop_ready = false;
        break;
      }
      case TGP_LMHEAD: {
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, g, dout, nullptr, M, dout, 0, 0u, 1.0f, c->seed, s.dstep,
                        (uint32_t)l, r0, opptr(c, L.dYop, r0, dout), dout, true, nullptr));
        c->kernels++;
        EpiParams e2 = e;
        e2.mode = EPI_STORE;
        e2.out0 = s.dh;
        e2.ld0 = din;
        e2.split_f = din;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 2), dout, din, din}, true,
                         Opnd{L.dYop, c->max_batch, dout, dout}, nullptr, false, din, M, dout, r0, dout, true, e2));
        TGP_TRY(ln_bwd_any(c, s, pdl() && c->use_pdl, s.dh, xin, L.mean[slot], L.rstd[slot], mparam(s, L, 0), nullptr,
                           dx, M, din, L.pg + po * din, L.pbt + po * din));
        dyop_ready = false;
        break;
      }
      case TGP_TRANSFORMER: {
        const int d = din, H = L.L.d_hidden, d3 = 3 * din;
        const float p = L.L.dropout;
        const uint32_t th = drop_thresh(p);
        const float dsc = p > 0 ? 1.0f / (1.0f - p) : 1.0f;
        // MLP branch: dm = g o keep3 -> bf16 dY operand (+ b2 partial)
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, g, d, nullptr, M, d, 0, th, dsc, c->seed, s.dstep,
                        (uint32_t)l + (3u << 16), r0, opptr(c, L.dYop, r0, d), d, true, L.pb2 + po * d));
        c->kernels++;
        EpiParams e1 = e;
        e1.mode = EPI_ACT_BWD;
        e1.act = TGP_ACT_GELU;
        e1.zbuf = L.z[slot];
        e1.ldz = H;
        e1.op = opptr(c, L.dAop, r0, H);
        e1.ld_op = H;
        e1.colsum = L.pb + po * H;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 10), d, H, H}, true, Opnd{L.dYop, c->max_batch, d, d},
                         nullptr, false, H, M, d, r0, d, true, e1));
        EpiParams es = e;
        es.mode = EPI_STORE;
        es.out0 = s.dh;
        es.ld0 = d;
        es.split_f = d;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 8), H, d, d}, true, Opnd{L.dAop, c->max_batch, H, H},
                         nullptr, false, d, M, H, r0, H, true, es));
        // dx1 = g + LN2_bwd(dh2), kept in dx until the end of the layer
        TGP_TRY(ln_bwd_any(c, s, pdl() && c->use_pdl, s.dh, L.x1[slot], L.mean2[slot], L.rstd2[slot], mparam(s, L, 6),
                           g, dx, M, d, L.pg2 + po * d, L.pbt2 + po * d));
        // attention branch: da = dx1 o keep2 -> bf16 operand (+ bo partial); dctx = da Wo
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, dx, d, nullptr, M, d, 0, th, dsc, c->seed, s.dstep,
                        (uint32_t)l + (2u << 16), r0, opptr(c, L.dX1op, r0, d), d, true, L.po + po * d));
        c->kernels++;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 4), d, d, d}, true, Opnd{L.dX1op, c->max_batch, d, d},
                         nullptr, false, d, M, d, r0, d, true, es));
        TGP_TRY(attn_bwd(s.comp, opptr(c, L.QKVop, r0, d3), opptr(c, L.CTXop, r0, d), s.dh, L.lse[slot], s.attnD, M, d,
                         L.L.n_heads, L.L.seq, r0, th, dsc, c->seed, s.dstep, (uint32_t)l + (1u << 16), s.tbuf));
        c->kernels += 3;
        TGP_TRY(colwise(s.comp, false, s.tbuf, d3, nullptr, M, d3, 0, 0u, 1.0f, c->seed, s.dstep, (uint32_t)l, r0,
                        opptr(c, L.dQKVop, r0, d3), d3, true, L.pq + po * d3));
        c->kernels++;
        TGP_TRY(run_gemm(c, s, pdl(), Opnd{wparam(c, s, L, 2), d3, d, d}, true, Opnd{L.dQKVop, c->max_batch, d3, d3},
                         nullptr, false, d, M, d3, r0, d3, true, es));
        // dx = dx1 + LN1_bwd(dh1) (in place: each element read and written by the same thread)
        TGP_TRY(ln_bwd_any(c, s, pdl() && c->use_pdl, s.dh, xin, L.mean[slot], L.rstd[slot], mparam(s, L, 0), dx, dx, M,
                           d, L.pg + po * d, L.pbt + po * d));
        dyop_ready = false;
        break;
      }
      case TGP_LAYERNORM: {
        // dx = LN_bwd(dy) with the per-16-row dgamma / dbeta column partials of micro-batch i
        TGP_TRY(ln_bwd_any(c, s, pdl() && c->use_pdl, g, xin, L.mean[slot], L.rstd[slot], mparam(s, L, 0), nullptr, dx,
                           M, din, L.pg + po * din, L.pbt + po * din));
        dyop_ready = false;
        break;
      }
      case TGP_DROPOUT: {  // dx = dy * keep / (1 - p), the same mask (same site, counters and step)
        const float p = L.L.dropout;
        TGP_TRY(colwise(s.comp, pdl() && c->use_pdl, g, dout, nullptr, M, dout, 0, drop_thresh(p),
                        p > 0 ? 1.0f / (1.0f - p) : 1.0f, c->seed, s.dstep, (uint32_t)l, r0, dx, din, false, nullptr));
        c->kernels++;
        dyop_ready = false;
        break;
      }
      case TGP_BATCHNORM: {
        TGP_TRY(bn_bwd(s.comp, g, xin, L.z[slot], L.bn_mu + pbn * din, L.bn_rstd + pbn * din, mparam(s, L, 0), M, din,
                       L.L.act, dx, L.pg + po * din, L.pb + po * din));
        c->kernels++;
        first_kernel = false;
        dyop_ready = false;
        break;
      }
    }
    if (s.prof_ev) TGP_CUDA_TRY(cudaEventRecord(s.prof_ev[(s.l1 - s.l0) + (s.l1 - 1 - l)], s.comp));
    g = dx;
  }
  return 0;
}

// W_j: deferred weight gradients g^j = sum_i g_i^j as one GEMM per weight over the stacked
// micro-batches, plus fixed-order reductions of the per-micro-batch column partials.
// Descriptors of the fused W_j + SGD GEMMs for batch B (the operand maps have K = B rows: TMA
// zero-fills past them), uploaded on the compute stream (stream-ordered before the W task).
static int ensure_ws(tgp_ctx* c, Stage& s, int B) {
  if (s.ws_B == B || s.ws_layers.empty()) return 0;
  s.ws_host.assign(2 * s.ws_layers.size(), WsGemm{});
  int tile0 = 0;
  for (size_t q = 0; q < s.ws_layers.size(); ++q) {
    const LayerRT& L = c->layers[s.ws_layers[q]];
    const int d = L.L.d_in, H = L.L.d_hidden;
    WsGemm& g1 = s.ws_host[2 * q];
    WsGemm& g2 = s.ws_host[2 * q + 1];
    // dW1[h][k] = sum_r dA[r][h] LN(x)[r][k];  dW2[f][h] = sum_r dY[r][f] G[r][h]
    if (!wgrad_sgd_desc(&g1, L.dAop, H, L.Hop, d, mparam(s, L, 2), s.shadow + L.poff[2], d, H, d, B) ||
        !wgrad_sgd_desc(&g2, L.dYop, d, L.Gop, H, mparam(s, L, 4), s.shadow + L.poff[4], H, d, H, B))
      return TGP_E_CUDA;
    g1.tile0 = tile0;
    tile0 += g1.tiles;
    g2.tile0 = tile0;
    tile0 += g2.tiles;
  }
  TGP_CUDA_TRY(cudaMemcpyAsync(s.ws_dev, s.ws_host.data(), s.ws_host.size() * sizeof(WsGemm), cudaMemcpyHostToDevice,
                               s.comp));
  s.ws_B = B;
  return 0;
}

// W_j.  fused: SGD applied here (tgp_backward_step): the fused weight matrices' dW accumulators update
// the master / shadow directly (wgrad_sgd), the other parameters' gradients are stored as usual and
// then stepped by sgd_segments; requires fresh gradients.
static int exec_wgrad(tgp_ctx* c, Stage& s, int B, bool fused = false) {
  const bool acc = !s.grads_fresh;
  for (int l = s.l0; l < s.l1; ++l) {
    LayerRT& L = c->layers[l];
    if (fused && std::find(s.ws_layers.begin(), s.ws_layers.end(), l) != s.ws_layers.end()) continue;
    const int din = L.L.d_in, dout = L.L.d_out;
    EpiParams e{};
    e.mode = EPI_DW;
    e.accumulate = acc ? 1 : 0;
    switch (L.L.kind) {
      case TGP_LINEAR:
      case TGP_MERGE: {
        const int K = din + L.d_skip;
        e.dw = gparam(s, L, 0);
        e.ldw = K;
        // dW[m = out][n = in] = sum_k dZ[k][m] X[k][n]
        TGP_TRY(run_gemm(c, s, false, Opnd{L.Zop, B, dout, dout}, true, Opnd{L.Xop, B, din, din}, nullptr, true, dout,
                         din, B, 0, B, false, e));
        if (L.L.kind == TGP_MERGE) {
          const Route& R = c->routes[L.L.pop_route];
          e.dw = gparam(s, L, 0) + din;
          TGP_TRY(run_gemm(c, s, false, Opnd{L.Zop, B, dout, dout}, true, Opnd{s.self.skip_in[R.id], B, R.width, R.width},
                           nullptr, true, dout, R.width, B, 0, B, false, e));
        }
        break;
      }
      case TGP_RESMLP: {
        const int H = L.L.d_hidden;
        e.dw = gparam(s, L, 2);
        e.ldw = din;
        TGP_TRY(run_gemm(c, s, false, Opnd{L.dAop, B, H, H}, true, Opnd{L.Hop, B, din, din}, nullptr, true, H, din, B, 0,
                         B, false, e));
        e.dw = gparam(s, L, 4);
        e.ldw = H;
        TGP_TRY(run_gemm(c, s, false, Opnd{L.dYop, B, dout, dout}, true, Opnd{L.Gop, B, H, H}, nullptr, true, dout, H, B,
                         0, B, false, e));
        break;
      }
      case TGP_EMBED:
        TGP_TRY(embed_wgrad(s.comp, s.self.fwd_in, s.d_in, B, L.dE, dout, L.L.vocab, L.L.seq, L.emb_scratch,
                            gparam(s, L, 0), gparam(s, L, 1), acc));
        c->kernels += 5;
        break;
      case TGP_LMHEAD:
        e.dw = gparam(s, L, 2);
        e.ldw = din;
        TGP_TRY(run_gemm(c, s, false, Opnd{L.dYop, B, dout, dout}, true, Opnd{L.Hop, B, din, din}, nullptr, true, dout,
                         din, B, 0, B, false, e));
        break;
      case TGP_TRANSFORMER: {
        const int d = din, H = L.L.d_hidden, d3 = 3 * din;
        struct {
          int k;
          void *a, *b;
          int M, N;
        } gw[4] = {{2, L.dQKVop, L.Hop, d3, d}, {4, L.dX1op, L.CTXop, d, d}, {8, L.dAop, L.H2op, H, d},
                   {10, L.dYop, L.Gop, d, H}};
        for (auto& q : gw) {
          e.dw = gparam(s, L, q.k);
          e.ldw = q.N;
          TGP_TRY(run_gemm(c, s, false, Opnd{q.a, B, q.M, q.M}, true, Opnd{q.b, B, q.N, q.N}, nullptr, true, q.M, q.N,
                           B, 0, B, false, e));
        }
        break;
      }
      case TGP_BATCHNORM:
      case TGP_LAYERNORM:
      case TGP_DROPOUT:
        break;
    }
  }
  // every bias / LayerNorm / BatchNorm column-partial reduction of the partition in one launch
  if (s.n_red > 0) {
    TGP_TRY(reduce_partials_multi(s.comp, (const RedItem*)s.red_items, s.n_red, s.red_maxd, c->m * c->pb, acc));
    c->kernels++;
  }
  if (fused) {
    if (!s.ws_layers.empty()) {
      TGP_TRY(wgrad_sgd(s.comp, s.ws_dev, s.ws_host.data(), (int)s.ws_host.size(), s.dlr));
      c->kernels++;
    }
    TGP_TRY(sgd_segments(s.comp, s.master, s.grad, s.shadow, s.seg_dev, s.n_seg, s.seg_maxlen, s.dlr));
    c->kernels++;
  }
  s.grads_fresh = false;
  return 0;
}

// ---------------------------------------------------------------------------- task graphs
// Each task's kernel sequence is captured once into a CUDA graph (per micro-batch, per batch size)
// and replayed: one host launch per task instead of ~3 per layer.
template <typename Fn>
static int run_task(tgp_ctx* c, Stage& s, TaskGraph& tg, int B, Fn&& fn, cudaStream_t st = nullptr, int mode = 0) {
  if (!st) st = s.comp;
  if (!c->use_graphs) return fn();
  if (tg.exec && tg.B == B && tg.mode == mode) {
    TGP_CUDA_TRY(cudaGraphLaunch(tg.exec, st));
    c->kernels += tg.kernels;
    return 0;
  }
  if (tg.exec) {
    cudaGraphExecDestroy(tg.exec);
    tg.exec = nullptr;
  }
  const int64_t k0 = c->kernels;
  TGP_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  int rc = fn();
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(st, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  TGP_CUDA_TRY(ce);
  ce = cudaGraphInstantiate(&tg.exec, graph, 0);
  cudaGraphDestroy(graph);
  TGP_CUDA_TRY(ce);
  tg.B = B;
  tg.mode = mode;
  tg.kernels = c->kernels - k0;
  c->kernels = k0;
  TGP_CUDA_TRY(cudaGraphLaunch(tg.exec, st));
  c->kernels += tg.kernels;
  return 0;
}

// ============================================================================ waits / transport
static int wait_flag(tgp_ctx* c, cudaStream_t st, uint32_t* flag, uint32_t v) {
  const Driver* d = driver();
  if (!d) return TGP_E_CUDA;
  unsigned flags = CU_STREAM_WAIT_VALUE_GEQ;
  if (c->can_flush) flags |= CU_STREAM_WAIT_VALUE_FLUSH;
  TGP_CU_TRY(d->streamWaitValue32((CUstream)st, (CUdeviceptr)flag, v, flags));
  return 0;
}

// transport "auto" (2): copy engine from this message size up, SM push kernel below -- the crossover
// measured on B200 (profiles/round2_transport_sweep.txt: push 4.7 us vs CE 5.7 us at 4 KiB, CE 6.2 us
// vs push 7.3 us at 16 KiB and flat to 4 MiB)
constexpr int64_t kCeMinBytes = 16384;

static int write_flag(cudaStream_t st, uint32_t* flag, uint32_t v) {
  const Driver* d = driver();
  if (!d) return TGP_E_CUDA;
  TGP_CU_TRY(d->streamWriteValue32((CUstream)st, (CUdeviceptr)flag, v, CU_STREAM_WRITE_VALUE_DEFAULT));
  return 0;
}

// 4-byte value into device memory, ordered on the stream (no host staging buffer: asynchronous calls
// may return before it executes)
static int put_u32(cudaStream_t st, void* dst, uint32_t v) { return write_flag(st, (uint32_t*)dst, v); }


static void trace_begin(tgp_ctx* c, Stage& s, cudaStream_t st, int stream_id, int kind, int i, cudaEvent_t* a) {
  if (!c->trace) return;
  cudaEventCreate(a);
  cudaEventRecord(*a, st);
  (void)s;
  (void)stream_id;
  (void)kind;
  (void)i;
}
static void trace_end(tgp_ctx* c, Stage& s, cudaStream_t st, int stream_id, int kind, int i, cudaEvent_t a) {
  if (!c->trace) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, st);
  c->trace_recs.push_back(TraceRec{s.j, stream_id, kind, i, a, b});
}

static void micro_rows(const tgp_ctx* c, int B, int i, int* r0, int* M) {
  // split the B / unit samples (reading Z7), rows = samples x unit (unit = seq tokens for C5)
  const int U = c->unit, S = B / U;
  const int q = S / c->m, r = S % c->m;
  const int ii = i - 1;
  *r0 = (ii * q + std::min(ii, r)) * U;
  *M = (q + (ii < r ? 1 : 0)) * U;
}

// an event of stage s's device (reused every call; the waits bind at enqueue time)
static cudaEvent_t abl_event(Stage& s) {
  if (s.abl_next == s.abl_events.size()) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(s.dev);
    cudaEvent_t e = nullptr;
    const cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaSetDevice(cur);
    if (err != cudaSuccess) {
      set_error("cudaEventCreate failed: %s", cudaGetErrorString(err));
      return nullptr;
    }
    s.abl_events.push_back(e);
  }
  return s.abl_events[s.abl_next++];
}

// partitions that push data into partition j (receive arena writers)
static std::vector<int> writers_of(const tgp_ctx* c, int j) {
  std::vector<int> w;
  if (j > 0) w.push_back(j - 1);
  if (j + 1 < c->n) w.push_back(j + 1);
  for (const Route& r : c->routes) {
    if (r.src == r.dst) continue;
    if (r.dst == j) w.push_back(r.src);
    if (r.src == j) w.push_back(r.dst);
  }
  std::sort(w.begin(), w.end());
  w.erase(std::unique(w.begin(), w.end()), w.end());
  return w;
}

// Issue one schedule record whose actor is local.  Copies ride on the producer's copy streams and
// end with a flag release on the consumer; computes wait on their receive flags on the compute
// stream (the consumer never blocks the producer).
// NVTX ranges (host issue side; SURVEY 5 tracing, Fig. 7): one range per tgp_* call and
// per issued task, named after the schedule record ("F i=3 j=2", "COPY_B i=1 2->1", "W j=1"), so a
// profiler timeline lines the host issue order up against the device work.  Header-only NVTX 3: a
// no-op pointer check when no tool is attached.  Option "nvtx" (default 1).
struct NvtxRange {
  bool on;
  NvtxRange(const tgp_ctx* c, const char* name) : on(c->nvtx) {
    if (on) nvtxRangePushA(name);
  }
  ~NvtxRange() {
    if (on) nvtxRangePop();
  }
};
static const char* kind_name(int k) {
  static const char* names[] = {"F", "F'", "B", "COPY_F", "COPY_B", "SKIP_F", "SKIP_B", "W"};
  return (k >= 0 && k < 8) ? names[k] : "?";
}

static int issue_task(tgp_ctx* c, const Rec& rc, int B, std::vector<std::vector<char>>& first_push);
static int issue(tgp_ctx* c, const Rec& rc, int B, std::vector<std::vector<char>>& first_push) {
  if (!c->nvtx) return issue_task(c, rc, B, first_push);
  char name[64];
  if (rc.kind == K_W)
    snprintf(name, sizeof(name), "W j=%d", rc.j);
  else if (rc.kind >= K_COPY_F)
    snprintf(name, sizeof(name), "%s i=%d %d->%d r=%d", kind_name(rc.kind), rc.i, rc.src, rc.dst, rc.route);
  else
    snprintf(name, sizeof(name), "%s i=%d j=%d", kind_name(rc.kind), rc.i, rc.j);
  NvtxRange r(c, name);
  return issue_task(c, rc, B, first_push);
}

static int issue_task(tgp_ctx* c, const Rec& rc, int B, std::vector<std::vector<char>>& first_push) {
  const int i = rc.i;
  int r0 = 0, M = 0;
  if (i > 0) micro_rows(c, B, i, &r0, &M);
  const uint32_t seq = c->seq;
  switch (rc.kind) {
    case K_COPY_F:
    case K_COPY_B:
    case K_SKIP_F:
    case K_SKIP_B: {
      const int src = rc.src - 1, dst = rc.dst - 1;
      Stage* sp = c->local[src];
      if (!sp) return 0;  // actor is the source; remote source -> nothing to issue here
      Stage& s = *sp;
      const bool skip = rc.kind == K_SKIP_F || rc.kind == K_SKIP_B;
      if ((rc.kind == K_COPY_F && fuse_fwd(c, s, M)) || (rc.kind == K_COPY_B && fuse_bwd(c, s, M))) {
        // fused with the producing task (f3): the task kernel wrote the consumer's slab and flag
        c->copy_bytes += (int64_t)M * (rc.kind == K_COPY_F ? s.d_out : s.d_in) * 4;
        c->copy_msgs++;
        c->issue_log.push_back(rc);
        return 0;
      }
      cudaStream_t st = skip ? s.cskip : s.cact;
      cudaEvent_t ev = (rc.kind == K_COPY_F || rc.kind == K_SKIP_F) ? s.fdone[i - 1] : s.bdone[i - 1];
      if (c->abl_streams) {
        // Table 1 "no copy streams" ablation: the copy rides on the producer's compute stream and,
        // like a default-stream copy (Fig. 5), first waits for all work issued so far on the
        // consumer's compute stream
        st = s.comp;
        cudaEvent_t e = abl_event(*c->local[dst]);
        if (!e) return TGP_E_CUDA;
        TGP_CUDA_TRY(cudaEventRecord(e, c->local[dst]->comp));
        TGP_CUDA_TRY(cudaStreamWaitEvent(st, e, 0));
      }
      TGP_CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
      if (!first_push[src][dst]) {
        // the consumer must have finished the previous call before its receive slots are reused
        TGP_TRY(wait_flag(c, st, flag_done(c, s.self, dst), seq - 1));
        first_push[src][dst] = 1;
      }
      const ArenaView& pv = c->view[dst];
      if (c->drop_push_part == src && rc.kind == K_COPY_F) return 0;  // watchdog test: the message is lost
      if (c->delay_push_ns) {  // negative-control tests: make a missing receive wait observable
        TGP_TRY(spin(st, c->delay_push_ns));
        c->kernels++;
      }
      cudaEvent_t ta = nullptr;
      trace_begin(c, s, st, skip ? 2 : 1, rc.kind, i, &ta);
      uint32_t* ctr = s.counters + (skip ? 1 : 0);
      int64_t nbytes = 0;
      const int64_t msg_bytes = (int64_t)M * (rc.kind == K_COPY_F ? s.d_out : s.d_in) * 4;
      const bool use_ce = c->transport == 1 || (c->transport == 2 && msg_bytes >= kCeMinBytes);
      if ((rc.kind == K_COPY_F || rc.kind == K_COPY_B) && use_ce) {
        // copy-engine transport: DMA copy, then a stream memory write of the flag (the driver orders it
        // after the copy with a memory barrier: CU_STREAM_WRITE_VALUE_DEFAULT)
        const bool fw = rc.kind == K_COPY_F;
        const int w = fw ? s.d_out : s.d_in;
        nbytes = (int64_t)M * w * 4;
        const float* from = (fw ? s.out : s.dx_out) + (size_t)r0 * w;
        float* to = (fw ? pv.fwd_in : pv.grad_in) + (size_t)r0 * w;
        TGP_CUDA_TRY(cudaMemcpyAsync(to, from, (size_t)nbytes, cudaMemcpyDefault, st));
        TGP_TRY(write_flag(st, fw ? flag_fwd(pv, i) : flag_grad(c, pv, i), seq));
      } else if (rc.kind == K_COPY_F) {
        nbytes = (int64_t)M * s.d_out * 4;
        TGP_TRY(push_rows(st, s.out + (size_t)r0 * s.d_out, pv.fwd_in + (size_t)r0 * s.d_out, false,
                          (int64_t)M * s.d_out, ctr, flag_fwd(pv, i), seq));
      } else if (rc.kind == K_COPY_B) {
        nbytes = (int64_t)M * s.d_in * 4;
        TGP_TRY(push_rows(st, s.dx_out + (size_t)r0 * s.d_in, pv.grad_in + (size_t)r0 * s.d_in, false,
                          (int64_t)M * s.d_in, ctr, flag_grad(c, pv, i), seq));
      } else if (rc.kind == K_SKIP_F) {
        // portal: stash partition -> pop partition; relay (ablation): hop src -> dst through the
        // relay slots of the partitions in between
        const Route& R = c->routes[rc.route];
        nbytes = (int64_t)M * R.width * op_size(c);
        void* from = src == R.src ? s.skip_send[R.id] : s.relay_skip[R.id];
        void* to = dst == R.dst ? pv.skip_in[R.id] : c->local[dst]->relay_skip[R.id];
        if (!from || !to) {
          set_error("skip route %d: no buffer for hop %d -> %d", R.id, src, dst);
          return TGP_E_STATE;
        }
        TGP_TRY(push_bytes(st, opptr(c, from, r0, R.width), opptr(c, to, r0, R.width), nbytes, ctr,
                           flag_skip(c, pv, R.id, i), seq));
      } else {
        const Route& R = c->routes[rc.route];
        nbytes = (int64_t)M * R.width * 4;
        float* from = src == R.dst ? s.dskip_send[R.id] : s.relay_dskip[R.id];
        float* to = dst == R.src ? pv.dskip_in[R.id] : c->local[dst]->relay_dskip[R.id];
        if (!from || !to) {
          set_error("skip route %d: no gradient buffer for hop %d -> %d", R.id, src, dst);
          return TGP_E_STATE;
        }
        TGP_TRY(push_rows(st, from + (size_t)r0 * R.width, to + (size_t)r0 * R.width, false, (int64_t)M * R.width, ctr,
                          flag_dskip(c, pv, R.id, i), seq));
      }
      if (c->abl_streams) {  // the consumer's later work waits for the copy (default-stream semantics)
        cudaEvent_t e = abl_event(s);
        if (!e) return TGP_E_CUDA;
        TGP_CUDA_TRY(cudaEventRecord(e, st));
        TGP_CUDA_TRY(cudaStreamWaitEvent(c->local[dst]->comp, e, 0));
      }
      c->copy_bytes += nbytes;
      c->copy_msgs++;
      c->kernels++;
      trace_end(c, s, st, skip ? 2 : 1, rc.kind, i, ta);
      c->issue_log.push_back(rc);
      return 0;
    }
    case K_F:
    case K_RECOMPUTE:
    case K_B: {
      const int j = rc.j - 1;
      Stage* sp = c->local[j];
      if (!sp) return 0;
      Stage& s = *sp;
      const bool stream_task = use_stream(c, s, M);
      if (stream_task && s.st_micro_B != B) TGP_TRY(st_build_desc(c, s, B));
      if (rc.kind == K_RECOMPUTE && s.pair_ok && s.hoisted[i] == 1) {
        // F'_{i,j} was issued on lane 1 beside B_{i+1,j} (see K_B): only the record remains
        c->issue_log.push_back(rc);
        return 0;
      }
      // F' / B pairing: F'_{i-1,j} depends only on the stage input and the weights, not on B_{i,j},
      // so it is hoisted onto lane 1 and runs beside B_{i,j}, both on half grids; issued before B's
      // gradient wait so it does not wait for the downstream partition
      bool paired = false;
      if (rc.kind == K_B && !stream_task && s.pair_layer && c->pair && c->order_seed == 0 && !c->relay &&
          !c->abl_streams && i >= 2 &&
          checkpointed(i - 1, c->m, c->ckpt) && !s.hoisted[i - 1]) {
        // per-layer partitions: the same hoist with full-size kernels on lane 1 (exec_forward launches
        // on s.comp, so the lanes are swapped around its issue / graph capture)
        int pr0 = 0, pM = 0;
        micro_rows(c, B, i - 1, &pr0, &pM);
        TGP_CUDA_TRY(cudaEventRecord(s.ev_pair, s.comp));  // after B_{i+1,j}, the last reader of the slot
        TGP_CUDA_TRY(cudaStreamWaitEvent(s.comp2, s.ev_pair, 0));
        cudaEvent_t tr = nullptr;
        trace_begin(c, s, s.comp2, 3, K_RECOMPUTE, i - 1, &tr);
        std::swap(s.comp, s.comp2);
        const int rcode = run_task(c, s, s.gR2[i - 2], B, [&] { return exec_forward(c, s, i - 1, pr0, pM); }, s.comp);
        std::swap(s.comp, s.comp2);
        TGP_TRY(rcode);
        trace_end(c, s, s.comp2, 3, K_RECOMPUTE, i - 1, tr);
        TGP_CUDA_TRY(cudaEventRecord(s.rdone[i - 2], s.comp2));
        s.hoisted[i - 1] = 1;
      }
      if (rc.kind == K_B && stream_task && s.pair_ok && !s.pair_layer && c->pair && c->order_seed == 0 && i >= 2 &&
          checkpointed(i - 1, c->m, c->ckpt) && !s.hoisted[i - 1]) {
        int pr0 = 0, pM = 0;
        micro_rows(c, B, i - 1, &pr0, &pM);
        if (use_stream(c, s, pM)) {
          TGP_CUDA_TRY(cudaEventRecord(s.ev_pair, s.comp));  // after B_{i+1,j}, the last reader of the slot
          TGP_CUDA_TRY(cudaStreamWaitEvent(s.comp2, s.ev_pair, 0));
          cudaEvent_t tr = nullptr;
          trace_begin(c, s, s.comp2, 3, K_RECOMPUTE, i - 1, &tr);
          TGP_TRY(run_task(c, s, s.gR2[i - 2], B, [&] { return exec_task_stream(c, s, i - 1, pr0, pM, false, 2); },
                           s.comp2));
          trace_end(c, s, s.comp2, 3, K_RECOMPUTE, i - 1, tr);  // before rdone: B_{i-1} starts after it
          TGP_CUDA_TRY(cudaEventRecord(s.rdone[i - 2], s.comp2));
          s.hoisted[i - 1] = 1;
          paired = true;
        }
      }
      if (rc.kind == K_F && j > 0 && c->skip_wait_part != j) TGP_TRY(wait_flag(c, s.comp, flag_fwd(s.self, i), seq));
      // relay (ablation): a partition between stash and pop takes the skip tensor as a tuple input
      // of F and its gradient as a tuple input of B
      auto relays = [&](const Route& R) { return c->relay && R.src < j && j < R.dst; };
      if (rc.kind == K_F)
        for (const Route& R : c->routes)
          if ((R.dst == j && R.src != j) || relays(R)) TGP_TRY(wait_flag(c, s.comp, flag_skip(c, s.self, R.id, i), seq));
      if (rc.kind == K_B) {
        if (j < c->n - 1 && c->skip_wait_part != j) TGP_TRY(wait_flag(c, s.comp, flag_grad(c, s.self, i), seq));
        for (const Route& R : c->routes)
          if ((R.src == j && R.dst != j) || relays(R)) TGP_TRY(wait_flag(c, s.comp, flag_dskip(c, s.self, R.id, i), seq));
      }
      if (rc.kind == K_B && s.pair_ok && s.hoisted[i] == 1) TGP_CUDA_TRY(cudaStreamWaitEvent(s.comp, s.rdone[i - 1], 0));
      if (rc.kind == K_RECOMPUTE && s.pair_ok) s.hoisted[i] = 2;  // issued in place
      // fused send: the task writes the neighbour's receive slab, which the neighbour must have
      // finished using in the previous call (R2; the push path does this wait on its copy stream)
      const bool send = (rc.kind == K_F && fuse_fwd(c, s, M)) || (rc.kind == K_B && fuse_bwd(c, s, M));
      const int nb = rc.kind == K_B ? j - 1 : j + 1;
      if (send && !first_push[j][nb]) {
        TGP_TRY(wait_flag(c, s.comp, flag_done(c, s.self, nb), seq - 1));
        first_push[j][nb] = 1;
      }
      float* send_to = nullptr;
      uint32_t* send_flag = nullptr;
      if (send && rc.kind == K_F) {
        send_to = c->view[nb].fwd_in + (size_t)r0 * s.d_out;
        send_flag = flag_fwd(c->view[nb], i);
      } else if (send) {
        send_to = c->view[nb].grad_in + (size_t)r0 * s.d_in;
        send_flag = flag_grad(c, c->view[nb], i);
      }
      // a checkpointed F keeps only its output (F' recomputes the intermediates before B reads them;
      // F and F' have separate task graphs)
      const bool f_keep = !(rc.kind == K_F && checkpointed(i, c->m, c->ckpt) && c->dead_stash);
      cudaEvent_t ta = nullptr;
      trace_begin(c, s, s.comp, 0, rc.kind, i, &ta);
      if (rc.kind == K_B && (paired || send)) {
        TGP_TRY(run_task(c, s, paired ? s.gB2[i - 1] : s.gB[i - 1], B,
                         [&] { return exec_task_stream(c, s, i, r0, M, true, paired ? 1 : 0, send_to, send_flag); },
                         nullptr, send ? 1 : 0));
        TGP_CUDA_TRY(cudaEventRecord(s.bdone[i - 1], s.comp));
      } else if (rc.kind == K_B) {
        TGP_TRY(run_task(c, s, s.gB[i - 1], B, [&] { return exec_backward(c, s, i, r0, M); }));
        TGP_CUDA_TRY(cudaEventRecord(s.bdone[i - 1], s.comp));
      } else if (send) {  // F_{i,j} sending its output
        TGP_TRY(run_task(c, s, s.gF[i - 1], B,
                         [&] { return exec_task_stream(c, s, i, r0, M, false, 0, send_to, send_flag, f_keep); }, nullptr, 1));
        TGP_CUDA_TRY(cudaEventRecord(s.fdone[i - 1], s.comp));
      } else {
        // F without a send, or F' (never sends; with a sending F it has its own graph)
        TaskGraph& tg = rc.kind == K_RECOMPUTE ? s.gR[i - 1] : s.gF[i - 1];
        TGP_TRY(run_task(c, s, tg, B, [&] { return exec_forward(c, s, i, r0, M, rc.kind == K_RECOMPUTE || f_keep); }));
        if (rc.kind == K_F) TGP_CUDA_TRY(cudaEventRecord(s.fdone[i - 1], s.comp));
      }
      trace_end(c, s, s.comp, 0, rc.kind, i, ta);
      c->issue_log.push_back(rc);
      return 0;
    }
    case K_W: {
      const int j = rc.j - 1;
      Stage* sp = c->local[j];
      if (!sp) return 0;
      Stage& s = *sp;
      cudaEvent_t ta = nullptr;
      trace_begin(c, s, s.comp, 0, rc.kind, 0, &ta);
      if (c->fuse_sgd && s.grads_fresh && c->bf16) {
        // W_j + SGD (tgp_backward_step): the learning rate is a device scalar, so the graph replays
        TGP_TRY(ensure_ws(c, s, B));
        uint32_t lr_bits;
        std::memcpy(&lr_bits, &c->lr_host, 4);
        TGP_TRY(put_u32(s.comp, s.dlr, lr_bits));
        TGP_TRY(run_task(c, s, s.gWs, B, [&] { return exec_wgrad(c, s, B, true); }));
        s.grads_fresh = true;  // consumed by the fused step
      } else if (s.grads_fresh) {
        // the W graph bakes in the accumulate flag -> only replay when grads are fresh
        TGP_TRY(run_task(c, s, s.gW, B, [&] { return exec_wgrad(c, s, B); }));
        s.grads_fresh = false;
      } else {
        TGP_TRY(exec_wgrad(c, s, B));
      }
      if (c->fuse_sgd && !s.grads_fresh) {  // tgp_backward_step without the fused path: W_j, then SGD
        TGP_TRY(sgd_step(s.comp, s.master, s.grad, s.shadow, s.n_elems, c->lr_host));
        c->kernels++;
        s.grads_fresh = true;
      }
      trace_end(c, s, s.comp, 0, rc.kind, 0, ta);
      c->issue_log.push_back(rc);
      return 0;
    }
  }
  return 0;
}

// Bounded host wait for every local stream of the call ("a handshake wait past the
// watchdog -> TGP_E_TIMEOUT"; the host issues, the device waits).  A lost message or
// flag leaves a consumer stream in cuStreamWaitValue32 forever; past `watchdog_ms` the call returns
// TGP_E_TIMEOUT instead of hanging.  It first tries to release every local receive flag far ahead of
// any sequence number from a fresh stream and to drain the device (bounded); the context is failed
// either way (the call's results are garbage).  Measured on B200: while a stream-memory wait is
// pending the release kernel may not get to run (profiles/diag/wd_dbg.py), so when the device does
// not drain the context is also marked wedged: tgp_destroy then skips every CUDA call that could
// block and leaks the device memory to process exit, where the driver reclaims it.
static bool streams_idle(tgp_ctx* c) {
  for (Stage* q : c->local) {
    if (!q) continue;
    cudaSetDevice(q->dev);
    for (cudaStream_t st : {q->comp, q->cact, q->cskip, q->comp2 ? q->comp2 : q->comp})
      if (cudaStreamQuery(st) == cudaErrorNotReady) return false;
  }
  return true;
}

static int sync_with_watchdog(tgp_ctx* c) {
  const auto t0 = std::chrono::steady_clock::now();
  auto ms_since = [](std::chrono::steady_clock::time_point t) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
  };
  for (int j = 0; j < c->n; ++j) {
    Stage* sp = c->local[j];
    if (!sp) continue;
    TGP_CUDA_TRY(cudaSetDevice(sp->dev));
    for (cudaStream_t st : {sp->comp, sp->cact, sp->cskip, sp->comp2 ? sp->comp2 : sp->comp}) {
      while (true) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) break;
        if (e != cudaErrorNotReady) {
          set_error("CUDA error: %s", cudaGetErrorString(e));
          return TGP_E_CUDA;
        }
        if (c->watchdog_ms > 0 && ms_since(t0) > (double)c->watchdog_ms) {
          for (Stage* q : c->local) {
            if (!q) continue;
            cudaSetDevice(q->dev);
            cudaStream_t rs = nullptr;
            if (cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking) == cudaSuccess)
              fill_flags(rs, q->self.flags, n_flags(c), c->seq + 0x40000000u);  // stream leaked if wedged
          }
          const auto t1 = std::chrono::steady_clock::now();
          bool idle = false;
          while (!(idle = streams_idle(c)) && ms_since(t1) < 2000.0)
            std::this_thread::sleep_for(std::chrono::microseconds(100));
          c->failed = true;
          c->wedged = !idle;
          set_error("watchdog: partition %d (device %d) did not complete the call within %lld ms (a lost message or "
                    "flag); %s -- destroy the context",
                    j, sp->dev, (long long)c->watchdog_ms,
                    idle ? "waits released, device drained" : "device did not drain (resources leak to process exit)");
          return TGP_E_TIMEOUT;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    }
  }
  return 0;
}

// Timeline records of the finished calls (needs their events complete: after a host wait).
static void drain_trace(tgp_ctx* c) {
  for (auto& t : c->trace_recs) {
    Stage* s = c->local[t.part];
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, s->ev_epoch, t.a);
    cudaEventElapsedTime(&b, s->ev_epoch, t.b);
    int64_t rec[6] = {t.part, t.stream, t.kind, t.i, (int64_t)(a * 1e6), (int64_t)(b * 1e6)};
    c->timeline.insert(c->timeline.end(), rec, rec + 6);
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  c->trace_recs.clear();
}

// Asynchronous stream-ordered calls (tgp_*_async).  enter: every local partition's
// compute stream waits for the work the caller queued on `st` before the call (its inputs' producers);
// leave: each partition joins its other lanes (comp2, copy streams) into comp, and `st` waits for every
// partition, so whatever the caller queues next on `st` sees the call's results.  No host wait.
static int async_enter(tgp_ctx* c, cudaStream_t st) {
  int dev = -1;
  if (cudaStreamGetDevice(st, &dev) != cudaSuccess) {
    cudaGetLastError();
    TGP_CUDA_TRY(cudaGetDevice(&dev));
  }
  if (!c->ev_user || c->ev_user_dev != dev) {
    TGP_CUDA_TRY(cudaSetDevice(dev));
    if (c->ev_user) cudaEventDestroy(c->ev_user);
    c->ev_user = nullptr;
    TGP_CUDA_TRY(cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming));
    c->ev_user_dev = dev;
  }
  TGP_CUDA_TRY(cudaSetDevice(dev));
  TGP_CUDA_TRY(cudaEventRecord(c->ev_user, st));
  for (Stage* s : c->local)
    if (s) {
      TGP_CUDA_TRY(cudaSetDevice(s->dev));
      TGP_CUDA_TRY(cudaStreamWaitEvent(s->comp, c->ev_user, 0));
    }
  c->async_call = true;
  c->ustream = st;
  return 0;
}

static int async_leave(tgp_ctx* c) {
  cudaStream_t st = c->ustream;
  c->async_call = false;
  c->ustream = nullptr;
  for (Stage* s : c->local) {
    if (!s) continue;
    TGP_CUDA_TRY(cudaSetDevice(s->dev));
    const cudaStream_t lanes[3] = {s->comp2, s->cact, s->cskip};
    for (int k = 0; k < 3; ++k)
      if (lanes[k]) {
        TGP_CUDA_TRY(cudaEventRecord(s->ev_join[k], lanes[k]));
        TGP_CUDA_TRY(cudaStreamWaitEvent(s->comp, s->ev_join[k], 0));
      }
    TGP_CUDA_TRY(cudaEventRecord(s->ev_done, s->comp));
  }
  TGP_CUDA_TRY(cudaSetDevice(c->ev_user_dev));
  for (Stage* s : c->local)
    if (s) TGP_CUDA_TRY(cudaStreamWaitEvent(st, s->ev_done, 0));
  return 0;
}

static int finish_call(tgp_ctx* c) {
  // tell every partition that writes into a local partition that this call is done on it
  for (int j = 0; j < c->n; ++j) {
    Stage* sp = c->local[j];
    if (!sp) continue;
    for (int k : writers_of(c, j)) {
      TGP_TRY(signal_flag(sp->comp, flag_done(c, c->view[k], j), c->seq));
      c->kernels++;
    }
  }
  if (c->async_call) return 0;  // the caller's stream is joined by async_leave; tgp_sync waits
  TGP_TRY(sync_with_watchdog(c));
  if (c->trace) drain_trace(c);
  return 0;
}

static int begin_call(tgp_ctx* c) {
  c->seq++;
  for (Stage* s : c->local)
    if (s) s->abl_next = 0;
  for (Stage* s : c->local)
    if (s) {  // the fused-send flags carry the call's sequence number (read on the device)
      TGP_CUDA_TRY(cudaSetDevice(s->dev));
      TGP_TRY(put_u32(s->comp, s->dseq, c->seq));
    }
  for (int j = 0; j < c->n; ++j) {
    Stage* sp = c->local[j];
    if (!sp) continue;
    TGP_CUDA_TRY(cudaSetDevice(sp->dev));
    TGP_CUDA_TRY(cudaEventRecord(sp->ev_start, sp->comp));
    // copy streams must not run ahead of the call's start (events of the previous call)
    TGP_CUDA_TRY(cudaStreamWaitEvent(sp->cact, sp->ev_start, 0));
    TGP_CUDA_TRY(cudaStreamWaitEvent(sp->cskip, sp->ev_start, 0));
    if (sp->comp2) TGP_CUDA_TRY(cudaStreamWaitEvent(sp->comp2, sp->ev_start, 0));
  }
  return 0;
}

// ============================================================================ ABI
extern "C" {

const char* tgp_last_error(void) { return get_error(); }

tgp_status tgp_balance(const double* cost, int32_t L, int32_t n, int32_t* out) {
  if (!cost || !out || L < 1 || n < 1 || n > L) {
    set_error("tgp_balance: need 1 <= n_parts <= n_layers");
    return TGP_E_INVALID;
  }
  std::vector<int> tmp(n);
  if (!balance_minmax(cost, L, n, tmp.data())) {
    set_error("tgp_balance failed");
    return TGP_E_INVALID;
  }
  for (int j = 0; j < n; ++j) out[j] = tmp[j];
  return TGP_OK;
}

tgp_status tgp_profile_size(const tgp_layer* layers, int32_t L, int32_t rows, double* out) {
  if (!layers || !out || L < 1 || rows < 1) {
    set_error("tgp_profile_size: need layers, n_layers >= 1, rows >= 1");
    return TGP_E_INVALID;
  }
  for (int l = 0; l < L; ++l) {
    const tgp_layer& x = layers[l];
    const double di = x.d_in, dout = x.d_out, H = x.d_hidden;
    double skip = 0.0;
    if (x.kind == TGP_MERGE)
      for (int q = 0; q < L; ++q)
        if (layers[q].stash_route >= 0 && layers[q].stash_route == x.pop_route) skip = layers[q].d_out;
    double params = 0.0;
    switch (x.kind) {
      case TGP_LINEAR: params = dout * di + dout; break;
      case TGP_MERGE: params = dout * (di + skip) + dout; break;
      case TGP_RESMLP: params = 2 * di + H * di + H + dout * H + dout; break;
      case TGP_BATCHNORM:
      case TGP_LAYERNORM: params = 2 * di; break;
      case TGP_DROPOUT: params = 0.0; break;
      case TGP_EMBED: params = ((double)x.vocab + x.seq) * dout; break;
      case TGP_TRANSFORMER: params = 2 * di + 3 * di * di + 3 * di + di * di + di + 2 * di + H * di + H + di * H + di; break;
      case TGP_LMHEAD: params = 2 * di + dout * di; break;
      default:
        set_error("tgp_profile_size: layer %d has unknown kind %d", l, x.kind);
        return TGP_E_INVALID;
    }
    out[l] = 8.0 * params + (double)rows * dout * 4.0;
  }
  return TGP_OK;
}

tgp_status tgp_split(int32_t B, int32_t m, int32_t* sizes) {
  if (!sizes || m < 1 || m > B) {
    set_error("tgp_split: need 1 <= m <= B (m=%d B=%d)", m, B);
    return TGP_E_INVALID;
  }
  std::vector<int> t(m);
  split_sizes(B, m, t.data());
  for (int i = 0; i < m; ++i) sizes[i] = t[i];
  return TGP_OK;
}

static tgp_status schedule_impl(const char* who, int32_t m, int32_t n, tgp_checkpoint ckpt, const int32_t* routes,
                                int32_t n_routes, bool relay, uint64_t order_seed, int32_t* rec, int64_t cap,
                                int64_t* n_rec) {
  if (m < 1 || n < 1 || (int)ckpt < 0 || (int)ckpt > 2 || n_routes < 0 || (n_routes > 0 && !routes)) {
    set_error("%s: bad arguments", who);
    return TGP_E_INVALID;
  }
  std::vector<std::pair<int, int>> r;
  for (int q = 0; q < n_routes; ++q) {
    if (routes[2 * q] < 1 || routes[2 * q + 1] < routes[2 * q] || routes[2 * q + 1] > n) {
      set_error("%s: route %d must satisfy 1 <= src <= dst <= n", who, q);
      return TGP_E_INVALID;
    }
    r.emplace_back(routes[2 * q], routes[2 * q + 1]);
  }
  auto recs = emit_schedule(m, n, (int)ckpt, r, relay);
  if (order_seed) {
    std::vector<Rec> f, w;
    for (const Rec& x : recs) (x.phase == 0 ? f : w).push_back(x);
    auto b = unordered_backward(m, n, (int)ckpt, r, relay, order_seed);
    recs = f;
    for (const Rec& x : b) recs.push_back(x);
    for (const Rec& x : w)
      if (x.phase == 2) recs.push_back(x);
  }
  if (n_rec) *n_rec = (int64_t)recs.size();
  if (rec) {
    if (cap < (int64_t)recs.size()) {
      set_error("%s: cap %lld < %zu records", who, (long long)cap, recs.size());
      return TGP_E_INVALID;
    }
    memcpy(rec, recs.data(), recs.size() * sizeof(Rec));
  }
  return TGP_OK;
}

tgp_status tgp_schedule(int32_t m, int32_t n, tgp_checkpoint ckpt, const int32_t* routes, int32_t n_routes,
                        int32_t* rec, int64_t cap, int64_t* n_rec) {
  return schedule_impl("tgp_schedule", m, n, ckpt, routes, n_routes, false, 0, rec, cap, n_rec);
}

tgp_status tgp_schedule_ablation(int32_t m, int32_t n, tgp_checkpoint ckpt, const int32_t* routes, int32_t n_routes,
                                 int32_t relay, uint64_t order_seed, int32_t* rec, int64_t cap, int64_t* n_rec) {
  return schedule_impl("tgp_schedule_ablation", m, n, ckpt, routes, n_routes, relay != 0, order_seed, rec, cap, n_rec);
}

}  // extern "C"

#include "runtime_create.inc"
