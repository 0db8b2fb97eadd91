// Persistent weight-streaming task kernel: ONE launch executes a whole GPipe compute task of a
// partition made of pre-LN residual MLP blocks -- F_{i,j} / F'_{i,j} (PAPER.md Eq. F_{i,j},
// P:52-55; recompute P:105) or B_{i,j} (Eq. B_{i,j}) -- for one micro-batch of
// M <= 16 rows.
//
// Why: at 16 rows per micro-batch every dense layer is a weight-streaming GEMM (arithmetic
// intensity 15.9 FLOP/B): the task is a chain of 2 dependent 32 MiB weight reads
// per block.  As separate kernels, every boundary drains and refills the HBM pipe.  Here the weight
// stream of every CTA is static and independent of the activations, so it runs ahead continuously
// across all GEMMs of the task; only the tiny activation operand of a GEMM waits for its producers,
// and it is loaded once per phase (this rank's K quarter x 16 or 32 rows).
//
// Two-level weight buffer (so the stream keeps running while a phase waits for its activations):
// TMA lands 16 KB weight tiles in a shared-memory ring; four copy warps move every landed tile into
// a ring of 12 TMEM slots (ld.shared -> tcgen05.st, the A-operand layout: one output feature per
// lane, two bf16 of K per 32-bit column) and free its shared stage at once; the MMA reads A from
// TMEM (tcgen05.mma A-in-TMEM, B = activations in shared memory).  The bytes in flight per SM are
// bounded by the shared ring, the time a CTA can keep streaming through a dependency wait by both
// rings (17 - 22 tiles); that matters most on the half grid, where a CTA streams 32 tiles per
// phase.  (tcgen05.cp would do the copy on the in-order tensor pipe, where it measured slower.)
//
// Work split (grid = C clusters x 4 CTAs, one CTA per SM):
//  * every GEMM phase has out-features F (H or d) in 128-row slabs; a cluster owns NV slabs (NV = 1:
//    the full grid, C = max(d, H) / 128; NV = 2: the half grid of a PAIRED task, runtime.cu: F'_{i-1}
//    runs beside B_i, each on half the SMs); its 4 CTAs split K in quarters (swap-AB tcgen05.mma
//    M = 128 features x N = 16 rows, fp32 in TMEM).  A unit = (phase, slab); the weight stream and
//    the MMAs go unit by unit, and the two slabs of a phase have their own epilogue warp groups, so
//    their epilogues (and dependency waits) run side by side;
//  * split-K partials are reduced inside the cluster: each rank pushes 32-feature slices of its
//    TMEM tile into the owning rank's shared memory with st.async (completion on the owner's
//    mbarrier); the owner sums the 4 sources in fixed rank order (deterministic -> F' == F
//    bitwise on either grid, reading Z21) and runs the epilogue for its 32 features x 16 rows;
//  * dependencies are counters (one 128-byte line each): an owner signals "my 32 outputs of
//    phase p are written" with a release increment on the counter of the K-quarter they fall in;
//    a CTA of the next phase polls only the counter of its own K-quarter before the TMA load of its
//    activation operand.  Row reductions (LayerNorm statistics forward, LayerNorm backward sums)
//    go through per-32-feature chunk statistics and one global counter, combined in fixed order.
//
// Phases.  Forward, block l (ids are dependency counters):
//   input y of block l (x for l = 0): operand gamma (y - mu~) bf16 (id 1 + 3l, quarters) and LN
//                                     chunk statistics (id 3 + 3l, global)
//   GEMM1 a = LN(y) W1^T + b1, LayerNorm folded (see ln_produce) -> g = dropout(GELU(a)) bf16
//                                                                   (id 2 + 3l)
//   GEMM2 y' = y + g W2^T + b2 -> the next block's operand and statistics (ids 4 + 3l, 6 + 3l)
// Backward, k = 0..L-1 over blocks l = L-1-k:
//   [k = 0] dY_top bf16 + db2 column sums (id 1)
//   dG = dY W2 -> dA = dG * dropout' * GELU'(a) bf16, db1 column sums       (id 2 + 3k)
//   dH = dA W1 -> LN backward row sums (id 3 + 3k) -> dx = gy + LN_bwd(dH);
//                 dgamma, dbeta column sums; [l > 0] dY_{l-1} = dx bf16, db2 sums (id 4 + 3k)
#include <cuda_bf16.h>

#include <type_traits>

#include "common.cuh"
#include "host.h"
#include "kernels.h"
#include "task_stream.h"

namespace tgp {

namespace {
constexpr int SK = 4;                       // split-K ranks per cluster
constexpr int ST_A = 16384;                 // 128 x 64 bf16 weight tile
constexpr int KB_MAX = 16;                  // k-blocks of 64 per phase and CTA (K <= 4096)
// Shared-memory layout (the backward's dG phases have 32-row operands; a receive buffer per
// epilogue group and TMEM accumulator buffer):
//   ring NST x 16 KB | activation operand 16 x ATILE | receive NV x 2 x RECV | misc 8 KB
//   forward : ATILE 2 KB, RECV  8 KB, NST 10 (NV = 1) / 9 (NV = 2)       -> 208 KB + misc
//   backward: ATILE 4 KB, RECV 16 KB, NST  7 (NV = 1) / 5 (NV = 2)       -> 208 KB + misc
template <bool BWD, int NV>
struct StCfg {
  static constexpr int NST = BWD ? (NV == 2 ? 5 : 7) : (NV == 2 ? 9 : 10);
  static constexpr int ATILE = BWD ? 4096 : 2048;
  static constexpr int NCOLMAX = BWD ? 32 : 16;
  static constexpr int RECV = SK * 32 * NCOLMAX * 4;
  static constexpr int OFF_ACT = NST * ST_A;
  static constexpr int OFF_RECV = OFF_ACT + KB_MAX * ATILE;
  static constexpr int OFF_BAR = OFF_RECV + NV * 2 * RECV;
  static constexpr int SMEM = OFF_BAR + 8192 + 1024;
  // TMEM: one accumulator of 32 columns per epilogue group, then NSLOT weight slots of 32 columns.
  // A group's consecutive units are consecutive phases, and phase p + 1's activations exist only after
  // every owner's epilogue of phase p -- which drained the accumulator first -- so a second
  // accumulator buffer would never be used concurrently; its 32 columns hold one more weight slot.
  // (NCOLMAX columns: 16 rows forward, the backward's 32-row [u | n] dG operand)
  static constexpr int ACC = NV * NCOLMAX;
  static constexpr int NSLOT = (512 - ACC) / 32;  // 15, except 14 on the half grid of a backward task
};
constexpr int ST_SMEM_MAX = StCfg<false, 1>::SMEM > StCfg<true, 2>::SMEM ? StCfg<false, 1>::SMEM : StCfg<true, 2>::SMEM;
// warps: TMA, MMA, poller, NV epilogue groups of 4, 4 copy -> 352 (NV = 1) / 480 (NV = 2) threads
template <int NV>
constexpr int st_threads() { return (3 + 4 * NV + 4) * 32; }
constexpr int CNT_STRIDE = 32;   // uints between counters (one 128-byte line each)
static_assert(StCfg<false, 1>::SMEM <= 227 * 1024 && StCfg<false, 2>::SMEM <= 227 * 1024 &&
                  StCfg<true, 1>::SMEM <= 227 * 1024 && StCfg<true, 2>::SMEM <= 227 * 1024,
              "stream kernel shared memory");
}  // namespace

TGP_DEV unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
TGP_DEV void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Acquire side of a counter that a relaxed poll has seen reach its target: one ld.acquire re-read of
// the counter (LDG.STRONG + L1 invalidate) instead of a full fence (MEMBAR.ALL.GPU, which also waits
// for the warp's outstanding memory operations).  The counter only grows within a task and every
// increment is a release RMW, so the acquire synchronises with all of them.
TGP_DEV void acquire_counter(const unsigned* p) {
#ifndef TGP_ST_FENCE_ACQ
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  (void)v;
#else
  (void)p;
  fence_acq_rel_gpu();
#endif
}
TGP_DEV void st_release_cta_u32(uint32_t saddr, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
TGP_DEV uint32_t ld_acquire_cta_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}
TGP_DEV void dbg_stamp(const STask& t, int p, int slot) {
  if (!t.dbg) return;
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  t.dbg[((size_t)blockIdx.x * 2 * t.L + p) * ST_DBG_SLOTS + slot] = v;
}

TGP_DEV uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
TGP_DEV uint4 lds_u128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}
// 32 lanes x 32 bit, 32 consecutive columns per thread (thread = lane of its warp's quadrant)
TGP_DEV void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
TGP_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// 16 lanes x 4 x 256 bit: per 8-column chunk c (registers 4c .. 4c + 3) thread t writes lane t/4
// (r0, r1) and lane t/4 + 8 (r2, r3), columns 8c + 2(t%4), +1
TGP_DEV void tmem_st_16x256b_x4(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// four 8x8 b16 matrices, transposed: thread t gets {M[2(t%4)][t/4], M[2(t%4)+1][t/4]} of matrix i in
// register i; threads 8i..8i+7 give the row addresses of matrix i
TGP_DEV void ldsm_x4_trans(uint32_t a, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a)
               : "memory");
}

template <typename T>
TGP_DEV T wsum32(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Ph {
  const CUtensorMap* A;  // the phase's weight matrix (tensor map of the layout the phase streams)
  const CUtensorMap* B;  // its activation operand
  int K, F;              // contraction length, output features
};

TGP_DEV Ph phase_of(const STask& t, int p) {
  const int k = p >> 1, sub = p & 1;
  const int l = t.bwd ? t.L - 1 - k : k;
  const SLayer& Ly = t.layers[l];
  if (!t.bwd) return sub ? Ph{&Ly.w2k, &Ly.gop, t.H, t.d} : Ph{&Ly.w1k, &Ly.ygm, t.d, t.H};
  return sub ? Ph{&Ly.w1m, &Ly.daop, t.H, t.d} : Ph{&Ly.w2m, &Ly.ucm, t.d, t.H};
}

template <bool BWD, int NV>
__global__ void __launch_bounds__(st_threads<NV>(), 1) task_stream_kernel(const __grid_constant__ STask t) {
  using Cfg = StCfg<BWD, NV>;
  constexpr int NST = Cfg::NST, ATILE = Cfg::ATILE, RECV = Cfg::RECV, OFF_BAR = Cfg::OFF_BAR;
  constexpr int NSLOT = Cfg::NSLOT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* act = smem + Cfg::OFF_ACT;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);  // [NST] weight tile landed in the ring
  uint64_t* empty = full + 16;   // [NST] ring stage read by the copy warps (4 arrivals)
  uint64_t* aempty = empty + 16; // [NSLOT <= 16] TMEM weight slot consumed by the MMAs (commit)
  uint64_t* tfull = aempty + 16; // [2 groups][2] TMEM accumulator ready (index 2 g)
  uint64_t* tempty = tfull + 4;  // [2][2] TMEM accumulator drained (128 arrivals; index 2 g)
  uint64_t* rbar = tempty + 4;   // [2][2] split-K partials of a unit received (owner)
  uint64_t* bfull = rbar + 4;    // activation operand of the current phase landed (TMA)
  uint64_t* bempty = bfull + 1;  // activation operand consumed (commit after the phase's MMAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int cl = blockIdx.x / SK, ncl = gridDim.x / SK;
  auto slab_of = [&](int v) { return cl + v * ncl; };  // v = epilogue group
  const int NP = 2 * t.L, NU = NP * NV;
  const int d = t.d, H = t.H, M = t.M;
  auto unit_active = [&](int u) { return slab_of(u % NV) * 128 < phase_of(t, u / NV).F; };
  // rows of a phase's activation operand / MMA N: the backward's dG phases take [u | n] (32 rows,
  // LayerNorm backward folded, see the backward epilogue), every other phase the 16 micro-batch rows
  auto ncol = [&](int p) { return (BWD && !(p & 1)) ? 32 : 16; };
  // active units of this CTA in order (NU past the end), and per epilogue group
  uint16_t* act_list = reinterpret_cast<uint16_t*>(smem + OFF_BAR + 5120);  // [<= 256]
  uint16_t* grp_list = act_list + 256;                                      // [2][<= 128]
  auto nth_active = [&](int k) { return k < NU ? (int)act_list[k] : NU; };
  auto nth_group = [&](int g, int k) { return NV == 1 ? nth_active(k) : (k < NP ? (int)grp_list[g * 128 + k] : NU); };
  // phases < *released have their activation dependency met (written by the poller warp with
  // st.release.cta after its gpu-scope acquire; read by the producer with ld.acquire.cta)
  const uint32_t released = smem_u32(smem + OFF_BAR + 6144);
  // loaded phases whose MMAs have started (MMA issuer, st.release.cta; read by the copy warps)
  const uint32_t mstart = smem_u32(smem + OFF_BAR + 6176);
  auto recv_bytes = [&](int u) { return (uint32_t)(SK * 32 * ncol(u / NV) * 4); };
  auto cnt = [&](int id, int q) { return t.cnt + ((size_t)id * 5 + q) * CNT_STRIDE; };

  if (warp == 0 && lane == 0) {
    int na = 0, ng[2] = {0, 0};
    for (int u = 0; u < NU; ++u)
      if (unit_active(u)) {
        act_list[na++] = (uint16_t)u;
        if (NV == 2) grp_list[(u % NV) * 128 + ng[u % NV]++] = (uint16_t)u;
      }
    for (int k = na; k < NU; ++k) act_list[k] = (uint16_t)NU;
    if (NV == 2)
      for (int g = 0; g < 2; ++g)
        for (int k = ng[g]; k < 128; ++k) grp_list[g * 128 + k] = (uint16_t)NU;
    st_release_cta_u32(released, 0u);
    st_release_cta_u32(mstart, 0u);
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    for (int s = 0; s < NSLOT; ++s) mbar_init(&aempty[s], 1);
    for (int w = 0; w < 4; ++w) st_release_cta_u32(smem_u32(smem + OFF_BAR + 6160 + 4 * w), 0u);
    for (int b = 0; b < 4; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
      mbar_init(&rbar[b], 1);
    }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    fence_barrier_init();
    // first use of each receive buffer: 4 sources x 32 features x ncol rows x 4 B
    for (int g = 0; g < NV; ++g)
      for (int b = 0; b < 2; ++b) {
        const int u = nth_group(g, b);
        if (u < NU) mbar_arrive_expect_tx(&rbar[g * 2 + b], recv_bytes(u));
      }
  }
  // TMEM: [0, 32 NSLOT): NSLOT weight slots of 32 columns; then group g's fp32 accumulator at
  // 32 NSLOT + NCOLMAX g (16 or 32 columns)
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // every rank's receive barriers are initialised before any st.async
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first(), pol_b = policy_evict_last();
      auto next_unit = [&](int u) {
        while (u < NU && !unit_active(u)) ++u;
        return u;
      };
      auto next_phase = [&](int p) {  // first phase >= p with an active unit
        while (p < NP) {
          bool any = false;
#pragma unroll
          for (int v = 0; v < NV; ++v) any = any || unit_active(p * NV + v);
          if (any) break;
          ++p;
        }
        return p;
      };
      int wu = next_unit(0), wkb = 0, it = 0;  // weight cursor: unit, k-block, ring tile
      int rp = next_phase(0), nb = 0;          // next phase whose activations are to be loaded; loads issued
      while (wu < NU || rp < NP) {
        bool progress = false;
        while (wu < NU) {  // weights: run ahead as far as the ring allows
          const int s = it % NST, r = it / NST;
          if (!mbar_test_wait(smem_u32(&empty[s]), (uint32_t)((r & 1) ^ 1))) break;
          if (t.inflight && (int)t.inflight < NST && it >= (int)t.inflight) {
            // at most `inflight` weight tiles in flight: tile it - inflight has landed (its stage is
            // not re-armed before tile it - inflight + NST > it is issued, so the parity is unambiguous)
            const int o = it - (int)t.inflight;
            if (!mbar_test_wait(smem_u32(&full[o % NST]), (uint32_t)((o / NST) & 1))) break;
          }
          const int wp = wu / NV, slab = slab_of(wu % NV);
          const Ph P = phase_of(t, wp);
          const int nkb = P.K / (SK * 64);
          const int kc = (rank * nkb + wkb) * 64;
          if (wkb == 0) dbg_stamp(t, wp, 1);
          if (wkb == nkb - 1) dbg_stamp(t, wp, 2);
          uint8_t* dst = ring + s * ST_A;
          mbar_arrive_expect_tx(&full[s], (uint32_t)ST_A);
          if (!BWD) {
            tma_load_2d(P.A, &full[s], dst, kc, slab * 128, pol_w);
          } else {
            tma_load_2d(P.A, &full[s], dst, slab * 128, kc, pol_w);
            tma_load_2d(P.A, &full[s], dst + 8192, slab * 128 + 64, kc, pol_w);
          }
          ++it;
          progress = true;
          if (++wkb == nkb) {
            wkb = 0;
            wu = next_unit(wu + 1);
          }
        }
        // activations of phase rp: once released (poller) and the previous phase's MMAs have
        // consumed the single activation buffer
        if (rp < NP && (int)ld_acquire_cta_u32(released) > rp &&
            (nb == 0 || mbar_test_wait(smem_u32(bempty), (uint32_t)((nb - 1) & 1)))) {
          asm volatile("fence.proxy.async.global;" ::: "memory");
          dbg_stamp(t, rp, 0);
          const Ph P = phase_of(t, rp);
          const int nkb = P.K / (SK * 64);
          // forward GEMM1 reads the [16][d] task scratch gamma (y - mu~), the backward's dG the [32][d]
          // scratch [u | n] (both row 0), all others the stash rows of the micro-batch
          const int row = !(rp & 1) ? 0 : t.r0;
          mbar_arrive_expect_tx(bfull, (uint32_t)(nkb * 128 * ncol(rp)));
          for (int kb = 0; kb < nkb; ++kb) tma_load_2d(P.B, bfull, act + kb * ATILE, (rank * nkb + kb) * 64, row, pol_b);
          ++nb;
          rp = next_phase(rp + 1);
          progress = true;
        }
        if (!progress) __nanosleep(t.sleep_ns);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ------------------------------------------------------------ MMA issuer (single thread)
      // A (weights) from the TMEM slots, B (activations) from the phase's activation buffer;
      // accumulator of unit u in its group's double buffer
      const uint32_t idesc16 = make_idesc_bf16(128, 16, false, false);
      const uint32_t idesc32 = make_idesc_bf16(128, 32, false, false);
      const uint32_t act0 = smem_u32(act);
      const uint32_t copied = smem_u32(smem + OFF_BAR + 6160);
      int g = 0, ready = 0, nload = 0, ng[2] = {0, 0};
      for (int k = 0; k < NU; ++k) {
        const int u = nth_active(k);
        if (u >= NU) break;
        const int p = u / NV, grp = u % NV;
        const bool first = k == 0 || nth_active(k - 1) / NV != p;  // first / last unit of its phase
        const int un = nth_active(k + 1);
        const bool last = un >= NU || un / NV != p;
        const int nkb = phase_of(t, p).K / (SK * 64);
        const uint32_t idesc = ncol(p) == 32 ? idesc32 : idesc16;
        mbar_wait(&tempty[grp * 2], (uint32_t)((ng[grp] & 1) ^ 1));
        if (first) {
          mbar_wait(bfull, (uint32_t)(nload & 1));
          if constexpr (NV == 1 && !BWD) st_release_cta_u32(mstart, (uint32_t)(nload + 1));
        }
        tc_fence_after();
        const uint32_t dacc = tmem + (uint32_t)(NSLOT * 32 + grp * Cfg::NCOLMAX);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int slot = g % NSLOT;
          if (g >= ready) {
            // tiles [0, ready) are in TMEM: the minimum over the four copy warps' counters (one
            // shared-memory acquire instead of an mbarrier probe per tile, which costs ~200 clk
            // between MMAs)
            do {
              ready = 0x7fffffff;
#pragma unroll
              for (int w = 0; w < 4; ++w) ready = min(ready, (int)ld_acquire_cta_u32(copied + 4u * w));
            } while (ready <= g);
            tc_fence_after();
          }
          if (kb == 0) dbg_stamp(t, p, 3);
          if (kb == nkb / 2) dbg_stamp(t, p, 10);
          const uint32_t ta = tmem + (uint32_t)(slot * 32);
          const uint32_t b = act0 + (uint32_t)(kb * ATILE);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_bf16_ts(dacc, ta + (uint32_t)(kk * 8), make_sdesc_sw128(b + kk * 32, 16, 1024), idesc,
                           (kb | kk) ? 1u : 0u);
          tc_commit(&aempty[slot]);  // the slot is free once its 4 MMAs completed
        }
        dbg_stamp(t, p, 4);
        tc_commit(&tfull[grp * 2]);
        if (last) {
          tc_commit(bempty);
          ++nload;
        }
        ++ng[grp];
      }
    }
    __syncwarp();
  } else if (warp >= 3 + 4 * NV) {
    // ------------------------------------------------------------ copy warps: ring -> TMEM slots
    // Warp w may access TMEM lanes 32 (w % 4) ..; lane f = 32 (w % 4) + lane of the slot holds
    // output feature f of the slab: A[f][k] for the tile's 64 k as 32 columns of bf16 pairs (low
    // half = even k), the K-major A-in-TMEM layout of tcgen05.mma (tc_mma_bf16_ts).
    const int q = warp & 3, f = 32 * q + lane;
    const uint32_t copied = smem_u32(smem + OFF_BAR + 6160);  // [4] tiles this copy warp has in TMEM
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16);
    const uint32_t ring0 = smem_u32(ring);
    int g = 0;
    int pord = -1, lastp = -1, dph = 0;  // loaded-phase ordinal of the tile, MMA-complete phases
    for (int k = 0; k < NU; ++k) {
      const int u = nth_active(k);
      if (u >= NU) break;
      const int p = u / NV;
      if (p != lastp) {
        ++pord;
        lastp = p;
      }
      const int nkb = phase_of(t, p).K / (SK * 64);
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % NST, r = g / NST;
        const int slot = g % NSLOT, rs = g / NSLOT;
        mbar_wait(&full[s], (uint32_t)(r & 1));
        uint32_t v[32];
        const uint32_t base = ring0 + (uint32_t)(s * ST_A);
        if (!BWD) {
          // K-major tile [128 f][64 k], 128-byte rows, 16-byte chunk c of row f at chunk c ^ (f & 7)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 w = lds_u128(base + (uint32_t)(f * 128 + ((c ^ (f & 7)) << 4)));
            v[4 * c] = w.x;
            v[4 * c + 1] = w.y;
            v[4 * c + 2] = w.z;
            v[4 * c + 3] = w.w;
          }
        } else {
          // MN-major tile: two [64 k][64 f] halves of 8 KB, element (k, f) of half f / 64 in 128-byte
          // row k, 16-byte chunk ((f % 64) / 8) ^ (k & 7), position f % 8 (the transpose of A).
          // Transposed 8x8 loads straight into the 16x256b TMEM-store fragment: chunk (h2, cc) =
          // lanes 32q + 16 h2 + [0, 16) (feature groups jj = 4q + 2 h2 + {0, 1}) x k-pair columns
          // 8 cc + [0, 8).  Matrix i = (jj offset i / 2, k rows 16 cc + {0,1,4,5,8,9,12,13} + 2 (i % 2)),
          // so thread t receives k pairs 8 cc + 2 (t % 4) (+ 1) of features 8 jj + t / 4: registers
          // v[4 (4 h2 + cc) ..] = r0..r3 of tcgen05.st.16x256b.
          const int mi = lane >> 3, ri = lane & 7;
          const int kr = ((ri >> 1) << 2) + (ri & 1) + 2 * (mi & 1);
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int jj = 4 * q + 2 * h2 + (mi >> 1);
            const uint32_t hb = base + (uint32_t)((jj >> 3) * 8192);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              const int k = 16 * cc + kr;
              ldsm_x4_trans(hb + (uint32_t)(k * 128 + (((jj & 7) ^ (k & 7)) << 4)), v + 4 * (4 * h2 + cc));
            }
          }
        }
        // the stage goes back to the TMA (async proxy) only after these generic-proxy reads: without
        // the fence (and the "memory" clobbers of lds_*, which keep the compiler from sinking the
        // loads below the arrive) the next tile could land before a copy warp has read this one --
        // a race that showed as non-deterministic forward results at d = 4096
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // the ring stage is free (the tile is in registers)
        mbar_wait(&aempty[slot], (uint32_t)((rs & 1) ^ 1));
        if constexpr (NV == 1 && !BWD) {
          // full-grid forward: a tile of a LATER phase waits while the current phase's MMAs run (its
          // tcgen05.st would share TMEM bandwidth with their A-operand reads; F task 512 -> 481 us);
          // tiles of the running phase go at once.  Not on the half grid of a paired task, whose 32
          // tiles per phase need every copy slot (measured: paired F' + B 976 -> 1196 us), and not in
          // the backward, whose heavier tile copies leave a CTA that fell behind no way to catch up:
          // one straggler CTA per launch, 2.5-3 us late in every phase (B 582 -> 517 us without it,
          // profiles/r7/r8p_summary.txt)
          while (true) {
            const int st = (int)ld_acquire_cta_u32(mstart);
            while (dph < st && mbar_test_wait(smem_u32(bempty), (uint32_t)(dph & 1))) ++dph;
            if (!(st > dph && pord >= st)) break;
          }
        }
        tc_fence_after();
        if (!BWD) {
          tmem_st32(trow + (uint32_t)(slot * 32), v);
        } else {
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) tmem_st_16x256b_x4(trow + ((uint32_t)(16 * h2) << 16) + (uint32_t)(slot * 32), v + 16 * h2);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          st_release_cta_u32(copied + 4u * (uint32_t)q, (uint32_t)(g + 1));
          if (q == 0 && kb == nkb - 1) dbg_stamp(t, p, 11);
        }
      }
    }
  } else if (warp == 2) {
    if (lane == 0) {
      // ------------------------------------------------------------ dependency poller
      // for every phase with an active unit, in order: wait for its activation-operand counter,
      // then publish
      int lastp = -1;
      for (int k = 0; k < NU; ++k) {
        const int u = nth_active(k);
        if (u >= NU) break;
        const int p = u / NV;
        if (p == lastp) continue;
        lastp = p;
        const unsigned need = (unsigned)(phase_of(t, p).K / 128);
        const unsigned* dep = cnt(1 + 3 * (p >> 1) + (p & 1), rank);
        while (ld_relaxed_u32(dep) < need) __nanosleep(t.sleep_ns);
        acquire_counter(dep);
        st_release_cta_u32(released, (uint32_t)(p + 1));
      }
    }
    __syncwarp();
  } else if (warp < 3 + 4 * NV) {
    // ------------------------------------------------------------ epilogue group g (128 threads)
    // Owner item: feature fo = slab*128 + rank*32 + lane of the phase's out space (slab = the
    // group's slab), rows 4*ew .. 4*ew+3.  Warp w reads TMEM lane quadrant w % 4.
    const int g = (warp - 3) >> 2;
    const int et = threadIdx.x - 96 - 128 * g, ew = et >> 5, lg = warp & 3;
    const int slab = slab_of(g);
    const int fo = slab * 128 + rank * 32 + lane;
    const int chunk = slab * SK + rank;  // 32-feature chunk index of the owner slice
    const bool own_d = slab * 128 < d, own_h = slab * 128 < H;
    float* grp = reinterpret_cast<float*>(smem + OFF_BAR + 1024 + g * 2048);
    float* rmu = grp;       // [16] row statistics
    float* rrs = grp + 16;  // [16]
    float* rmp = grp + 32;  // [16] forward: mu~ of the current block (previous block's input mean)
    float* rsb = grp + 48;  // [16] backward: rstd of the LN whose backward feeds the current dG
    float* cs = grp + 64;   // [3][4][32] column-sum partials
    float* recv = reinterpret_cast<float*>(smem + Cfg::OFF_RECV + g * 2 * RECV);  // [2][SK][32][ncols]
    int n = 0, cur_p = 0;
    auto epi_bar = [g] {
      if (g == 0)
        asm volatile("bar.sync 1, 128;" ::: "memory");
      else
        asm volatile("bar.sync 2, 128;" ::: "memory");
    };
    // stamps (diagnostics) only for the phase's operand signal, not the statistics signals (q == 4)
    auto signal = [&](int id, int q) {
      if (et == 0 && q < 4) dbg_stamp(t, cur_p, 9);
      epi_bar();
      if (et == 0 && q < 4) dbg_stamp(t, cur_p, 12);  // all 128 threads stored (barrier passed)
      if (et == 0) {
        // release: the epilogue barrier orders the other threads' stores before this reduction
        asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(cnt(id, q)), "r"(1u) : "memory");
        if (q < 4) dbg_stamp(t, cur_p, 7);
      }
    };
    auto wait_cnt = [&](int id, int q, unsigned need) {
      if (et == 0) {
        while (ld_relaxed_u32(cnt(id, q)) < need) __nanosleep(t.sleep_ns);
        acquire_counter(cnt(id, q));
        dbg_stamp(t, cur_p, 8);
      }
      epi_bar();
    };
    // column sums over the 16 rows of up to 3 values per thread (fixed order: rows within a quad,
    // then quads), written by warp 0 of the group to dst[k][fo]
    auto colsums = [&](const float* v0, const float* v1, const float* v2, float* d0, float* d1, float* d2) {
      const float* v[3] = {v0, v1, v2};
      float* dd[3] = {d0, d1, d2};
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (v[k]) cs[(k * 4 + ew) * 32 + lane] = ((v[k][0] + v[k][1]) + v[k][2]) + v[k][3];
      epi_bar();
      if (ew == 0) {
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (v[k] && dd[k])
            dd[k][fo] = ((cs[(k * 4) * 32 + lane] + cs[(k * 4 + 1) * 32 + lane]) + cs[(k * 4 + 2) * 32 + lane]) +
                        cs[(k * 4 + 3) * 32 + lane];
      }
      epi_bar();
    };
    // result of the group's current unit for (fo, rows 4ew..4ew+3) [and, 32-column phases, columns
    // 16 + 4ew..]: TMEM -> push 32-feature slices to their owners -> fixed-order sum of the 4 sources
    auto gemm_result = [&](auto NC, float* acc, float* acc2) {
      const int buf = n & 1, u = n >> 1;
      constexpr int nc = decltype(NC)::value, nq = nc / 4;
      mbar_wait(&tfull[g * 2], (uint32_t)(n & 1));
      tc_fence_after();
      if (et == 0) dbg_stamp(t, cur_p, 5);
      float v[32];
      const uint32_t ta = tmem + (uint32_t)(NSLOT * 32 + g * Cfg::NCOLMAX) + ((uint32_t)(lg * 32) << 16);
      tmem_ld16(ta, v);
      if constexpr (nc == 32) tmem_ld16(ta + 16, v + 16);
      tc_fence_before();
      mbar_arrive(&tempty[g * 2]);
      const uint32_t rb = smem_u32(recv + buf * (RECV / 4));
      const uint32_t dbar = mapa_shared(smem_u32(&rbar[g * 2 + buf]), (uint32_t)lg);
#pragma unroll
      for (int q = 0; q < nq; ++q) {
        const uint32_t idx = (uint32_t)((rank * 32 + lane) * nq + (q ^ (lane & (nq - 1))));
        st_async_f32x4(mapa_shared(rb + idx * 16u, (uint32_t)lg),
                       make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]), dbar);
      }
      mbar_wait(&rbar[g * 2 + buf], (uint32_t)(u & 1));
      if (et == 0) dbg_stamp(t, cur_p, 6);
      const float4* r4 = reinterpret_cast<const float4*>(recv + buf * (RECV / 4));
#pragma unroll
      for (int h = 0; h < nc / 16; ++h) {
        const int q = ew + 4 * h;
        float4 a = r4[(0 * 32 + lane) * nq + (q ^ (lane & (nq - 1)))];
#pragma unroll
        for (int s = 1; s < SK; ++s) {
          const float4 b = r4[(s * 32 + lane) * nq + (q ^ (lane & (nq - 1)))];
          a.x += b.x;
          a.y += b.y;
          a.z += b.z;
          a.w += b.w;
        }
        float* o = h ? acc2 : acc;
        o[0] = a.x;
        o[1] = a.y;
        o[2] = a.z;
        o[3] = a.w;
      }
      // re-arm for this buffer's next use (its pushes come only after every owner signalled
      // this unit, i.e. after the reads above)
      if (et == 0) {
        const int un = nth_group(g, n + 2);
        if (un < NU) mbar_arrive_expect_tx(&rbar[g * 2 + buf], recv_bytes(un));
      }
      ++n;
    };
    // consumer side: wait for all chunk statistics of block l's input, combine them in fixed order
    // (identical in every CTA and group) into rmu / rrs; the previous means move to rmp (mu~ of
    // block l; for block 0 the exact mean, see ln_produce_first).
    auto ln_rows = [&](int l) {
      const int J = d / 32;
      const float* st = t.stats + (size_t)l * J * 32;
      wait_cnt(3 + 3 * l, 4, (unsigned)J);
      const int rr = et >> 3, jl = et & 7;
      float2 sv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int j = jl + 8 * u;
        sv[u] = j < J ? __ldcg(reinterpret_cast<const float2*>(st + ((size_t)j * 16 + rr) * 2)) : make_float2(0.f, 0.f);
      }
      float mu = 0.0f;
#pragma unroll
      for (int u = 0; u < 16; ++u) mu += sv[u].x;
      mu += __shfl_xor_sync(0xffffffffu, mu, 4);
      mu += __shfl_xor_sync(0xffffffffu, mu, 2);
      mu += __shfl_xor_sync(0xffffffffu, mu, 1);
      mu /= (float)J;
      float m2 = 0.0f;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (jl + 8 * u < J) {
          const float dm = sv[u].x - mu;
          m2 += sv[u].y + 32.0f * dm * dm;
        }
      m2 += __shfl_xor_sync(0xffffffffu, m2, 4);
      m2 += __shfl_xor_sync(0xffffffffu, m2, 2);
      m2 += __shfl_xor_sync(0xffffffffu, m2, 1);
      const float rs = 1.0f / sqrtf(m2 / (float)d + 1e-5f);
      if (jl == 0) {
        rmp[rr] = l == 0 ? mu : rmu[rr];  // block 0: operand centred on its exact mean
        rmu[rr] = mu;
        rrs[rr] = rs;
        if (t.keep && blockIdx.x == 0 && g == 0 && rr < M) {
          t.micro[l].mean[rr] = mu;
          t.micro[l].rstd[rr] = rs;
        }
      }
      epi_bar();
    };
    // Forward LayerNorm folded into GEMM1 (reading R3 in DESIGN.md).  With mu, rs the statistics
    // of the block input y and mu~ the input mean of the previous block (0 for the first):
    //   a = LN(y) W1^T + b1 = rs (sum_k bf16(gamma_k (y_k - mu~)) W1[h][k] - (mu - mu~) c_h) + e_h
    // with c_h = sum_k gamma_k W1[h][k], e_h = sum_k beta_k W1[h][k] + b1[h] (task_stream_fold).  The
    // GEMM1 operand needs no row statistics, so the statistics exchange overlaps GEMM1 instead of
    // preceding it; the exact LN output (dW1 stash) and mean / rstd are written off the critical path.
    //
    // producer side (owners of the block input, d-space): the operand gamma (y - mu~), the quarter
    // counter (operand), then the chunk statistics and the global counter.  mut[e] = mu~ of row 4ew+e.
    auto ln_chunk_stats = [&](const float* y, int l) {
      float* st = t.stats + (size_t)l * (d / 32) * 32;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = 4 * ew + e;
        const float mu = wsum32(y[e]) * (1.0f / 32.0f);
        const float dv = y[e] - mu;
        const float m2 = wsum32(dv * dv);
        if (lane == 0) *reinterpret_cast<float2*>(st + ((size_t)chunk * 16 + r) * 2) = make_float2(mu, m2);
      }
    };
    auto ln_produce = [&](const float* y, const float* mut, int l, float gm, __nv_bfloat16* yg) {
      // the operand first (critical path: the next GEMM1's activation tiles), statistics after
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = 4 * ew + e;
        yg[(size_t)r * d + fo] = __float2bfloat16_rn(r < M ? gm * (y[e] - mut[e]) : 0.0f);
      }
      signal(1 + 3 * l, fo / (d / 4));
      ln_chunk_stats(y, l);
      signal(3 + 3 * l, 4);
    };
    // block 0 of the task: no previous block mean to centre on, and the stage input may sit far off
    // zero (row mean >> row std), where bf16(gamma y) would lose the (y - mu) digits.  So the chunk
    // statistics go first, every producer waits for all of them and centres the operand on the exact
    // mean (mu~ = mu, the correction term vanishes).  One exchange more, only at the task start.
    auto ln_produce_first = [&](const float* y, float gm, __nv_bfloat16* yg) {
      ln_chunk_stats(y, 0);
      signal(3, 4);
      ln_rows(0);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = 4 * ew + e;
        yg[(size_t)r * d + fo] = __float2bfloat16_rn(r < M ? gm * (y[e] - rmu[r]) : 0.0f);
      }
      signal(1, fo / (d / 4));
    };
    // exact LN output of the thread's own d-space item (dW1 operand stash, read by W_j only)
    auto ln_stash = [&](const float* y, int l) {
      const SLayer& Ly = t.layers[l];
      const float gm = Ly.gamma[fo], b = Ly.beta[fo];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int r = 4 * ew + e;
        if (t.keep && r < M) t.micro[l].hop[(size_t)r * d + fo] = __float2bfloat16_rn(gm * ((y[e] - rmu[r]) * rrs[r]) + b);
      }
    };

    if (!BWD) {
      // ---------------------------------------------------------------- forward task
      float yk[4] = {0.f, 0.f, 0.f, 0.f};  // the thread's d-space item of the current block input
      if (own_d) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 4 * ew + e;
          yk[e] = r < M ? __ldcg(t.micro[0].x + (size_t)r * d + fo) : 0.0f;
        }
        ln_produce_first(yk, t.layers[0].gamma[fo], t.layers[0].yg);
      }
      for (int l = 0; l < t.L; ++l) {
        const SLayer& Ly = t.layers[l];
        const SMicro& Mi = t.micro[l];
        cur_p = 2 * l;
        if (own_h) {  // GEMM1 epilogue: a = rs (acc - (mu - mu~) c) + e; g = dropout(GELU(a))
          // every descriptor field the epilogue needs is loaded before the wait (no pointer chase
          // through global memory after the GEMM result)
          const float cf = Ly.cfold[fo], ef = Ly.efold[fo];
          const uint32_t dth = Ly.drop_thresh, site = Ly.site;
          const float dsc = Ly.drop_scale;
          const uint32_t step = dth ? *t.step : 0u;
          __nv_bfloat16* const gop = Mi.gop;
          float* const aout = Mi.a;
          ln_rows(l);  // while GEMM1 streams: its row statistics are only needed by this epilogue
          float acc[4];
          gemm_result(std::integral_constant<int, 16>{}, acc, nullptr);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            if (r >= M) continue;
            const float z = rrs[r] * (acc[e] - (rmu[r] - rmp[r]) * cf) + ef;
            acc[e] = z;
            float gv = gelu_f(z);
            if (dth) {
              const uint64_t idx = (uint64_t)(t.r0 + r) * (uint64_t)H + (uint64_t)fo;
              gv = dropout_keep(t.seed, step, site, idx, dth) ? gv * dsc : 0.0f;
            }
            gop[(size_t)r * H + fo] = __float2bfloat16_rn(gv);
          }
          signal(2 + 3 * l, fo / (H / 4));
          // read only by the backward task / W_j: stored off the critical path
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (t.keep && 4 * ew + e < M) aout[(size_t)(4 * ew + e) * H + fo] = acc[e];
        } else if (own_d) {
          ln_rows(l);
        }
        if (own_d) ln_stash(yk, l);
        cur_p = 2 * l + 1;
        if (own_d) {  // GEMM2 epilogue: y = x + acc + b2, then the next block's LN operand
          const float b2 = Ly.b2[fo];
          const bool more = l + 1 < t.L;
          const float gnext = more ? t.layers[l + 1].gamma[fo] : 0.0f;
          __nv_bfloat16* const yg = Ly.yg;
          float* const yout = (t.y_send && l + 1 == t.L) ? t.y_send : Mi.y;  // fused send: the consumer's slab
          float acc[4];
          gemm_result(std::integral_constant<int, 16>{}, acc, nullptr);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            yk[e] = r < M ? acc[e] + b2 + yk[e] : 0.0f;
          }
          if (more) {
            float mut[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) mut[e] = rmu[4 * ew + e];
            ln_produce(yk, mut, l + 1, gnext, yg);
          }
          // the residual stream is read by this thread (next block) and later tasks only
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if ((t.keep || l + 1 == t.L) && 4 * ew + e < M) yout[(size_t)(4 * ew + e) * d + fo] = yk[e];
        }
      }
    } else {
      // ---------------------------------------------------------------- backward task
      // LayerNorm backward folded into the next dG (reading R4 in DESIGN.md).  With u = gy + rs dn
      // and n the normalised input of block l:  dx = u - rs (m1 + m2 n),  m1 = mean_f(dn),
      // m2 = mean_f(dn n), so the dG GEMM of block l-1 runs on the 32-row operand [u | n] (N = 32)
      // and its epilogue corrects per row:  dG = acc_u - rs (m1 c2_h + m2 acc_n),  c2_h = sum_k
      // W2[k][h] (task_stream_fold).  [u | n] needs no row reduction, so the LayerNorm-backward
      // sums overlap dG's weight stream; the exact dx (dW2 operand stash, db2 partials, residual
      // gradient, message) is formed off the critical path.
      const int L = t.L;
      __nv_bfloat16* const uc = t.layers[0].uc;  // [32][d] task scratch [u | n]
      // rmu / rrs / rsb: m1, m2, rstd of the LayerNorm whose backward feeds the current dG (0 for
      // the top block, whose dG operand is the exact incoming gradient)
      if (et < 16) rmu[et] = rrs[et] = rsb[et] = 0.0f;
      epi_bar();
      // combine the LN-backward chunk sums of backward step kk (row sums of dn, dn n) -> rmu, rrs
      auto bwd_rows = [&](int kk, int lb) {
        const int J = d / 32;
        const float* st = t.stats + (size_t)kk * J * 32;
        wait_cnt(3 + 3 * kk, 4, (unsigned)J);
        const int rr = et >> 3, jl = et & 7;
        float s1 = 0.0f, s2 = 0.0f;
        for (int j = jl; j < J; j += 8) {
          const float2 v = __ldcg(reinterpret_cast<const float2*>(st + ((size_t)j * 16 + rr) * 2));
          s1 += v.x;
          s2 += v.y;
        }
        s1 += __shfl_xor_sync(0xffffffffu, s1, 4);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
        s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 4);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        if (jl == 0) {
          rmu[rr] = s1 / (float)d;
          rrs[rr] = s2 / (float)d;
          rsb[rr] = rr < M ? t.micro[lb].rstd[rr] : 0.0f;
        }
        epi_bar();
      };
      float gyv[4] = {0.f, 0.f, 0.f, 0.f};  // d-space item of the incoming gradient of the current block
      if (own_d) {  // top block: exact dY (stash + db2 column sums), operand [gy | 0]
        const SMicro& Mi = t.micro[L - 1];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int r = 4 * ew + e;
          gyv[e] = r < M ? __ldcg(t.gy_top + (size_t)r * d + fo) : 0.0f;
          const __nv_bfloat16 gb = __float2bfloat16_rn(gyv[e]);
          if (r < M) Mi.dyop[(size_t)r * d + fo] = gb;
          uc[(size_t)r * d + fo] = gb;
          uc[(size_t)(16 + r) * d + fo] = __float2bfloat16_rn(0.0f);
        }
        signal(1, fo / (d / 4));
        colsums(gyv, nullptr, nullptr, Mi.pb2, nullptr, nullptr);
      }
      for (int k = 0; k < L; ++k) {
        const int l = L - 1 - k;
        const SLayer& Ly = t.layers[l];
        const SMicro& Mi = t.micro[l];
        cur_p = 2 * k;
        if (own_h) {  // dG epilogue: row correction, dA = dG * dropout mask * GELU'(a)
          if (!own_d && k > 0) bwd_rows(k - 1, l + 1);
          const uint32_t dth = Ly.drop_thresh, site = Ly.site;
          const float dsc = Ly.drop_scale;
          const uint32_t step = dth ? *t.step : 0u;
          const float c2 = Ly.c2fold[fo];
          __nv_bfloat16* const daop = Mi.daop;
          float* const pb = Mi.pb;
          float av[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            av[e] = r < M ? Mi.a[(size_t)r * H + fo] : 0.0f;
          }
          float acc[4], accn[4], da[4];
          gemm_result(std::integral_constant<int, 32>{}, acc, accn);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            da[e] = 0.0f;
            if (r >= M) continue;
            float dg = acc[e] - rsb[r] * (rmu[r] * c2 + rrs[r] * accn[e]);
            if (dth) {
              const uint64_t idx = (uint64_t)(t.r0 + r) * (uint64_t)H + (uint64_t)fo;
              dg = dropout_keep(t.seed, step, site, idx, dth) ? dg * dsc : 0.0f;
            }
            da[e] = dg * gelu_df(av[e]);
            daop[(size_t)r * H + fo] = __float2bfloat16_rn(da[e]);
          }
          signal(2 + 3 * k, fo / (H / 4));
          colsums(da, nullptr, nullptr, pb, nullptr, nullptr);
        }
        cur_p = 2 * k + 1;
        if (own_d) {  // dH epilogue: u = gy + rs dn and n for the next dG; LN-backward sums; exact dx
          const float gam = Ly.gamma[fo];
          float nv[4], rsv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            if (r < M) {
              const float mu = Mi.mean[r];
              rsv[e] = Mi.rstd[r];
              nv[e] = (Mi.x[(size_t)r * d + fo] - mu) * rsv[e];
            } else {
              nv[e] = rsv[e] = 0.0f;
            }
          }
          float* const pg = Mi.pg;
          float* const pbt = Mi.pbt;
          __nv_bfloat16* const dyn = l > 0 ? t.micro[l - 1].dyop : nullptr;
          float* const pb2n = l > 0 ? t.micro[l - 1].pb2 : nullptr;
          float dh[4], dhn[4], dn[4], uv[4];
          gemm_result(std::integral_constant<int, 16>{}, dh, nullptr);
          const int J = d / 32;
          float* st = t.stats + (size_t)k * J * 32;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            if (r >= M) dh[e] = 0.0f;
            dhn[e] = dh[e] * nv[e];
            dn[e] = dh[e] * gam;
            uv[e] = r < M ? gyv[e] + rsv[e] * dn[e] : 0.0f;
          }
          if (l > 0) {  // the next dG's operand first (critical path)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int r = 4 * ew + e;
              uc[(size_t)r * d + fo] = __float2bfloat16_rn(uv[e]);
              uc[(size_t)(16 + r) * d + fo] = __float2bfloat16_rn(nv[e]);
            }
            signal(4 + 3 * k, fo / (d / 4));
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float s1 = wsum32(dn[e]);
            const float s2 = wsum32(dn[e] * nv[e]);
            if (lane == 0) *reinterpret_cast<float2*>(st + ((size_t)chunk * 16 + 4 * ew + e) * 2) = make_float2(s1, s2);
          }
          signal(3 + 3 * k, 4);
          colsums(dhn, dh, nullptr, pg, pbt, nullptr);
          // exact dx = u - rs (m1 + m2 n): the next block's residual gradient and dW2 operand
          bwd_rows(k, l);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * ew + e;
            gyv[e] = r < M ? uv[e] - rsv[e] * (rmu[r] + nv[e] * rrs[r]) : 0.0f;
          }
          if (l > 0) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int r = 4 * ew + e;
              if (r < M) dyn[(size_t)r * d + fo] = __float2bfloat16_rn(gyv[e]);
            }
            colsums(gyv, nullptr, nullptr, pb2n, nullptr, nullptr);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (4 * ew + e < M) t.dx_bottom[(size_t)(4 * ew + e) * d + fo] = gyv[e];
          }
        }
      }
    }
  }
  __syncthreads();
  cluster_sync();
  if (warp == 1) tmem_dealloc(tmem, 512);
  // the last CTA to finish resets every dependency counter for the next task (no other CTA polls
  // any more once all have arrived here; the kernel boundary publishes the zeros)
  const int ncnt = (3 * t.L + 3) * 5;
  unsigned* done = t.cnt + (size_t)ncnt * CNT_STRIDE;
  __shared__ int last;
  if (threadIdx.x == 0) {
    unsigned prev;
    if (t.send_flag) {
      // fused send: this CTA's stores into the consumer's receive slab (ordered before this thread by
      // the barrier above) become visible at system scope before its arrival is counted
      asm volatile("atom.add.acq_rel.sys.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(done) : "memory");
    } else {
      __threadfence();
      prev = atomicAdd(done, 1u);
    }
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    for (int k = threadIdx.x; k < ncnt; k += blockDim.x) t.cnt[(size_t)k * CNT_STRIDE] = 0u;
    if (threadIdx.x == 0) {
      *done = 0u;
      if (t.send_flag)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(t.send_flag), "r"(*t.send_seq) : "memory");
    }
  }
}

// c[h] = sum_k gamma[k] W1[h][k], e[h] = sum_k beta[k] W1[h][k] + b1[h]: one warp per row, lanes
// stride the row in 8-element vectors, fixed-order sums (deterministic)
__global__ void __launch_bounds__(256) task_stream_fold_kernel(const SLayer* __restrict__ layers, int d, int H) {
  const SLayer& Ly = layers[blockIdx.y];
  if (blockIdx.z == 1) {
    // column sums of W2 [d][H], stage 1: block (row chunk kc of 256 rows, column block) -> partial
    // sums of 8 columns per thread over the chunk's rows (fixed order) into c2part[L][d/256][H]
    const int cb = H / (8 * 256) > 0 ? H / (8 * 256) : 1;  // column blocks of 2048 columns
    const int kc = blockIdx.x / cb, col0 = ((blockIdx.x % cb) * 256 + threadIdx.x) * 8;
    if (kc * 256 >= d || col0 >= H) return;
    const __nv_bfloat16* __restrict__ W2 = Ly.w2;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int k = kc * 256; k < kc * 256 + 256; ++k) {
      const uint4 raw = *reinterpret_cast<const uint4*>(W2 + (size_t)k * H + col0);
      const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(w2[q]);
        a[2 * q] += f.x;
        a[2 * q + 1] += f.y;
      }
    }
    float* part = Ly.c2part + (size_t)kc * H + col0;
#pragma unroll
    for (int q = 0; q < 8; ++q) part[q] = a[q];
    return;
  }
  const __nv_bfloat16* __restrict__ W = Ly.w1;
  const float* __restrict__ gamma = Ly.gamma;
  const float* __restrict__ beta = Ly.beta;
  const int h = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (h >= H) return;
  float sc = 0.0f, se = 0.0f;
#pragma unroll 4
  for (int k = lane * 8; k < d; k += 256) {
    const uint4 raw = *reinterpret_cast<const uint4*>(W + (size_t)h * d + k);
    const __nv_bfloat162* w2 = reinterpret_cast<const __nv_bfloat162*>(&raw);
    const float4 g0 = *reinterpret_cast<const float4*>(gamma + k), g1 = *reinterpret_cast<const float4*>(gamma + k + 4);
    const float4 b0 = *reinterpret_cast<const float4*>(beta + k), b1v = *reinterpret_cast<const float4*>(beta + k + 4);
    const float2 w0 = __bfloat1622float2(w2[0]), w1 = __bfloat1622float2(w2[1]);
    const float2 w2f = __bfloat1622float2(w2[2]), w3 = __bfloat1622float2(w2[3]);
    sc += g0.x * w0.x + g0.y * w0.y + g0.z * w1.x + g0.w * w1.y + g1.x * w2f.x + g1.y * w2f.y + g1.z * w3.x + g1.w * w3.y;
    se += b0.x * w0.x + b0.y * w0.y + b0.z * w1.x + b0.w * w1.y + b1v.x * w2f.x + b1v.y * w2f.y + b1v.z * w3.x +
          b1v.w * w3.y;
  }
  sc = wsum32(sc);
  se = wsum32(se);
  if (lane == 0) {
    const_cast<float*>(Ly.cfold)[h] = sc;
    const_cast<float*>(Ly.efold)[h] = se + Ly.b1[h];
  }
}

// column sums of W2, stage 2: fixed-order sum of the d/256 chunk partials
__global__ void __launch_bounds__(256) task_stream_fold2_kernel(const SLayer* __restrict__ layers, int d, int H) {
  const SLayer& Ly = layers[blockIdx.y];
  const int h = blockIdx.x * 256 + threadIdx.x;
  if (h >= H) return;
  float acc = 0.0f;
  for (int kc = 0; kc < d / 256; ++kc) acc += Ly.c2part[(size_t)kc * H + h];
  const_cast<float*>(Ly.c2fold)[h] = acc;
}

int task_stream_fold(cudaStream_t st, const SLayer* layers, int L, int d, int H) {
  task_stream_fold_kernel<<<dim3((H + 7) / 8, L, 2), 256, 0, st>>>(layers, d, H);
  task_stream_fold2_kernel<<<dim3((H + 255) / 256, L), 256, 0, st>>>(layers, d, H);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    set_error("task_stream_fold launch: %s", cudaGetErrorString(err));
    return -3;
  }
  return 0;
}

// ---------------------------------------------------------------------------------------- host
int task_stream_smem() { return ST_SMEM_MAX; }
int task_stream_counter_bytes(int L) { return ((3 * L + 3) * 5 + 1) * CNT_STRIDE * 4; }

template <bool BWD, int NV>
static bool stream_attr_one() {
  cudaError_t e = cudaFuncSetAttribute(task_stream_kernel<BWD, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       StCfg<BWD, NV>::SMEM);
  if (e != cudaSuccess) {
    set_error("task_stream smem attribute: %s", cudaGetErrorString(e));
    return false;
  }
  cudaFuncSetAttribute(task_stream_kernel<BWD, NV>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  return true;
}

static bool stream_attr() {
  static int done = 0;  // per process (the attribute is per device; the runtime sets it on first use)
  if (!done) {
    if (!stream_attr_one<false, 1>() || !stream_attr_one<false, 2>() || !stream_attr_one<true, 1>() ||
        !stream_attr_one<true, 2>())
      return false;
    done = 1;
  }
  return true;
}

static void stream_cfg(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, int clusters, int smem, cudaStream_t st,
                       int threads = st_threads<1>()) {
  cfg = cudaLaunchConfig_t{};
  cfg.gridDim = dim3(clusters * SK, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = SK;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
}

int task_stream_max_clusters(int dev) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(dev);
  int n = 0;
  if (stream_attr()) {
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    stream_cfg(cfg, at, 1, ST_SMEM_MAX, nullptr);
    if (cudaOccupancyMaxActiveClusters(&n, task_stream_kernel<false, 1>, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();
  cudaSetDevice(cur);
  return n;
}

int task_stream_launch(cudaStream_t st, const STask& t, int clusters) {
  if (!stream_attr()) return -3;
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute at[1];
  cudaError_t e;
  if (t.bwd) {
    if (t.nv == 2) {
      stream_cfg(cfg, at, clusters, StCfg<true, 2>::SMEM, st, st_threads<2>());
      e = cudaLaunchKernelEx(&cfg, task_stream_kernel<true, 2>, t);
    } else {
      stream_cfg(cfg, at, clusters, StCfg<true, 1>::SMEM, st);
      e = cudaLaunchKernelEx(&cfg, task_stream_kernel<true, 1>, t);
    }
  } else {
    if (t.nv == 2) {
      stream_cfg(cfg, at, clusters, StCfg<false, 2>::SMEM, st, st_threads<2>());
      e = cudaLaunchKernelEx(&cfg, task_stream_kernel<false, 2>, t);
    } else {
      stream_cfg(cfg, at, clusters, StCfg<false, 1>::SMEM, st);
      e = cudaLaunchKernelEx(&cfg, task_stream_kernel<false, 1>, t);
    }
  }
  if (e != cudaSuccess) {
    set_error("task_stream launch (%d clusters, nv %d): %s", clusters, t.nv, cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

}  // namespace tgp
