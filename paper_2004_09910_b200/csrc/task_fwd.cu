// Persistent forward-task kernel: one cooperative launch executes F_{i,j} (and F'_{i,j}) for a
// partition made of pre-LN residual MLP blocks (PAPER.md Eq. F_{i,j}).
//
// Why: a micro-batch task is a chain of 2 dependent weight-streaming GEMMs per block (M = 16 rows).
// As separate kernels, every GEMM boundary idles HBM for several microseconds (grid drain, launch,
// ring restart; profiles/r1*_gemm_timeline).  Here every CTA (one per SM) owns a contiguous range of
// the flattened (128-row slab, 64-wide k-block) space of EVERY GEMM phase -- the same range size for
// all phases -- and its TMA weight ring runs ahead continuously across phases: only the small
// activation operand (B) of the next phase waits for the grid barrier.
//
// Phases per block l (barrier ids in parentheses; a barrier k completes when the global counter
// reaches G*k):
//   [l = 0 only] row statistics of x (1), normalise x -> h = LN(x) bf16 (2)
//   GEMM1 partial tiles (3+5l) -> owner epilogue: a = acc + b1, g = drop(GELU(a)) bf16 (4+5l)
//   GEMM2 partial tiles (5+5l) -> owner epilogue: y = acc + b2 + x, + LN chunk stats of y (6+5l)
//   [l < L-1] combine stats, normalise y -> h_{l+1} (7+5l)
// Determinism: fixed work assignment, split-K partials summed in ascending CTA order, LN statistics
// combined (Chan et al.) in fixed chunk order -> F' reproduces F bit-exactly (reading Z21).
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "host.h"
#include "kernels.h"
#include "task_fwd.h"

namespace tgp {

constexpr int PT_A = 16384;             // 128 x 64 bf16 weight tile (one ring stage)
constexpr int PT_B = 2048;              // 16 x 64 bf16 activation tile
constexpr int PT_STAGES = 11;           // weight ring
constexpr int PT_BT = 16;               // activation tiles of one phase (the CTA's whole B share)
constexpr int PT_SMEM = PT_STAGES * PT_A + PT_BT * PT_B + 1024 + 8192;

TGP_DEV unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Grid barrier: one cumulative arrival counter.  (Measured: spreading arrivals over 8 counters
// 128 B apart makes every poll 8 loads and floods L2 -- slower overall.)
constexpr int PT_NCTR = 1;
TGP_DEV unsigned bar_count(const unsigned* bar) { return ld_acquire_u32(bar); }
TGP_DEV int lo_of(int c, int T, int G) { return (int)(((long long)c * T) / G); }
// the CTA owning flat k-block x: lo(c) <= x < lo(c+1) (skips CTAs with empty ranges); `lot` is the
// shared table of range starts lo(0..G) (no 64-bit division on the hot path)
TGP_DEV int owner_of(int x, const int* lot, int T, int G) {
  int c = (x * G) / T;
  if (c >= G) c = G - 1;
  while (c > 0 && lot[c] > x) --c;
  while (c + 1 < G && lot[c + 1] <= x) ++c;
  return c;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// diagnostics (t.dbg != nullptr only): per CTA, per GEMM phase g < 128, up to 8 event stamps
TGP_DEV void dbg_stamp(const PTask& t, int c, int g, int slot) {
  if (!t.dbg || g >= 128) return;
  unsigned long long tt;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
  t.dbg[(size_t)gridDim.x * 512 + 256 + ((size_t)c * 128 + g) * 8 + slot] = tt;
}

template <typename T>
TGP_DEV T wsum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(192, 1) task_fwd_kernel(const PTask t) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* bbuf = smem + PT_STAGES * PT_A;  // [PT_BT] activation tiles of the current phase
  uint64_t* full = reinterpret_cast<uint64_t*>(bbuf + PT_BT * PT_B);
  uint64_t* empty = full + PT_STAGES;
  uint64_t* tfull = empty + PT_STAGES;   // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* bfull = tempty + 2;          // [1] activation tiles of a phase landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [4 warps][4 rows][2]
  float* rmu = red + 32;                                  // [16]
  float* rrs = rmu + 16;                                  // [16]
  int* lot = reinterpret_cast<int*>(rrs + 16);            // [G + 1] range starts (G <= 255)
  float* stg = reinterpret_cast<float*>(lot + 256);       // [1024] staged LN chunk statistics

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x, c = blockIdx.x;
  const int L = t.L, d = t.d, H = t.H, M = t.M;
  // every GEMM phase has T = (H/128)*(d/64) = (d/128)*(H/64) flat k-blocks
  const int T = (H / 128) * (d / 64);
  const int lo = lo_of(c, T, G), hi = lo_of(c + 1, T, G), nit = hi - lo;
  const int total = 2 * L * nit;
  for (int q = threadIdx.x; q <= G; q += blockDim.x) lot[q] = lo_of(q, T, G);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < PT_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tfull[1], 1);
    mbar_init(&tempty[0], 128);
    mbar_init(&tempty[1], 128);
    mbar_init(bfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      // ------------------------------------------------------------ TMA producer
      const uint64_t pol_w = policy_evict_first(), pol_b = policy_evict_last();
      int ia = 0, gb = 0;
      unsigned level = 0;  // highest barrier observed complete (avoid an L2 round trip per check)
      while (ia < total || gb < 2 * L) {
        bool progress = false;
        // activations of the next phase first: all of this CTA's B tiles at once, as soon as the
        // phase that produces them has completed (which also implies the previous phase's MMAs,
        // the only readers of bbuf, are done)
        if (gb < 2 * L) {
          const unsigned need = (gb & 1) ? (unsigned)(4 + 5 * (gb >> 1)) : (unsigned)(2 + 5 * (gb >> 1));
          if (level < need) {
            const unsigned v = bar_count(t.bar) / (unsigned)G;
            if (v >= need) {
              level = v;
              asm volatile("fence.proxy.async.global;" ::: "memory");
            }
          }
          if (level >= need) {
            const PLayer& P = t.layers[gb >> 1];
            const int kbs = (gb & 1) ? H / 64 : d / 64;
            mbar_arrive_expect_tx(bfull, (uint32_t)(nit * PT_B));
            for (int q = 0; q < nit; ++q)
              tma_load_2d((gb & 1) ? &P.tmG : &P.tmH, bfull, bbuf + q * PT_B, ((lo + q) % kbs) * 64, t.r0, pol_b);
            dbg_stamp(t, c, gb, 0);
            ++gb;
            progress = true;
          }
        }
        while (ia < total) {  // weights: run ahead as far as the ring allows
          const int s = ia % PT_STAGES, r = ia / PT_STAGES;
          if (!mbar_test_wait(smem_u32(&empty[s]), (r & 1) ^ 1)) break;
          const int g = ia / nit, x = lo + ia % nit;
          const PLayer& P = t.layers[g >> 1];
          const int kbs = (g & 1) ? H / 64 : d / 64;
          mbar_arrive_expect_tx(&full[s], PT_A);
          tma_load_2d((g & 1) ? &P.tmW2 : &P.tmW1, &full[s], smem + s * PT_A, (x % kbs) * 64, (x / kbs) * 128, pol_w);
          if (ia % nit == 0) dbg_stamp(t, c, g, 7);
          if (ia % nit == nit - 1) dbg_stamp(t, c, g, 2);
          ++ia;
          progress = true;
          if (gb < 2 * L && g >= gb) break;  // re-check the activation barrier between weight loads
        }
        if (!progress) __nanosleep(64);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = make_idesc_bf16(128, 16, false, false);
      int it = 0, buf = 0;
      int use[2] = {0, 0};
      for (int g = 0; g < 2 * L; ++g) {
        const int kbs = (g & 1) ? H / 64 : d / 64;
        int x = lo;
        while (x < hi) {
          const int slab = x / kbs;
          const int xe = min(hi, (slab + 1) * kbs);
          mbar_wait(&tempty[buf], (use[buf] & 1) ^ 1);
          ++use[buf];
          tc_fence_after();
          const uint32_t dacc = tmem + (uint32_t)(buf * 32);
          for (int xx = x; xx < xe; ++xx, ++it) {
            const int s = it % PT_STAGES, r = it / PT_STAGES;
            mbar_wait(&full[s], r & 1);
            tc_fence_after();
            if (xx == lo) {
              mbar_wait(bfull, (uint32_t)(g & 1));  // this phase's activation tiles
              tc_fence_after();
              dbg_stamp(t, c, g, 3);
            }
            const uint32_t a = smem_u32(smem + s * PT_A), b = smem_u32(bbuf + (xx - lo) * PT_B);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tc_mma_bf16(dacc, make_sdesc_sw128(a + kk * 32, 16, 1024), make_sdesc_sw128(b + kk * 32, 16, 1024), idesc,
                          (xx != x || kk) ? 1u : 0u);
            tc_commit(&empty[s]);
          }
          tc_commit(&tfull[buf]);
          if (xe == hi) dbg_stamp(t, c, g, 4);
          buf ^= 1;
          x = xe;
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue warps (128 threads)
    const int et = threadIdx.x - 64;
    const int lg = warp & 3;
    const int fl = lg * 32 + lane;  // TMEM lane = feature within the slab
    const int ew = et >> 5;         // epilogue warp index for reductions
    int buf = 0;
    int seen[2] = {0, 0};
    // The counter is cumulative, so an arrival at barrier k is only allowed once barrier k-1 is
    // complete -- otherwise a CTA with no work in a phase could run ahead and its arrivals would
    // count towards an earlier barrier.  Then "counter >= G*k" <=> every CTA arrived at 1..k.
    auto arrive = [&](unsigned k) {
      epi_bar();
      if (et == 0) {
        while (bar_count(t.bar) < (unsigned)G * (k - 1)) __nanosleep(32);
        if (t.dbg && k < 256) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          t.dbg[((size_t)c * 256 + k) * 2] = tt;
        }
        __threadfence();
        atomicAdd(t.bar + 32 * (c % PT_NCTR), 1u);
        if (t.dbg && k < 256 && bar_count(t.bar) == (unsigned)G * k) {  // ~last arrival: completion time
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          t.dbg[(size_t)G * 512 + k] = tt;
        }
      }
    };
    auto wait = [&](unsigned k) {
      if (et == 0) {
        while (bar_count(t.bar) < (unsigned)G * k) __nanosleep(32);
        if (t.dbg && k < 256) {
          unsigned long long tt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
          t.dbg[((size_t)c * 256 + k) * 2 + 1] = tt;
        }
      }
      epi_bar();
    };
    // LN chunk statistics of one 128-item chunk: thread holds 4 row values v[e]; writes (mean, M2)
    // per row to stats[chunk][e]
    auto chunk_stats = [&](const float* v, int chunk) {
      float mw[4], qw[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        mw[e] = wsum(v[e]) * (1.0f / 32.0f);
        const float dd = v[e] - mw[e];
        qw[e] = wsum(dd * dd);
      }
      if (lane == 0)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          red[(ew * 4 + e) * 2] = mw[e];
          red[(ew * 4 + e) * 2 + 1] = qw[e];
        }
      epi_bar();
      if (et < 4) {
        float mu = 0.0f;
        for (int w = 0; w < 4; ++w) mu += red[(w * 4 + et) * 2];
        mu *= 0.25f;
        float m2 = 0.0f;
        for (int w = 0; w < 4; ++w) {
          const float dm = red[(w * 4 + et) * 2] - mu;
          m2 += red[(w * 4 + et) * 2 + 1] + 32.0f * dm * dm;
        }
        t.stats[(chunk * 4 + et) * 2] = mu;
        t.stats[(chunk * 4 + et) * 2 + 1] = m2;
      }
      epi_bar();
    };
    // wait for barrier kw, combine the d/128 chunk statistics of each row (fixed order) and
    // normalise rows of src.  gamma / beta of the first item are fetched before the barrier; the
    // chunk statistics are pulled into smem by all 128 threads at once (one L2 round trip).
    auto normalise = [&](const float* src, const PLayer& P, unsigned kw) {
      const int d4 = d / 4;
      const int gi0 = c * 128 + et;
      float4 pg = make_float4(0.f, 0.f, 0.f, 0.f), pb = pg;
      if (gi0 < M * d4) {
        pg = reinterpret_cast<const float4*>(P.gamma)[gi0 % d4];
        pb = reinterpret_cast<const float4*>(P.beta)[gi0 % d4];
      }
      wait(kw);
      const int J = d / 128;
      const bool staged = J * 16 * 2 <= 1024;
      if (staged) {
        for (int u = et; u < J * 32; u += 128) stg[u] = __ldcg(&t.stats[u]);
        epi_bar();
      }
      auto st_mu = [&](int q, int j, int e) { return staged ? stg[((q * J + j) * 4 + e) * 2] : __ldcg(&t.stats[((q * J + j) * 4 + e) * 2]); };
      auto st_m2 = [&](int q, int j, int e) {
        return staged ? stg[((q * J + j) * 4 + e) * 2 + 1] : __ldcg(&t.stats[((q * J + j) * 4 + e) * 2 + 1]);
      };
      {
        // 8 threads per row: strided partial sums, then a fixed xor-tree over the 8 lanes
        const int rr = et >> 3, jl = et & 7, q = rr >> 2, e = rr & 3;
        float mu = 0.0f;
        for (int j = jl; j < J; j += 8) mu += st_mu(q, j, e);
        mu += __shfl_xor_sync(0xffffffffu, mu, 4);
        mu += __shfl_xor_sync(0xffffffffu, mu, 2);
        mu += __shfl_xor_sync(0xffffffffu, mu, 1);
        mu /= (float)J;
        float m2 = 0.0f;
        for (int j = jl; j < J; j += 8) {
          const float dm = st_mu(q, j, e) - mu;
          m2 += st_m2(q, j, e) + 128.0f * dm * dm;
        }
        m2 += __shfl_xor_sync(0xffffffffu, m2, 4);
        m2 += __shfl_xor_sync(0xffffffffu, m2, 2);
        m2 += __shfl_xor_sync(0xffffffffu, m2, 1);
        const float rs = 1.0f / sqrtf(m2 / (float)d + 1e-5f);
        if (jl == 0) {
          rmu[rr] = mu;
          rrs[rr] = rs;
          if (c == 0 && rr < M) {
            P.mean[rr] = mu;
            P.rstd[rr] = rs;
          }
        }
      }
      epi_bar();
      for (int gi = gi0; gi < M * d4; gi += G * 128) {
        const int r = gi / d4, c4 = gi % d4;
        const float4 v = __ldcg(reinterpret_cast<const float4*>(src + (size_t)r * d) + c4);
        const float4 ga = gi == gi0 ? pg : reinterpret_cast<const float4*>(P.gamma)[c4];
        const float4 be = gi == gi0 ? pb : reinterpret_cast<const float4*>(P.beta)[c4];
        const float mu = rmu[r], rs = rrs[r];
        __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(P.hop + (size_t)r * d + c4 * 4);
        o[0] = __floats2bfloat162_rn(ga.x * ((v.x - mu) * rs) + be.x, ga.y * ((v.y - mu) * rs) + be.y);
        o[1] = __floats2bfloat162_rn(ga.z * ((v.z - mu) * rs) + be.z, ga.w * ((v.w - mu) * rs) + be.w);
      }
    };

    // ---- block 0 input: statistics of x, then h_0 = LN(x)
    {
      const PLayer& P0 = t.layers[0];
      for (int gi = c * 128 + et; gi < d * 4; gi += G * 128) {
        const int f = gi % d, q = gi / d;
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (4 * q + e < M) ? __ldcg(P0.x + (size_t)(4 * q + e) * d + f) : 0.0f;
        chunk_stats(v, gi / 128);
      }
      arrive(1);
      normalise(P0.x, P0, 1);
      arrive(2);
    }
    for (int l = 0; l < L; ++l) {
      const PLayer& P = t.layers[l];
      for (int sub = 0; sub < 2; ++sub) {
        const int g = 2 * l + sub;
        const int kbs = sub ? H / 64 : d / 64;
        const int Mout = sub ? d : H;
        float* ws = t.ws + (size_t)(g & 1) * t.ws_stride;
        // (1) partial tiles of my segments -> workspace slot (slab, c - owner(first k-block of slab))
        int x = lo;
        while (x < hi) {
          const int slab = x / kbs;
          const int xe = min(hi, (slab + 1) * kbs);
          mbar_wait(&tfull[buf], seen[buf] & 1);
          ++seen[buf];
          tc_fence_after();
          if (et == 0 && x == lo) dbg_stamp(t, c, g, 5);
          if (et == 0 && xe == hi) dbg_stamp(t, c, g, 6);
          float v[16];
          tmem_ld16(tmem + (uint32_t)(buf * 32) + ((uint32_t)(lg * 32) << 16), v);
          tc_fence_before();
          mbar_arrive(&tempty[buf]);
          buf ^= 1;
          const int seg = c - owner_of(slab * kbs, lot, T, G);
          float4* dst = reinterpret_cast<float4*>(ws + ((size_t)slab * t.segmax + seg) * 2048);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q * 128 + fl] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          x = xe;
        }
        // operands of my first owner item that do not depend on this phase: fetched before the
        // barrier so only the partial-tile loads remain on the critical path
        const int gi0 = c * 128 + et;
        float pre_b = 0.0f, pre_x[4] = {0.f, 0.f, 0.f, 0.f};
        if (gi0 < Mout * 4) {
          const int f0 = gi0 % Mout, q0 = gi0 / Mout;
          pre_b = sub ? P.b2[f0] : P.b1[f0];
          if (sub)
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (4 * q0 + e < M) pre_x[e] = __ldcg(P.x + (size_t)(4 * q0 + e) * d + f0);
        }
        arrive(3 + 5 * l + 2 * sub);
        wait(3 + 5 * l + 2 * sub);
        // (2) owner epilogue over items (feature f, row quad q)
        for (int gi = gi0; gi < Mout * 4; gi += G * 128) {
          const int f = gi % Mout, q = gi / Mout;
          const bool first = gi == gi0;
          const float bias = first ? pre_b : (sub ? P.b2[f] : P.b1[f]);
          const int slab = f >> 7, f128 = f & 127;
          const int c0 = owner_of(slab * kbs, lot, T, G), c1 = owner_of(slab * kbs + kbs - 1, lot, T, G);
          const float4* base = reinterpret_cast<const float4*>(ws + (size_t)slab * t.segmax * 2048) + q * 128 + f128;
          float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
          // issue up to 8 partial-tile loads at once, then add them in ascending CTA order
          for (int cb = c0; cb <= c1; cb += 8) {
            float4 p[8];
            bool v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int cc = cb + u;
              v[u] = cc <= c1 && lot[cc + 1] != lot[cc];  // empty range: wrote nothing
              p[u] = v[u] ? __ldcg(base + (size_t)(cc - c0) * 512) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (v[u]) {
                a.x += p[u].x;
                a.y += p[u].y;
                a.z += p[u].z;
                a.w += p[u].w;
              }
          }
          const float av[4] = {a.x, a.y, a.z, a.w};
          float yv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int r = 4 * q + e;
            yv[e] = 0.0f;
            if (r >= M) continue;
            if (!sub) {
              const float z = av[e] + bias;
              P.a[(size_t)r * H + f] = z;
              float gv = gelu_f(z);
              if (P.drop_thresh) {
                const uint64_t idx = (uint64_t)(t.r0 + r) * (uint64_t)H + (uint64_t)f;
                gv = dropout_keep(t.seed, *t.step, P.site, idx, P.drop_thresh) ? gv * P.drop_scale : 0.0f;
              }
              P.gop[(size_t)r * H + f] = __float2bfloat16_rn(gv);
            } else {
              const float y = av[e] + bias + (first ? pre_x[e] : __ldcg(P.x + (size_t)r * d + f));
              P.y[(size_t)r * d + f] = y;
              yv[e] = y;
            }
          }
          if (sub && l + 1 < L) chunk_stats(yv, gi / 128);
        }
        arrive(4 + 5 * l + 2 * sub);
      }
      if (l + 1 < L) {
        normalise(P.y, t.layers[l + 1], 6 + 5 * l);
        arrive(7 + 5 * l);
      }
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 64);
}

// ---------------------------------------------------------------------------------------- host
int task_fwd_smem() { return PT_SMEM; }
int task_fwd_max_phase_tiles() { return PT_BT; }

int task_fwd_launch(cudaStream_t st, const PTask& t, int grid) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(task_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM);
    if (e != cudaSuccess) {
      set_error("task_fwd smem attribute: %s", cudaGetErrorString(e));
      return -3;
    }
    attr = true;
  }
  cudaError_t e = cudaMemsetAsync(t.bar, 0, sizeof(unsigned) * 32 * PT_NCTR, st);
  if (e != cudaSuccess) {
    set_error("task_fwd barrier reset: %s", cudaGetErrorString(e));
    return -3;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(192, 1, 1);
  cfg.dynamicSmemBytes = PT_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barrier)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, task_fwd_kernel, t);
  if (e != cudaSuccess) {
    set_error("task_fwd launch (grid %d): %s", grid, cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

int task_fwd_max_grid(int dev) {
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(task_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PT_SMEM);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, task_fwd_kernel, 192, PT_SMEM);
  const char* ov = getenv("TGP_PT_GRID");  // diagnostics only
  if (ov && atoi(ov) > 0 && atoi(ov) <= sms) return atoi(ov);
  return sms * (per > 0 ? 1 : 0);
}

}  // namespace tgp
