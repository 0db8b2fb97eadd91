// tcgen05 / TMA bf16 GEMM kernel (see gemm_tc.cuh for the design) and its host launcher.
#include <algorithm>
#include <cstdlib>

#include "epilogue.cuh"
#include "gemm_tc.cuh"
#include "host.h"
#include "kernels.h"

#ifndef TGP_SKINNY_SMEM
#define TGP_SKINNY_SMEM 163840
#endif
#ifndef TGP_W128_SMEM
#define TGP_W128_SMEM 131072
#endif

namespace tgp {

#ifdef TGP_GEMM_TIMING
// Debug instrumentation (variant builds only): per-CTA %globaltimer stamps of the last launches.
__device__ unsigned long long g_ts[8192][12];
__device__ unsigned int g_ts_next;
TGP_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TGP_TS(slot) \
  do { if (ts_row >= 0) g_ts[ts_row][slot] = gtimer(); } while (0)
#else
#define TGP_TS(slot) do {} while (0)
#endif

template <int BN>
struct TcCfg {
  static constexpr int BK = 64;
  static constexpr int A_BYTES = 128 * BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  // One CTA per SM (320 threads at ~100 registers): skinny (weight-streaming) tiles take a deep
  // pipeline (160 KB: 9 - 12 stages; measured better than two 90 KB CTAs per SM overlapping across
  // the PDL boundary, profiles/r6/); BN = 128 tiles (65 - 128-row micro-batches, C3 at m = 4) take 4
  // stages next to the push reduction's 64 KB receive region; wide tiles (dW) take the whole SM.
  static constexpr int BUDGET = BN <= 64 ? TGP_SKINNY_SMEM : BN == 128 ? TGP_W128_SMEM : 196608;
  static constexpr int STAGES = (BUDGET / STAGE) > 12 ? 12 : (BUDGET / STAGE);
  static constexpr int RED_BYTES = 128 * BN * 4;           // fp32 partial tile (float4 quads)
  static constexpr int CS_BYTES = (BN / 4) * 128 * 4;      // column-sum partials [quad][feature]
  // skinny tiles reduce split-K by pushing partials into a dedicated receive region (one cluster
  // barrier); wide tiles pull from the (aliased) stage buffers instead
  static constexpr bool PUSH = BN <= 128;
  static constexpr int RECV_BYTES = PUSH ? RED_BYTES : 0;
  static constexpr int DATA = PUSH ? STAGES * STAGE
                                   : ((STAGES * STAGE > RED_BYTES + CS_BYTES) ? STAGES * STAGE : RED_BYTES + CS_BYTES);
  static constexpr int BAR_OFF = DATA + RECV_BYTES + (PUSH ? CS_BYTES : 0);
  static constexpr int SMEM = BAR_OFF + 1024 + 256;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  // the push epilogue stages the whole partial tile in the (idle) pipeline buffers
  static_assert(!PUSH || RED_BYTES <= STAGES * STAGE, "split-K staging must fit the pipeline buffers");
};

TGP_DEV void tma_store_2d(const void* desc, const void* smem, int32_t c0, int32_t c1, bool reduce_add) {
  if (reduce_add)
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(desc),
                 "r"(c0), "r"(c1), "r"(smem_u32(smem))
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(desc), "r"(c0),
                 "r"(c1), "r"(smem_u32(smem))
                 : "memory");
}
TGP_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
TGP_DEV void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// warps: 0 TMA, 1 MMA, 2..5 TMEM epilogue (lane quadrants), 6..9 helpers: the split-K tail of the
// push-reduced tiles is instruction-bound, so all 8 epilogue warps finish its work items
constexpr int TC_THREADS = 320;
constexpr int TC_FIN = TC_THREADS - 64;  // threads finishing push-reduced work items

template <int BN, bool A_MN, bool B_MN, int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                   const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmD,
                   const GemmParams p) {
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* rbar = tfull + 1;  // split-K receive region complete (PUSH tiles)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.z;
#ifdef TGP_GEMM_TIMING
  __shared__ int ts_row_s;
  if (threadIdx.x == 0) ts_row_s = (int)(atomicAdd(&g_ts_next, 1u) % 8192u);
  __syncthreads();
  const int ts_row = ts_row_s;
  if (threadIdx.x == 0) g_ts[ts_row][0] = gtimer();
#endif
  const int nkb_total = p.K / C::BK;
  const int kb0 = blockIdx.y * p.kb_per_split;
  const int kb1 = min(kb0 + p.kb_per_split, nkb_total);
  const int nkb = kb1 > kb0 ? kb1 - kb0 : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB0);
    tma_prefetch_desc(&tmB1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    if (C::PUSH && MODE != EPI_DW) {
      // every byte of the receive region is written once by the S cluster ranks' st.async
      mbar_init(rbar, 1);
      fence_barrier_init();
      mbar_arrive_expect_tx(rbar, (uint32_t)C::RED_BYTES);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  griddep_launch();
  // receive barriers of all cluster ranks must be initialised before anyone pushes into them:
  // arrive now, wait right before the first push (the whole mainloop in between)
  constexpr bool push_red = C::PUSH && MODE != EPI_DW;
  if (push_red) cluster_arrive();

  // owner-epilogue operands of a thread's first two work items, gathered during the mainloop (PUSH
  // tiles); the tail loop stays rolled and requests item k + 2's operands before finishing item k.
  // (Unrolling every item's epilogue overflowed the instruction cache: at BN = 128 half the warp
  // samples were no_instructions, profiles/r6/.)
  EpiPre pre[2][4];
  auto stage_a = [&](int s) { return smem + s * C::STAGE; };
  auto stage_b = [&](int s) { return smem + s * C::STAGE + C::A_BYTES; };
  const int m0 = m_tile * 128;
  const int nb = n_tile * BN;

  if (warp == 0) {
    if (elect_one()) {
      // ---------------- TMA producer
      const uint64_t pol_a = p.a_is_weight ? policy_evict_first() : policy_evict_last();
      const uint64_t pol_b = policy_evict_last();
      auto load_a = [&](int s, int kb) {
        const int k = kb * C::BK;
        if (A_MN) {
          tma_load_2d(&tmA, &full[s], stage_a(s), m0, k, pol_a);
          tma_load_2d(&tmA, &full[s], stage_a(s) + 8192, m0 + 64, k, pol_a);
        } else {
          tma_load_2d(&tmA, &full[s], stage_a(s), k, m0, pol_a);
        }
      };
      auto load_b = [&](int s, int kb) {
        const int k = kb * C::BK;
        const bool second = k >= p.k_seg;
        const CUtensorMap* tm = second ? &tmB1 : &tmB0;
        const int kk = second ? k - p.k_seg : k;
        if (B_MN) {
#pragma unroll
          for (int c = 0; c < BN / 64; ++c) tma_load_2d(tm, &full[s], stage_b(s) + c * 8192, p.n0 + nb + c * 64, kk, pol_b);
        } else {
          tma_load_2d(tm, &full[s], stage_b(s), kk, p.n0 + nb, pol_b);
        }
      };
      int pre = 0;
      if (p.a_is_weight) {
        // weights do not depend on the previous kernel: start streaming them before the wait
        pre = nkb < C::STAGES ? nkb : C::STAGES;
        for (int it = 0; it < pre; ++it) {
          mbar_arrive_expect_tx(&full[it], C::STAGE);
          load_a(it, kb0 + it);
        }
        if (p.a_l2pf) {
          for (int it = pre; it < nkb; ++it) {
            const int k = (kb0 + it) * C::BK;
            if (A_MN) {
              tma_prefetch_l2_2d(&tmA, m0, k);
              tma_prefetch_l2_2d(&tmA, m0 + 64, k);
            } else {
              tma_prefetch_l2_2d(&tmA, k, m0);
            }
          }
        }
      }
      griddep_wait();
      TGP_TS(1);
      for (int it = 0; it < pre; ++it) load_b(it, kb0 + it);
      for (int it = pre; it < nkb; ++it) {
        const int s = it % C::STAGES, r = it / C::STAGES;
        mbar_wait(&empty[s], (r & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], C::STAGE);
        load_a(s, kb0 + it);
        load_b(s, kb0 + it);
      }
      if (p.pf_bytes > 0) {
        const int64_t ncta = (int64_t)gridDim.x * gridDim.y * gridDim.z;
        const int64_t cid = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        const int64_t chunk = ((p.pf_bytes + ncta - 1) / ncta + 255) & ~int64_t(255);
        const int64_t beg = cid * chunk;
        const int64_t end = beg + chunk < p.pf_bytes ? beg + chunk : p.pf_bytes;
        const char* base = reinterpret_cast<const char*>(p.pf_ptr);
        for (int64_t o = beg; o < end; o += 65536) {
          const uint32_t sz = (uint32_t)((end - o) < 65536 ? (end - o) : 65536);
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + o), "r"(sz) : "memory");
        }
      }
    }
    // reconverge before the .aligned cluster barriers below (only one lane ran the producer loop)
    __syncwarp();
    if (push_red) cluster_wait();
  } else if (warp == 1) {
    if (elect_one()) {
      // ---------------- MMA issuer (single thread)
      constexpr uint32_t idesc = make_idesc_bf16(128, BN, A_MN, B_MN);
      for (int it = 0; it < nkb; ++it) {
        const int s = it % C::STAGES, r = it / C::STAGES;
        mbar_wait(&full[s], r & 1);
        tc_fence_after();
        const uint32_t a_base = smem_u32(stage_a(s));
        const uint32_t b_base = smem_u32(stage_b(s));
#pragma unroll
        for (int kk = 0; kk < C::BK / 16; ++kk) {
          const uint64_t ad = A_MN ? make_sdesc_sw128(a_base + kk * 2048, 8192, 1024)
                                   : make_sdesc_sw128(a_base + kk * 32, 16, 1024);
          const uint64_t bd = B_MN ? make_sdesc_sw128(b_base + kk * 2048, 8192, 1024)
                                   : make_sdesc_sw128(b_base + kk * 32, 16, 1024);
          tc_mma_bf16(tmem, ad, bd, idesc, (it | kk) != 0);
        }
        tc_commit(&empty[s]);
      }
      TGP_TS(2);
      if (nkb > 0)
        tc_commit(tfull);
      else
        mbar_arrive(tfull);
    }
    __syncwarp();
    if (push_red) cluster_wait();
  } else {
    // ---------------- epilogue warps 2..5: TMEM -> registers (6..9: helpers, see TC_THREADS)
    griddep_wait();
    if (push_red) {
      // gather the owner-side epilogue operands (bias, residual, pre-activation, dropout mask) now,
      // while the mainloop streams: the tail after the split-K exchange is then arithmetic + stores
      const int S = gridDim.y, lrpr = 8 - __ffs(S), rpr = 1 << lrpr, rank = (int)cluster_ctarank();
      const int et = (int)threadIdx.x - 64;
      const int nvalid = min(BN, p.N - nb), nq = (nvalid + 3) >> 2;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int it = et + TC_FIN * t;
        if (it < rpr * nq) {
          const int fll = it & (rpr - 1), q = it >> lrpr, f = m0 + rank * rpr + fll;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (f < p.M && 4 * q + e < nvalid) pre[t][e] = epi_load<MODE>(p.epi, f, nb + 4 * q + e);
        }
      }
    }
    // helpers (warps 6..9) share the TMEM lane quadrant of warp - 4 and take every other column chunk
    // of the split-K push; the other tile kinds use warps 2..5 only
    const bool helper = warp >= 6;
    if (!helper || push_red) {
    mbar_wait(tfull, 0);
    tc_fence_after();
    if (threadIdx.x == 64) TGP_TS(3);
    const int lg = warp & 3;  // TMEM lane group accessible to this warp
    const int fl = lg * 32 + lane;
    const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16);
    if constexpr (MODE == EPI_DW) {
      // fp32 tile -> shared memory (128-byte swizzled [128 rows][32 cols] chunks, double-buffered
      // in the now idle pipeline stages) -> TMA tensor store, or TMA reduce-add into the existing
      // gradient when accumulating (the read-modify-write happens in L2); full 128-byte row
      // segments instead of 32 row-strided 16-byte stores per warp instruction
      const bool leader = threadIdx.x == 64;
      const bool acc = p.epi.accumulate != 0;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint8_t* buf = smem + (c & 1) * 16384;
        if (c >= 2) {
          if (leader) bulk_wait_read<1>();  // the store issued from this buffer has read it
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
        float v[32];
        tmem_ld16(taddr + c * 32, v);
        tmem_ld16(taddr + c * 32 + 16, v + 16);
        if (nkb == 0) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.0f;
        }
        uint8_t* row = buf + fl * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(row + ((q ^ (fl & 7)) << 4)) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        fence_proxy_async();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (leader && nb + c * 32 < p.N) {
          tma_store_2d(&tmD, buf, nb + c * 32, m0, acc);
          bulk_commit();
        }
      }
      if (leader) bulk_wait_read<0>();
    } else if constexpr (C::PUSH) {
      // push: every rank sends the slice of its partial tile owned by rank `owner` (features
      // [owner*rpr, +rpr)) into the owner's dedicated receive region, slot = source rank:
      // quad (src, c, fll, q) at float4 ((src*(BN/16) + c)*rpr + fll)*4 + (q ^ (fll & 3)).
      const int lrpr = 8 - __ffs((int)gridDim.y), rpr = 1 << lrpr;  // split S = 128 / rpr, a power of two
      const int owner = fl >> lrpr, fll = fl & (rpr - 1), src = (int)cluster_ctarank();
      const uint32_t recv = smem_u32(smem + C::DATA);
      // stage the partial tile in this CTA's (now idle) pipeline buffers, owner slice by owner slice in
      // the receive layout, then ONE bulk DSMEM copy per owner (S copies of BN * rpr * 4 bytes)
      // instead of a 16-byte st.async per float4 (C3 m = 8: 24.1 -> 23.2 ms/step, m = 4: 16.15 -> 15.97)
      const uint32_t slice = (uint32_t)(BN * rpr * 4);  // bytes of one source's slice at an owner
      const uint32_t stage0 = smem_u32(smem);
#pragma unroll 1
      for (int c = helper ? 1 : 0; c < BN / 16; c += 2) {
        float v[16];
        tmem_ld16(taddr + c * 16, v);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t idx = (uint32_t)((c * rpr + fll) * 4 + (q ^ (fll & 3)));
          const float4 val =
              nkb ? make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stage0 + (uint32_t)owner * slice + idx * 16u),
                       "f"(val.x), "f"(val.y), "f"(val.z), "f"(val.w)
                       : "memory");
        }
      }
      fence_proxy_async();
      asm volatile("bar.sync 1, %0;" ::"n"(TC_FIN) : "memory");
      cluster_wait();  // every rank's receive barrier is initialised (arrived right after setup)
      {
        const int S = (int)gridDim.y, et0 = (int)threadIdx.x - 64;
        if (et0 < S) {
          const uint32_t o = (uint32_t)et0;
          const uint32_t dst = mapa_shared(recv + (uint32_t)src * slice, o);
          const uint32_t mb = mapa_shared(smem_u32(rbar), o);
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
              "r"(stage0 + o * slice), "r"(slice), "r"(mb)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
      }

      if (threadIdx.x == 64) TGP_TS(5);
    } else {
      // partial tile -> own smem as float4 quads: quad (chunk c, feature fl, q) at
      // ((c*128 + fl)*4 + (q ^ (fl & 3))), the XOR spreading a warp's stores over the banks
      float4* red4 = reinterpret_cast<float4*>(smem);
#pragma unroll 1
      for (int c = 0; c < BN / 16; ++c) {
        float v[16];
        tmem_ld16(taddr + c * 16, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          red4[(c * 128 + fl) * 4 + (q ^ (fl & 3))] =
              nkb ? make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    }  // !helper || push_red
  }
  tc_fence_before();

  if constexpr (MODE != EPI_DW && C::PUSH) {
    // ---------------- wait for the S ranks' partials (local mbarrier), then a purely local
    // fixed-order (source-rank) sum
    if (threadIdx.x >= 64) mbar_wait(rbar, 0);
    if (threadIdx.x == 64) TGP_TS(6);
    const int S = gridDim.y;
    const int rank = (int)cluster_ctarank();
    const int lrpr = 8 - __ffs(S), rpr = 1 << lrpr;  // S is a power of two <= 8
    const int et = (int)threadIdx.x - 64;
    const int nvalid = min(BN, p.N - nb);
    const int nq = (nvalid + 3) >> 2;
    const float4* recv4 = reinterpret_cast<const float4*>(smem + C::DATA);
    float* cs = reinterpret_cast<float*>(smem + C::DATA + C::RECV_BYTES);
    const bool want_cs = MODE == EPI_ACT_BWD && p.epi.colsum;
    if (et >= 0) {
      // one work item = (feature, 4-row quad): fixed source-rank order sum, then the epilogue with
      // operands requested two items ahead (the first two during the mainloop)
      auto item = [&](int it, const EpiPre* pq) {
        const int fll = it & (rpr - 1), q = it >> lrpr;
        const int f = m0 + rank * rpr + fll;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int s = 0; s < S; ++s) {
          const float4 t = recv4[((s * (BN / 16) + (q >> 2)) * rpr + fll) * 4 + ((q & 3) ^ (fll & 3))];
          a.x += t.x;
          a.y += t.y;
          a.z += t.z;
          a.w += t.w;
        }
        const float av[4] = {a.x, a.y, a.z, a.w};
        if (threadIdx.x == 64 && it == et) TGP_TS(8);
        const float part = f < p.M ? epi_finish_rows<MODE, 4>(p.epi, f, nb + 4 * q, min(4, nvalid - 4 * q), av, pq) : 0.0f;
        if (want_cs) cs[q * rpr + fll] = part;
        if (threadIdx.x == 64 && it == et) TGP_TS(9);
      };
      auto gather = [&](int it, EpiPre* pq) {
        if (it >= rpr * nq) return;
        const int fll = it & (rpr - 1), q = it >> lrpr, f = m0 + rank * rpr + fll;
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (f < p.M && 4 * q + e < nvalid) pq[e] = epi_load<MODE>(p.epi, f, nb + 4 * q + e);
      };
#pragma unroll 1
      for (int it = et; it < rpr * nq; it += TC_FIN) {
        EpiPre nx[4];
        gather(it + 2 * TC_FIN, nx);
        item(it, pre[0]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          pre[0][e] = pre[1][e];
          pre[1][e] = nx[e];
        }
      }
      if (want_cs) {
        asm volatile("bar.sync 1, %0;" ::"n"(TC_FIN) : "memory");  // the epilogue threads only
        if (et < rpr) {
          const int f = m0 + rank * rpr + et;
          float s = 0.0f;
          for (int q = 0; q < nq; ++q) s += cs[q * rpr + et];
          if (f < p.M) p.epi.colsum[(int64_t)(nb / 16) * p.M + f] = s;
        }
      }
    }
    if (threadIdx.x == 64) TGP_TS(7);
  } else if constexpr (MODE != EPI_DW) {
    // ---------------- deterministic split-K reduction through DSMEM, fixed rank order.
    // Rank r finalises features [r*128/S, (r+1)*128/S); work item = (feature, 4-row quad); all S
    // remote quads are requested before the fixed-order sum.
    cluster_sync();
    const int S = gridDim.y;
    const int rank = (int)cluster_ctarank();
    const int lrpr = 8 - __ffs(S), rpr = 1 << lrpr;  // S is a power of two <= 8
    const int et = (int)threadIdx.x - 64;
    const int nvalid = min(BN, p.N - nb);
    const int nq = (nvalid + 3) >> 2;
    float* cs = reinterpret_cast<float*>(smem + C::RED_BYTES);  // [q][feature] column-sum partials
    const bool want_cs = MODE == EPI_ACT_BWD && p.epi.colsum;
    if (et >= 0 && et < 128) {  // warps 2..5
      const uint32_t base = smem_u32(smem);
      // UNR work items per thread per round: their global epilogue operands (residual rows,
      // saved pre-activations) are all requested before any is consumed, so the loads' latency
      // overlaps (one item at a time left the epilogue waiting on each 4-element gather)
      constexpr int UNR = 4;
#pragma unroll 1
      for (int it0 = et; it0 < rpr * nq; it0 += 128 * UNR) {
        EpiPre pq[UNR][4];
        float av[UNR][4];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int it = it0 + 128 * u;
          if (it >= rpr * nq) break;
          const int fll = it & (rpr - 1), q = it >> lrpr;
          const int fl = rank * rpr + fll;
          const int f = m0 + fl;
          const uint32_t off = (uint32_t)(((q >> 2) * 128 + fl) * 4 + ((q & 3) ^ (fl & 3))) * 16u;
          float4 t[8];
#pragma unroll
          for (int s = 0; s < 8; ++s)
            if (s < S) t[s] = ld_dsmem_f32x4(mapa_shared(base + off, (uint32_t)s));
          float4 a = t[0];
#pragma unroll
          for (int s = 1; s < 8; ++s)
            if (s < S) {
              a.x += t[s].x;
              a.y += t[s].y;
              a.z += t[s].z;
              a.w += t[s].w;
            }
          av[u][0] = a.x;
          av[u][1] = a.y;
          av[u][2] = a.z;
          av[u][3] = a.w;
          if (f < p.M) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (4 * q + e < nvalid) pq[u][e] = epi_load<MODE>(p.epi, f, nb + 4 * q + e);
          }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int it = it0 + 128 * u;
          if (it >= rpr * nq) break;
          const int fll = it & (rpr - 1), q = it >> lrpr;
          const int f = m0 + rank * rpr + fll;
          float part = 0.0f;
          if (f < p.M) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (4 * q + e < nvalid) part += epi_finish<MODE>(p.epi, f, nb + 4 * q + e, av[u][e], pq[u][e]);
          }
          if (want_cs) cs[q * rpr + fll] = part;
        }
      }
      if (want_cs) {
        asm volatile("bar.sync 1, 128;" ::: "memory");  // the 128 epilogue threads only
        if (et < rpr) {
          const int f = m0 + rank * rpr + et;
          float s = 0.0f;
          for (int q = 0; q < nq; ++q) s += cs[q * rpr + et];
          if (f < p.M) p.epi.colsum[(int64_t)(nb / 16) * p.M + f] = s;
        }
      }
    }
    cluster_sync();
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
  if (threadIdx.x == 0) TGP_TS(4);
}

// ---------------------------------------------------------------------------------- host side
bool make_map(CUtensorMap* map, const TcMat& t, int box_inner, int box_outer, bool l2_promote) {
  const Driver* d = driver();
  if (!d) return false;
  cuuint64_t dims[2] = {(cuuint64_t)t.cols, (cuuint64_t)t.rows};
  cuuint64_t strides[1] = {(cuuint64_t)t.ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = d->tensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(t.ptr), dims,
                                       strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                       CU_TENSOR_MAP_SWIZZLE_128B,
                                       l2_promote ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): rows=%lld cols=%lld ld=%lld box=%dx%d", (int)r,
              (long long)t.rows, (long long)t.cols, (long long)t.ld, box_inner, box_outer);
    return false;
  }
  return true;
}

template <int BN, bool A_MN, bool B_MN, int MODE>
static int launch_tc(cudaStream_t st, bool pdl, const CUtensorMap& a, const CUtensorMap& b0, const CUtensorMap& b1,
                     const CUtensorMap& dmap, const GemmParams& p, int S, int ntiles) {
  using C = TcCfg<BN>;
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN, MODE>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute(smem=%d): %s", C::SMEM, cudaGetErrorString(e));
      return -3;
    }
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.M + 127) / 128, S, ntiles);
  cfg.blockDim = dim3(TC_THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 1;
  attrs[0].val.clusterDim.y = S;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, b0, b1, dmap, p);
  if (e != cudaSuccess) {
    set_error("gemm_tc launch (BN=%d A_MN=%d B_MN=%d grid=%d,%d,%d): %s", BN, (int)A_MN, (int)B_MN, (p.M + 127) / 128, S,
              ntiles, cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

int gemm_tc(cudaStream_t st, bool pdl, const TcMat& A, bool a_mn, const TcMat& B0, const TcMat* B1, bool b_mn,
            GemmParams p, int splits) {
  if (p.M % 64 || p.K % 64 || p.M <= 0 || p.N <= 0) {
    // M % 64: the last 128-row tile may be half empty (TMA zero-fills, the epilogue masks f >= M)
    set_error("gemm_tc: unsupported shape M=%d N=%d K=%d (need M%%64==0, K%%64==0)", p.M, p.N, p.K);
    return -5;
  }
  const bool dw = p.epi.mode == EPI_DW;
  int BN;
  if (dw) {
    BN = p.N >= 256 ? 256 : (p.N >= 128 ? 128 : 64);
    if (p.N % 64 && b_mn) {
      set_error("gemm_tc dW: N=%d must be a multiple of 64", p.N);
      return -5;
    }
  } else {
    BN = p.N <= 16 ? 16 : p.N <= 32 ? 32 : p.N <= 64 ? 64 : 128;
  }
  const int ntiles = (p.N + BN - 1) / BN;
  const int nkb = p.K / 64;
  int S = 1;
  if (!dw) {
    const int mt = (p.M + 127) / 128;
    S = splits > 0 ? splits : env_int("TGP_SPLITK", 0);
    if (S <= 0) {
      // ~one wave of 148 CTAs (measured: in the full step, split 4 beats split 8 at C2 although an
      // isolated PDL-chained GEMM prefers 8 -- profiles/gemm_timeline.py)
      S = (148 + mt * ntiles / 2) / (mt * ntiles);
    }
    S = std::max(1, std::min(S, 8));
    S = std::min(S, nkb);
    while (128 % S) --S;  // rows-per-rank must divide the 128-row tile
  }
  p.kb_per_split = (nkb + S - 1) / S;
  S = (nkb + p.kb_per_split - 1) / p.kb_per_split;
  while (128 % S) {  // keep 128 divisible by S after re-balancing
    ++p.kb_per_split;
    S = (nkb + p.kb_per_split - 1) / p.kb_per_split;
  }
  if (!B1) p.k_seg = p.K;

  CUtensorMap ma, mb0, mb1;
  if (!make_map(&ma, A, 64, a_mn ? 64 : 128)) return -3;
  const int b_outer = b_mn ? 64 : BN;
  if (!make_map(&mb0, B0, 64, b_outer)) return -3;
  if (B1) {
    if (!make_map(&mb1, *B1, 64, b_outer)) return -3;
  } else {
    mb1 = mb0;
  }
  CUtensorMap md = mb0;  // dW: fp32 [M][ldw] output, box {32 cols, 128 rows}, 128-byte swizzle
  if (dw) {
    const Driver* drv = driver();
    if (!drv) return -3;
    cuuint64_t dims[2] = {(cuuint64_t)p.N, (cuuint64_t)p.M};
    cuuint64_t strides[1] = {(cuuint64_t)p.epi.ldw * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = drv->tensorMapEncodeTiled(&md, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p.epi.dw, dims, strides, box, es,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("dW output tensor map failed (%d): M=%d N=%d ldw=%lld", (int)r, p.M, p.N, (long long)p.epi.ldw);
      return -3;
    }
  }
  // instantiated for the (operand majors, epilogue mode) pairs the runtime uses: forward
  // W[out][in] x X[rows][in] (K-major, K-major), backward W^T x dY (MN-major, K-major), deferred dW
  // dY^T x X (MN-major, MN-major)
  const int mode = p.epi.mode;
#define TGP_LAUNCH_M(BNv, AM, BM, MD) \
  if (BN == BNv && a_mn == AM && b_mn == BM && mode == MD) return launch_tc<BNv, AM, BM, MD>(st, pdl, ma, mb0, mb1, md, p, S, ntiles);
#define TGP_LAUNCH(BNv)                                  \
  TGP_LAUNCH_M(BNv, false, false, EPI_LINEAR_FWD)        \
  TGP_LAUNCH_M(BNv, false, false, EPI_RESID_FWD)         \
  TGP_LAUNCH_M(BNv, false, false, EPI_STORE)             \
  TGP_LAUNCH_M(BNv, true, false, EPI_ACT_BWD)            \
  TGP_LAUNCH_M(BNv, true, false, EPI_STORE)
  if (!dw) {
    TGP_LAUNCH(16)
    TGP_LAUNCH(32)
    TGP_LAUNCH(64)
    TGP_LAUNCH(128)
    TGP_LAUNCH(256)
  } else {
    TGP_LAUNCH_M(64, true, true, EPI_DW)
    TGP_LAUNCH_M(128, true, true, EPI_DW)
    TGP_LAUNCH_M(256, true, true, EPI_DW)
  }
#undef TGP_LAUNCH_M
#undef TGP_LAUNCH
  set_error("gemm_tc: no instantiation for BN=%d a_mn=%d b_mn=%d mode=%d", BN, (int)a_mn, (int)b_mn, mode);
  return -5;
}

}  // namespace tgp

#ifdef TGP_GEMM_TIMING
extern "C" int tgp_debug_timestamps(unsigned long long* out, int cap, int reset) {
  unsigned int n = 0;
  cudaMemcpyFromSymbol(&n, tgp::g_ts_next, 4);
  const int m = (int)(n < (unsigned)cap ? n : (unsigned)cap);
  cudaMemcpyFromSymbol(out, tgp::g_ts, (size_t)m * 12 * 8);
  if (reset) {
    unsigned int z = 0;
    cudaMemcpyToSymbol(tgp::g_ts_next, &z, 4);
  }
  return m;
}
#endif
