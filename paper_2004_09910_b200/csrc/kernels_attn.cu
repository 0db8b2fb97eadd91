// GPT-2-shaped stage kernels (C5, BASELINE.json configs[4]): causal multi-head
// attention forward / backward, token + position embedding forward and its deterministic deferred
// weight gradient, and the token cross-entropy loss.  The formulas are the textbook ones the oracle
// states (oracle/model.py header; reading Z13); dropout uses the same Philox decision as every other
// site (O8), on the [n_seq, n_heads, seq, seq] probability tensor for attention.
//
// Attention: head dim 64, 64-row query / key tiles, one CTA of 4 warps per (tile, head, sequence),
// bf16 mma.sync m16n8k16 with fp32 accumulation (the tiles are 64 x 64: too small for a 128-row
// tcgen05 MMA per warp group), flash-style online softmax.  Backward recomputes P
// from the saved log-sum-exp and splits into a dK/dV kernel (per key tile, loop over query tiles)
// and a dQ kernel (per query tile, loop over key tiles): every output element is written by exactly
// one thread, no atomics, so the backward is deterministic.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "host.h"
#include "kernels_gpt.h"

namespace tgp {

namespace {

#ifndef TGP_ATTN_MINB
#define TGP_ATTN_MINB 1
#endif
constexpr int HD = 64;     // head dim
constexpr int TILE = 64;   // query / key tile
constexpr int PITCH = 72;  // smem row pitch (bf16 elements): conflict-free fragment loads
constexpr float LOG2E = 1.4426950408889634f;

TGP_DEV void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
TGP_DEV uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
TGP_DEV uint32_t ld32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

// 64 rows x 64 bf16 columns from global (row stride ld elements) into smem [64][PITCH]; optionally
// also the transpose into smem T[64][PITCH] (T[c][r] = X[r][c]).
TGP_DEV void load_tile(const __nv_bfloat16* g, int64_t ld, __nv_bfloat16* S, __nv_bfloat16* T) {
  for (int q = threadIdx.x; q < TILE * 8; q += blockDim.x) {
    const int r = q >> 3, c8 = (q & 7) * 8;
    const uint4 v = *reinterpret_cast<const uint4*>(g + (int64_t)r * ld + c8);
    if (S) *reinterpret_cast<uint4*>(S + r * PITCH + c8) = v;
    if (T) {
      const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int k = 0; k < 8; ++k) T[(c8 + k) * PITCH + r] = e[k];
    }
  }
}
// same from fp32 global (converted to bf16)
TGP_DEV void load_tile_f32(const float* g, int64_t ld, __nv_bfloat16* S, __nv_bfloat16* T) {
  for (int q = threadIdx.x; q < TILE * 16; q += blockDim.x) {
    const int r = q >> 4, c4 = (q & 15) * 4;
    const float4 v = *reinterpret_cast<const float4*>(g + (int64_t)r * ld + c4);
    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __nv_bfloat16 b = __float2bfloat16_rn(e[k]);
      if (S) S[r * PITCH + c4 + k] = b;
      if (T) T[(c4 + k) * PITCH + r] = b;
    }
  }
}
// A fragments (16 rows starting at row0, k = 64) of a [64][PITCH] smem tile
TGP_DEV void load_afrag(const __nv_bfloat16* S, int row0, uint32_t (*a)[4]) {
  const int g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    a[kc][0] = ld32(S + (row0 + g) * PITCH + kc * 16 + 2 * t);
    a[kc][1] = ld32(S + (row0 + g + 8) * PITCH + kc * 16 + 2 * t);
    a[kc][2] = ld32(S + (row0 + g) * PITCH + kc * 16 + 8 + 2 * t);
    a[kc][3] = ld32(S + (row0 + g + 8) * PITCH + kc * 16 + 8 + 2 * t);
  }
}
TGP_DEV void ldsm_x4(uint32_t* r, const __nv_bfloat16* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
TGP_DEV void ldsm_x4_t(uint32_t* r, const __nv_bfloat16* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
// acc[nt][4] (+)= A(16 x 64, fragments a) * B^T, B element (n, k) = Bs[n][k] for n < 64.  B fragments
// by ldmatrix: matrix i of an x4 = 8 rows n x 8 columns k at k offset 8i (b0 / b1 of two k-chunks).
TGP_DEV void mma_row_tile(float (*acc)[4], const uint32_t (*a)[4], const __nv_bfloat16* Bs) {
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    uint32_t b[8];
    ldsm_x4(b, Bs + (nt * 8 + (l & 7)) * PITCH + (l >> 3) * 8);
    ldsm_x4(b + 4, Bs + (nt * 8 + (l & 7)) * PITCH + 32 + (l >> 3) * 8);
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) mma16816(acc[nt], a[kc], b[2 * kc], b[2 * kc + 1]);
  }
}
// acc[dt][4] += P(16 x 64 keys, accumulator layout p[nt][4]) * X, X element (k, n) = Xs[k][n] (row-major
// [64 k][64 n] tile): B fragments by ldmatrix.trans (matrix i: k rows 8(i&1).., n columns 8(i>>1)..).
TGP_DEV void mma_p_tile(float (*acc)[4], const float (*p)[4], const __nv_bfloat16* Xs) {
  const int l = threadIdx.x & 31;
#pragma unroll
  for (int kc = 0; kc < 4; ++kc) {
    uint32_t a[4];
    a[0] = pack2(p[2 * kc][0], p[2 * kc][1]);
    a[1] = pack2(p[2 * kc][2], p[2 * kc][3]);
    a[2] = pack2(p[2 * kc + 1][0], p[2 * kc + 1][1]);
    a[3] = pack2(p[2 * kc + 1][2], p[2 * kc + 1][3]);
#pragma unroll
    for (int dp = 0; dp < 4; ++dp) {
      uint32_t b[4];
      ldsm_x4_t(b, Xs + (kc * 16 + ((l >> 3) & 1) * 8 + (l & 7)) * PITCH + (2 * dp + (l >> 4)) * 8);
      mma16816(acc[2 * dp], a, b[0], b[1]);
      mma16816(acc[2 * dp + 1], a, b[2], b[3]);
    }
  }
}

struct AttnArgs {
  const __nv_bfloat16* qkv;  // [rows][3d] (q | k | v), rows pre-offset to the micro-batch
  int64_t ldq;
  int d, nh, seq;
  int64_t seq0;  // global sequence index of row 0 (dropout counters)
  float scale_log2;  // log2(e) / sqrt(64)
  float scale;       // 1 / sqrt(64)
  uint32_t thresh;
  float dscale;
  uint64_t seed;
  const uint32_t* step;
  uint32_t site;
};

// Keep bits of a 64-key tile for the accumulator layout (rows q0 and q0 + 8 of this thread, keys
// kbase + nt*8 + 2t + {0, 1}): one Philox call yields the 4 words of 4 consecutive keys (the flat
// index is a multiple of 4 at every 4-key group because seq % 64 == 0), so the two lanes t, t^1 that
// share a group split the rows -- even t draws row q0, odd t row q0 + 8 -- and swap halves with one
// shuffle: 8 Philox calls per thread per tile instead of 32.  Bit (nt*4 + c) = keep of element [nt][c].
TGP_DEV uint32_t attn_keep_tile(const AttnArgs& A, int s, int h, int q0, int kbase) {
  const int t = threadIdx.x & 3;
  const int qm = q0 + (t & 1) * 8;
  const uint64_t rowbase = (((uint64_t)(A.seq0 + s) * A.nh + h) * A.seq + qm) * A.seq;
  const uint2 key = make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32));
  const uint32_t step = *A.step;
  uint32_t bits = 0;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const uint64_t qi = (rowbase + kbase + nt * 8 + (t >> 1) * 4) >> 2;
    const uint4 o = philox4x32_10(make_uint4((uint32_t)qi, (uint32_t)(qi >> 32), A.site, step), key);
    const uint32_t mine = ((o.x >> 8) >= A.thresh ? 1u : 0u) | ((o.y >> 8) >= A.thresh ? 2u : 0u) |
                          ((o.z >> 8) >= A.thresh ? 4u : 0u) | ((o.w >> 8) >= A.thresh ? 8u : 0u);
    const uint32_t other = __shfl_xor_sync(0xffffffffu, mine, 1);
    const uint32_t r0 = (t & 1) ? other : mine, r1 = (t & 1) ? mine : other;  // groups of rows q0, q0 + 8
    const int off = (t & 1) * 2;  // this lane's keys 2t, 2t+1 inside the 4-key group
    bits |= (((r0 >> off) & 3u) | (((r1 >> off) & 3u) << 2)) << (nt * 4);
  }
  return bits;
}

// Same for the transposed accumulator layout of the dK/dV kernel (rows = keys k0 + {0, 8} with
// k0 = kbase + g, columns = queries qbase + nt*8 + 2t + {0, 1}).  The 4 consecutive keys of a Philox
// group sit in the 4 lanes g = 4j..4j+3 (same t); lane j of the quartet draws the groups of
// element c = j for every nt, then 4 shuffles hand every lane its own key's bit of each group.
TGP_DEV uint32_t attn_keep_tile_t(const AttnArgs& A, int s, int h, int kbase_w, int qbase) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, j = g & 3;
  const uint2 key = make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32));
  const uint32_t step = *A.step;
  const uint64_t hb = ((uint64_t)(A.seq0 + s) * A.nh + h) * A.seq;
  const int kgrp = kbase_w + (g & ~3) + (j >> 1) * 8;  // key group of element c = j
  uint32_t W = 0;
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) {
    const int q = qbase + nt * 8 + 2 * t + (j & 1);
    const uint64_t qi = ((hb + q) * A.seq + kgrp) >> 2;
    const uint4 o = philox4x32_10(make_uint4((uint32_t)qi, (uint32_t)(qi >> 32), A.site, step), key);
    W |= (((o.x >> 8) >= A.thresh ? 1u : 0u) | ((o.y >> 8) >= A.thresh ? 2u : 0u) |
          ((o.z >> 8) >= A.thresh ? 4u : 0u) | ((o.w >> 8) >= A.thresh ? 8u : 0u))
         << (nt * 4);
  }
  uint32_t bits = 0;
#pragma unroll
  for (int sl = 0; sl < 4; ++sl) {
    const uint32_t V = __shfl_sync(0xffffffffu, W, (((g & ~3) + sl) << 2) | t);
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) bits |= ((V >> (nt * 4 + j)) & 1u) << (nt * 4 + sl);
  }
  return bits;
}


// Work items of the forward: (query tile, key-tile range, part).  Causal rows are unequal (query tile
// qt sees qt + 1 key tiles), and one micro-batch is one sequence, so a launch holds only
// 25 heads x 16 tiles: the longest CTA (16 key tiles) bounded the kernel at ~2x the average.  Long
// rows are therefore split into parts of <= KS key tiles (heaviest first); split rows write
// unnormalised partial (O, m, l) and attn_fwd_merge_kernel combines the parts in fixed order.
constexpr int FWD_MAX_ITEMS = 256, FWD_MAX_PARTS = 4, PART_STRIDE = HD + 2;
struct FwdItems {
  uint32_t it[FWD_MAX_ITEMS];  // qt | kt0 << 8 | kt1 << 16 | part << 24 (bit 31: split row)
};

__global__ void __launch_bounds__(128, TGP_ATTN_MINB) attn_fwd_kernel(AttnArgs A, __nv_bfloat16* __restrict__ ctx, int64_t ldc,
                                                       float* __restrict__ lse, const FwdItems items,
                                                       float* __restrict__ part_buf) {
  __shared__ __align__(16) __nv_bfloat16 Qs[TILE * PITCH], Ks[TILE * PITCH], Vs[TILE * PITCH];
  const uint32_t item = items.it[blockIdx.x];
  const int qt = item & 0xFF, kt0 = (item >> 8) & 0xFF, kt1 = (item >> 16) & 0xFF, part = (item >> 24) & 0x7F;
  const bool split = (item >> 31) != 0;
  const int h = blockIdx.y, s = blockIdx.z;
  const int w = threadIdx.x >> 5, g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
  const int64_t base = (int64_t)s * A.seq;
  load_tile(A.qkv + (base + qt * TILE) * A.ldq + h * HD, A.ldq, Qs, nullptr);
  __syncthreads();
  uint32_t qa[4][4];
  load_afrag(Qs, w * 16, qa);
  float m2[2] = {-INFINITY, -INFINITY}, l[2] = {0.0f, 0.0f};
  float o[8][4] = {};
  const int q0 = qt * TILE + w * 16 + g;
  for (int kt = kt0; kt <= kt1; ++kt) {
    __syncthreads();
    load_tile(A.qkv + (base + kt * TILE) * A.ldq + A.d + h * HD, A.ldq, Ks, nullptr);
    load_tile(A.qkv + (base + kt * TILE) * A.ldq + 2 * A.d + h * HD, A.ldq, Vs, nullptr);
    __syncthreads();
    float sc[8][4] = {};
    mma_row_tile(sc, qa, Ks);
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int key = kt * TILE + nt * 8 + 2 * t + (c & 1), q = q0 + (c >> 1) * 8;
        float v = sc[nt][c] * A.scale_log2;
        if (key > q) v = -INFINITY;
        sc[nt][c] = v;
        mx[c >> 1] = fmaxf(mx[c >> 1], v);
      }
    float alpha[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
      const float mn = fmaxf(m2[r], mx[r]);
      alpha[r] = exp2f(m2[r] - mn);
      m2[r] = mn;
      l[r] *= alpha[r];
    }
    const uint32_t kb = A.thresh ? attn_keep_tile(A, s, h, q0, kt * TILE) : 0xFFFFFFFFu;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float p = exp2f(sc[nt][c] - m2[c >> 1]);
        l[c >> 1] += p;
        if (A.thresh) p = ((kb >> (nt * 4 + c)) & 1u) ? p * A.dscale : 0.0f;
        sc[nt][c] = p;
      }
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      o[dt][0] *= alpha[0];
      o[dt][1] *= alpha[0];
      o[dt][2] *= alpha[1];
      o[dt][3] *= alpha[1];
    }
    mma_p_tile(o, sc, Vs);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
  }
  if (split) {  // unnormalised partial of this key range
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int64_t row = base + q0 + r * 8;
      float* pb = part_buf + ((row * A.nh + h) * FWD_MAX_PARTS + part) * PART_STRIDE;
#pragma unroll
      for (int dt = 0; dt < 8; ++dt)
        *reinterpret_cast<float2*>(pb + dt * 8 + 2 * t) = make_float2(o[dt][2 * r], o[dt][2 * r + 1]);
      if (t == 0) {
        pb[HD] = m2[r];
        pb[HD + 1] = l[r];
      }
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t row = base + q0 + r * 8;
    const float inv = 1.0f / l[r];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt)
      *reinterpret_cast<uint32_t*>(ctx + row * ldc + h * HD + dt * 8 + 2 * t) =
          pack2(o[dt][2 * r] * inv, o[dt][2 * r + 1] * inv);
    if (t == 0) lse[row * A.nh + h] = m2[r] + log2f(l[r]);  // log2 domain
  }
}

// Combine the parts of split rows (fixed part order): one warp per (row, head), 2 columns per lane.
__global__ void attn_fwd_merge_kernel(const float* __restrict__ part_buf, int seq, int nh, int q_first, int nparts_max,
                                      int ks, int nrows, __nv_bfloat16* __restrict__ ctx, int64_t ldc,
                                      float* __restrict__ lse) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= nrows * nh) return;
  const int h = wid % nh, rr = wid / nh;           // rr enumerates the split rows of every sequence
  const int per_seq = seq - q_first;
  const int s = rr / per_seq, q = q_first + rr % per_seq;
  const int np = (q / TILE) / ks + 1;              // parts of this query tile
  const int64_t row = (int64_t)s * seq + q;
  const float* pb = part_buf + (row * nh + h) * FWD_MAX_PARTS * PART_STRIDE;
  float m = -INFINITY;
  for (int p = 0; p < np; ++p) m = fmaxf(m, pb[p * PART_STRIDE + HD]);
  float lt = 0.0f, o0 = 0.0f, o1 = 0.0f;
  for (int p = 0; p < np; ++p) {
    const float sc = exp2f(pb[p * PART_STRIDE + HD] - m);
    lt += pb[p * PART_STRIDE + HD + 1] * sc;
    o0 += pb[p * PART_STRIDE + 2 * lane] * sc;
    o1 += pb[p * PART_STRIDE + 2 * lane + 1] * sc;
  }
  const float inv = 1.0f / lt;
  *reinterpret_cast<uint32_t*>(ctx + row * ldc + h * HD + 2 * lane) = pack2(o0 * inv, o1 * inv);
  if (lane == 0) lse[row * nh + h] = m + log2f(lt);
  (void)nparts_max;
}

// ---------------------------------------------------------------------------------------------
// tcgen05 forward (seq % 128 == 0): one CTA of 4 warps per (128-query tile, head, sequence); thread
// = query row = TMEM lane, so the softmax statistics of a row are thread-local.  Per 128-key tile:
// S = Q K^T (tcgen05.mma 128x128x64, fp32 in TMEM) -> registers -> mask, online softmax, Philox
// dropout -> P (bf16) into a 128-byte-swizzled K-major smem tile -> O_tile = P V (tcgen05.mma
// 128x64x128, V read MN-major) -> registers, O = alpha O + O_tile.  K / V tiles double-buffered with
// cp.async into the swizzled layout; Q, K and P are K-major operands, V an MN-major one.  Same
// arithmetic as the mma.sync kernel up to accumulation order (both sides bf16 operands, fp32 sums).
TGP_DEV void cp_async16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(g) : "memory");
}
TGP_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
TGP_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int TCQ = 128;
constexpr int TC_SMEM = 16384 * 7 + 64 + 1024 + 1024;  // Q, K[2], V[2], P (2 chunks), barriers, row exchange + align

// row r, 16-byte chunk c of a [rows][64] bf16 tile in the SW128 layout
TGP_DEV uint32_t sw_off(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }
TGP_DEV void load_sw_tile(const __nv_bfloat16* g, int64_t ld, uint8_t* S) {
  for (int q = threadIdx.x; q < TCQ * 8; q += blockDim.x) {
    const int r = q >> 3, c = q & 7;
    cp_async16(S + sw_off(r, c), g + (int64_t)r * ld + c * 8);
  }
}

#ifndef TGP_ATTN_TC_MINB
#define TGP_ATTN_TC_MINB 1
#endif
__global__ void __launch_bounds__(256, TGP_ATTN_TC_MINB) attn_fwd_tc_kernel(AttnArgs A, __nv_bfloat16* __restrict__ ctx, int64_t ldc,
                                                          float* __restrict__ lse) {
  // 8 warps: warp w reads TMEM lane quadrant (w & 3) and owns key half / output-column half (w >> 2)
  // of its rows, so two threads share a query row (row max and sum combined through smem)
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = sm;
  uint8_t* Ks0 = sm + 16384;
  uint8_t* Vs0 = sm + 3 * 16384;
  uint8_t* Ps = sm + 5 * 16384;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 7 * 16384);  // [0] S done, [1] PV done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  float* xch = reinterpret_cast<float*>(sm + 7 * 16384 + 64);  // [2][128] row max / sum halves
  const int qt = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int hf = w >> 2, row = (w & 3) * 32 + lane;
  const int64_t base = (int64_t)s * A.seq;
  const int q = qt * TCQ + row;
  const __nv_bfloat16* Kg = A.qkv + base * A.ldq + A.d + h * HD;
  const __nv_bfloat16* Vg = A.qkv + base * A.ldq + 2 * A.d + h * HD;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (w == 0) tmem_alloc(tslot, 256);
  load_sw_tile(A.qkv + (base + qt * TCQ) * A.ldq + h * HD, A.ldq, Qs);
  load_sw_tile(Kg, A.ldq, Ks0);
  load_sw_tile(Vg, A.ldq, Vs0);
  cp_async_commit();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
  constexpr uint32_t idS = make_idesc_bf16(128, 128, false, false);
  constexpr uint32_t idO = make_idesc_bf16(128, 64, false, true);
  const uint64_t rowbase = (((uint64_t)(A.seq0 + s) * A.nh + h) * A.seq + q) * A.seq;
  const uint2 pkey = make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32));
  const uint32_t pstep = A.thresh ? *A.step : 0u;
  float m2 = -INFINITY, l = 0.0f;
  float o[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) o[i] = 0.0f;
  const int nkt = qt + 1;
  for (int kt = 0; kt < nkt; ++kt) {
    const int st = kt & 1;
    uint8_t* Ks = Ks0 + st * 16384;
    uint8_t* Vs = Vs0 + st * 16384;
    if (kt + 1 < nkt) {
      load_sw_tile(Kg + (int64_t)(kt + 1) * TCQ * A.ldq, A.ldq, Ks0 + (st ^ 1) * 16384);
      load_sw_tile(Vg + (int64_t)(kt + 1) * TCQ * A.ldq, A.ldq, Vs0 + (st ^ 1) * 16384);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        tc_mma_bf16(tS, make_sdesc_sw128(smem_u32(Qs) + kk * 32, 16, 1024), make_sdesc_sw128(smem_u32(Ks) + kk * 32, 16, 1024),
                    idS, kk > 0);
      tc_commit(&bar[0]);
    }
    mbar_wait(&bar[0], (uint32_t)(kt & 1));
    tc_fence_after();
    float sv[64];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld16(tS + lane_off + hf * 64 + c * 16, sv + c * 16);
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const int key = kt * TCQ + hf * 64 + j;
      const float v = key <= q ? sv[j] * A.scale_log2 : -INFINITY;
      sv[j] = v;
      mx = fmaxf(mx, v);
    }
    xch[hf * 128 + row] = mx;
    __syncthreads();
    mx = fmaxf(xch[row], xch[128 + row]);
    const float mn = fmaxf(m2, mx);
    const float alpha = exp2f(m2 - mn);
    m2 = mn;
    l *= alpha;
#pragma unroll
    for (int g4 = 0; g4 < 16; ++g4) {
      uint32_t kb = 0xFu;
      if (A.thresh) {
        const uint64_t qi = (rowbase + (uint64_t)(kt * TCQ + hf * 64 + 4 * g4)) >> 2;
        const uint4 ph = philox4x32_10(make_uint4((uint32_t)qi, (uint32_t)(qi >> 32), A.site, pstep), pkey);
        kb = ((ph.x >> 8) >= A.thresh ? 1u : 0u) | ((ph.y >> 8) >= A.thresh ? 2u : 0u) |
             ((ph.z >> 8) >= A.thresh ? 4u : 0u) | ((ph.w >> 8) >= A.thresh ? 8u : 0u);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 4 * g4 + e;
        float p = exp2f(sv[j] - mn);
        l += p;
        if (A.thresh) p = ((kb >> e) & 1u) ? p * A.dscale : 0.0f;
        sv[j] = p;
      }
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {  // this half's 64 keys = K-chunk hf of P
      uint4 v;
      v.x = pack2(sv[8 * c], sv[8 * c + 1]);
      v.y = pack2(sv[8 * c + 2], sv[8 * c + 3]);
      v.z = pack2(sv[8 * c + 4], sv[8 * c + 5]);
      v.w = pack2(sv[8 * c + 6], sv[8 * c + 7]);
      *reinterpret_cast<uint4*>(Ps + hf * 16384 + sw_off(row, c)) = v;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] *= alpha;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        tc_mma_bf16(tO, make_sdesc_sw128(smem_u32(Ps) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    make_sdesc_sw128(smem_u32(Vs) + kk * 2048, 8192, 1024), idO, kk > 0);
      tc_commit(&bar[1]);
    }
    mbar_wait(&bar[1], (uint32_t)(kt & 1));
    tc_fence_after();
    float pv[32];
    tmem_ld16(tO + lane_off + hf * 32, pv);
    tmem_ld16(tO + lane_off + hf * 32 + 16, pv + 16);
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] += pv[i];
  }
  xch[hf * 128 + row] = l;  // (the last tile's reads of xch finished before the PV barrier)
  __syncthreads();
  const float lt = xch[row] + xch[128 + row];
  const float inv = 1.0f / lt;
  __nv_bfloat16* orow = ctx + (base + q) * ldc + h * HD + hf * 32;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint4 v;
    v.x = pack2(o[8 * c] * inv, o[8 * c + 1] * inv);
    v.y = pack2(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
    v.z = pack2(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
    v.w = pack2(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
    *reinterpret_cast<uint4*>(orow + 8 * c) = v;
  }
  if (hf == 0) lse[(base + q) * A.nh + h] = m2 + log2f(lt);
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 256);
}

// ---------------------------------------------------------------- tcgen05 attention backward
// The same VJP as attn_bwd_dkv_kernel / attn_bwd_dq_kernel (P recomputed from the saved log-sum-exp,
// dS = Pd o (dPd - D), D = rowsum(dO o O); oracle/model.py _attn_bwd), on 128 x 128 tiles with every
// product on the 5th-generation tensor cores: S = Q K^T and dP = dO V^T with the query as the MMA M
// side (TMEM lane = query row), then the transposed products dV += Pd^T dO, dK += dS^T Q (dK/dV
// kernel) or dQ += dS K (dQ kernel) read Pd / dS back from shared memory as MN-major operands, so no
// transpose is ever materialised.  8 warps: warp w reads TMEM lane quadrant w & 3 and handles key
// half w >> 2 of its query row (the forward's layout); one thread issues the MMAs.  Every output
// element is accumulated by one CTA in a fixed order: deterministic.
constexpr int BTC_SMEM_KV = 16384 * 8 + 64 + 1024;  // K, V, Q, dO, Pd (2 chunks), dS (2 chunks), barriers
constexpr int BTC_SMEM_Q = 16384 * 6 + 64 + 1024;   // Q, dO, K, V, dS (2 chunks), barriers

// fp32 [128][64] rows (row stride ld) -> bf16 SW128 tile (the K-major operand layout)
TGP_DEV void load_sw_tile_f32(const float* g, int64_t ld, uint8_t* S) {
  for (int q = threadIdx.x; q < TCQ * 8; q += blockDim.x) {
    const int r = q >> 3, c = q & 7;
    const float4 a = *reinterpret_cast<const float4*>(g + (int64_t)r * ld + c * 8);
    const float4 b = *reinterpret_cast<const float4*>(g + (int64_t)r * ld + c * 8 + 4);
    uint4 v;
    v.x = pack2(a.x, a.y);
    v.y = pack2(a.z, a.w);
    v.z = pack2(b.x, b.y);
    v.w = pack2(b.z, b.w);
    *reinterpret_cast<uint4*>(S + sw_off(r, c)) = v;
  }
}

// Pd and dS of this thread's 64 keys (half hf) of query row q for key tile kt, from the S and dP
// accumulators in TMEM, written as bf16 into [128 q][128 k] tiles (two SW128 chunks of 64 keys).
// Pd: the dropped-out probability (what dV sees); dS = P (dPd - D) with dPd the dropped-out dP.
TGP_DEV void attn_bwd_tc_probs(const AttnArgs& A, uint32_t tS, uint32_t tdP, int row, int hf, int q, int kt,
                               float lse_q, float D_q, uint64_t rowbase, uint32_t pstep, uint8_t* Pd, uint8_t* dS) {
  const uint2 pkey = make_uint2((uint32_t)A.seed, (uint32_t)(A.seed >> 32));
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {  // 16 keys at a time
    float sv[16], dv[16];
    tmem_ld16(tS + hf * 64 + c * 16, sv);
    tmem_ld16(tdP + hf * 64 + c * 16, dv);
    float pv[16], gv[16];
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) {
      const int key0 = kt * TCQ + hf * 64 + c * 16 + 4 * g4;
      uint32_t kb = 0xFu;
      if (A.thresh) {
        const uint64_t qi = (rowbase + (uint64_t)key0) >> 2;
        const uint4 ph = philox4x32_10(make_uint4((uint32_t)qi, (uint32_t)(qi >> 32), A.site, pstep), pkey);
        kb = ((ph.x >> 8) >= A.thresh ? 1u : 0u) | ((ph.y >> 8) >= A.thresh ? 2u : 0u) |
             ((ph.z >> 8) >= A.thresh ? 4u : 0u) | ((ph.w >> 8) >= A.thresh ? 8u : 0u);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = 4 * g4 + e;
        const float p = key0 + e <= q ? exp2f(sv[j] * A.scale_log2 - lse_q) : 0.0f;
        float pd = p, dpd = dv[j];
        if (A.thresh) {
          const bool keep = (kb >> e) & 1u;
          pd = keep ? p * A.dscale : 0.0f;
          dpd = keep ? dpd * A.dscale : 0.0f;
        }
        pv[j] = pd;
        gv[j] = p * (dpd - D_q);
      }
    }
#pragma unroll
    for (int h8 = 0; h8 < 2; ++h8) {
      uint4 a, b;
      a.x = pack2(pv[8 * h8], pv[8 * h8 + 1]);
      a.y = pack2(pv[8 * h8 + 2], pv[8 * h8 + 3]);
      a.z = pack2(pv[8 * h8 + 4], pv[8 * h8 + 5]);
      a.w = pack2(pv[8 * h8 + 6], pv[8 * h8 + 7]);
      b.x = pack2(gv[8 * h8], gv[8 * h8 + 1]);
      b.y = pack2(gv[8 * h8 + 2], gv[8 * h8 + 3]);
      b.z = pack2(gv[8 * h8 + 4], gv[8 * h8 + 5]);
      b.w = pack2(gv[8 * h8 + 6], gv[8 * h8 + 7]);
      const uint32_t off = hf * 16384 + sw_off(row, 2 * c + h8);
      if (Pd) *reinterpret_cast<uint4*>(Pd + off) = a;
      *reinterpret_cast<uint4*>(dS + off) = b;
    }
  }
}

// dK, dV of one 128-key tile: loop over the query tiles at or after it.
__global__ void __launch_bounds__(256, 1) attn_bwd_dkv_tc_kernel(AttnArgs A, const float* __restrict__ dO, int64_t ldo,
                                                                 const float* __restrict__ lse, const float* __restrict__ D,
                                                                 float* __restrict__ dqkv, int64_t ldg) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Ks = sm;
  uint8_t* Vs = sm + 16384;
  uint8_t* Qs = sm + 2 * 16384;
  uint8_t* Os = sm + 3 * 16384;  // dO (bf16)
  uint8_t* Ps = sm + 4 * 16384;  // Pd [128 q][128 k]
  uint8_t* Gs = sm + 6 * 16384;  // dS [128 q][128 k]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 8 * 16384);  // [0] S, dP done; [1] dV, dK done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int kt = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int hf = w >> 2, row = (w & 3) * 32 + lane;
  const int nq = A.seq / TCQ;
  const int64_t base = (int64_t)s * A.seq;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (w == 0) tmem_alloc(tslot, 512);
  load_sw_tile(A.qkv + (base + kt * TCQ) * A.ldq + A.d + h * HD, A.ldq, Ks);
  load_sw_tile(A.qkv + (base + kt * TCQ) * A.ldq + 2 * A.d + h * HD, A.ldq, Vs);
  cp_async_commit();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
  const uint32_t tS = tmem + lane_off, tdP = tmem + 128 + lane_off;
  constexpr uint32_t idSS = make_idesc_bf16(128, 128, false, false);  // S, dP: K-major Q / dO and K / V
  constexpr uint32_t idT = make_idesc_bf16(128, 64, true, true);      // dV, dK: MN-major Pd^T / dS^T and dO / Q
  const uint32_t pstep = A.thresh ? *A.step : 0u;
  for (int qt = kt; qt < nq; ++qt) {
    const int it = qt - kt;
    if (it > 0) mbar_wait(&bar[1], (uint32_t)((it - 1) & 1));  // the previous dV / dK MMAs read Q, dO, Pd, dS
    load_sw_tile(A.qkv + (base + qt * TCQ) * A.ldq + h * HD, A.ldq, Qs);
    cp_async_commit();
    load_sw_tile_f32(dO + (base + qt * TCQ) * ldo + h * HD, ldo, Os);
    const int q = qt * TCQ + row;
    const float lse_q = lse[(base + q) * A.nh + h], D_q = D[(base + q) * A.nh + h];
    cp_async_wait<0>();
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        tc_mma_bf16(tmem, make_sdesc_sw128(smem_u32(Qs) + kk * 32, 16, 1024), make_sdesc_sw128(smem_u32(Ks) + kk * 32, 16, 1024),
                    idSS, kk > 0);
        tc_mma_bf16(tmem + 128, make_sdesc_sw128(smem_u32(Os) + kk * 32, 16, 1024),
                    make_sdesc_sw128(smem_u32(Vs) + kk * 32, 16, 1024), idSS, kk > 0);
      }
      tc_commit(&bar[0]);
    }
    mbar_wait(&bar[0], (uint32_t)(it & 1));
    tc_fence_after();
    const uint64_t rowbase = (((uint64_t)(A.seq0 + s) * A.nh + h) * A.seq + q) * A.seq;
    attn_bwd_tc_probs(A, tS, tdP, row, hf, q, kt, lse_q, D_q, rowbase, pstep, Ps, Gs);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // K = the 128 queries, 16 per MMA
        tc_mma_bf16(tmem + 256, make_sdesc_sw128(smem_u32(Ps) + kk * 2048, 16384, 1024),
                    make_sdesc_sw128(smem_u32(Os) + kk * 2048, 8192, 1024), idT, (it | kk) ? 1u : 0u);
        tc_mma_bf16(tmem + 320, make_sdesc_sw128(smem_u32(Gs) + kk * 2048, 16384, 1024),
                    make_sdesc_sw128(smem_u32(Qs) + kk * 2048, 8192, 1024), idT, (it | kk) ? 1u : 0u);
      }
      tc_commit(&bar[1]);
    }
  }
  mbar_wait(&bar[1], (uint32_t)((nq - 1 - kt) & 1));
  tc_fence_after();
  // TMEM lane = key row of the tile; this thread writes 32 of the 64 head columns of dK and dV
  float dv[32], dk[32];
  tmem_ld16(tmem + 256 + lane_off + hf * 32, dv);
  tmem_ld16(tmem + 256 + lane_off + hf * 32 + 16, dv + 16);
  tmem_ld16(tmem + 320 + lane_off + hf * 32, dk);
  tmem_ld16(tmem + 320 + lane_off + hf * 32 + 16, dk + 16);
  const int64_t grow = base + kt * TCQ + row;
  float* kdst = dqkv + grow * ldg + A.d + h * HD + hf * 32;
  float* vdst = dqkv + grow * ldg + 2 * A.d + h * HD + hf * 32;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    *reinterpret_cast<float4*>(kdst + 4 * c) =
        make_float4(dk[4 * c] * A.scale, dk[4 * c + 1] * A.scale, dk[4 * c + 2] * A.scale, dk[4 * c + 3] * A.scale);
    *reinterpret_cast<float4*>(vdst + 4 * c) = make_float4(dv[4 * c], dv[4 * c + 1], dv[4 * c + 2], dv[4 * c + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 512);
}

// dQ of one 128-query tile: loop over the key tiles at or before it.
__global__ void __launch_bounds__(256, 1) attn_bwd_dq_tc_kernel(AttnArgs A, const float* __restrict__ dO, int64_t ldo,
                                                                const float* __restrict__ lse, const float* __restrict__ D,
                                                                float* __restrict__ dqkv, int64_t ldg) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* Qs = sm;
  uint8_t* Os = sm + 16384;
  uint8_t* Ks = sm + 2 * 16384;
  uint8_t* Vs = sm + 3 * 16384;
  uint8_t* Gs = sm + 4 * 16384;  // dS [128 q][128 k]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6 * 16384);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  const int qt = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, s = blockIdx.z;  // heaviest first
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int hf = w >> 2, row = (w & 3) * 32 + lane;
  const int64_t base = (int64_t)s * A.seq;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  if (w == 0) tmem_alloc(tslot, 512);
  load_sw_tile(A.qkv + (base + qt * TCQ) * A.ldq + h * HD, A.ldq, Qs);
  cp_async_commit();
  load_sw_tile_f32(dO + (base + qt * TCQ) * ldo + h * HD, ldo, Os);
  const int q = qt * TCQ + row;
  const float lse_q = lse[(base + q) * A.nh + h], D_q = D[(base + q) * A.nh + h];
  const uint64_t rowbase = (((uint64_t)(A.seq0 + s) * A.nh + h) * A.seq + q) * A.seq;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
  const uint32_t tS = tmem + lane_off, tdP = tmem + 128 + lane_off;
  constexpr uint32_t idSS = make_idesc_bf16(128, 128, false, false);
  constexpr uint32_t idQ = make_idesc_bf16(128, 64, false, true);  // dQ: K-major dS, MN-major K
  const uint32_t pstep = A.thresh ? *A.step : 0u;
  for (int kt = 0; kt <= qt; ++kt) {
    if (kt > 0) mbar_wait(&bar[1], (uint32_t)((kt - 1) & 1));  // the previous dQ MMAs read K and dS
    load_sw_tile(A.qkv + (base + kt * TCQ) * A.ldq + A.d + h * HD, A.ldq, Ks);
    load_sw_tile(A.qkv + (base + kt * TCQ) * A.ldq + 2 * A.d + h * HD, A.ldq, Vs);
    cp_async_commit();
    cp_async_wait<0>();
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        tc_mma_bf16(tmem, make_sdesc_sw128(smem_u32(Qs) + kk * 32, 16, 1024), make_sdesc_sw128(smem_u32(Ks) + kk * 32, 16, 1024),
                    idSS, kk > 0);
        tc_mma_bf16(tmem + 128, make_sdesc_sw128(smem_u32(Os) + kk * 32, 16, 1024),
                    make_sdesc_sw128(smem_u32(Vs) + kk * 32, 16, 1024), idSS, kk > 0);
      }
      tc_commit(&bar[0]);
    }
    mbar_wait(&bar[0], (uint32_t)(kt & 1));
    tc_fence_after();
    attn_bwd_tc_probs(A, tS, tdP, row, hf, q, kt, lse_q, D_q, rowbase, pstep, nullptr, Gs);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)  // K = the 128 keys, 16 per MMA
        tc_mma_bf16(tmem + 256, make_sdesc_sw128(smem_u32(Gs) + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                    make_sdesc_sw128(smem_u32(Ks) + kk * 2048, 8192, 1024), idQ, (kt | kk) ? 1u : 0u);
      tc_commit(&bar[1]);
    }
  }
  mbar_wait(&bar[1], (uint32_t)(qt & 1));
  tc_fence_after();
  float dq[32];
  tmem_ld16(tmem + 256 + lane_off + hf * 32, dq);
  tmem_ld16(tmem + 256 + lane_off + hf * 32 + 16, dq + 16);
  float* qdst = dqkv + (base + q) * ldg + h * HD + hf * 32;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(qdst + 4 * c) =
        make_float4(dq[4 * c] * A.scale, dq[4 * c + 1] * A.scale, dq[4 * c + 2] * A.scale, dq[4 * c + 3] * A.scale);
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tmem, 512);
}

// D[row][h] = sum_c dO[row][h*64 + c] * O[row][h*64 + c]  (= rowsum(P o dP), the softmax VJP term)
__global__ void attn_bwd_prep_kernel(const float* __restrict__ dO, const __nv_bfloat16* __restrict__ O, int64_t ld,
                                     int rows, int nh, float* __restrict__ D) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= rows * nh) return;
  const int r = wid / nh, h = wid % nh;
  const float2 a = *reinterpret_cast<const float2*>(dO + (int64_t)r * ld + h * HD + 2 * lane);
  const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(O + (int64_t)r * ld + h * HD + 2 * lane);
  float v = a.x * __low2float(b) + a.y * __high2float(b);
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) D[wid] = v;
}

// dK, dV of one key tile: loop over the query tiles at or after it.
__global__ void __launch_bounds__(128, TGP_ATTN_MINB) attn_bwd_dkv_kernel(AttnArgs A, const float* __restrict__ dO, int64_t ldo,
                                                           const float* __restrict__ lse, const float* __restrict__ D,
                                                           float* __restrict__ dqkv, int64_t ldg) {
  __shared__ __align__(16) __nv_bfloat16 Qs[TILE * PITCH], Os[TILE * PITCH];
  __shared__ float ls[TILE], Ds[TILE];
  const int kt = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int w = threadIdx.x >> 5, g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
  const int64_t base = (int64_t)s * A.seq;
  const int nq = A.seq / TILE;
  load_tile(A.qkv + (base + kt * TILE) * A.ldq + A.d + h * HD, A.ldq, Qs, nullptr);
  load_tile(A.qkv + (base + kt * TILE) * A.ldq + 2 * A.d + h * HD, A.ldq, Os, nullptr);
  __syncthreads();
  uint32_t ka[4][4], va[4][4];
  load_afrag(Qs, w * 16, ka);
  load_afrag(Os, w * 16, va);
  float dk[8][4] = {}, dv[8][4] = {};
  const int k0 = kt * TILE + w * 16 + g;
  for (int qt = kt; qt < nq; ++qt) {
    __syncthreads();
    load_tile(A.qkv + (base + qt * TILE) * A.ldq + h * HD, A.ldq, Qs, nullptr);
    load_tile_f32(dO + (base + qt * TILE) * ldo + h * HD, ldo, Os, nullptr);
    if (threadIdx.x < TILE) {
      ls[threadIdx.x] = lse[(base + qt * TILE + threadIdx.x) * A.nh + h];
      Ds[threadIdx.x] = D[(base + qt * TILE + threadIdx.x) * A.nh + h];
    }
    __syncthreads();
    float p[8][4] = {}, dp[8][4] = {};
    mma_row_tile(p, ka, Qs);   // S^T[key][q]
    mma_row_tile(dp, va, Os);  // dP^T[key][q] = V dO^T
    float pd[8][4];
    const uint32_t kb = A.thresh ? attn_keep_tile_t(A, s, h, kt * TILE + w * 16, qt * TILE) : 0xFFFFFFFFu;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int ql = nt * 8 + 2 * t + (c & 1), q = qt * TILE + ql, key = k0 + (c >> 1) * 8;
        const float pr = key <= q ? exp2f(p[nt][c] * A.scale_log2 - ls[ql]) : 0.0f;
        float dpv = dp[nt][c];
        float pdv = pr;
        if (A.thresh) {
          const bool keep = (kb >> (nt * 4 + c)) & 1u;
          pdv = keep ? pr * A.dscale : 0.0f;
          dpv = keep ? dpv * A.dscale : 0.0f;
        }
        pd[nt][c] = pdv;
        p[nt][c] = pr * (dpv - Ds[ql]);  // dS^T
      }
    mma_p_tile(dv, pd, Os);  // dV += Pd^T dO
    mma_p_tile(dk, p, Qs);   // dK += dS^T Q
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t row = base + k0 + r * 8;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      const int col = h * HD + dt * 8 + 2 * t;
      *reinterpret_cast<float2*>(dqkv + row * ldg + A.d + col) =
          make_float2(dk[dt][2 * r] * A.scale, dk[dt][2 * r + 1] * A.scale);
      *reinterpret_cast<float2*>(dqkv + row * ldg + 2 * A.d + col) = make_float2(dv[dt][2 * r], dv[dt][2 * r + 1]);
    }
  }
}

// dQ of one query tile: loop over the key tiles at or before it.
__global__ void __launch_bounds__(128, TGP_ATTN_MINB) attn_bwd_dq_kernel(AttnArgs A, const float* __restrict__ dO, int64_t ldo,
                                                          const float* __restrict__ lse, const float* __restrict__ D,
                                                          float* __restrict__ dqkv, int64_t ldg) {
  __shared__ __align__(16) __nv_bfloat16 Ks[TILE * PITCH], Vs[TILE * PITCH];
  const int qt = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int w = threadIdx.x >> 5, g = (threadIdx.x & 31) >> 2, t = threadIdx.x & 3;
  const int64_t base = (int64_t)s * A.seq;
  load_tile(A.qkv + (base + qt * TILE) * A.ldq + h * HD, A.ldq, Ks, nullptr);
  load_tile_f32(dO + (base + qt * TILE) * ldo + h * HD, ldo, Vs, nullptr);
  __syncthreads();
  uint32_t qa[4][4], oa[4][4];
  load_afrag(Ks, w * 16, qa);
  load_afrag(Vs, w * 16, oa);
  const int q0 = qt * TILE + w * 16 + g;
  float ls[2], Dr[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    ls[r] = lse[(base + q0 + r * 8) * A.nh + h];
    Dr[r] = D[(base + q0 + r * 8) * A.nh + h];
  }
  float dq[8][4] = {};
  for (int kt = 0; kt <= qt; ++kt) {
    __syncthreads();
    load_tile(A.qkv + (base + kt * TILE) * A.ldq + A.d + h * HD, A.ldq, Ks, nullptr);
    load_tile(A.qkv + (base + kt * TILE) * A.ldq + 2 * A.d + h * HD, A.ldq, Vs, nullptr);
    __syncthreads();
    float p[8][4] = {}, dp[8][4] = {};
    mma_row_tile(p, qa, Ks);   // S
    mma_row_tile(dp, oa, Vs);  // dP = dO V^T
    const uint32_t kb = A.thresh ? attn_keep_tile(A, s, h, q0, kt * TILE) : 0xFFFFFFFFu;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int key = kt * TILE + nt * 8 + 2 * t + (c & 1), q = q0 + (c >> 1) * 8;
        const float pr = key <= q ? exp2f(p[nt][c] * A.scale_log2 - ls[c >> 1]) : 0.0f;
        float dpv = dp[nt][c];
        if (A.thresh) dpv = ((kb >> (nt * 4 + c)) & 1u) ? dpv * A.dscale : 0.0f;
        p[nt][c] = pr * (dpv - Dr[c >> 1]);  // dS
      }
    mma_p_tile(dq, p, Ks);  // dQ += dS K
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int64_t row = base + q0 + r * 8;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt)
      *reinterpret_cast<float2*>(dqkv + row * ldg + h * HD + dt * 8 + 2 * t) =
          make_float2(dq[dt][2 * r] * A.scale, dq[dt][2 * r + 1] * A.scale);
  }
}

AttnArgs make_args(const void* qkv, int rows, int d, int nh, int seq, int64_t row_global0, uint32_t thresh,
                   float dscale, uint64_t seed, const uint32_t* step, uint32_t site) {
  AttnArgs A;
  A.qkv = (const __nv_bfloat16*)qkv;
  A.ldq = 3 * (int64_t)d;
  A.d = d;
  A.nh = nh;
  A.seq = seq;
  A.seq0 = row_global0 / seq;
  A.scale = 0.125f;
  A.scale_log2 = 0.125f * LOG2E;
  A.thresh = thresh;
  A.dscale = dscale;
  A.seed = seed;
  A.step = step;
  A.site = site;
  (void)rows;
  return A;
}


// ------------------------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const float* __restrict__ ids, int64_t ldi, const float* __restrict__ wte,
                                 const float* __restrict__ wpe, int d, int seq, int64_t row_global0, uint32_t thresh,
                                 float dscale, uint64_t seed, const uint32_t* step, uint32_t site, float* __restrict__ y) {
  const int r = blockIdx.x;
  const int64_t id = (int64_t)__float2int_rn(ids[(int64_t)r * ldi]);
  const int64_t pos = (row_global0 + r) % seq;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float v = wte[id * d + c] + wpe[pos * d + c];
    if (thresh) v = dropout_keep(seed, *step, site, (uint64_t)(row_global0 + r) * d + c, thresh) ? v * dscale : 0.0f;
    y[(int64_t)r * d + c] = v;
  }
}

// deterministic dW_te: counting sort of the token rows by id, each vocabulary row sums its rows in
// ascending order (no floating-point atomics)
__global__ void embed_count_kernel(const float* __restrict__ ids, int64_t ldi, int rows, int* cnt) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    atomicAdd(cnt + __float2int_rn(ids[(int64_t)r * ldi]), 1);
}
__global__ void embed_scan_kernel(const int* __restrict__ cnt, int V, int* start, int* cursor) {
  __shared__ int tot[1024];
  const int per = (V + blockDim.x - 1) / blockDim.x;
  const int a = threadIdx.x * per, b = min(V, a + per);
  int s = 0;
  for (int v = a; v < b; ++v) s += cnt[v];
  tot[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < (int)blockDim.x; ++i) {
      const int x = tot[i];
      tot[i] = run;
      run += x;
    }
  }
  __syncthreads();
  int run = tot[threadIdx.x];
  for (int v = a; v < b; ++v) {
    start[v] = run;
    cursor[v] = run;
    run += cnt[v];
  }
}
__global__ void embed_fill_kernel(const float* __restrict__ ids, int64_t ldi, int rows, int* cursor, int* list) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x)
    list[atomicAdd(cursor + __float2int_rn(ids[(int64_t)r * ldi]), 1)] = r;
}
// one CTA per vocabulary row: sort its bucket (ascending row), sum the rows
__global__ void embed_wte_kernel(const int* __restrict__ cnt, const int* __restrict__ start, int* list,
                                 const float* __restrict__ dE, int d, float* __restrict__ dwte, int accumulate) {
  const int v = blockIdx.x, n = cnt[v];
  int* L = list + start[v];
  if (threadIdx.x == 0)
    for (int i = 1; i < n; ++i) {  // insertion sort (buckets hold ~B/V rows)
      const int x = L[i];
      int j = i - 1;
      while (j >= 0 && L[j] > x) {
        L[j + 1] = L[j];
        --j;
      }
      L[j + 1] = x;
    }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = accumulate ? dwte[(int64_t)v * d + c] : 0.0f;
    for (int i = 0; i < n; ++i) s += dE[(int64_t)L[i] * d + c];
    dwte[(int64_t)v * d + c] = s;
  }
}
__global__ void embed_wpe_kernel(const float* __restrict__ dE, int rows, int d, int seq, float* __restrict__ dwpe,
                                 int accumulate) {
  const int p = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float s = accumulate ? dwpe[(int64_t)p * d + c] : 0.0f;
    for (int r = p; r < rows; r += seq) s += dE[(int64_t)r * d + c];
    dwpe[(int64_t)p * d + c] = s;
  }
}

// ------------------------------------------------------------------------------- cross-entropy
__global__ void ce_row_kernel(const float* __restrict__ y, int64_t ldy, const int* __restrict__ tgt, int V, int T,
                              float* __restrict__ dy, double* __restrict__ part) {
  // one pass for the row maximum and the rescaled exponential sum (online softmax, per thread then a
  // fixed-order combination), one pass writing dy: 2 reads of the logits instead of 3
  __shared__ float shm[32], shs[32];
  __shared__ float bm, bs;
  const int r = blockIdx.x;
  const float* yr = y + (int64_t)r * ldy;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float m = -INFINITY, se = 0.0f;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float v = yr[c];
    if (v > m) {
      se = se * __expf(m - v) + 1.0f;
      m = v;
    } else {
      se += __expf(v - m);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, se, o);
    const float mn = fmaxf(m, m2);
    se = (m == -INFINITY ? 0.0f : se * __expf(m - mn)) + (m2 == -INFINITY ? 0.0f : s2 * __expf(m2 - mn));
    m = mn;
  }
  if (lane == 0) {
    shm[w] = m;
    shs[w] = se;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = shm[0];
    for (int i = 1; i < nw; ++i) mm = fmaxf(mm, shm[i]);
    float ss = 0.0f;
    for (int i = 0; i < nw; ++i) ss += shm[i] == -INFINITY ? 0.0f : shs[i] * __expf(shm[i] - mm);  // fixed order
    bm = mm;
    bs = ss;
  }
  __syncthreads();
  const float mx = bm, sum = bs;
  const int tg = tgt[r];
  const float inv = 1.0f / sum, invT = 1.0f / (float)T;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float p = __expf(yr[c] - mx) * inv;
    dy[(int64_t)r * ldy + c] = (p - (c == tg ? 1.0f : 0.0f)) * invT;
  }
  if (threadIdx.x == 0) part[r] = (double)mx + log((double)sum) - (double)yr[tg];
}
__global__ void ce_final_kernel(const double* part, int T, double* loss) {
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < T; ++i) s += part[i];
    loss[0] = s / (double)T;
  }
}

template <typename Kern, typename... Args>
int launch(const char* name, Kern k, dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  k<<<grid, block, 0, st>>>(args...);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch: %s", name, cudaGetErrorString(e));
    return -3;
  }
  return 0;
}

}  // namespace

static int g_attn_tc = -1;  // -1: environment (TGP_ATTN_TC), else option "attn_tc"
void attn_set_tc(int on) { g_attn_tc = on; }
// tcgen05 attention (forward and backward, seq % 128 == 0) is the default; TGP_ATTN_TC=0 or option
// attn_tc = 0 selects the mma.sync kernels (kept for comparison and for seq % 128 != 0)
static bool attn_tc_on() {
  static const bool tc_env = [] {
    const char* e = getenv("TGP_ATTN_TC");
    return !(e && e[0] == '0');
  }();
  return g_attn_tc < 0 ? tc_env : g_attn_tc != 0;
}

bool attn_shape_ok(int rows, int d, int nh, int seq) {
  return nh > 0 && d == nh * HD && seq % TILE == 0 && seq > 0 && rows % seq == 0;
}

int attn_fwd(cudaStream_t st, const void* qkv, int rows, int d, int nh, int seq, int64_t row_global0,
             uint32_t thresh, float dscale, uint64_t seed, const uint32_t* step, uint32_t site, void* ctx,
             float* lse, float* part_buf) {
  if (!attn_shape_ok(rows, d, nh, seq)) {
    set_error("attention: need d = 64 * n_heads, seq %% 64 == 0, rows %% seq == 0 (d=%d nh=%d seq=%d rows=%d)", d,
              nh, seq, rows);
    return TGP_E_UNSUPPORTED;
  }
  AttnArgs A = make_args(qkv, rows, d, nh, seq, row_global0, thresh, dscale, seed, step, site);
  if (attn_tc_on() && seq % TCQ == 0) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
      if (e != cudaSuccess) {
        set_error("attn_fwd_tc smem attribute: %s", cudaGetErrorString(e));
        return TGP_E_CUDA;
      }
      attr = true;
    }
    attn_fwd_tc_kernel<<<dim3(seq / TCQ, nh, rows / seq), 256, TC_SMEM, st>>>(A, (__nv_bfloat16*)ctx, (int64_t)d, lse);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("attn_fwd_tc launch: %s", cudaGetErrorString(e));
      return TGP_E_CUDA;
    }
    return 0;
  }
  const int nq = seq / TILE;
  int ks = 8;
  while ((nq + ks - 1) / ks > FWD_MAX_PARTS) ks *= 2;
  if (!part_buf) ks = nq;  // no scratch: one item per query tile
  FwdItems items{};
  int n = 0;
  // heaviest first: items of ks key tiles, then the shorter remainders, in descending length
  for (int len = ks; len >= 1; --len)
    for (int qt = nq - 1; qt >= 0; --qt) {
      const int np = qt / ks + 1;
      for (int p = 0; p < np; ++p) {
        const int a = p * ks, b = std::min(qt, a + ks - 1);
        if (b - a + 1 != len) continue;
        if (n >= FWD_MAX_ITEMS) {
          set_error("attention: seq %d needs more than %d forward work items", seq, FWD_MAX_ITEMS);
          return TGP_E_UNSUPPORTED;
        }
        items.it[n++] = (uint32_t)qt | ((uint32_t)a << 8) | ((uint32_t)b << 16) | ((uint32_t)p << 24) |
                        (np > 1 ? 0x80000000u : 0u);
      }
    }
  TGP_TRY(launch("attn_fwd", attn_fwd_kernel, dim3(n, nh, rows / seq), dim3(128), st, A, (__nv_bfloat16*)ctx,
                 (int64_t)d, lse, items, part_buf));
  if (ks >= nq) return 0;
  const int q_first = ks * TILE, nrows = (rows / seq) * (seq - q_first);
  return launch("attn_fwd_merge", attn_fwd_merge_kernel, dim3((nrows * nh + 3) / 4), dim3(128), st,
                (const float*)part_buf, seq, nh, q_first, FWD_MAX_PARTS, ks, nrows, (__nv_bfloat16*)ctx, (int64_t)d, lse);
}

int attn_bwd(cudaStream_t st, const void* qkv, const void* ctx, const float* dO, const float* lse, float* Dbuf,
             int rows, int d, int nh, int seq, int64_t row_global0, uint32_t thresh, float dscale, uint64_t seed,
             const uint32_t* step, uint32_t site, float* dqkv) {
  if (!attn_shape_ok(rows, d, nh, seq)) {
    set_error("attention backward: unsupported shape");
    return TGP_E_UNSUPPORTED;
  }
  AttnArgs A = make_args(qkv, rows, d, nh, seq, row_global0, thresh, dscale, seed, step, site);
  const int warps = rows * nh;
  TGP_TRY(launch("attn_bwd_prep", attn_bwd_prep_kernel, dim3((warps + 3) / 4), dim3(128), st, dO,
                 (const __nv_bfloat16*)ctx, (int64_t)d, rows, nh, Dbuf));
  if (attn_tc_on() && seq % TCQ == 0) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(attn_bwd_dkv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BTC_SMEM_KV);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(attn_bwd_dq_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BTC_SMEM_Q);
      if (e != cudaSuccess) {
        set_error("attn_bwd_tc smem attribute: %s", cudaGetErrorString(e));
        return TGP_E_CUDA;
      }
      attr = true;
    }
    attn_bwd_dkv_tc_kernel<<<dim3(seq / TCQ, nh, rows / seq), 256, BTC_SMEM_KV, st>>>(A, dO, (int64_t)d, lse,
                                                                                   (const float*)Dbuf, dqkv, 3 * (int64_t)d);
    attn_bwd_dq_tc_kernel<<<dim3(seq / TCQ, nh, rows / seq), 256, BTC_SMEM_Q, st>>>(A, dO, (int64_t)d, lse,
                                                                                 (const float*)Dbuf, dqkv, 3 * (int64_t)d);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("attn_bwd_tc launch: %s", cudaGetErrorString(e));
      return TGP_E_CUDA;
    }
    return 0;
  }
  TGP_TRY(launch("attn_bwd_dkv", attn_bwd_dkv_kernel, dim3(seq / TILE, nh, rows / seq), dim3(128), st, A, dO,
                 (int64_t)d, lse, (const float*)Dbuf, dqkv, 3 * (int64_t)d));
  return launch("attn_bwd_dq", attn_bwd_dq_kernel, dim3(seq / TILE, nh, rows / seq), dim3(128), st, A, dO, (int64_t)d,
                lse, (const float*)Dbuf, dqkv, 3 * (int64_t)d);
}

int embed_fwd(cudaStream_t st, const float* ids, int64_t ldi, int rows, const float* wte, const float* wpe, int d,
              int seq, int64_t row_global0, uint32_t thresh, float dscale, uint64_t seed, const uint32_t* step,
              uint32_t site, float* y) {
  return launch("embed_fwd", embed_fwd_kernel, dim3(rows), dim3(256), st, ids, ldi, wte, wpe, d, seq, row_global0,
                thresh, dscale, seed, step, site, y);
}

int embed_wgrad(cudaStream_t st, const float* ids, int64_t ldi, int rows, const float* dE, int d, int V, int seq,
                int* scratch, float* dwte, float* dwpe, bool accumulate) {
  int* cnt = scratch;
  int* start = cnt + V;
  int* cursor = start + V;
  int* list = cursor + V;
  TGP_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * (size_t)V, st));
  TGP_TRY(launch("embed_count", embed_count_kernel, dim3(std::min(1024, (rows + 255) / 256)), dim3(256), st, ids,
                 ldi, rows, cnt));
  TGP_TRY(launch("embed_scan", embed_scan_kernel, dim3(1), dim3(1024), st, (const int*)cnt, V, start, cursor));
  TGP_TRY(launch("embed_fill", embed_fill_kernel, dim3(std::min(1024, (rows + 255) / 256)), dim3(256), st, ids, ldi,
                 rows, cursor, list));
  TGP_TRY(launch("embed_wte", embed_wte_kernel, dim3(V), dim3(128), st, (const int*)cnt, (const int*)start, list, dE,
                 d, dwte, (int)accumulate));
  return launch("embed_wpe", embed_wpe_kernel, dim3(seq), dim3(128), st, dE, rows, d, seq, dwpe, (int)accumulate);
}

int ce_loss_grad(cudaStream_t st, const float* y, int64_t ldy, const int* tgt, int T, int V, float* dy,
                 double* part, double* loss_dev) {
  TGP_TRY(launch("ce_row", ce_row_kernel, dim3(T), dim3(256), st, y, ldy, tgt, V, T, dy, part));
  return launch("ce_final", ce_final_kernel, dim3(1), dim3(32), st, (const double*)part, T, loss_dev);
}

}  // namespace tgp
