// Element-wise GEMM epilogues shared by the tcgen05 GEMM and the fp32 SIMT GEMM (both product
// kernels).  Row r is the micro-batch-local row, f the output feature; all row-indexed pointers in
// EpiParams are pre-offset to the micro-batch's first row.
#pragma once
#include "common.cuh"
#include "gemm_tc.cuh"

namespace tgp {

TGP_DEV void store_op(const EpiParams& e, int r, int f, float v) {
  if (e.op_bf16)
    reinterpret_cast<__nv_bfloat16*>(e.op)[(int64_t)r * e.ld_op + f] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(e.op)[(int64_t)r * e.ld_op + f] = v;
}

// The epilogue in two halves, specialised on the mode at compile time (the tcgen05 GEMM is
// instantiated per mode, which keeps its tail a few dozen straight-line instructions: the generic
// switch cost ~1 us per CTA in instruction-fetch stalls, profiles/gemm_timeline.py).  epi_load gathers
// everything an output element needs besides its accumulator (bias, residual, saved pre-activation,
// dropout decision) -- the GEMM issues it during its mainloop, off the kernel's serial tail;
// epi_finish does the arithmetic and the stores.  epi_apply = both back to back (bit-identical).
struct EpiPre {
  float a = 0.0f, b = 0.0f;
  bool keep = true;
};

// WITH_KEEP = false: the caller supplies EpiPre::keep itself (gemm_wide draws the dropout bits of
// 4 features x 4 rows per Philox call and shares them across lanes)
template <int MODE, bool WITH_KEEP = true>
TGP_DEV EpiPre epi_load(const EpiParams& e, int f, int r) {
  EpiPre q;
  if constexpr (MODE == EPI_LINEAR_FWD) {
    q.a = e.bias ? e.bias[f] : 0.0f;
  } else if constexpr (MODE == EPI_RESID_FWD) {
    q.a = e.bias ? e.bias[f] : 0.0f;
    q.b = e.res[(int64_t)r * e.ld_res + f];
  } else if constexpr (MODE == EPI_ACT_BWD) {
    if (e.act) q.a = e.zbuf[(int64_t)r * e.ldz + f];
  }
  if constexpr (WITH_KEEP && (MODE == EPI_LINEAR_FWD || MODE == EPI_ACT_BWD || MODE == EPI_RESID_FWD)) {
    if (e.drop_thresh) {
      const uint64_t idx = (uint64_t)(e.row_global0 + r) * (uint64_t)e.drop_width + (uint64_t)f;
      q.keep = dropout_keep(e.seed, *e.step, e.site, idx, e.drop_thresh);
    }
  }
  return q;
}

// Finishes one accumulator value; returns the value contributed to the column sum (EPI_ACT_BWD),
// else 0.
template <int MODE>
TGP_DEV float epi_finish(const EpiParams& e, int f, int r, float v, const EpiPre& q) {
  if constexpr (MODE == EPI_LINEAR_FWD) {
    const float z = v + q.a;
    if (e.zbuf) e.zbuf[(int64_t)r * e.ldz + f] = z;
    float y = act_f(e.act, z);
    if (e.drop_thresh) y = q.keep ? y * e.drop_scale : 0.0f;
    if (e.out0) e.out0[(int64_t)r * e.ld0 + f] = y;
    if (e.op) store_op(e, r, f, y);
    return 0.0f;
  } else if constexpr (MODE == EPI_RESID_FWD) {
    float br = v + q.a;  // residual branch (dropout on the branch: GPT-2 blocks)
    if (e.drop_thresh) br = q.keep ? br * e.drop_scale : 0.0f;
    const float y = br + q.b;
    e.out0[(int64_t)r * e.ld0 + f] = y;
    if (e.op) store_op(e, r, f, y);
    return 0.0f;
  } else if constexpr (MODE == EPI_ACT_BWD) {
    float d = v;
    if (e.drop_thresh) d = q.keep ? d * e.drop_scale : 0.0f;
    if (e.act) d *= act_df(e.act, q.a);
    if (e.op) store_op(e, r, f, d);
    if (e.out0) e.out0[(int64_t)r * e.ld0 + f] = d;
    return d;
  } else if constexpr (MODE == EPI_STORE) {
    if (f < e.split_f)
      e.out0[(int64_t)r * e.ld0 + f] = v;
    else
      e.out1[(int64_t)r * e.ld1 + (f - e.split_f)] = v;
    return 0.0f;
  } else {
    return 0.0f;
  }
}

// epi_finish for rows r0 .. r0 + n - 1 (n <= NR) of one feature: the same arithmetic per element,
// with the flag tests and the row addressing done once per call (the GEMM tails are issue-bound:
// ~120 instructions per element through epi_finish in the skinny split-K tail, profiles/r6/)
template <int MODE, int NR>
TGP_DEV float epi_finish_rows(const EpiParams& e, int f, int r0, int n, const float* v, const EpiPre* q,
                              float part = 0.0f) {
  // part: running column sum (EPI_ACT_BWD) the rows are added to, in row order
  const bool drop = e.drop_thresh != 0;
  const float ds = e.drop_scale;
  auto put_op = [&](float (&y)[NR]) {
    if (!e.op) return;
    if (e.op_bf16) {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(e.op) + (int64_t)r0 * e.ld_op + f;
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < n) o[(int64_t)j * e.ld_op] = __float2bfloat16_rn(y[j]);
    } else {
      float* o = reinterpret_cast<float*>(e.op) + (int64_t)r0 * e.ld_op + f;
#pragma unroll
      for (int j = 0; j < NR; ++j)
        if (j < n) o[(int64_t)j * e.ld_op] = y[j];
    }
  };
  if constexpr (MODE == EPI_LINEAR_FWD) {
    float* zp = e.zbuf ? e.zbuf + (int64_t)r0 * e.ldz + f : nullptr;
    float* op0 = e.out0 ? e.out0 + (int64_t)r0 * e.ld0 + f : nullptr;
    const int act = e.act;
    float y[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const float z = v[j] + q[j].a;
      if (zp && j < n) zp[(int64_t)j * e.ldz] = z;
      float t = act_f(act, z);
      if (drop) t = q[j].keep ? t * ds : 0.0f;
      y[j] = t;
      if (op0 && j < n) op0[(int64_t)j * e.ld0] = t;
    }
    put_op(y);
  } else if constexpr (MODE == EPI_RESID_FWD) {
    float* op0 = e.out0 + (int64_t)r0 * e.ld0 + f;
    float y[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      float br = v[j] + q[j].a;  // residual branch (dropout on the branch: GPT-2 blocks)
      if (drop) br = q[j].keep ? br * ds : 0.0f;
      y[j] = br + q[j].b;
      if (j < n) op0[(int64_t)j * e.ld0] = y[j];
    }
    put_op(y);
  } else if constexpr (MODE == EPI_ACT_BWD) {
    float* op0 = e.out0 ? e.out0 + (int64_t)r0 * e.ld0 + f : nullptr;
    const int act = e.act;
    float y[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      float d = v[j];
      if (drop) d = q[j].keep ? d * ds : 0.0f;
      if (act) d *= act_df(act, q[j].a);
      y[j] = d;
      if (j < n) {
        if (op0) op0[(int64_t)j * e.ld0] = d;
        part += d;
      }
    }
    put_op(y);
  } else if constexpr (MODE == EPI_STORE) {
    float* o = f < e.split_f ? e.out0 + (int64_t)r0 * e.ld0 + f : e.out1 + (int64_t)r0 * e.ld1 + (f - e.split_f);
    const int64_t ld = f < e.split_f ? e.ld0 : e.ld1;
#pragma unroll
    for (int j = 0; j < NR; ++j)
      if (j < n) o[(int64_t)j * ld] = v[j];
  }
  return part;
}

template <int MODE>
TGP_DEV float epi_apply(const EpiParams& e, int f, int r, float v) {
  return epi_finish<MODE>(e, f, r, v, epi_load<MODE>(e, f, r));
}

// Runtime-mode dispatch (fp32 SIMT GEMM).
TGP_DEV float epi_apply(const EpiParams& e, int f, int r, float v) {
  switch (e.mode) {
    case EPI_LINEAR_FWD:
      return epi_apply<EPI_LINEAR_FWD>(e, f, r, v);
    case EPI_RESID_FWD:
      return epi_apply<EPI_RESID_FWD>(e, f, r, v);
    case EPI_ACT_BWD:
      return epi_apply<EPI_ACT_BWD>(e, f, r, v);
    case EPI_STORE:
      return epi_apply<EPI_STORE>(e, f, r, v);
    default:
      return 0.0f;
  }
}

}  // namespace tgp
