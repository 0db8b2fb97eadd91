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

// Applies the epilogue to one accumulator value; returns the value contributed to the column sum
// (EPI_ACT_BWD), else 0.
TGP_DEV float epi_apply(const EpiParams& e, int f, int r, float v) {
  switch (e.mode) {
    case EPI_LINEAR_FWD: {
      float z = v + (e.bias ? e.bias[f] : 0.0f);
      if (e.zbuf) e.zbuf[(int64_t)r * e.ldz + f] = z;
      float y = act_f(e.act, z);
      if (e.drop_thresh) {
        uint64_t idx = (uint64_t)(e.row_global0 + r) * (uint64_t)e.drop_width + (uint64_t)f;
        y = dropout_keep(e.seed, *e.step, e.site, idx, e.drop_thresh) ? y * e.drop_scale : 0.0f;
      }
      if (e.out0) e.out0[(int64_t)r * e.ld0 + f] = y;
      if (e.op) store_op(e, r, f, y);
      return 0.0f;
    }
    case EPI_RESID_FWD: {
      float y = v + (e.bias ? e.bias[f] : 0.0f) + e.res[(int64_t)r * e.ld_res + f];
      e.out0[(int64_t)r * e.ld0 + f] = y;
      if (e.op) store_op(e, r, f, y);
      return 0.0f;
    }
    case EPI_ACT_BWD: {
      float d = v;
      if (e.drop_thresh) {
        uint64_t idx = (uint64_t)(e.row_global0 + r) * (uint64_t)e.drop_width + (uint64_t)f;
        d = dropout_keep(e.seed, *e.step, e.site, idx, e.drop_thresh) ? d * e.drop_scale : 0.0f;
      }
      if (e.act) d *= act_df(e.act, e.zbuf[(int64_t)r * e.ldz + f]);
      if (e.op) store_op(e, r, f, d);
      if (e.out0) e.out0[(int64_t)r * e.ld0 + f] = d;
      return d;
    }
    case EPI_STORE: {
      if (f < e.split_f)
        e.out0[(int64_t)r * e.ld0 + f] = v;
      else
        e.out1[(int64_t)r * e.ld1 + (f - e.split_f)] = v;
      return 0.0f;
    }
    default:
      return 0.0f;
  }
}

}  // namespace tgp
