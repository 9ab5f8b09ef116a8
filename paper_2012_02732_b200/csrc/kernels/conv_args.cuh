// Arguments of the implicit-GEMM convolution kernels (conv.cu, conv1x1.cu),
// decoded from the op descriptor's params / ptrs (runtime/ops.h).
#pragma once

#include "common.cuh"

namespace sw {

struct ConvArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w;
  const float* __restrict__ bias;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, pre_relu, has_res;
  int64_t in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  int M, Kdim, split;
  Epi epi;
};

static inline ConvArgs conv_args(const sw_op_desc& op) {
  const int64_t* p = op.params;
  ConvArgs a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.w = reinterpret_cast<const float*>(op.ptrs[PT_W]);
  a.bias = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K];
  a.R = (int)p[SP_R]; a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.in_sn = p[SP_IN_SN]; a.in_sh = p[SP_IN_SH]; a.in_sw = p[SP_IN_SW]; a.in_sc = p[SP_IN_SC];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  a.M = a.N * a.P * a.Q;
  a.Kdim = a.R * a.S * a.C;
  a.split = p[SP_SPLIT_K] > 1 ? (int)p[SP_SPLIT_K] : 1;
  a.epi = Epi{a.bias, a.res, a.out, a.M, a.K, a.P, a.Q, a.act, a.has_res, 0,
              a.out_sn, a.out_sh, a.out_sw, a.out_sc, a.res_sn, a.res_sh, a.res_sw, a.res_sc};
  a.epi.vec = epi_vec_ok(op.ptrs[PT_OUT], a.out_sn, a.out_sh, a.out_sw, a.out_sc, op.ptrs[PT_BIAS],
                         a.has_res != 0, op.ptrs[PT_RES], a.res_sn, a.res_sh, a.res_sw, a.res_sc) ? 1 : 0;
  return a;
}

}  // namespace sw
