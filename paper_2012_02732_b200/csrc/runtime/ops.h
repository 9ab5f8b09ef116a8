// Op table layout shared by the engine runtime and the sm_100a kernels.
//
// Every task of the AoT schedule is one sw_op_desc: a kernel kind, a tile
// variant picked at prepare time, 32 int64 params and 8 device pointers.
// Tensors are described by a base pointer plus element strides (N, H, W, C),
// which is how zero-copy concat (producers writing channel slices of one
// buffer), broadcast (stride 0) and NCHW inputs are expressed without copies.
#pragma once

#include <cstdint>

#include "../../../include/streamweave_b200.h"

namespace sw {

enum KernelKind : int32_t {
  K_CONV = 1,        // dense conv / 1x1 conv / linear as implicit GEMM (fp32)
  K_DWCONV = 2,      // depthwise conv (groups == C, multiplier 1)
  K_POOL = 3,        // max / avg pool (k x k), optional fused residual add
  K_ELTWISE = 4,     // add / mul / affine / copy over up to 3 broadcastable operands
  K_GLOBAL_POOL = 5, // global average pool over H x W
  K_CONV_TC = 6,     // dense conv / GEMM on tcgen05 tensor cores (3xTF32)
  K_CONCAT = 7,      // unfused channel concat of up to 7 dense NHWC inputs
  K_SEPCONV = 8,     // fused depthwise k x k → pointwise 1x1
};
// K_CONCAT params: 0 N, 1 H, 2 W, 3 n_in, 4 C_total, 5 out channel stride,
// 6 out pixel stride, 8.. C_i; ptrs 0..6 inputs, 7 output.

enum Act : int32_t { ACT_NONE = 0, ACT_RELU = 1, ACT_RELU6 = 2, ACT_SILU = 3, ACT_SIGMOID = 4 };

enum EltOp : int32_t { EW_ADD = 0, EW_MUL = 1, EW_AFFINE = 2, EW_COPY = 3 };

// Spatial ops (K_CONV, K_DWCONV, K_POOL, K_CONV_TC): params index
enum SpatialParam : int {
  SP_N = 0, SP_H, SP_W, SP_C,          // input dims
  SP_P, SP_Q, SP_K,                    // output dims (K = out channels)
  SP_R, SP_S, SP_STRIDE_H, SP_STRIDE_W,
  SP_PAD_H, SP_PAD_W,                  // top / left padding (may be negative)
  SP_ACT, SP_PRE_RELU,                 // epilogue act; ReLU applied to inputs on load
  SP_IN_SN, SP_IN_SH, SP_IN_SW, SP_IN_SC,
  SP_OUT_SN, SP_OUT_SH, SP_OUT_SW,     // output channel stride: SP_OUT_SC
  SP_RES_SN, SP_RES_SH, SP_RES_SW,     // residual (added before act), channel stride SP_RES_SC
  SP_HAS_RES,
  SP_POOL_MODE,                        // 0 max, 1 avg
  SP_COUNT_PAD,                        // avg: count_include_pad
  SP_PAD_BOTTOM, SP_PAD_RIGHT,         // avg count_include_pad window clamp
  SP_SPLIT_K,                          // K_CONV: split-K cluster size (1 = none)
  SP_OUT_SC,                           // output channel stride (1 = NHWC, H*W = NCHW output)
  SP_RES_SC,                           // residual channel stride (0 → 1)
  SP_KPAD,                             // K_CONV_TC: row stride of the pre-split weights
  SP_DW_ACT                            // K_SEPCONV: activation between depthwise and pointwise
};
// K_SEPCONV: PT_W / PT_BIAS = pointwise [K][C] / [K]; PT_WS = depthwise
// weights [R][S][C]; PT_DW_BIAS = depthwise bias [C]; spatial params describe
// the depthwise geometry, SP_K the pointwise output channels.
constexpr int PT_DW_BIAS = 6;
// ptrs: 0 in, 1 out, 2 weight [K][R][S][C], 3 bias, 4 residual, 5 workspace,
// 6/7 tcgen05 weights pre-split into TF32 hi / lo, [K][Kpad]
enum SpatialPtr : int { PT_IN = 0, PT_OUT, PT_W, PT_BIAS, PT_RES, PT_WS, PT_W_TC_HI, PT_W_TC_LO };

// K_ELTWISE / K_GLOBAL_POOL params
enum EwParam : int {
  EW_N = 0, EW_H, EW_W, EW_C, EW_OP, EW_ACT,
  EW_A_SN, EW_A_SH, EW_A_SW, EW_A_SC,
  EW_B_SN, EW_B_SH, EW_B_SW, EW_B_SC,
  EW_C_SN, EW_C_SH, EW_C_SW, EW_C_SC,
  EW_O_SN, EW_O_SH, EW_O_SW, EW_O_SC,
  EW_NIN,       // number of tensor operands (1..3)
  EW_PRE_RELU,  // global pool: relu on load
};
// ptrs: 0 a, 1 b, 2 c, 3 out, 4 scale, 5 shift
enum EwPtr : int { EP_A = 0, EP_B, EP_C, EP_OUT, EP_SCALE, EP_SHIFT };

// Launch one op on a stream (kernels/*.cu). Returns cudaError_t as int.
int launch_conv(const sw_op_desc& op, void* stream);
int launch_null(void* stream);  // diagnostic empty task
int launch_conv_pw(const sw_op_desc& op, int variant, void* stream);  // conv variants 16..21
int launch_conv_tc(const sw_op_desc& op, void* stream);
int launch_dwconv(const sw_op_desc& op, void* stream);
int launch_pool(const sw_op_desc& op, void* stream);
int launch_eltwise(const sw_op_desc& op, void* stream);
int launch_global_pool(const sw_op_desc& op, void* stream);
int launch_concat(const sw_op_desc& op, void* stream);
void init_tc_kernels();
void init_simt_kernels();
void init_pw_kernels();
int launch_sepconv(const sw_op_desc& op, void* stream);
void init_sep_kernels();

}  // namespace sw
