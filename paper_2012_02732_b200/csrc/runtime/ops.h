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
  // training (csrc/kernels/train.cu; paper_2012_02732_b200/train.py)
  K_BN_STATS = 9,       // batch statistics (+ running-stat update) of an NHWC map
  K_BN_APPLY = 10,      // normalise + affine (+ residual) + act
  K_BN_BWD_REDUCE = 11, // dgamma / dbeta (through the activation derivative)
  K_BN_BWD_APPLY = 12,  // dx of batch norm (+ accumulate)
  K_DW_DGRAD = 13,      // depthwise conv input gradient (+ accumulate)
  K_DW_WGRAD = 14,      // depthwise conv weight gradient
  K_GEMM = 15,          // strided / implicit-im2col GEMM with deterministic split-K
  K_XENT = 16,          // softmax cross-entropy: mean loss + dlogits
  K_SGD = 17,           // SGD with momentum + weight decay over the flat parameters
  K_ALLREDUCE = 18,     // NCCL average of the flat gradient buffer (engine-owned comm)
  K_EW_BWD = 19,        // activation / broadcast-mul backward (EfficientNet SE)
  K_TRANSPOSE = 20,     // out[c][r] = in[r][c] (1x1 weights for the dgrad conv)
  K_GEMM_REDUCE = 21,   // fold K_GEMM split partials (+ bias, + res): wide splits
  K_BN_FWD = 22,        // fused K_BN_STATS + K_BN_APPLY (per-channel-block barrier)
  K_BN_BWD = 23,        // fused K_BN_BWD_REDUCE + K_BN_BWD_APPLY (per-channel-block barrier)
  K_SEP2 = 24,          // NASNet separable block: two chained sepconvs in one cluster kernel
};

// K_SEP2 extra params (after the SpatialParam block; spatial params describe
// the FIRST sepconv's input / stride / pad, SP_P/SP_Q the map both stages
// share, SP_K the final channels, SP_ACT / residual the second pointwise's
// epilogue, SP_PRE_RELU the first depthwise's input ReLU, SP_SPLIT_K the
// cluster size = row bands per image)
enum Sep2Param : int {
  S2_MID = 36,      // channels between the two sepconvs
  S2_ACT1,          // activation after the first pointwise (+ folded BN)
  S2_DW_ACT1,       // activation after the first depthwise
  S2_DW_ACT2,       // activation after the second depthwise
  S2_PRE_RELU2,     // ReLU on load of the intermediate
  S2_OFF_DW1,       // offsets (floats) into the packed weights (PT_W):
  S2_OFF_PW1,       //   dw1 [k][k][C], pw1 [C][MID], b1 [MID], db1 [C] (or -1),
  S2_OFF_B1,        //   dw2 [k][k][MID], pw2 [MID][K], b2 [K], db2 [MID] (or -1)
  S2_OFF_DB1,
  S2_OFF_DW2,
  S2_OFF_PW2,
  S2_OFF_B2,
  S2_OFF_DB2,
};
// K_SEP2 ptrs: PT_IN, PT_OUT, PT_W (packed weights), PT_RES

// Batch-norm kinds (K_BN_*): params index
enum BnParam : int {
  BN_M = 0,      // pixels N*H*W
  BN_C,          // channels
  BN_HW,         // pixels per image (dOut broadcast decomposition)
  BN_ACT,        // activation after the affine
  BN_HAS_RES,    // APPLY: + residual (before act); BWD_APPLY: accumulate into res
  BN_EPS,        // float bits
  BN_MOMENTUM,   // float bits (running stats)
  BN_GRID,       // CTAs of the reduce kinds (workspace = GRID * 2 * C doubles + ticket)
  BN_DO_SN,      // dOut image stride
  BN_DO_SP,      // dOut pixel stride (0 = broadcast over H*W, e.g. global-pool backward)
  BN_DO_SCALE,   // float bits: dOut multiplier (1/HW for global-pool backward)
  BN_LD,         // pixel stride of y / out / res
};
// STATS ptrs: 0 y, 1 stats out [mean C | invstd C], 2 running [mean C | var C], 7 ws
// APPLY ptrs: 0 y, 1 stats, 2 gamma [gamma C | beta C], 3 res, 4 out
// BWD_REDUCE ptrs: 0 dOut, 1 y, 2 stats, 3 gamma|beta, 4 dgamma|dbeta, 7 ws
// BWD_APPLY ptrs: 0 dOut, 1 y, 2 stats, 3 gamma|beta, 4 dgamma|dbeta, 5 res, 6 out
// K_BN_FWD ptrs: 0 y, 1 stats, 2 running, 3 gamma|beta, 4 res, 5 out, 7 ws
// K_BN_BWD ptrs: as BWD_APPLY + 7 ws.  The fused kinds keep all BN_GRID x
// ceil(C/32) CTAs co-resident (cooperative launch) and meet at a barrier per
// channel block between the reduction and the elementwise pass.

// K_DW_DGRAD / K_DW_WGRAD reuse the SpatialParam geometry (SP_N..SP_PAD_W, the
// forward op's dims: input N,H,W,C → output P,Q); dense NHWC.
// DGRAD ptrs: 0 dY, 1 dX out, 2 W [R][S][C], 4 res (SP_HAS_RES accumulate)
// WGRAD ptrs: 0 dY, 1 dW out [R][S][C], 2 X, 5 ws; SP_SPLIT_K = CTAs
// (workspace = CTAs * R*S*C floats + ticket)

// K_GEMM: C[i,j] = sum_r A(i,r) B(r,j) (+ bias[j]) (+ res[i,j])
enum GemmParam : int {
  GM_M = 0, GM_N, GM_K,          // i < M, j < N, r < K
  GM_A_I, GM_A_R,                // A(i,r) = A[i*a_i + r*a_r]
  GM_B_R, GM_B_J,                // B(r,j) = B[r*b_r + j*b_j]  (GM_IM2COL = 0)
  GM_C_I,                        // C[i*c_i + j]
  GM_SPLIT,                      // split of r over gridDim.z (deterministic ticket reduce)
  GM_HAS_RES,                    // accumulate: C = AB + res (res may alias C)
  GM_IM2COL,                     // 1: B(r=pixel, j=(rr,ss,c)) gathered from a conv input
  GM_X_N, GM_X_H, GM_X_W, GM_X_C, GM_X_P, GM_X_Q, GM_X_R, GM_X_S,
  GM_X_STRIDE, GM_X_PAD,
  GM_X_SN, GM_X_SH, GM_X_SW, GM_X_SC,
  GM_PARTIALS_ONLY,              // 1: split CTAs only store partials; a K_GEMM_REDUCE task folds them
};
// ptrs: 0 A, 1 B, 2 C, 3 bias, 4 res, 5 ws (split > 1: split*tiles*64*64 floats + tiles tickets)
// K_GEMM_REDUCE: same params/ptrs as the K_GEMM whose partials it folds (ws
// layout [tile][split][64x64]); 8 partial lanes x 32 outputs per CTA.

// K_XENT params: 0 N, 1 classes, 2 logits row stride; ptrs 0 logits, 1 labels (int32),
// 2 loss (1 float), 3 dlogits [N][classes]
// K_SGD params: 0 n, 1 lr, 2 momentum, 3 weight decay (float bits); ptrs 0 params,
// 1 grads, 2 momentum buffer
// K_ALLREDUCE params: 0 count (floats); ptrs 0 buffer (in place)
// K_TRANSPOSE params: 0 rows, 1 cols; ptrs 0 in [rows][cols], 1 out [cols][rows]
// K_EW_BWD params: 0 N, 1 HW, 2 C, 3 mode (0 act-backward: dx = dy*act'(z) [+res];
// 1 mul-backward: dx = dy*s[n,c] [+res]; 2 mul-backward to the scale: ds[n,c] =
// sum_hw dy*x, then act'(z_s) applied; 3 broadcast: dx = s[n,c]*scale [+res]
// (global-pool backward)), 4 act, 5 has_res, 6 scale (float bits);
// ptrs 0 dy, 1 z/x, 2 s, 3 res, 4 out, 5 z_s
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
  SP_DW_ACT,                           // K_SEPCONV: activation between depthwise and pointwise
  SP_POOL_MUL                          // K_POOL: integer output multiplier (0 → 1): twin pools merged
};
// K_CONV / K_CONV_TC: which packed weight image PT_WS holds for the
// weight-streaming variants (conv_tcs.cu): 0 = 3xTF32 hi|lo (variants 6000 +
// NT), 1 = bf16 (variants 7000 + NT, the engine's precision="bf16" path)
constexpr int SP_WS_KIND = 49;
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
int launch_io_copy(void* dst, const void* src, int64_t bytes, void* stream);  // staging copy as a kernel
int set_io_copy_node(void* exec, void* node, void* dst, const void* src, int64_t bytes);  // re-point it
int launch_l2_prefetch(const void* p, int64_t bytes, void* stream);  // warm L2 with the weights
int launch_conv_pw(const sw_op_desc& op, int variant, void* stream);  // conv variants 16..21
int launch_conv_tc(const sw_op_desc& op, void* stream);
int launch_dwconv(const sw_op_desc& op, void* stream);
int launch_pool(const sw_op_desc& op, void* stream);
int launch_eltwise(const sw_op_desc& op, void* stream);
int launch_global_pool(const sw_op_desc& op, void* stream);
int launch_concat(const sw_op_desc& op, void* stream);
void init_tc_kernels();
// K_CONV_TC variants 6000 + NT: weight-streaming swap-AB tcgen05 conv for
// few output pixels (conv_tcs.cu)
int launch_conv_tcs(const sw_op_desc& op, void* stream);
void init_tcs_kernels();
// K_CONV_TC variants 8000 + BN: large-batch pointwise conv, persistent
// warp-specialised tcgen05 GEMM with double-buffered TMEM (conv_pw_tc.cu)
int launch_conv_pw_tc(const sw_op_desc& op, void* stream);
void init_pw_tc_kernels();
void init_simt_kernels();
void init_pw_kernels();
int launch_sepconv(const sw_op_desc& op, void* stream);
void init_sep_kernels();
// K_SEPCONV variant SEP_TC_VARIANT: depthwise + tcgen05 pointwise, persistent
// warp-specialised (sepconv_tc.cu); PT_W_TC_LO = the packed 3xTF32 pointwise
// weight images [block][hi | lo][Cpad/4][BN][4] (engine.py sep_tc_layout)
constexpr int SEP_TC_VARIANT = 100;
int launch_sepconv_tc(const sw_op_desc& op, void* stream);
// sep_rows.cu: row-staged fused sepconv for thin wide maps (variants 20..23)
int launch_sep_rows(const sw_op_desc& op, void* stream);
int launch_pool_rows(const sw_op_desc& op, void* stream);  // K_POOL variant 2
void init_sep_rows_kernels();
void init_sep_tc_kernels();
int launch_train(const sw_op_desc& op, void* stream);  // K_BN_* .. K_SGD, K_EW_BWD
int launch_sep2(const sw_op_desc& op, void* stream);   // K_SEP2 (sep2.cu)
void init_sep2_kernels();

}  // namespace sw
