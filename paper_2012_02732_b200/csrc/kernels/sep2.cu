// NASNet separable block in ONE kernel (K_SEP2):
//   [relu] → dw1 k×k (stride s) → pw1 (+ folded BN) → act1 → [relu]
//          → dw2 k×k (stride 1, same padding) → pw2 (+ folded BN) (+ residual) → act2
//
// Two chained sepconv tasks cost two graph nodes on the NASNet critical path
// (conv_1x1 → sep → sep per cell, profiles/r01_tasks_nasnet_bs1.txt); here the
// intermediate map never leaves the chip.  One thread-block CLUSTER per image:
// CTA r owns a band of output rows.  Stage 1 computes the intermediate rows of
// its band (all channels) into shared memory; after a cluster barrier, stage 2
// reads the k/2 halo rows of the second depthwise straight from the
// neighbouring CTAs' shared memory (DSMEM), then runs the second pointwise and
// the epilogue.  A second cluster barrier keeps every band alive until its
// neighbours have read their halo.
//
// Latency-oriented (batch-1 maps are 7²..56²): depthwise filters are staged in
// shared memory before the PDL wait; pointwise GEMMs are thread-per-output
// dot products over smem rows with coalesced weight reads (weights stored
// [C][K]).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sw {

namespace {

struct Sep2Args {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ pack;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, sh, sw, ph, pw, mid;
  int pre_relu1, dw_act1, act1, pre_relu2, dw_act2, act2, has_res, rows;
  int64_t in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  int64_t o_dw1, o_pw1, o_b1, o_db1, o_dw2, o_pw2, o_b2, o_db2;
};

}  // namespace

template <int KS>
__global__ void __launch_bounds__(256) sep2_kernel(Sep2Args a) {
  extern __shared__ __align__(16) float smem[];
  const int C = a.C, MID = a.mid, Q = a.Q;
  const int BPX = a.rows * Q;  // pixels of one band
  float* wd1 = smem;                        // [KS*KS][C]
  float* wd2 = wd1 + KS * KS * C;           // [KS*KS][MID]
  float* D1 = wd2 + KS * KS * MID;          // [BPX][C]    first depthwise
  float* Y = D1 + BPX * C;                  // [BPX][MID]  intermediate band (read by the peers)
  float* D2 = Y + BPX * MID;                // [BPX][MID]  second depthwise
  const int tid = threadIdx.x;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int nb = blockIdx.y;
  const int r0 = rank * a.rows;
  const int nrows = max(0, min(a.P, r0 + a.rows) - r0);
  const int npx = nrows * Q;

  // constants before the PDL wait
  for (int e = tid; e < KS * KS * C; e += 256) wd1[e] = __ldg(a.pack + a.o_dw1 + e);
  for (int e = tid; e < KS * KS * MID; e += 256) wd2[e] = __ldg(a.pack + a.o_dw2 + e);
  pdl_trigger();
  pdl_wait();
  __syncthreads();

  // ---- stage 1a: first depthwise (stride s) for the band, all C channels ----
  const float* inb = a.in + nb * a.in_sn;
  for (int e = tid; e < npx * C; e += 256) {
    const int c = e % C, px = e / C;
    const int p = r0 + px / Q, q = px % Q;
    const int ih0 = p * a.sh - a.ph, iw0 = q * a.sw - a.pw;
    float acc = a.o_db1 >= 0 ? __ldg(a.pack + a.o_db1 + c) : 0.f;
#pragma unroll
    for (int r = 0; r < KS; ++r) {
      const int ih = ih0 + r;
      const bool rok = (unsigned)ih < (unsigned)a.H;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int iw = iw0 + s;
        const bool ok = rok && (unsigned)iw < (unsigned)a.W;
        float x = __ldg(inb + (ok ? ih * a.in_sh + iw * a.in_sw + c * a.in_sc : 0));
        if (a.pre_relu1) x = fmaxf(x, 0.f);
        acc = fmaf(ok ? x : 0.f, wd1[(r * KS + s) * C + c], acc);
      }
    }
    D1[px * C + c] = apply_act(acc, a.dw_act1);
  }
  __syncthreads();
  // ---- stage 1b: first pointwise → intermediate band Y ----
  const float* pw1 = a.pack + a.o_pw1;  // [C][MID]
  for (int e = tid; e < npx * MID; e += 256) {
    const int j = e % MID, px = e / MID;
    float acc = __ldg(a.pack + a.o_b1 + j);
    const float* d = D1 + px * C;
#pragma unroll 4
    for (int c = 0; c < C; ++c) acc = fmaf(d[c], __ldg(pw1 + c * MID + j), acc);
    acc = apply_act(acc, a.act1);
    if (a.pre_relu2) acc = fmaxf(acc, 0.f);
    Y[px * MID + j] = acc;
  }
  cluster.sync();  // every band of the intermediate map is in its CTA's smem

  // ---- stage 2a: second depthwise (stride 1, same padding), halo via DSMEM ----
  const int pad2 = KS / 2;
  for (int e = tid; e < npx * MID; e += 256) {
    const int j = e % MID, px = e / MID;
    const int p = r0 + px / Q, q = px % Q;
    float acc = a.o_db2 >= 0 ? __ldg(a.pack + a.o_db2 + j) : 0.f;
#pragma unroll
    for (int r = 0; r < KS; ++r) {
      const int pp = p + r - pad2;
      if ((unsigned)pp >= (unsigned)a.P) continue;
      const int owner = pp / a.rows;
      const float* yb = owner == rank ? Y : cluster.map_shared_rank(Y, owner);
      const float* yrow = yb + (pp - owner * a.rows) * Q * MID + j;
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int qq = q + s - pad2;
        if ((unsigned)qq >= (unsigned)Q) continue;
        acc = fmaf(yrow[qq * MID], wd2[(r * KS + s) * MID + j], acc);
      }
    }
    D2[px * MID + j] = apply_act(acc, a.dw_act2);
  }
  __syncthreads();
  // ---- stage 2b: second pointwise + residual + act → out ----
  const float* pw2 = a.pack + a.o_pw2;  // [MID][K]
  for (int e = tid; e < npx * a.K; e += 256) {
    const int k = e % a.K, px = e / a.K;
    const int p = r0 + px / Q, q = px % Q;
    float acc = __ldg(a.pack + a.o_b2 + k);
    const float* d = D2 + px * MID;
#pragma unroll 4
    for (int j = 0; j < MID; ++j) acc = fmaf(d[j], __ldg(pw2 + j * a.K + k), acc);
    if (a.has_res) acc += a.res[nb * a.res_sn + p * a.res_sh + q * a.res_sw + k * a.res_sc];
    a.out[nb * a.out_sn + p * a.out_sh + q * a.out_sw + k * a.out_sc] = apply_act(acc, a.act2);
  }
  cluster.sync();  // the peers have read my halo rows
}

static Sep2Args sep2_args(const sw_op_desc& op) {
  const int64_t* p = op.params;
  Sep2Args a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.pack = reinterpret_cast<const float*>(op.ptrs[PT_W]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K]; a.R = (int)p[SP_R];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W]; a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.mid = (int)p[S2_MID];
  a.pre_relu1 = (int)p[SP_PRE_RELU]; a.dw_act1 = (int)p[S2_DW_ACT1]; a.act1 = (int)p[S2_ACT1];
  a.pre_relu2 = (int)p[S2_PRE_RELU2]; a.dw_act2 = (int)p[S2_DW_ACT2]; a.act2 = (int)p[SP_ACT];
  a.has_res = (int)p[SP_HAS_RES];
  a.in_sn = p[SP_IN_SN]; a.in_sh = p[SP_IN_SH]; a.in_sw = p[SP_IN_SW]; a.in_sc = p[SP_IN_SC];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  a.o_dw1 = p[S2_OFF_DW1]; a.o_pw1 = p[S2_OFF_PW1]; a.o_b1 = p[S2_OFF_B1]; a.o_db1 = p[S2_OFF_DB1];
  a.o_dw2 = p[S2_OFF_DW2]; a.o_pw2 = p[S2_OFF_PW2]; a.o_b2 = p[S2_OFF_B2]; a.o_db2 = p[S2_OFF_DB2];
  const int cl = p[SP_SPLIT_K] > 0 ? (int)p[SP_SPLIT_K] : 1;
  a.rows = (a.P + cl - 1) / cl;
  return a;
}

static size_t sep2_smem(const Sep2Args& a, int ks) {
  const size_t bpx = (size_t)a.rows * a.Q;
  return 4 * ((size_t)ks * ks * (a.C + a.mid) + bpx * (a.C + 2 * (size_t)a.mid));
}

constexpr int kSep2SmemMax = 227 * 1024;

// SP_SPLIT_K = cluster size (bands per image, <= 16)
int launch_sep2(const sw_op_desc& op, void* stream) {
  Sep2Args a = sep2_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int cl = op.params[SP_SPLIT_K] > 0 ? (int)op.params[SP_SPLIT_K] : 1;
  if (cl > 16 || a.R != (int)op.params[SP_S]) return (int)cudaErrorInvalidValue;
  const size_t smem = sep2_smem(a, a.R);
  if (smem > (size_t)kSep2SmemMax) return (int)cudaErrorInvalidValue;
  const dim3 grid(1, (unsigned)a.N, (unsigned)cl);  // one cluster (along z) per image
  switch (a.R) {
    case 3: return (int)launch_k(sep2_kernel<3>, grid, dim3(256), smem, st, (unsigned)cl, a);
    case 5: return (int)launch_k(sep2_kernel<5>, grid, dim3(256), smem, st, (unsigned)cl, a);
    case 7: return (int)launch_k(sep2_kernel<7>, grid, dim3(256), smem, st, (unsigned)cl, a);
    default: return (int)cudaErrorInvalidValue;
  }
}

void init_sep2_kernels() {
  cudaFuncSetAttribute(sep2_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSep2SmemMax);
  cudaFuncSetAttribute(sep2_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSep2SmemMax);
  cudaFuncSetAttribute(sep2_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSep2SmemMax);
  cudaFuncSetAttribute(sep2_kernel<3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(sep2_kernel<5>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(sep2_kernel<7>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

}  // namespace sw
