// Dense convolution / 1x1 convolution / linear as an implicit GEMM on the
// fp32 SIMT pipe (the fp32-exact path; the tensor-core path is conv_tc.cu).
//
//   GEMM view: M = N*P*Q output pixels, Ncol = K output channels,
//              Kdim = R*S*C with k = (r*S + s)*C + c (weights [K][R][S][C]).
//   Epilogue:  v = acc + bias[k] (+ residual) -> act -> strided store, so
//              BN (folded into weights/bias), ReLU/ReLU6/SiLU, residual adds
//              and zero-copy concat (output channel slice + pixel stride)
//              never touch HBM twice.
//   Split-K:   a thread-block cluster of `split` CTAs along grid z each owns
//              a K slice; partial tiles are reduced through distributed
//              shared memory (DSMEM) and every rank finishes a slice of the
//              tile, so deep-K / small-M layers (batch 1) fill the 148 SMs
//              with one deterministic kernel and no workspace.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

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
};

static ConvArgs conv_args(const sw_op_desc& op) {
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
  return a;
}

__device__ __forceinline__ void conv_epilogue_store(const ConvArgs& a, int m, int n, float v) {
  int q = m % a.Q;
  int t = m / a.Q;
  int pp = t % a.P;
  int nb = t / a.P;
  v += a.bias ? a.bias[n] : 0.f;
  if (a.has_res) v += a.res[nb * a.res_sn + pp * a.res_sh + q * a.res_sw + n * a.res_sc];
  a.out[nb * a.out_sn + pp * a.out_sh + q * a.out_sw + n * a.out_sc] = apply_act(v, a.act);
}

// BM x BN output tile, 4x4 micro-tile per thread, BK = 16, register-staged
// double buffering of the smem tiles.
template <int BM, int BN>
__global__ void __launch_bounds__((BM / 4) * (BN / 4))
conv_simt_kernel(ConvArgs a) {
  constexpr int BK = 16;
  constexpr int NT = (BM / 4) * (BN / 4);
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = BN * BK / NT;
  constexpr int PAD = 4;
  static_assert(NT % BK == 0, "kk must be fixed per thread");
  constexpr int TILE_FLOATS = 2 * BK * (BM + PAD) + 2 * BK * (BN + PAD);
  constexpr int SMEM_FLOATS = TILE_FLOATS > BM * BN ? TILE_FLOATS : BM * BN;
  __shared__ __align__(16) float smem[SMEM_FLOATS];
  float* As = smem;                           // [2][BK][BM+PAD]
  float* Bs = smem + 2 * BK * (BM + PAD);     // [2][BK][BN+PAD]

  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int kk = tid % BK;

  // K range of this split (cluster rank == blockIdx.z)
  const int ksteps_total = (a.Kdim + BK - 1) / BK;
  const int per = (ksteps_total + a.split - 1) / a.split;
  const int ks_begin = blockIdx.z * per;
  const int ks_end = min(ksteps_total, ks_begin + per);

  // per-thread pixel decode for the A loads (fixed across K)
  int64_t a_base[A_PER];
  int a_ih[A_PER], a_iw[A_PER];
  bool a_ok[A_PER];
#pragma unroll
  for (int i = 0; i < A_PER; ++i) {
    int mm = (tid + i * NT) / BK;
    int m = m0 + mm;
    a_ok[i] = m < a.M;
    int mq = a_ok[i] ? m : 0;
    int q = mq % a.Q;
    int t = mq / a.Q;
    int p = t % a.P;
    int nb = t / a.P;
    a_base[i] = nb * a.in_sn;
    a_ih[i] = p * a.sh - a.ph;
    a_iw[i] = q * a.sw - a.pw;
  }
  float ra[A_PER], rb[B_PER];

  auto load_tiles = [&](int kstep) {
    int k = kstep * BK + kk;
    bool kin = k < a.Kdim;
    int c = 0, r = 0, s = 0;
    if (kin) {
      c = k % a.C;
      int rs = k / a.C;
      s = rs % a.S;
      r = rs / a.S;
    }
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      float v = 0.f;
      int ih = a_ih[i] + r, iw = a_iw[i] + s;
      if (kin && a_ok[i] && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W) {
        v = __ldg(a.in + a_base[i] + ih * a.in_sh + iw * a.in_sw + c * a.in_sc);
        if (a.pre_relu) v = fmaxf(v, 0.f);
      }
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      int nn = (tid + i * NT) / BK;
      int n = n0 + nn;
      rb[i] = (kin && n < a.K) ? __ldg(a.w + (int64_t)n * a.Kdim + k) : 0.f;
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int i = 0; i < A_PER; ++i) As[(buf * BK + kk) * (BM + PAD) + (tid + i * NT) / BK] = ra[i];
#pragma unroll
    for (int i = 0; i < B_PER; ++i) Bs[(buf * BK + kk) * (BN + PAD) + (tid + i * NT) / BK] = rb[i];
  };

  const int ty = tid / (BN / 4);
  const int tx = tid % (BN / 4);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  if (ks_begin < ks_end) {
    load_tiles(ks_begin);
    store_tiles(0);
    __syncthreads();
    for (int ks = ks_begin; ks < ks_end; ++ks) {
      int buf = (ks - ks_begin) & 1;
      if (ks + 1 < ks_end) load_tiles(ks + 1);
#pragma unroll
      for (int k2 = 0; k2 < BK; ++k2) {
        float4 av = *reinterpret_cast<const float4*>(&As[(buf * BK + k2) * (BM + PAD) + ty * 4]);
        float4 bv = *reinterpret_cast<const float4*>(&Bs[(buf * BK + k2) * (BN + PAD) + tx * 4]);
        float ai[4] = {av.x, av.y, av.z, av.w};
        float bj[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ai[i], bj[j], acc[i][j]);
      }
      if (ks + 1 < ks_end) store_tiles(buf ^ 1);
      __syncthreads();
    }
  }

  if (a.split == 1) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int m = m0 + ty * 4 + i;
      if (m >= a.M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int n = n0 + tx * 4 + j;
        if (n < a.K) conv_epilogue_store(a, m, n, acc[i][j]);
      }
    }
    return;
  }

  // split-K: reduce partial tiles across the cluster through DSMEM.
  cg::cluster_group cluster = cg::this_cluster();
  float* part = smem;  // BM*BN floats, reuses the operand tiles
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) part[(ty * 4 + i) * BN + tx * 4 + j] = acc[i][j];
  cluster.sync();
  const int rank = (int)cluster.block_rank();
  const int nranks = (int)cluster.num_blocks();
  const int chunk = (BM * BN + nranks - 1) / nranks;
  const int e_begin = rank * chunk;
  const int e_end = min(BM * BN, e_begin + chunk);
  for (int e = e_begin + tid; e < e_end; e += NT) {
    int mm = e / BN, nn = e % BN;
    int m = m0 + mm, n = n0 + nn;
    if (m >= a.M || n >= a.K) continue;
    float v = 0.f;
    for (int r = 0; r < nranks; ++r) v += cluster.map_shared_rank(part, r)[e];
    conv_epilogue_store(a, m, n, v);
  }
  cluster.sync();
}

// Small-M 1x1 conv / linear (batch-1 classifier heads, 1x1-spatial layers):
// one warp per output channel streams its weight row once with 128-bit loads.
template <int MAXM>
__global__ void __launch_bounds__(256) conv_gemv_kernel(ConvArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.K) return;
  const int n = warp;
  const float* wrow = a.w + (int64_t)n * a.Kdim;
  int64_t base[MAXM];
  for (int m = 0; m < a.M; ++m) {
    int q = m % a.Q;
    int t = m / a.Q;
    int p = t % a.P;
    int nb = t / a.P;
    base[m] = nb * a.in_sn + (int64_t)(p * a.sh - a.ph) * a.in_sh + (int64_t)(q * a.sw - a.pw) * a.in_sw;
  }
  float acc[MAXM];
#pragma unroll
  for (int m = 0; m < MAXM; ++m) acc[m] = 0.f;
  const bool vec = (a.in_sc == 1) && ((a.Kdim & 3) == 0) && ((reinterpret_cast<uintptr_t>(wrow) & 15) == 0);
  if (vec) {
    for (int k = lane * 4; k < a.Kdim; k += 128) {
      float4 wv = __ldg(reinterpret_cast<const float4*>(wrow + k));
#pragma unroll
      for (int m = 0; m < MAXM; ++m) {
        if (m < a.M) {
          const float* src = a.in + base[m] + k;
          float x0 = __ldg(src), x1 = __ldg(src + 1), x2 = __ldg(src + 2), x3 = __ldg(src + 3);
          if (a.pre_relu) {
            x0 = fmaxf(x0, 0.f); x1 = fmaxf(x1, 0.f); x2 = fmaxf(x2, 0.f); x3 = fmaxf(x3, 0.f);
          }
          acc[m] += wv.x * x0 + wv.y * x1 + wv.z * x2 + wv.w * x3;
        }
      }
    }
  } else {
    for (int k = lane; k < a.Kdim; k += 32) {
      float wv = __ldg(wrow + k);
#pragma unroll
      for (int m = 0; m < MAXM; ++m) {
        if (m < a.M) {
          float x = __ldg(a.in + base[m] + k * a.in_sc);
          if (a.pre_relu) x = fmaxf(x, 0.f);
          acc[m] = fmaf(wv, x, acc[m]);
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < MAXM; ++m) {
    float v = acc[m];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[m] = v;
  }
  if (lane == 0)
    for (int m = 0; m < a.M; ++m) conv_epilogue_store(a, m, n, acc[m]);
}

// variant: 0 = 64x64, 1 = 32x64, 2 = 32x32, 3 = 128x64, 8 = gemv (M <= 8, 1x1)
int launch_conv(const sw_op_desc& op, void* stream) {
  ConvArgs a = conv_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  if (op.variant == 8) {
    if (a.M > 8 || a.R != 1 || a.S != 1) return (int)cudaErrorInvalidValue;
    int blocks = (int)cdiv((int64_t)a.K * 32, 256);
    conv_gemv_kernel<8><<<blocks, 256, 0, st>>>(a);
    return (int)cudaGetLastError();
  }
  int bm = 64, bn = 64;
  switch (op.variant) {
    case 1: bm = 32; bn = 64; break;
    case 2: bm = 32; bn = 32; break;
    case 3: bm = 128; bn = 64; break;
    default: break;
  }
  dim3 grid((unsigned)cdiv(a.M, bm), (unsigned)cdiv(a.K, bn), (unsigned)a.split);
  int threads = (bm / 4) * (bn / 4);
  void (*fn)(ConvArgs) = nullptr;
  switch (op.variant) {
    case 1: fn = conv_simt_kernel<32, 64>; break;
    case 2: fn = conv_simt_kernel<32, 32>; break;
    case 3: fn = conv_simt_kernel<128, 64>; break;
    default: fn = conv_simt_kernel<64, 64>; break;
  }
  if (a.split == 1) {
    fn<<<grid, threads, 0, st>>>(a);
    return (int)cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)a.split;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return (int)cudaLaunchKernelEx(&cfg, fn, a);
}

}  // namespace sw
