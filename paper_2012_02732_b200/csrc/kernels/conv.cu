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

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// BM x BN output tile, 4x4 micro-tile per thread, BK = 16, STAGES-deep
// cp.async (LDGSTS) pipeline: the im2col gather of STAGES-1 future K tiles is
// in flight while the current tile is multiplied, so a layer costs about one
// memory round trip instead of one per K tile (batch-1 layers are latency-,
// not FLOP-bound).  Out-of-range taps are zero-filled by cp.async itself.
template <int BM, int BN, bool PRE>
__global__ void __launch_bounds__((BM / 4) * (BN / 4))
conv_simt_kernel(ConvArgs a) {
  // Code size matters as much as FLOPs here: at batch 1 every CTA starts on
  // a cold SM, so loops outside the FMA micro-kernel stay rolled and the
  // epilogue is one smem-staged loop shared with the split-K reduction.
  constexpr int BK = 16;
  constexpr int STAGES = 4;
  constexpr int NT = (BM / 4) * (BN / 4);
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = BN * BK / NT;
  constexpr int PAD = 4;
  static_assert(NT % BK == 0, "kk must be fixed per thread");
  extern __shared__ __align__(16) float smem[];
  float* As = smem;                                // [STAGES][BK][BM+PAD]
  float* Bs = smem + STAGES * BK * (BM + PAD);     // [STAGES][BK][BN+PAD]

  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int kk = tid % BK;
  const int row = tid / BK;  // + i * (NT / BK)

  // K range of this split (cluster rank == blockIdx.z)
  const int ksteps_total = (a.Kdim + BK - 1) / BK;
  const int per = (ksteps_total + a.split - 1) / a.split;
  const int ks_begin = blockIdx.z * per;
  const int nsteps = max(0, min(ksteps_total, ks_begin + per) - ks_begin);

  // per-thread pixel decode for the A loads (fixed across K)
  int a_base[A_PER], a_ih[A_PER], a_iw[A_PER];
#pragma unroll
  for (int i = 0; i < A_PER; ++i) {
    int m = m0 + row + i * (NT / BK);
    int q = m % a.Q;
    int t = m / a.Q;
    int p = t % a.P;
    int nb = t / a.P;
    a_base[i] = nb * (int)a.in_sn;
    a_ih[i] = m < a.M ? p * a.sh - a.ph : -(1 << 28);  // out-of-range row: never valid
    a_iw[i] = q * a.sw - a.pw;
  }
  const int in_sh = (int)a.in_sh, in_sw = (int)a.in_sw, in_sc = (int)a.in_sc;

  // cp.async gather of K tile `kstep` into pipeline buffer `buf`
  auto issue = [&](int kstep, int buf) {
    const int k = kstep * BK + kk;
    const bool kin = k < a.Kdim;
    const int c = k % a.C;
    const int rs = k / a.C;
    const int s = rs % a.S;
    const int r = rs / a.S;
    float* as = As + (buf * BK + kk) * (BM + PAD) + row;
    float* bs = Bs + (buf * BK + kk) * (BN + PAD) + row;
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      const int ih = a_ih[i] + r, iw = a_iw[i] + s;
      const bool ok = kin && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
      const float* src = a.in + (ok ? a_base[i] + ih * in_sh + iw * in_sw + c * in_sc : 0);
      cp_async4(as + i * (NT / BK), src, ok);
    }
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      const int n = n0 + row + i * (NT / BK);
      const bool ok = kin && n < a.K;
      cp_async4(bs + i * (NT / BK), a.w + (ok ? (size_t)n * a.Kdim + k : 0), ok);
    }
  };

  const int ty = tid / (BN / 4);
  const int tx = tid % (BN / 4);
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  pdl_trigger();
  pdl_wait();
#pragma unroll 1
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nsteps) issue(ks_begin + st, st);
    cp_async_commit();
  }
#pragma unroll 1
  for (int it = 0; it < nsteps; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // tile `it` landed for everyone; buffer (it-1)%STAGES is free
    const int nxt = it + STAGES - 1;
    if (nxt < nsteps) issue(ks_begin + nxt, nxt % STAGES);
    cp_async_commit();
    const float* at = As + (it % STAGES) * BK * (BM + PAD) + ty * 4;
    const float* bt = Bs + (it % STAGES) * BK * (BN + PAD) + tx * 4;
#pragma unroll 4
    for (int k2 = 0; k2 < BK; ++k2) {
      float4 av = *reinterpret_cast<const float4*>(at + k2 * (BM + PAD));
      float4 bv = *reinterpret_cast<const float4*>(bt + k2 * (BN + PAD));
      if (PRE) {
        av.x = fmaxf(av.x, 0.f); av.y = fmaxf(av.y, 0.f); av.z = fmaxf(av.z, 0.f); av.w = fmaxf(av.w, 0.f);
      }
      const float ai[4] = {av.x, av.y, av.z, av.w};
      const float bj[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(ai[i], bj[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // stage the tile in smem (reusing the operand buffers), then one rolled
  // epilogue loop; split-K ranks of a cluster reduce through DSMEM first
  float* part = smem;  // [BM][BN]
#pragma unroll
  for (int i = 0; i < 4; ++i)
    *reinterpret_cast<float4*>(&part[(ty * 4 + i) * BN + tx * 4]) =
        make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
  int e_begin = 0, e_end = BM * BN, nranks = 1;
  cg::cluster_group cluster = cg::this_cluster();
  if (a.split > 1) {
    cluster.sync();
    nranks = (int)cluster.num_blocks();
    const int chunk = (BM * BN + nranks - 1) / nranks;
    e_begin = (int)cluster.block_rank() * chunk;
    e_end = min(BM * BN, e_begin + chunk);
  } else {
    __syncthreads();
  }
#pragma unroll 1
  for (int e = e_begin + tid; e < e_end; e += NT) {
    const int m = m0 + e / BN, n = n0 + e % BN;
    if (m >= a.M || n >= a.K) continue;
    float v = part[e];
    if (nranks > 1) {
      v = 0.f;
#pragma unroll 1
      for (int r = 0; r < nranks; ++r) v += cluster.map_shared_rank(part, r)[e];
    }
    conv_epilogue_store(a, m, n, v);
  }
  if (a.split > 1) cluster.sync();
}


// Small-M 1x1 conv / linear (batch-1 classifier heads, 1x1-spatial layers):
// one warp per output channel streams its weight row once with 128-bit loads.
template <int MAXM>
__global__ void __launch_bounds__(256) conv_gemv_kernel(ConvArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  pdl_trigger();
  pdl_wait();
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
#pragma unroll 1
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
  if (lane == 0) {
#pragma unroll
    for (int m = 0; m < MAXM; ++m)
      if (m < a.M) conv_epilogue_store(a, m, n, acc[m]);
  }
}

static size_t simt_smem_bytes(int bm, int bn) {
  const size_t tile = 4 * 16 * (size_t)(bm + 4) + 4 * 16 * (size_t)(bn + 4);  // STAGES * BK * (B? + PAD)
  const size_t part = (size_t)bm * bn;
  return 4 * (tile > part ? tile : part);
}

void init_simt_kernels() {
  const int cfgs[4][2] = {{64, 64}, {32, 64}, {32, 32}, {128, 64}};
  void (*fns[4][2])(ConvArgs) = {
      {conv_simt_kernel<64, 64, false>, conv_simt_kernel<64, 64, true>},
      {conv_simt_kernel<32, 64, false>, conv_simt_kernel<32, 64, true>},
      {conv_simt_kernel<32, 32, false>, conv_simt_kernel<32, 32, true>},
      {conv_simt_kernel<128, 64, false>, conv_simt_kernel<128, 64, true>}};
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 2; ++j)
      cudaFuncSetAttribute(fns[i][j], cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)simt_smem_bytes(cfgs[i][0], cfgs[i][1]));
}

// variant: 0 = 64x64, 1 = 32x64, 2 = 32x32, 3 = 128x64, 8 = gemv (M <= 8, 1x1)
int launch_conv(const sw_op_desc& op, void* stream) {
  ConvArgs a = conv_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  if (op.variant == 8) {
    if (a.M > 8 || a.R != 1 || a.S != 1) return (int)cudaErrorInvalidValue;
    int blocks = (int)cdiv((int64_t)a.K * 32, 256);
    return (int)launch_k(conv_gemv_kernel<8>, dim3(blocks), dim3(256), 0, st, 1, a);
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
  const bool pre = a.pre_relu != 0;
  switch (op.variant) {
    case 1: fn = pre ? conv_simt_kernel<32, 64, true> : conv_simt_kernel<32, 64, false>; break;
    case 2: fn = pre ? conv_simt_kernel<32, 32, true> : conv_simt_kernel<32, 32, false>; break;
    case 3: fn = pre ? conv_simt_kernel<128, 64, true> : conv_simt_kernel<128, 64, false>; break;
    default: fn = pre ? conv_simt_kernel<64, 64, true> : conv_simt_kernel<64, 64, false>; break;
  }
  const size_t smem = simt_smem_bytes(bm, bn);
  return (int)launch_k(fn, grid, dim3(threads), smem, st, (unsigned)a.split, a);
}

}  // namespace sw
