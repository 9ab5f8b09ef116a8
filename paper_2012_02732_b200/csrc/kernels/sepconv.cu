// Fused separable convolution: depthwise k x k → (bias, act) → pointwise 1x1
// → (bias, residual, act) in ONE kernel (NASNet sep-convs, MobileNetV2
// dw → project).  The depthwise result for the CTA's pixel tile never leaves
// shared memory, and the graph loses one node per separable conv — at batch 1
// the graph executor issues roughly one kernel node per microsecond
// (tools/microbench.cu), so node count is latency.
//
// CTA = 256 threads, tile = 16 output pixels x 32 output channels:
//   1. cp.async prefetch of the first pointwise-weight chunk;
//   2. depthwise for all C_in channels of the 16 pixels into smem D[c][px]
//      (branch-free unrolled taps, 128-bit NHWC loads when C % 4 == 0);
//   3. pointwise GEMM D^T x W over C_in (all weight chunks requested by
//      cp.async at kernel start, before the PDL wait), 1x2 micro-tile;
//   4. smem-staged rolled epilogue (bias, residual, activation, strided store).
#include "common.cuh"

namespace sw {

namespace {

constexpr int SEP_BM = 16;
constexpr int SEP_BN = 32;
constexpr int SEP_BK = 16;
constexpr int SEP_THREADS = 256;

struct SepArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w_pw;   // [K][C]
  const float* __restrict__ b_pw;   // [K] or null
  const float* __restrict__ w_dw;   // [R][S][C]
  const float* __restrict__ b_dw;   // [C] or null
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, dw_act, pre_relu, has_res, M, vec;
  int in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
};

__device__ __forceinline__ void cp4(float* dst, const float* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

}  // namespace

template <int KS, bool VEC>
__global__ void __launch_bounds__(SEP_THREADS) sepconv_kernel(SepArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int Cp = (a.C + SEP_BK - 1) / SEP_BK * SEP_BK;  // D rows padded to the K chunk
  float* D = smem;                                      // [Cp][SEP_BM]
  float* Bs = smem + Cp * SEP_BM;                       // [Cp][SEP_BN]: every weight chunk
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * SEP_BM;
  const int n0 = blockIdx.y * SEP_BN;
  const int RR = KS ? KS : a.R;
  const int SS = KS ? KS : a.S;

  // pointwise weight chunk loader: thread → (k row, n col) pairs of a 16x32 chunk
  auto load_b = [&](int chunk, int buf) {
#pragma unroll
    for (int i = 0; i < (SEP_BK * SEP_BN) / SEP_THREADS; ++i) {
      const int e = tid + i * SEP_THREADS;
      const int kk = e % SEP_BK, nn = e / SEP_BK;
      const int c = chunk * SEP_BK + kk, n = n0 + nn;
      const bool ok = c < a.C && n < a.K;
      cp4(&Bs[(buf * SEP_BK + kk) * SEP_BN + nn], a.w_pw + (ok ? (size_t)n * a.C + c : 0), ok);
    }
    cp_commit();
  };
  // weights are constant: request every chunk before waiting on the producer,
  // so the whole pointwise operand is one round trip hidden behind the depthwise
  const int chunks = Cp / SEP_BK;
#pragma unroll 1
  for (int ch = 0; ch < chunks; ++ch) load_b(ch, ch);
  pdl_trigger();
  pdl_wait();

  // ---- depthwise into D[c][px] (zero for padded rows / pixels past M) ----
  constexpr int V = VEC ? 4 : 1;
  const int cgroups = Cp / V;
#pragma unroll 1
  for (int e = tid; e < SEP_BM * cgroups; e += SEP_THREADS) {
    const int cg = e % cgroups;
    const int px = e / cgroups;
    const int c = cg * V;
    const int m = m0 + px;
    float acc[V];
#pragma unroll
    for (int j = 0; j < V; ++j) acc[j] = 0.f;
    if (m < a.M && c < a.C) {
      const int q = m % a.Q;
      const int t = m / a.Q;
      const int p = t % a.P, nb = t / a.P;
      const float* base = a.in + nb * a.in_sn + c * a.in_sc;
      const int ih0 = p * a.sh - a.ph, iw0 = q * a.sw - a.pw;
#pragma unroll
      for (int r = 0; r < (KS ? KS : 1); ++r) {
#pragma unroll 1
        for (int r2 = 0; r2 < (KS ? 1 : RR); ++r2) {
          const int rr = KS ? r : r2;
          const int ih = ih0 + rr;
          const bool rok = (unsigned)ih < (unsigned)a.H;
#pragma unroll
          for (int s = 0; s < (KS ? KS : 1); ++s) {
#pragma unroll 1
            for (int s2 = 0; s2 < (KS ? 1 : SS); ++s2) {
              const int ss = KS ? s : s2;
              const int iw = iw0 + ss;
              const bool ok = rok && (unsigned)iw < (unsigned)a.W;
              const float* src = base + (ok ? ih * a.in_sh + iw * a.in_sw : 0);
              const float* wsrc = a.w_dw + (rr * SS + ss) * a.C + c;
              if constexpr (VEC) {
                float4 x = __ldg(reinterpret_cast<const float4*>(src));
                const float4 w = __ldg(reinterpret_cast<const float4*>(wsrc));
                if (a.pre_relu) {
                  x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
                }
                const float msk = ok ? 1.f : 0.f;
                acc[0] = fmaf(x.x * msk, w.x, acc[0]);
                acc[1] = fmaf(x.y * msk, w.y, acc[1]);
                acc[2] = fmaf(x.z * msk, w.z, acc[2]);
                acc[3] = fmaf(x.w * msk, w.w, acc[3]);
              } else {
                float x = __ldg(src);
                if (a.pre_relu) x = fmaxf(x, 0.f);
                acc[0] = fmaf(ok ? x : 0.f, __ldg(wsrc), acc[0]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float v = acc[j] + (a.b_dw ? a.b_dw[c + j] : 0.f);
        acc[j] = apply_act(v, a.dw_act);
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j) D[(c + j) * SEP_BM + px] = acc[j];
  }

  // ---- pointwise GEMM: out[px][n] = sum_c D[c][px] * W[n][c] ----
  const int ty = tid / (SEP_BN / 2);  // 0..15 → output row (pixel) ty
  const int tx = tid % (SEP_BN / 2);  // 0..15 → cols tx*2, tx*2+1
  float o0 = 0.f, o1 = 0.f;
  cp_wait<0>();
  __syncthreads();  // D complete and all weight chunks landed
#pragma unroll 1
  for (int ch = 0; ch < chunks; ++ch) {
    const float* bt = Bs + ch * SEP_BK * SEP_BN + tx * 2;
    const float* at = D + ch * SEP_BK * SEP_BM + ty;
#pragma unroll 4
    for (int k = 0; k < SEP_BK; ++k) {
      const float av = at[k * SEP_BM];
      const float2 bv = *reinterpret_cast<const float2*>(bt + k * SEP_BN);
      o0 = fmaf(av, bv.x, o0);
      o1 = fmaf(av, bv.y, o1);
    }
  }
  __syncthreads();

  // ---- epilogue (tile through smem, rolled, coalesced along channels) ----
  float* part = Bs;  // [SEP_BM][SEP_BN] fits in the weight buffer (>= 16 x 32)
  part[ty * SEP_BN + tx * 2] = o0;
  part[ty * SEP_BN + tx * 2 + 1] = o1;
  __syncthreads();
#pragma unroll 2
  for (int e = tid; e < SEP_BM * SEP_BN; e += SEP_THREADS) {
    const int m = m0 + e / SEP_BN, n = n0 + e % SEP_BN;
    if (m >= a.M || n >= a.K) continue;
    const int q = m % a.Q;
    const int t = m / a.Q;
    const int pp = t % a.P, nb = t / a.P;
    float v = part[e] + (a.b_pw ? a.b_pw[n] : 0.f);
    if (a.has_res) v += a.res[nb * a.res_sn + pp * a.res_sh + q * a.res_sw + n * a.res_sc];
    a.out[nb * a.out_sn + pp * a.out_sh + q * a.out_sw + n * a.out_sc] = apply_act(v, a.act);
  }
}

static SepArgs sep_args(const sw_op_desc& op) {
  const int64_t* p = op.params;
  SepArgs a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.w_pw = reinterpret_cast<const float*>(op.ptrs[PT_W]);
  a.b_pw = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.w_dw = reinterpret_cast<const float*>(op.ptrs[PT_WS]);
  a.b_dw = reinterpret_cast<const float*>(op.ptrs[PT_DW_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K];
  a.R = (int)p[SP_R]; a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.dw_act = (int)p[SP_DW_ACT];
  a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.in_sn = (int)p[SP_IN_SN]; a.in_sh = (int)p[SP_IN_SH]; a.in_sw = (int)p[SP_IN_SW]; a.in_sc = (int)p[SP_IN_SC];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  a.M = a.N * a.P * a.Q;
  a.vec = (a.C % 4 == 0) && a.in_sc == 1 && a.in_sn % 4 == 0 && a.in_sh % 4 == 0 && a.in_sw % 4 == 0 &&
          aligned16(op.ptrs[PT_IN]) && aligned16(op.ptrs[PT_WS]);
  return a;
}

size_t sepconv_smem_bytes(int C) {
  const int cp = (C + SEP_BK - 1) / SEP_BK * SEP_BK;
  return 4 * ((size_t)cp * SEP_BM + (size_t)cp * SEP_BN);
}

template <bool VEC>
static int launch_sep_ks(const SepArgs& a, int ks, dim3 grid, size_t smem, cudaStream_t st) {
  switch (ks) {
    case 3: return (int)launch_k(sepconv_kernel<3, VEC>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 5: return (int)launch_k(sepconv_kernel<5, VEC>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 7: return (int)launch_k(sepconv_kernel<7, VEC>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    default: return (int)launch_k(sepconv_kernel<0, VEC>, grid, dim3(SEP_THREADS), smem, st, 1, a);
  }
}

int launch_sepconv(const sw_op_desc& op, void* stream) {
  SepArgs a = sep_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  const size_t smem = sepconv_smem_bytes(a.C);
  if (smem > 227 * 1024) return (int)cudaErrorInvalidValue;
  dim3 grid((unsigned)cdiv(a.M, SEP_BM), (unsigned)cdiv(a.K, SEP_BN));
  const int ks = (a.R == a.S && (a.R == 3 || a.R == 5 || a.R == 7)) ? a.R : 0;
  return a.vec ? launch_sep_ks<true>(a, ks, grid, smem, st) : launch_sep_ks<false>(a, ks, grid, smem, st);
}

void init_sep_kernels() {
  const int maxb = 227 * 1024;
  void (*fns[])(SepArgs) = {sepconv_kernel<3, true>, sepconv_kernel<5, true>, sepconv_kernel<7, true>,
                            sepconv_kernel<0, true>, sepconv_kernel<3, false>, sepconv_kernel<5, false>,
                            sepconv_kernel<7, false>, sepconv_kernel<0, false>};
  for (auto f : fns) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, maxb);
}

}  // namespace sw
