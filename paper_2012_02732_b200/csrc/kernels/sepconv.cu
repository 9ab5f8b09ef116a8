// Fused separable convolution: depthwise k x k → (bias, act) → pointwise 1x1
// → (bias, residual, act) in ONE kernel (NASNet sep-convs, MobileNetV2
// dw → project).  The depthwise result for the CTA's pixel tile never leaves
// shared memory, and the graph loses one node per separable conv — at batch 1
// the graph executor issues roughly one kernel node per microsecond
// (tools/microbench.cu), so node count is latency.
//
// CTA = 256 threads, tile = BM output pixels x BN output channels (variants
// autotuned at prepare; a small BN means more CTAs but recomputes the
// depthwise tile per column block, a large BN the opposite):
//   1. cp.async of the pointwise weights (stored [C][K]) the tile needs and of the whole
//      depthwise filter, issued before the PDL wait (constants);
//   2. depthwise for all C_in channels of the BM pixels into smem D[c][px]
//      (branch-free unrolled taps, 128-bit NHWC loads, filter from smem);
//   3. pointwise GEMM D^T x W, TM x TN micro-tile per thread;
//   4. shared float4 tile epilogue (bias, residual, activation, strided store).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sw {

namespace {

constexpr int SEP_BK = 16;  // channel padding granule
constexpr int SEP_THREADS = 256;

struct SepArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w_pw;   // [K][C]
  const float* __restrict__ b_pw;   // [K] or null
  const float* __restrict__ w_dw;   // [R][S][C]
  const float* __restrict__ b_dw;   // [C] or null
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, dw_act, pre_relu, has_res, M, vec, wvec;
  int in_sn, in_sh, in_sw, in_sc;
  Epi epi;
};

__device__ __forceinline__ void cp4(float* dst, const float* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp16(float* dst, const float* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

}  // namespace

template <int KS, bool VEC, int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(SEP_THREADS) sepconv_kernel(SepArgs a) {
  static_assert((BM / TM) * (BN / TN) == SEP_THREADS, "256 threads");
  extern __shared__ __align__(16) float smem[];
  const int Cp = (a.C + SEP_BK - 1) / SEP_BK * SEP_BK;
  const int RR = KS ? KS : a.R;
  const int SS = KS ? KS : a.S;
  float* D = smem;                  // [BM][Cp]   depthwise tile, channels contiguous
  float* Bs = D + Cp * BM;          // [Cp][BN]   pointwise weights, columns contiguous
  float* Wd = Bs + Cp * BN;         // [RR*SS][Cp]
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;

  // constants first: the tile's pointwise columns (weights stored transposed,
  // [C][K], so the fill is coalesced and bank-conflict free) + the filter
  if (a.wvec) {
#pragma unroll 1
    for (int e = tid; e < Cp * (BN / 4); e += SEP_THREADS) {
      const int n4 = e % (BN / 4), c = e / (BN / 4);
      const int n = n0 + n4 * 4;
      const bool ok = c < a.C && n < a.K;  // K % 4 == 0: a group is all in or all out
      cp16(&Bs[c * BN + n4 * 4], a.w_pw + (ok ? (size_t)c * a.K + n : 0), ok);
    }
  } else {
#pragma unroll 1
    for (int e = tid; e < Cp * BN; e += SEP_THREADS) {
      const int nn = e % BN, c = e / BN;
      const int n = n0 + nn;
      const bool ok = c < a.C && n < a.K;
      cp4(&Bs[c * BN + nn], a.w_pw + (ok ? (size_t)c * a.K + n : 0), ok);
    }
  }
  if (VEC) {
#pragma unroll 1
    for (int e = tid; e < RR * SS * (Cp / 4); e += SEP_THREADS) {
      const int cg4 = e % (Cp / 4), tap = e / (Cp / 4);
      const bool ok = cg4 * 4 < a.C;
      cp16(&Wd[tap * Cp + cg4 * 4], a.w_dw + (ok ? tap * a.C + cg4 * 4 : 0), ok);
    }
  } else {
#pragma unroll 1
    for (int e = tid; e < RR * SS * Cp; e += SEP_THREADS) {
      const int c = e % Cp, tap = e / Cp;
      const bool ok = c < a.C;
      cp4(&Wd[tap * Cp + c], a.w_dw + (ok ? tap * a.C + c : 0), ok);
    }
  }
  cp_commit();
  pdl_trigger();
  pdl_wait();
  cp_wait_all();
  __syncthreads();

  // ---- depthwise into D[px][c] (zero for padded channels / pixels past M) ----
  constexpr int V = VEC ? 4 : 1;
  const int cgroups = Cp / V;
#pragma unroll 1
  for (int e = tid; e < BM * cgroups; e += SEP_THREADS) {
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
              const float* wsrc = &Wd[(rr * SS + ss) * Cp + c];
              if constexpr (VEC) {
                float4 x = __ldg(reinterpret_cast<const float4*>(src));
                const float4 w = *reinterpret_cast<const float4*>(wsrc);
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
                acc[0] = fmaf(ok ? x : 0.f, *wsrc, acc[0]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < V; ++j) acc[j] = apply_act(acc[j] + (a.b_dw ? a.b_dw[c + j] : 0.f), a.dw_act);
    }
    if constexpr (VEC) {
      *reinterpret_cast<float4*>(&D[px * Cp + c]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
      D[px * Cp + c] = acc[0];
    }
  }
  __syncthreads();

  // ---- pointwise GEMM: out[px][n] = sum_c D[c][px] * W[n][c] ----
  const int ty = tid / (BN / TN);
  const int tx = tid % (BN / TN);
  float o[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) o[i][j] = 0.f;
  const float* at = D + ty * TM * Cp;
  const float* bt = Bs + tx * TN;
#pragma unroll 4
  for (int k = 0; k < Cp; ++k) {
    float av[TM], bv[TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) av[i] = at[i * Cp + k];
#pragma unroll
    for (int j = 0; j < TN; ++j) bv[j] = bt[k * BN + j];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) o[i][j] = fmaf(av[i], bv[j], o[i][j]);
  }
  __syncthreads();  // D / Bs reads done; reuse D as the output tile

  float* part = D;  // [BM][BN] ≤ Cp*BM + Cp*BN floats
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) part[(ty * TM + i) * BN + tx * TN + j] = o[i][j];
  cg::cluster_group cluster = cg::this_cluster();
  tile_epilogue<BM, BN, SEP_THREADS>(a.epi, part, m0, n0, 1, cluster);
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
  a.M = a.N * a.P * a.Q;
  a.vec = (a.C % 4 == 0) && a.in_sc == 1 && a.in_sn % 4 == 0 && a.in_sh % 4 == 0 && a.in_sw % 4 == 0 &&
          aligned16(op.ptrs[PT_IN]) && aligned16(op.ptrs[PT_WS]);
  a.wvec = (a.K % 4 == 0) && aligned16(op.ptrs[PT_W]);
  const int64_t osn = p[SP_OUT_SN], osh = p[SP_OUT_SH], osw = p[SP_OUT_SW], osc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  const int64_t rsn = p[SP_RES_SN], rsh = p[SP_RES_SH], rsw = p[SP_RES_SW], rsc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  a.epi = Epi{a.b_pw, a.res, a.out, a.M, a.K, a.P, a.Q, a.act, a.has_res, 0, osn, osh, osw, osc, rsn, rsh, rsw, rsc};
  a.epi.vec = epi_vec_ok(op.ptrs[PT_OUT], osn, osh, osw, osc, op.ptrs[PT_BIAS], a.has_res != 0, op.ptrs[PT_RES],
                         rsn, rsh, rsw, rsc) ? 1 : 0;
  return a;
}

namespace {
struct SepCfg {
  int bm, bn;
};
// variant → tile (all 256 threads)
constexpr SepCfg kSep[] = {{16, 32}, {8, 64}, {16, 64}, {32, 32}, {8, 32}, {32, 64}};
constexpr int kNumSep = sizeof(kSep) / sizeof(kSep[0]);
constexpr int kSepSmemMax = 227 * 1024;
}  // namespace

static size_t sep_smem(int C, int R, int S, int bm, int bn) {
  const size_t cp = (size_t)(C + SEP_BK - 1) / SEP_BK * SEP_BK;
  const size_t body = cp * bm + cp * bn + (size_t)R * S * cp;
  const size_t part = (size_t)bm * bn;  // epilogue tile reuses the same buffer
  return 4 * (body > part ? body : part);
}

template <int KS, bool VEC>
static cudaError_t launch_sep_v(int v, const SepArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  switch (v) {
    case 1: return launch_k(sepconv_kernel<KS, VEC, 8, 64, 1, 2>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 2: return launch_k(sepconv_kernel<KS, VEC, 16, 64, 1, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 3: return launch_k(sepconv_kernel<KS, VEC, 32, 32, 2, 2>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 4: return launch_k(sepconv_kernel<KS, VEC, 8, 32, 1, 1>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 5: return launch_k(sepconv_kernel<KS, VEC, 32, 64, 2, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    default: return launch_k(sepconv_kernel<KS, VEC, 16, 32, 1, 2>, grid, dim3(SEP_THREADS), smem, st, 1, a);
  }
}

template <bool VEC>
static cudaError_t launch_sep_ks(int ks, int v, const SepArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  switch (ks) {
    case 3: return launch_sep_v<3, VEC>(v, a, grid, smem, st);
    case 5: return launch_sep_v<5, VEC>(v, a, grid, smem, st);
    case 7: return launch_sep_v<7, VEC>(v, a, grid, smem, st);
    default: return launch_sep_v<0, VEC>(v, a, grid, smem, st);
  }
}

int launch_sepconv(const sw_op_desc& op, void* stream) {
  SepArgs a = sep_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  const int v = (op.variant >= 0 && op.variant < kNumSep) ? op.variant : 0;
  const size_t smem = sep_smem(a.C, a.R, a.S, kSep[v].bm, kSep[v].bn);
  if (smem > (size_t)kSepSmemMax) return (int)cudaErrorInvalidValue;  // the autotuner skips it
  dim3 grid((unsigned)cdiv(a.M, kSep[v].bm), (unsigned)cdiv(a.K, kSep[v].bn));
  const int ks = (a.R == a.S && (a.R == 3 || a.R == 5 || a.R == 7)) ? a.R : 0;
  return (int)(a.vec ? launch_sep_ks<true>(ks, v, a, grid, smem, st) : launch_sep_ks<false>(ks, v, a, grid, smem, st));
}

template <int KS, bool VEC>
static void init_sep_ks() {
  cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 16, 32, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 8, 64, 1, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 16, 64, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 32, 32, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 8, 32, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 32, 64, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
}

void init_sep_kernels() {
  init_sep_ks<3, true>(); init_sep_ks<5, true>(); init_sep_ks<7, true>(); init_sep_ks<0, true>();
  init_sep_ks<3, false>(); init_sep_ks<5, false>(); init_sep_ks<7, false>(); init_sep_ks<0, false>();
}

}  // namespace sw
