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
#include "conv_args.cuh"

namespace cg = cooperative_groups;

namespace sw {

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

// BM x BN output tile computed by 256 threads with a TM x TN micro-tile each,
// BK = 16, 4-stage cp.async (LDGSTS) pipeline.  Batch-1 layers are tiny, so
// the variants are "wide and shallow": 8 warps per CTA and as little serial
// work per warp as possible (ncu: a 2-warp CTA spent 4.4K dependent
// instructions per warp at IPC 0.26).  Out-of-range taps are zero-filled by
// cp.async; the epilogue is one smem-staged rolled loop shared with the
// split-K DSMEM reduction, keeping the code an SM must fetch small.
template <int BM, int BN, int TM, int TN, bool PRE>
__global__ void __launch_bounds__(256)
conv_simt_kernel(ConvArgs a) {
  constexpr int BK = 16;
  constexpr int STAGES = 8;  // deep ring: a batch-1 K slice is in flight at once
  constexpr int NT = 256;
  static_assert((BM / TM) * (BN / TN) == NT, "256 threads per CTA");
  constexpr int A_PER = (BM * BK + NT - 1) / NT;
  constexpr int B_PER = (BN * BK + NT - 1) / NT;
  constexpr int PAD = 4;
  extern __shared__ __align__(16) float smem[];
  float* As = smem;                                // [STAGES][BK][BM+PAD]
  float* Bs = smem + STAGES * BK * (BM + PAD);     // [STAGES][BK][BN+PAD]

  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int kk = tid % BK;
  const int row = tid / BK;  // 0..15, + i * 16

  const int ksteps_total = (a.Kdim + BK - 1) / BK;
  const int per = (ksteps_total + a.split - 1) / a.split;
  const int ks_begin = blockIdx.z * per;
  const int nsteps = max(0, min(ksteps_total, ks_begin + per) - ks_begin);

  int a_base[A_PER], a_ih[A_PER], a_iw[A_PER];
#pragma unroll
  for (int i = 0; i < A_PER; ++i) {
    const int mm = row + i * 16;
    const int m = m0 + mm;
    const int q = m % a.Q;
    const int t = m / a.Q;
    a_base[i] = (t / a.P) * (int)a.in_sn;
    a_ih[i] = (m < a.M && mm < BM) ? (t % a.P) * a.sh - a.ph : -(1 << 28);
    a_iw[i] = q * a.sw - a.pw;
  }
  const int in_sh = (int)a.in_sh, in_sw = (int)a.in_sw, in_sc = (int)a.in_sc;

  // A (activations) and B (weights) halves of one ring stage; the weights of
  // the prologue stages are constants and go out before the PDL wait.
  auto issue_a = [&](int kstep, int buf) {
    const int k = kstep * BK + kk;
    const bool kin = k < a.Kdim;
    const int c = k % a.C;
    const int rs = k / a.C;
    const int s = rs % a.S;
    const int r = rs / a.S;
    float* as = As + (buf * BK + kk) * (BM + PAD) + row;
#pragma unroll
    for (int i = 0; i < A_PER; ++i) {
      if (row + i * 16 >= BM) break;
      const int ih = a_ih[i] + r, iw = a_iw[i] + s;
      const bool ok = kin && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
      cp_async4(as + i * 16, a.in + (ok ? a_base[i] + ih * in_sh + iw * in_sw + c * in_sc : 0), ok);
    }
  };
  auto issue_b = [&](int kstep, int buf) {
    const int k = kstep * BK + kk;
    const bool kin = k < a.Kdim;
    float* bs = Bs + (buf * BK + kk) * (BN + PAD) + row;
#pragma unroll
    for (int i = 0; i < B_PER; ++i) {
      if (row + i * 16 >= BN) break;
      const int n = n0 + row + i * 16;
      const bool ok = kin && n < a.K;
      cp_async4(bs + i * 16, a.w + (ok ? (size_t)n * a.Kdim + k : 0), ok);
    }
  };

  const int ty = tid / (BN / TN);
  const int tx = tid % (BN / TN);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  probe_begin();
#pragma unroll 1
  for (int st = 0; st < STAGES - 1; ++st)
    if (st < nsteps) issue_b(ks_begin + st, st);  // joins commit group 0
  pdl_trigger();
  probe_pt(1);
  pdl_wait();
  probe_pt(2);
#pragma unroll 1
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nsteps) issue_a(ks_begin + st, st);
    cp_async_commit();
  }
#pragma unroll 1
  for (int it = 0; it < nsteps; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // tile `it` landed for everyone; buffer (it-1)%STAGES is free
    if (it == 0) probe_pt(3);
    const int nxt = it + STAGES - 1;
    if (nxt < nsteps) {
      issue_a(ks_begin + nxt, nxt % STAGES);
      issue_b(ks_begin + nxt, nxt % STAGES);
    }
    cp_async_commit();
    const float* at = As + (it % STAGES) * BK * (BM + PAD) + ty * TM;
    const float* bt = Bs + (it % STAGES) * BK * (BN + PAD) + tx * TN;
#pragma unroll 4
    for (int k2 = 0; k2 < BK; ++k2) {
      float ai[TM], bj[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) ai[i] = PRE ? fmaxf(at[k2 * (BM + PAD) + i], 0.f) : at[k2 * (BM + PAD) + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bj[j] = bt[k2 * (BN + PAD) + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(ai[i], bj[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  probe_pt(4);

  float* part = smem;  // [BM][BN], reuses the operand buffers
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) part[(ty * TM + i) * BN + tx * TN + j] = acc[i][j];
  cg::cluster_group cluster = cg::this_cluster();
  tile_epilogue<BM, BN, NT>(a.epi, part, m0, n0, a.split, cluster);
  probe_end();
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

struct SimtCfg {
  int bm, bn;
  void (*fn[2])(ConvArgs);
};

#define SW_SIMT_CFG(BM, BN, TM, TN) \
  { BM, BN, { conv_simt_kernel<BM, BN, TM, TN, false>, conv_simt_kernel<BM, BN, TM, TN, true> } }

// variant → tile; all 256 threads.  8 = GEMV (M <= 8, 1x1).
static const SimtCfg kSimt[] = {
    SW_SIMT_CFG(64, 64, 4, 4),   // 0
    SW_SIMT_CFG(32, 64, 2, 4),   // 1
    SW_SIMT_CFG(32, 32, 2, 2),   // 2
    SW_SIMT_CFG(128, 64, 8, 4),  // 3
    SW_SIMT_CFG(16, 32, 1, 2),   // 4
    SW_SIMT_CFG(16, 64, 1, 4),   // 5
    SW_SIMT_CFG(16, 16, 1, 1),   // 6
    SW_SIMT_CFG(64, 32, 4, 2),   // 7
};
constexpr int kNumSimt = sizeof(kSimt) / sizeof(kSimt[0]);

// Direct convolution for thin layers (variant 9): K <= 32 output channels and
// R*S*C <= 576 (NASNet's stem: 3x3 s2 3→32 on the NCHW image, 1x1 32→11 /
// 44→22 at 111² / 56²).  A GEMM tile would be mostly padding there and the
// layer is memory bound: one thread per output pixel keeps all K
// accumulators in registers, the filter sits in shared memory as [rsc][K]
// (warp-uniform broadcast reads), and each pixel's outputs leave as one
// contiguous run (float4 when the layout allows).
// Dense pointwise layer with few input channels: the CTA's 128 input pixel
// rows are one contiguous block, staged into shared memory by coalesced
// float4 loads (a thread reading its own 128-B pixel row made every load
// instruction touch 32 lines).  Row stride DX floats, DX / 4 odd: the per-row
// float4 reads of a warp are conflict-free.
__host__ __device__ inline bool direct_stage_in(const ConvArgs& a) {
  return a.R == 1 && a.S == 1 && a.sh == 1 && a.sw == 1 && a.ph == 0 && a.pw == 0 && a.in_sc == 1 &&
         (a.C & 3) == 0 && a.C <= 32 && a.in_sw == a.C && a.in_sh == (int64_t)a.W * a.C &&
         a.in_sn == (int64_t)a.H * a.W * a.C && (reinterpret_cast<uintptr_t>(a.in) & 15) == 0;
}
__host__ __device__ inline int direct_stage_ld(int C) { return ((C / 4 + 1) & 1) ? C + 4 : C + 8; }

template <int KB, int KS>
__global__ void __launch_bounds__(128) conv_direct_kernel(ConvArgs a) {
  extern __shared__ float wsm[];  // [Kdim][KB] + bias[KB]
  const int tid = threadIdx.x;
  for (int e = tid; e < a.Kdim * KB; e += blockDim.x) {
    const int k = e % KB, j = e / KB;  // j = (r, s, c) in the [K][R][S][C] weight order
    wsm[e] = k < a.K ? __ldg(a.w + (int64_t)k * a.Kdim + j) : 0.f;
  }
  float* bsm = wsm + a.Kdim * KB;
  if (tid < KB) bsm[tid] = (a.bias && tid < a.K) ? __ldg(a.bias + tid) : 0.f;
  pdl_trigger();
  pdl_wait();
  __syncthreads();
  const int m0 = blockIdx.x * blockDim.x;
  const int m = min(m0 + tid, a.M - 1);  // tail threads recompute the last pixel (not stored)
  const int q = m % a.Q;
  const int t = m / a.Q;
  const int p = t % a.P, nb = t / a.P;
  float acc[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) acc[k] = bsm[k];
  const int ih0 = p * a.sh - a.ph, iw0 = q * a.sw - a.pw;
  const float* base = a.in + nb * a.in_sn;
  const bool cvec = a.in_sc == 1 && (a.C & 3) == 0;
  if constexpr (KS > 0) {
    // fixed k x k window, channel by channel: the KS*KS tap loads of a channel
    // are issued together from clamped addresses and masked (branch-free),
    // so a thread waits one memory round trip per channel, not per tap
#pragma unroll 1
    for (int c = 0; c < a.C; ++c) {
      float x[KS * KS];
#pragma unroll
      for (int r = 0; r < KS; ++r)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const int ih = ih0 + r, iw = iw0 + s;
          const bool ok = (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
          const float v = __ldg(base + (ok ? ih * a.in_sh + iw * a.in_sw : 0) + c * a.in_sc);
          x[r * KS + s] = ok ? (a.pre_relu ? fmaxf(v, 0.f) : v) : 0.f;
        }
#pragma unroll
      for (int r = 0; r < KS; ++r)
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const float4* w4 = reinterpret_cast<const float4*>(wsm + ((r * KS + s) * a.C + c) * KB);
          const float xv = x[r * KS + s];
#pragma unroll
          for (int k4 = 0; k4 < KB / 4; ++k4) {
            const float4 w = w4[k4];  // one 16-B shared load per 4 FMAs
            acc[4 * k4] = fmaf(xv, w.x, acc[4 * k4]);
            acc[4 * k4 + 1] = fmaf(xv, w.y, acc[4 * k4 + 1]);
            acc[4 * k4 + 2] = fmaf(xv, w.z, acc[4 * k4 + 2]);
            acc[4 * k4 + 3] = fmaf(xv, w.w, acc[4 * k4 + 3]);
          }
        }
    }
  } else if (direct_stage_in(a)) {
    float* xs = bsm + KB + 128 * (KB + 4);  // [128][DX], past the epilogue tile
    const int DX = direct_stage_ld(a.C);
    const int c4n = a.C / 4;
    for (int e = tid; e < 128 * c4n; e += 128) {
      const int px = e / c4n, ch = e - px * c4n;
      const int mm = min(m0 + px, a.M - 1);
      float4 v = __ldg(reinterpret_cast<const float4*>(a.in + (int64_t)mm * a.C) + ch);
      if (a.pre_relu) {
        v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
      }
      *reinterpret_cast<float4*>(&xs[px * DX + ch * 4]) = v;
    }
    __syncthreads();
    const float* xr = xs + tid * DX;
#pragma unroll 4
    for (int c = 0; c < a.C; c += 4) {
      const float4 x = *reinterpret_cast<const float4*>(xr + c);
      const float4* w4 = reinterpret_cast<const float4*>(wsm + c * KB);
      constexpr int G = KB / 4;
#pragma unroll
      for (int k4 = 0; k4 < G; ++k4) {
        const float4 w0 = w4[k4], w1 = w4[G + k4], w2 = w4[2 * G + k4], w3 = w4[3 * G + k4];
        acc[4 * k4] = fmaf(x.x, w0.x, fmaf(x.y, w1.x, fmaf(x.z, w2.x, fmaf(x.w, w3.x, acc[4 * k4]))));
        acc[4 * k4 + 1] = fmaf(x.x, w0.y, fmaf(x.y, w1.y, fmaf(x.z, w2.y, fmaf(x.w, w3.y, acc[4 * k4 + 1]))));
        acc[4 * k4 + 2] = fmaf(x.x, w0.z, fmaf(x.y, w1.z, fmaf(x.z, w2.z, fmaf(x.w, w3.z, acc[4 * k4 + 2]))));
        acc[4 * k4 + 3] = fmaf(x.x, w0.w, fmaf(x.y, w1.w, fmaf(x.z, w2.w, fmaf(x.w, w3.w, acc[4 * k4 + 3]))));
      }
    }
  } else {
#pragma unroll 1
    for (int r = 0; r < a.R; ++r) {
      const int ih = ih0 + r;
      if ((unsigned)ih >= (unsigned)a.H) continue;
#pragma unroll 1
      for (int s = 0; s < a.S; ++s) {
        const int iw = iw0 + s;
        if ((unsigned)iw >= (unsigned)a.W) continue;
        const float* src = base + ih * a.in_sh + iw * a.in_sw;
        const float* wr = wsm + ((r * a.S + s) * a.C) * KB;
        if (cvec) {
          // 16 channels of loads in flight per step
#pragma unroll 1
          for (int c0 = 0; c0 < a.C; c0 += 16) {
            float4 xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              xv[u] = c0 + 4 * u < a.C ? __ldg(reinterpret_cast<const float4*>(src + c0 + 4 * u))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = c0 + 4 * u;
              if (c >= a.C) break;
              float4 x = xv[u];
              if (a.pre_relu) {
                x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
              }
              const float4* w4 = reinterpret_cast<const float4*>(wr + c * KB);
              constexpr int G = KB / 4;
#pragma unroll
              for (int k4 = 0; k4 < G; ++k4) {
                const float4 w0 = w4[k4], w1 = w4[G + k4], w2 = w4[2 * G + k4], w3 = w4[3 * G + k4];
                acc[4 * k4] = fmaf(x.x, w0.x, fmaf(x.y, w1.x, fmaf(x.z, w2.x, fmaf(x.w, w3.x, acc[4 * k4]))));
                acc[4 * k4 + 1] = fmaf(x.x, w0.y, fmaf(x.y, w1.y, fmaf(x.z, w2.y, fmaf(x.w, w3.y, acc[4 * k4 + 1]))));
                acc[4 * k4 + 2] = fmaf(x.x, w0.z, fmaf(x.y, w1.z, fmaf(x.z, w2.z, fmaf(x.w, w3.z, acc[4 * k4 + 2]))));
                acc[4 * k4 + 3] = fmaf(x.x, w0.w, fmaf(x.y, w1.w, fmaf(x.z, w2.w, fmaf(x.w, w3.w, acc[4 * k4 + 3]))));
              }
            }
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < a.C; ++c) {
            float x = __ldg(src + c * a.in_sc);
            if (a.pre_relu) x = fmaxf(x, 0.f);
            const float4* w4 = reinterpret_cast<const float4*>(wr + c * KB);
#pragma unroll
            for (int k4 = 0; k4 < KB / 4; ++k4) {
              const float4 w = w4[k4];
              acc[4 * k4] = fmaf(x, w.x, acc[4 * k4]);
              acc[4 * k4 + 1] = fmaf(x, w.y, acc[4 * k4 + 1]);
              acc[4 * k4 + 2] = fmaf(x, w.z, acc[4 * k4 + 2]);
              acc[4 * k4 + 3] = fmaf(x, w.w, acc[4 * k4 + 3]);
            }
          }
        }
      }
    }
  }
  float* o = a.out + nb * a.out_sn + p * a.out_sh + q * a.out_sw;
  const float* rp = a.has_res ? a.res + nb * a.res_sn + p * a.res_sh + q * a.res_sw : nullptr;
  if (a.epi.vec && (a.K & 3) == 0) {
    // stage the CTA's [128 px][K] tile in smem, then store it with consecutive
    // threads on consecutive 16-byte chunks (a per-thread K-float run would
    // make every store instruction touch 32 different lines)
    float* tile = bsm + KB;  // [128][KB + 4]
    constexpr int LD = KB + 4;
#pragma unroll
    for (int k = 0; k < KB; ++k) tile[tid * LD + k] = acc[k];
    __syncthreads();
    const int npx = min(128, a.M - m0);
    const int g4 = a.K / 4;
    for (int e = tid; e < npx * g4; e += 128) {
      const int px = e / g4, k = (e % g4) * 4;
      const int mm = m0 + px;
      const int qq = mm % a.Q, tt = mm / a.Q;
      const int pp = tt % a.P, nn = tt / a.P;
      float4 v = *reinterpret_cast<const float4*>(&tile[px * LD + k]);
      if (a.has_res)
        v = f4add(v, *reinterpret_cast<const float4*>(a.res + nn * a.res_sn + pp * a.res_sh + qq * a.res_sw + k));
      *reinterpret_cast<float4*>(a.out + nn * a.out_sn + pp * a.out_sh + qq * a.out_sw + k) = act4(v, a.act);
    }
    return;
  }
  if (m0 + tid >= a.M) return;
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    if (k >= a.K) break;
    float v = acc[k];
    if (rp) v += rp[k * a.res_sc];
    o[k * a.out_sc] = apply_act(v, a.act);
  }
}

static size_t simt_smem_bytes(int bm, int bn) {
  const size_t tile = 8 * 16 * (size_t)(bm + 4) + 8 * 16 * (size_t)(bn + 4);  // STAGES * BK * (B? + PAD)
  const size_t part = (size_t)bm * bn;
  return 4 * (tile > part ? tile : part);
}

void init_simt_kernels() {
  cudaFuncSetAttribute(conv_direct_kernel<8, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (576 * 8 + 8 + 128 * (8 + 4) + 128 * 72) * 4);
  cudaFuncSetAttribute(conv_direct_kernel<16, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (576 * 16 + 16 + 128 * (16 + 4) + 128 * 72) * 4);
  cudaFuncSetAttribute(conv_direct_kernel<32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (576 * 32 + 32 + 128 * (32 + 4) + 128 * 72) * 4);
  cudaFuncSetAttribute(conv_direct_kernel<8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (576 * 8 + 8 + 128 * (8 + 4) + 128 * 72) * 4);
  cudaFuncSetAttribute(conv_direct_kernel<16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (576 * 16 + 16 + 128 * (16 + 4) + 128 * 72) * 4);
  cudaFuncSetAttribute(conv_direct_kernel<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (576 * 32 + 32 + 128 * (32 + 4) + 128 * 72) * 4);
  for (int i = 0; i < kNumSimt; ++i)
    for (int j = 0; j < 2; ++j)
    {
      cudaFuncSetAttribute(kSimt[i].fn[j], cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)simt_smem_bytes(kSimt[i].bm, kSimt[i].bn));
      // split-K clusters of 16 (weight-streaming layers at batch 1 want >8 CTAs per tile)
      cudaFuncSetAttribute(kSimt[i].fn[j], cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
}

int launch_conv(const sw_op_desc& op, void* stream) {
  ConvArgs a = conv_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  if (op.variant == 8) {
    if (a.M > 8 || a.R != 1 || a.S != 1) return (int)cudaErrorInvalidValue;
    int blocks = (int)cdiv((int64_t)a.K * 32, 256);
    return (int)launch_k(conv_gemv_kernel<8>, dim3(blocks), dim3(256), 0, st, 1, a);
  }
  if (op.variant == 9) {
    if (a.K > 32 || a.Kdim > 576 || a.split != 1) return (int)cudaErrorInvalidValue;
    const int kb = a.K <= 8 ? 8 : (a.K <= 16 ? 16 : 32);
    size_t smem = ((size_t)a.Kdim * kb + kb + 128 * (size_t)(kb + 4)) * sizeof(float);
    if (direct_stage_in(a)) smem += 128 * (size_t)direct_stage_ld(a.C) * sizeof(float);
    const dim3 grid((unsigned)cdiv(a.M, 128));
    const bool k3 = a.R == 3 && a.S == 3;
    if (kb == 8)
      return (int)(k3 ? launch_k(conv_direct_kernel<8, 3>, grid, dim3(128), smem, st, 1, a)
                      : launch_k(conv_direct_kernel<8, 0>, grid, dim3(128), smem, st, 1, a));
    if (kb == 16)
      return (int)(k3 ? launch_k(conv_direct_kernel<16, 3>, grid, dim3(128), smem, st, 1, a)
                      : launch_k(conv_direct_kernel<16, 0>, grid, dim3(128), smem, st, 1, a));
    return (int)(k3 ? launch_k(conv_direct_kernel<32, 3>, grid, dim3(128), smem, st, 1, a)
                    : launch_k(conv_direct_kernel<32, 0>, grid, dim3(128), smem, st, 1, a));
  }
  if (op.variant >= 16) return launch_conv_pw(op, op.variant - 16, stream);  // conv1x1.cu (TMA)
  if (op.variant < 0 || op.variant >= kNumSimt) return (int)cudaErrorInvalidValue;
  const SimtCfg& c = kSimt[op.variant];
  dim3 grid((unsigned)cdiv(a.M, c.bm), (unsigned)cdiv(a.K, c.bn), (unsigned)a.split);
  return (int)launch_k(c.fn[a.pre_relu ? 1 : 0], grid, dim3(256), simt_smem_bytes(c.bm, c.bn), st,
                       (unsigned)a.split, a);
}

}  // namespace sw
