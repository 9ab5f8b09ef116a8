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
//   2. depthwise for all C_in channels of the BM pixels into smem D[px][c] (rows padded by 4 floats)
//      (branch-free unrolled taps, 128-bit NHWC loads, filter from smem);
//   3. pointwise GEMM D^T x W, TM x TN micro-tile per thread;
//   4. shared float4 tile epilogue (bias, residual, activation, strided store).
#include <cooperative_groups.h>

#include "common.cuh"
#include "tma.cuh"

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

// Row-blocked depthwise (PX > 1, large batches): a thread owns PX adjacent
// output pixels of one row and slides the k-tap window along the input row in
// registers, so each input element is loaded once per row of taps instead of
// up to k times (7x7 s1: 10 loads for 4 outputs instead of 28 per tap row).
template <int KS, int SWC, int PX, int V, bool VEC>
__device__ __forceinline__ void dw_row_block(const SepArgs& a, const float* base, const float* Wd, int Cp, int c,
                                             int ih0, int iw0, float (&acc)[PX][V]) {
  constexpr int NW = (PX - 1) * SWC + KS;
#pragma unroll
  for (int r = 0; r < KS; ++r) {
    const int ih = ih0 + r;
    if ((unsigned)ih >= (unsigned)a.H) continue;
    float xr[NW][V];
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const int iw = iw0 + j;
      const bool ok = (unsigned)iw < (unsigned)a.W;
      const float* src = base + (ok ? ih * a.in_sh + iw * a.in_sw : 0);
      if constexpr (VEC) {
        float4 x = __ldg(reinterpret_cast<const float4*>(src));
        const float msk = ok ? 1.f : 0.f;
        xr[j][0] = x.x * msk; xr[j][1 % V] = x.y * msk; xr[j][2 % V] = x.z * msk; xr[j][3 % V] = x.w * msk;
      } else {
        xr[j][0] = ok ? __ldg(src) : 0.f;
      }
      if (a.pre_relu) {
#pragma unroll
        for (int v = 0; v < V; ++v) xr[j][v] = fmaxf(xr[j][v], 0.f);
      }
    }
#pragma unroll
    for (int s = 0; s < KS; ++s) {
      float w[V];
      if constexpr (VEC) {
        const float4 w4 = *reinterpret_cast<const float4*>(&Wd[(r * KS + s) * Cp + c]);
        w[0] = w4.x; w[1 % V] = w4.y; w[2 % V] = w4.z; w[3 % V] = w4.w;
      } else {
        w[0] = Wd[(r * KS + s) * Cp + c];
      }
#pragma unroll
      for (int px = 0; px < PX; ++px)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[px][v] = fmaf(xr[px * SWC + s][v], w[v], acc[px][v]);
    }
  }
}

template <int KS, bool VEC, int BM, int BN, int TM, int TN, int PX = 1>
__global__ void __launch_bounds__(SEP_THREADS, PX > 1 ? 4 : 0) sepconv_kernel(SepArgs a) {
  static_assert((BM / TM) * (BN / TN) == SEP_THREADS, "256 threads");
  extern __shared__ __align__(16) float smem[];
  const int Cp = (a.C + SEP_BK - 1) / SEP_BK * SEP_BK;
  const int RR = KS ? KS : a.R;
  const int SS = KS ? KS : a.S;
  const int DS = PX > 1 ? Cp + 4 : Cp;  // D row stride (padded: 4 consecutive rows hit 4 distinct bank quads)
  float* D = smem;                  // [BM][DS]   depthwise tile, channels contiguous
  float* Bs = D + DS * BM;          // [Cp][BN]   pointwise weights, columns contiguous
  float* Wd = Bs + Cp * BN;         // [RR*SS][Cp]
  const int tid = threadIdx.x;
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  probe_begin();

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
  probe_pt(1);
  pdl_wait();
  probe_pt(2);
  cp_wait_all();
  __syncthreads();
  probe_pt(3);

  // ---- depthwise into D[px][c] (zero for padded channels / pixels past M) ----
  constexpr int V = VEC ? 4 : 1;
  const int cgroups = Cp / V;
  if constexpr (PX > 1 && KS > 0) {
#pragma unroll 1
    for (int e = tid; e < (BM / PX) * cgroups; e += SEP_THREADS) {
      const int cg = e % cgroups;
      const int px0 = (e / cgroups) * PX;
      const int c = cg * V;
      const int m = m0 + px0;
      float acc[PX][V];
#pragma unroll
      for (int j = 0; j < PX; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[j][v] = 0.f;
      if (m < a.M && c < a.C) {
        const int q = m % a.Q;
        const int t = m / a.Q;
        const int p = t % a.P, nb = t / a.P;
        const float* base = a.in + nb * a.in_sn + c * a.in_sc;
        const int ih0 = p * a.sh - a.ph, iw0 = q * a.sw - a.pw;
        if (q + PX - 1 < a.Q && m + PX - 1 < a.M && a.sw <= 2) {
          if (a.sw == 1)
            dw_row_block<KS, 1, PX, V, VEC>(a, base, Wd, Cp, c, ih0, iw0, acc);
          else
            dw_row_block<KS, 2, PX, V, VEC>(a, base, Wd, Cp, c, ih0, iw0, acc);
        } else {
          // row wrap / ragged end: pixel by pixel (unrolled: acc stays in registers)
#pragma unroll
          for (int j = 0; j < PX; ++j) {
            const int mj = m + j;
            if (mj >= a.M) continue;
            const int qj = mj % a.Q, tj = mj / a.Q;
            const int pj = tj % a.P, nj = tj / a.P;
            const float* bj = a.in + nj * a.in_sn + c * a.in_sc;
            float one[1][V];
#pragma unroll
            for (int v = 0; v < V; ++v) one[0][v] = 0.f;
            if (a.sw == 1)
              dw_row_block<KS, 1, 1, V, VEC>(a, bj, Wd, Cp, c, pj * a.sh - a.ph, qj * a.sw - a.pw, one);
            else
              dw_row_block<KS, 2, 1, V, VEC>(a, bj, Wd, Cp, c, pj * a.sh - a.ph, qj * a.sw - a.pw, one);
#pragma unroll
            for (int v = 0; v < V; ++v) acc[j][v] = one[0][v];
          }
        }
#pragma unroll
        for (int j = 0; j < PX; ++j)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[j][v] = apply_act(acc[j][v] + (a.b_dw ? a.b_dw[c + v] : 0.f), a.dw_act);
      }
#pragma unroll
      for (int j = 0; j < PX; ++j) {
        if constexpr (VEC) {
          *reinterpret_cast<float4*>(&D[(px0 + j) * DS + c]) = make_float4(acc[j][0], acc[j][1 % V], acc[j][2 % V],
                                                                          acc[j][3 % V]);
        } else {
          D[(px0 + j) * DS + c] = acc[j][0];
        }
      }
    }
  } else
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
      *reinterpret_cast<float4*>(&D[px * DS + c]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
      D[px * DS + c] = acc[0];
    }
  }
  __syncthreads();
  probe_pt(4);

  // ---- pointwise GEMM: out[px][n] = sum_c D[px][c] * W[c][n] ----
  const int ty = tid / (BN / TN);
  const int tx = tid % (BN / TN);
  float o[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) o[i][j] = 0.f;
  const float* bt = Bs + tx * TN;
  // large tiles (PX > 1, batch >= 8): thread (ty, tx) owns pixel rows
  // ty + i * RS (interleaved, so the 4 row groups of a warp read 4
  // consecutive padded rows: conflict-free float4 loads); four channels per
  // step feed 4 * TM * TN FMAs.  Small tiles (batch 1) keep the scalar loop
  // over rows ty * TM + i, which measured faster there.
  constexpr int RS = PX > 1 ? BM / TM : 1;
  const int row0 = PX > 1 ? ty : ty * TM;
  const float* at = D + row0 * DS;
  if constexpr (PX > 1) {
#pragma unroll 2
    for (int k = 0; k < Cp; k += 4) {
      float4 av[TM];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = *reinterpret_cast<const float4*>(&at[i * RS * DS + k]);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float bv[TN];
        if constexpr (TN % 4 == 0) {
#pragma unroll
          for (int j = 0; j < TN; j += 4) {
            const float4 b4 = *reinterpret_cast<const float4*>(&bt[(k + kk) * BN + j]);
            bv[j] = b4.x; bv[j + 1] = b4.y; bv[j + 2] = b4.z; bv[j + 3] = b4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < TN; ++j) bv[j] = bt[(k + kk) * BN + j];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float a_ = kk == 0 ? av[i].x : kk == 1 ? av[i].y : kk == 2 ? av[i].z : av[i].w;
#pragma unroll
          for (int j = 0; j < TN; ++j) o[i][j] = fmaf(a_, bv[j], o[i][j]);
        }
      }
    }
  } else {
#pragma unroll 4
    for (int k = 0; k < Cp; ++k) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = at[i * DS + k];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = bt[k * BN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) o[i][j] = fmaf(av[i], bv[j], o[i][j]);
    }
  }
  __syncthreads();  // D / Bs reads done; reuse D as the output tile
  probe_pt(5);

  float* part = D;  // [BM][BN] ≤ DS*BM + Cp*BN floats
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) part[(row0 + i * RS) * BN + tx * TN + j] = o[i][j];
  cg::cluster_group cluster = cg::this_cluster();
  tile_epilogue<BM, BN, SEP_THREADS>(a.epi, part, m0, n0, 1, cluster);
  probe_end();
}

// ---------------------------------------------------------------------------
// TMA variant.  One CTA = BM output pixels of ONE output row x BN output
// channels.  Everything it reads arrives by TMA / bulk copies that complete on
// two mbarriers, issued by one thread:
//   constants (before the PDL wait): pointwise weight slab [C][BN] (2-D tensor
//     map over the transposed weights), depthwise filter [KS*KS][C] and both
//     biases (1-D bulk copies);
//   activations (after the wait): the input patch [KS][PCW][C] of the row
//     (4-D tensor map over NHWC with per-dim strides, so concat slices and
//     padding — out-of-bounds rows / columns are zero-filled by TMA — need no
//     address math) and the residual tile [BM][BN].
// The patch arrives in one memory round trip (the cp.async / ldg variants
// above keep only a few of the 25-49 taps in flight: ~5 µs of a 7x7).
// Depthwise from smem → D[c][px]; pointwise GEMM split over the 8 warps along
// C (16 independent FMAs per lane per channel instead of a 176-long chain);
// the warp partials are summed in the epilogue with bias, residual and act.
// ---------------------------------------------------------------------------
struct SepTmaGeo {
  int PCW;     // patch columns = (BM - 1) * stride + KS
  int CB;      // channels per patch chunk (≤ 256) and chunks
  int NCH;
  int CBW;     // weight rows per box (≤ 256) and boxes
  int NCW;
  int QT;      // column tiles per output row
  int CS;      // depthwise split: the column blocks of a row tile form a cluster of CS CTAs,
  int Cs;      //   rank r computes the depthwise for channels [r*Cs, (r+1)*Cs)
  int o_bs, o_wd, o_bdw, o_bpw, o_x, o_d, o_r, o_bar;  // smem offsets (floats)
  uint32_t bytes_const, bytes_act;
};

template <int KS, int SW, int BM, int BN>
__global__ void __launch_bounds__(SEP_THREADS)
sepconv_tma_kernel(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tw,
                   const __grid_constant__ CUtensorMap tres, SepArgs a, SepTmaGeo g) {
  static_assert(BN % 32 == 0 && BM % 4 == 0, "tile");
  constexpr int JN = BN / 32;              // pointwise columns per lane
  constexpr int PXT = 2;                   // depthwise output pixels per thread (row neighbours)
  constexpr int SPAN = (PXT - 1) * SW + KS;  // input columns they read per filter row
  extern __shared__ __align__(128) float smem[];
  float* Bs = smem + g.o_bs;
  float* Wd = smem + g.o_wd;
  float* bdw = smem + g.o_bdw;
  float* bpw = smem + g.o_bpw;
  float* Xs = smem + g.o_x;
  float* D = smem + g.o_d;  // [C][BM]
  float* Rs = smem + g.o_r;
  float* Pt = Xs;  // warp partials reuse the patch once the depthwise is done
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.o_bar);
  const uint32_t bar_c = su32(&bars[0]), bar_a = su32(&bars[1]), bar_d = su32(&bars[2]);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qt = blockIdx.x % g.QT;
  const int rowi = blockIdx.x / g.QT;  // nb * P + p
  const int p = rowi % a.P, nb = rowi / a.P;
  const int q0 = qt * BM;
  const int cb = blockIdx.y + blockIdx.z;  // column block (grid y, or cluster z when CS > 1)
  const int n0 = cb * BN;
  const int C = a.C;
  const int CS = g.CS;
  const int me = CS > 1 ? (int)cluster_rank() : 0;
  const int c_lo = CS > 1 ? me * g.Cs : 0;                   // this CTA's depthwise channels
  const int c_n = CS > 1 ? max(0, min(g.Cs, C - c_lo)) : C;
  probe_begin();

  if (tid == 0) {
    prefetch_tmap(&tin);
    prefetch_tmap(&tw);
    mbar_init1(bar_c);
    mbar_init1(bar_a);
    mbar_init1(bar_d);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_cta();
    // the peers push their depthwise slices into D: every channel but mine
    if (CS > 1) mbar_expect_tx(bar_d, (uint32_t)((C - c_n) * BM * 4));
    mbar_expect_tx(bar_c, g.bytes_const + (a.b_pw ? (uint32_t)(min(BN, a.K - n0) * 4) : 0u));
#pragma unroll 1
    for (int j = 0; j < g.NCW; ++j) tma_load_2d(su32(Bs + j * g.CBW * BN), &tw, n0, j * g.CBW, bar_c);
    bulk_g2s(su32(Wd), a.w_dw, (uint32_t)(KS * KS * C * 4), bar_c);
    if (a.b_dw) bulk_g2s(su32(bdw), a.b_dw, (uint32_t)(C * 4), bar_c);
    if (a.b_pw) bulk_g2s(su32(bpw), a.b_pw + n0, (uint32_t)(min(BN, a.K - n0) * 4), bar_c);
  }
  if (CS > 1) cluster_arrive_relaxed();  // my barriers are initialised (peers wait before pushing)
  pdl_trigger();
  probe_pt(1);
  pdl_wait();
  probe_pt(2);
  if (tid == 0) {
    mbar_expect_tx(bar_a, g.bytes_act);
    const int iw0 = q0 * SW - a.pw, ih0 = p * a.sh - a.ph;
#pragma unroll 1
    for (int j = 0; j < g.NCH; ++j)
      tma_load_4d(su32(Xs + j * KS * g.PCW * g.CB), &tin, c_lo + j * g.CB, iw0, ih0, nb, bar_a);
    if (a.has_res) tma_load_4d(su32(Rs), &tres, n0, q0, p, nb, bar_a);
  }
  __syncthreads();  // barrier inits visible before anyone polls them
  mbar_wait_parity(bar_c, 0);
  mbar_wait_parity(bar_a, 0);
  probe_pt(3);

  // shared ReLU applied once over the patch (not once per tap use)
  if (a.pre_relu) {
    float4* x4 = reinterpret_cast<float4*>(Xs);
    const int n4 = g.NCH * KS * g.PCW * g.CB / 4;
#pragma unroll 1
    for (int i = tid; i < n4; i += SEP_THREADS) {
      float4 v = x4[i];
      v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
      x4[i] = v;
    }
    __syncthreads();
  }
  probe_pt(8);

  // ---- depthwise for channels [c_lo, c_lo + c_n): D[c][px] ----
  // A thread owns 4 channels x PXT row neighbours: per filter row it loads the
  // SPAN input columns and KS filter taps once and reuses them in registers
  // (shared-memory bandwidth, not FMAs, bounds this phase).
  const int C4 = c_n >> 2;
  constexpr int PG = BM / PXT;
#pragma unroll 1
  for (int e = tid; e < PG * C4; e += SEP_THREADS) {
    const int cg = e % C4, pg = e / C4;
    const int cl = cg * 4;  // channel within the slice
    const int c = c_lo + cl;
    const int ch = cl / g.CB, cc = cl - ch * g.CB;
    const float* xb = Xs + (ch * KS * g.PCW + pg * PXT * SW) * g.CB + cc;
    const float* wb = Wd + c;
    float4 acc[PXT];
#pragma unroll
    for (int j = 0; j < PXT; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < KS; ++r) {
      float4 xr[SPAN], wr[KS];
#pragma unroll
      for (int t = 0; t < SPAN; ++t) xr[t] = *reinterpret_cast<const float4*>(xb + (r * g.PCW + t) * g.CB);
#pragma unroll
      for (int s2 = 0; s2 < KS; ++s2) wr[s2] = *reinterpret_cast<const float4*>(wb + (r * KS + s2) * C);
#pragma unroll
      for (int j = 0; j < PXT; ++j)
#pragma unroll
        for (int s2 = 0; s2 < KS; ++s2) {
          const float4 x = xr[j * SW + s2];
          acc[j].x = fmaf(x.x, wr[s2].x, acc[j].x);
          acc[j].y = fmaf(x.y, wr[s2].y, acc[j].y);
          acc[j].z = fmaf(x.z, wr[s2].z, acc[j].z);
          acc[j].w = fmaf(x.w, wr[s2].w, acc[j].w);
        }
    }
    const float4 bd = a.b_dw ? *reinterpret_cast<const float4*>(bdw + c) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < PXT; ++j) {
      const int px = pg * PXT + j;
      D[(c + 0) * BM + px] = apply_act(acc[j].x + bd.x, a.dw_act);
      D[(c + 1) * BM + px] = apply_act(acc[j].y + bd.y, a.dw_act);
      D[(c + 2) * BM + px] = apply_act(acc[j].z + bd.z, a.dw_act);
      D[(c + 3) * BM + px] = apply_act(acc[j].w + bd.w, a.dw_act);
    }
  }
  probe_pt(9);
  if (CS > 1) {
    // push my D slice into every peer's D (bulk DSMEM copies completing on
    // the peer's mbarrier), then wait for theirs — no cluster-wide barrier
    fence_proxy_async_cta();
    __syncthreads();
    cluster_wait();  // every peer initialised its barriers
    if (tid == 0 && c_n > 0) {
      const uint32_t src = su32(D + c_lo * BM);
#pragma unroll 1
      for (int r = 0; r < CS; ++r)
        if (r != me) bulk_s2peer(mapa_rank(src, (uint32_t)r), src, (uint32_t)(c_n * BM * 4), mapa_rank(bar_d, (uint32_t)r));
      bulk_commit();
    }
    mbar_wait_parity(bar_d, 0);
  } else {
    __syncthreads();
  }
  probe_pt(4);

  // ---- pointwise: warp w sums channels [w*C/8, (w+1)*C/8) for the whole tile ----
  float o[BM][JN];
#pragma unroll
  for (int i = 0; i < BM; ++i)
#pragma unroll
    for (int j = 0; j < JN; ++j) o[i][j] = 0.f;
  const int k0 = warp * C / 8, k1 = (warp + 1) * C / 8;
#pragma unroll 2
  for (int k = k0; k < k1; ++k) {
    float dv[BM];
#pragma unroll
    for (int i = 0; i < BM; i += 4) {
      const float4 t = *reinterpret_cast<const float4*>(D + k * BM + i);
      dv[i] = t.x; dv[i + 1] = t.y; dv[i + 2] = t.z; dv[i + 3] = t.w;
    }
    float bv[JN];
#pragma unroll
    for (int j = 0; j < JN; ++j) bv[j] = Bs[k * BN + lane + 32 * j];
#pragma unroll
    for (int i = 0; i < BM; ++i)
#pragma unroll
      for (int j = 0; j < JN; ++j) o[i][j] = fmaf(dv[i], bv[j], o[i][j]);
  }
#pragma unroll
  for (int i = 0; i < BM; ++i)
#pragma unroll
    for (int j = 0; j < JN; ++j) Pt[(warp * BM + i) * BN + lane + 32 * j] = o[i][j];
  __syncthreads();
  probe_pt(5);

  // ---- epilogue: sum the 8 warp partials, bias, residual, act, float4 store ----
  constexpr int GPR = BN / 4;
#pragma unroll 1
  for (int gi = tid; gi < BM * GPR; gi += SEP_THREADS) {
    const int px = gi / GPR, nn = (gi % GPR) * 4;
    const int q = q0 + px, n = n0 + nn;
    float4 t[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) t[w] = *reinterpret_cast<const float4*>(Pt + (w * BM + px) * BN + nn);
    float4 v = t[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) v = f4add(v, t[w]);
    if (a.b_pw) v = f4add(v, *reinterpret_cast<const float4*>(bpw + nn));
    if (a.has_res) v = f4add(v, *reinterpret_cast<const float4*>(Rs + px * BN + nn));
    if (q < a.Q && n < a.K)
      *reinterpret_cast<float4*>(a.out + nb * a.epi.out_sn + p * a.epi.out_sh + q * a.epi.out_sw + n) =
          act4(v, a.act);
  }
  probe_pt(6);
  if (CS > 1 && tid == 0) bulk_wait_read0();  // my pushes have read D before the CTA exits
  probe_end();
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
// row-blocked depthwise variants (4 pixels per thread), after the TMA ones
constexpr int kSepRowFirst = 11;
// (wide column tiles: the depthwise is recomputed once per column block, so
// K up to 128 per block keeps that redundancy low for 88 / 176-channel layers)
constexpr SepCfg kSepRow[] = {{64, 32}, {128, 32}, {64, 64}, {64, 128}, {32, 128}};
constexpr int kNumSepRow = 5;
constexpr int kSepSmemMax = 227 * 1024;
}  // namespace

static size_t sep_smem(int C, int R, int S, int bm, int bn) {
  const size_t cp = (size_t)(C + SEP_BK - 1) / SEP_BK * SEP_BK;
  const size_t body = (cp + 4) * bm + cp * bn + (size_t)R * S * cp;  // D rows padded by 4
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
    case 11: return launch_k(sepconv_kernel<KS, VEC, 64, 32, 2, 4, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 12: return launch_k(sepconv_kernel<KS, VEC, 128, 32, 4, 4, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 13: return launch_k(sepconv_kernel<KS, VEC, 64, 64, 4, 4, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 14: return launch_k(sepconv_kernel<KS, VEC, 64, 128, 4, 8, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
    case 15: return launch_k(sepconv_kernel<KS, VEC, 32, 128, 2, 8, 4>, grid, dim3(SEP_THREADS), smem, st, 1, a);
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

// ---- TMA variants (6..): tile (BM, BN) ----
namespace {
constexpr SepCfg kSepTma[] = {{4, 32}, {8, 32}, {8, 64}, {16, 32}, {16, 64}};
constexpr int kNumSepTma = sizeof(kSepTma) / sizeof(kSepTma[0]);
}  // namespace

static int round32(int x) { return (x + 31) / 32 * 32; }

// smem plan of the TMA kernel; false if the op cannot use it
static bool sep_tma_geo(const SepArgs& a, const sw_op_desc& op, int bm, int bn, SepTmaGeo* g, size_t* smem) {
  const int ks = a.R;
  if (a.R != a.S || (ks != 3 && ks != 5 && ks != 7)) return false;
  if (!a.vec || a.in_sc != 1 || !a.wvec || !a.epi.vec) return false;
  if (a.has_res && (op.params[SP_RES_SC] > 1 || (op.ptrs[PT_RES] & 15))) return false;
  if ((op.ptrs[PT_WS] & 15) || (op.ptrs[PT_DW_BIAS] & 15) || (op.ptrs[PT_BIAS] & 15)) return false;
  g->PCW = (bm - 1) * a.sw + ks;
  if (g->PCW > 256) return false;
  g->CB = a.C <= 256 ? a.C : 256;
  g->NCH = (a.C + g->CB - 1) / g->CB;
  g->CS = 1;
  g->Cs = a.C;
  if (op.params[SP_SPLIT_K] > 1) {  // cluster-split depthwise over the column blocks
    const int cs = (int)cdiv(a.K, bn);
    if (cs < 2 || cs > 8) return false;
    g->CS = cs;
    g->Cs = (int)cdiv(cdiv(a.C, cs), 4) * 4;
    if (g->Cs > 256) return false;
    g->CB = g->Cs;
    g->NCH = 1;
  }
  g->CBW = a.C <= 256 ? a.C : 256;
  g->NCW = (a.C + g->CBW - 1) / g->CBW;
  g->QT = (a.Q + bm - 1) / bm;
  const int bs = g->NCW * g->CBW * bn;
  const int patch = g->NCH * ks * g->PCW * g->CB;
  int o = 0;
  g->o_bs = o; o += round32(bs);
  g->o_wd = o; o += round32(ks * ks * a.C);
  g->o_bdw = o; o += round32(a.C);
  g->o_bpw = o; o += round32(bn);
  g->o_x = o; o += round32(patch > 8 * bm * bn ? patch : 8 * bm * bn);
  g->o_d = o; o += round32(a.C * bm);
  g->o_r = o; o += round32(bm * bn);
  g->o_bar = o; o += 32;
  *smem = (size_t)o * 4;
  if (*smem > (size_t)kSepSmemMax) return false;
  // weight boxes are always BN wide (out-of-range columns zero-filled); the
  // pointwise bias slice is added per CTA in the kernel
  g->bytes_const = (uint32_t)(bs + ks * ks * a.C + (a.b_dw ? a.C : 0)) * 4;
  g->bytes_act = (uint32_t)(patch + (a.has_res ? bm * bn : 0)) * 4;
  return true;
}

template <int KS, int SW, int BM, int BN>
static cudaError_t launch_sep_tma_t(const SepArgs& a, const sw_op_desc& op, cudaStream_t st) {
  SepTmaGeo g;
  size_t smem = 0;
  if (!sep_tma_geo(a, op, BM, BN, &g, &smem)) return cudaErrorInvalidValue;
  CUtensorMap tin, tw, tres;
  {
    const uint64_t dims[4] = {(uint64_t)a.C, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.N};
    const uint64_t str[3] = {(uint64_t)a.in_sw * 4, (uint64_t)a.in_sh * 4, (uint64_t)a.in_sn * 4};
    const uint32_t box[4] = {(uint32_t)g.CB, (uint32_t)g.PCW, (uint32_t)KS, 1};
    if (!encode_tmap_f32(&tin, a.in, 4, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.C};
    const uint64_t str[1] = {(uint64_t)a.K * 4};
    const uint32_t box[2] = {(uint32_t)BN, (uint32_t)g.CBW};
    if (!encode_tmap_f32(&tw, a.w_pw, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  if (a.has_res) {
    const uint64_t dims[4] = {(uint64_t)a.K, (uint64_t)a.Q, (uint64_t)a.P, (uint64_t)a.N};
    const uint64_t str[3] = {(uint64_t)a.epi.res_sw * 4, (uint64_t)a.epi.res_sh * 4, (uint64_t)a.epi.res_sn * 4};
    const uint32_t box[4] = {(uint32_t)BN, (uint32_t)BM, 1, 1};
    if (!encode_tmap_f32(&tres, a.res, 4, dims, str, box)) return cudaErrorInvalidValue;
  } else {
    tres = tw;  // unused
  }
  if (g.CS > 1) {  // one cluster (along z) per row tile
    dim3 grid((unsigned)(a.N * a.P * g.QT), 1, (unsigned)g.CS);
    return launch_k(sepconv_tma_kernel<KS, SW, BM, BN>, grid, dim3(SEP_THREADS), smem, st, (unsigned)g.CS, tin, tw,
                    tres, a, g);
  }
  dim3 grid((unsigned)(a.N * a.P * g.QT), (unsigned)cdiv(a.K, BN));
  return launch_k(sepconv_tma_kernel<KS, SW, BM, BN>, grid, dim3(SEP_THREADS), smem, st, 1, tin, tw, tres, a, g);
}

template <int KS, int SW>
static cudaError_t launch_sep_tma_ksw(int v, const SepArgs& a, const sw_op_desc& op, cudaStream_t st) {
  switch (v) {
    case 0: return launch_sep_tma_t<KS, SW, 4, 32>(a, op, st);
    case 1: return launch_sep_tma_t<KS, SW, 8, 32>(a, op, st);
    case 2: return launch_sep_tma_t<KS, SW, 8, 64>(a, op, st);
    case 3: return launch_sep_tma_t<KS, SW, 16, 32>(a, op, st);
    default: return launch_sep_tma_t<KS, SW, 16, 64>(a, op, st);
  }
}

template <int KS>
static cudaError_t launch_sep_tma_ks(int v, const SepArgs& a, const sw_op_desc& op, cudaStream_t st) {
  if (a.sw == 1) return launch_sep_tma_ksw<KS, 1>(v, a, op, st);
  if (a.sw == 2) return launch_sep_tma_ksw<KS, 2>(v, a, op, st);
  return cudaErrorInvalidValue;
}

int launch_sepconv(const sw_op_desc& op, void* stream) {
  if (op.variant == SEP_TC_VARIANT) return launch_sepconv_tc(op, stream);  // sepconv_tc.cu
  if (op.variant >= 20 && op.variant < 30) return launch_sep_rows(op, stream);  // sep_rows.cu
  SepArgs a = sep_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  if (op.variant >= kNumSep && op.variant < kNumSep + kNumSepTma) {
    const int v = op.variant - kNumSep;
    switch (a.R == a.S ? a.R : 0) {
      case 3: return (int)launch_sep_tma_ks<3>(v, a, op, st);
      case 5: return (int)launch_sep_tma_ks<5>(v, a, op, st);
      case 7: return (int)launch_sep_tma_ks<7>(v, a, op, st);
      default: return (int)cudaErrorInvalidValue;
    }
  }
  const int ks = (a.R == a.S && (a.R == 3 || a.R == 5 || a.R == 7)) ? a.R : 0;
  int v = (op.variant >= 0 && op.variant < kNumSep) ? op.variant : 0;
  SepCfg cfg = kSep[v];
  if (op.variant >= kSepRowFirst && op.variant < kSepRowFirst + kNumSepRow) {
    if (!ks || a.sw > 2) return (int)cudaErrorInvalidValue;  // row blocking needs a fixed k x k window
    v = op.variant;
    cfg = kSepRow[v - kSepRowFirst];
  }
  const size_t smem = sep_smem(a.C, a.R, a.S, cfg.bm, cfg.bn);
  if (smem > (size_t)kSepSmemMax) return (int)cudaErrorInvalidValue;  // the autotuner skips it
  dim3 grid((unsigned)cdiv(a.M, cfg.bm), (unsigned)cdiv(a.K, cfg.bn));
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
  if constexpr (KS > 0) {
    cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 64, 32, 2, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSepSmemMax);
    cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 128, 32, 4, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSepSmemMax);
    cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 64, 64, 4, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSepSmemMax);
    cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 64, 128, 4, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSepSmemMax);
    cudaFuncSetAttribute(sepconv_kernel<KS, VEC, 32, 128, 2, 8, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSepSmemMax);
  }
}

template <int KS, int SW>
static void init_sep_tma_ksw() {
  cudaFuncSetAttribute(sepconv_tma_kernel<KS, SW, 4, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_tma_kernel<KS, SW, 8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_tma_kernel<KS, SW, 8, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_tma_kernel<KS, SW, 16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
  cudaFuncSetAttribute(sepconv_tma_kernel<KS, SW, 16, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSepSmemMax);
}
template <int KS>
static void init_sep_tma_ks() {
  init_sep_tma_ksw<KS, 1>();
  init_sep_tma_ksw<KS, 2>();
}

void init_sep_kernels() {
  init_sep_tma_ks<3>(); init_sep_tma_ks<5>(); init_sep_tma_ks<7>();
  init_sep_ks<3, true>(); init_sep_ks<5, true>(); init_sep_ks<7, true>(); init_sep_ks<0, true>();
  init_sep_ks<3, false>(); init_sep_ks<5, false>(); init_sep_ks<7, false>(); init_sep_ks<0, false>();
}

}  // namespace sw
