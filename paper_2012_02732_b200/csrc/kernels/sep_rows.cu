// Row-staged fused separable convolution for thin, wide maps (NASNet stem
// cells at large batch: 11 / 22 / 32 channels on 111x111 and 56x56 maps).
//
// The pixel-tiled sepconv kernels gather the depthwise window of every
// output pixel from L1 / L2: at stride 2 with a 7x7 window on a 32-channel
// 111x111 map each input element is fetched ~3.5 times and the 11 / 22
// channel maps cannot use 128-bit loads at all (44-byte pixels), so those
// layers ran at 0.3-1.3 TB/s (r03l).  Here one CTA owns TH whole output rows
// of one image:
//   1. the pointwise weights [C][K], the depthwise filter and biases go to
//      shared memory before the PDL wait (constants);
//   2. the (TH-1)*stride + k input rows the tile needs are staged ONCE into
//      shared memory by cp.async, a channel chunk at a time, the next chunk
//      in flight while this one is convolved ([row][column][channel], zero
//      fill for the padding columns / rows / channels), with coalesced copies
//      whatever the channel count (ReLU applied as the window is read);
//   3. depthwise: a thread owns one channel (its k x k taps in registers)
//      and slides the window of PX adjacent output pixels along the staged
//      row in registers (scalar shared reads at compile-time offsets from a
//      per-item base; a pad every PX*stride columns so the lanes of a warp
//      hit distinct banks) into D[row][pixel][channel] (+ bias, act) —
//      shared traffic ~1.75 reads per output per tap row instead of the 7.5
//      float4 reads of a 4-channel-per-thread window (r03o: 74 % L1 busy);
//   4. pointwise: a thread owns one output pixel (its depthwise row in
//      registers, the weight rows broadcast from shared memory): bias,
//      residual, act, NHWC stores.
// Variants 20..23 (TH, PX) = (2, 8), (4, 8), (8, 8), (4, 4).
#include <algorithm>

#include "common.cuh"
#include "tma.cuh"

namespace sw {

namespace {

constexpr int SR_THREADS = 256;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(ok ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(su32(dst)), "l"(src), "r"(ok ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct SepRowsArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w_pw;  // [C][K]
  const float* __restrict__ b_pw;  // [K] or null
  const float* __restrict__ w_dw;  // [R][S][C]
  const float* __restrict__ b_dw;  // [C] or null
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, sh, sw, ph, pw, act, dw_act, pre_relu, has_res, in_vec;
  int64_t in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  // geometry (host-computed)
  int TH, Cp, CC, nch, IR, WP, RL, padG, QG;
  int o_wp, o_wd, o_bdw, o_bpw, o_d, o_x;  // float offsets into shared memory
};

}  // namespace

// pointwise + epilogue of the row tile: thread = output pixel, CQ channel
// quads of its depthwise row in registers; rows >= C4 of a padded case read
// the zero tail of D / Wp (allocated to 16 quads for that case)
template <int CQ>
__device__ __forceinline__ void sep_rows_pw(const SepRowsArgs& a, const float* D, const float4* Wp,
                                            const float* Bpw, int nb, int p0, int rows) {
  const int C4 = a.Cp / 4;
#pragma unroll 1
  for (int px = threadIdx.x; px < rows * a.Q; px += SR_THREADS) {
    const int q = px % a.Q;
    const int p = p0 + px / a.Q;
    float4 d[CQ];
    const float4* dr = reinterpret_cast<const float4*>(D + px * a.Cp);
#pragma unroll
    for (int i = 0; i < CQ; ++i) d[i] = i < C4 ? dr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    float* op = a.out + nb * a.out_sn + p * a.out_sh + q * a.out_sw;
    const float* rp = a.has_res ? a.res + nb * a.res_sn + p * a.res_sh + q * a.res_sw : nullptr;
#pragma unroll 1
    for (int k = 0; k < a.K; ++k) {
      const float4* wr = Wp + k * C4;
      float acc = Bpw[k];
#pragma unroll
      for (int i = 0; i < CQ; ++i) {
        const float4 wv = i < C4 ? wr[i] : make_float4(0.f, 0.f, 0.f, 0.f);
        acc = fmaf(d[i].x, wv.x, acc);
        acc = fmaf(d[i].y, wv.y, acc);
        acc = fmaf(d[i].z, wv.z, acc);
        acc = fmaf(d[i].w, wv.w, acc);
      }
      if (rp) acc += rp[k * a.res_sc];
      op[k * a.out_sc] = apply_act(acc, a.act);
    }
  }
}

template <int KS, int SW, int PX>
__global__ void __launch_bounds__(SR_THREADS) sep_rows_kernel(SepRowsArgs a) {
  constexpr int KK = KS * KS;
  constexpr int NW = (PX - 1) * SW + KS;
  constexpr int PS = PX * SW;  // staged columns per pixel group
  extern __shared__ __align__(16) float smem[];
  float4* Wp = reinterpret_cast<float4*>(smem + a.o_wp);  // [K][Cp/4] quads: pointwise row of output k
  float* Wd = smem + a.o_wd;                               // [Cp][KK]: taps of channel c
  float* Bdw = smem + a.o_bdw;                             // [Cp]
  float* Bpw = smem + a.o_bpw;                             // [K]
  float* D = smem + a.o_d;                                 // [TH][Q][Cp]
  float* X = smem + a.o_x;                                 // [buf][IR][RL]
  const int tid = threadIdx.x;
  const int tiles = (a.P + a.TH - 1) / a.TH;
  const int nb = blockIdx.x / tiles;
  const int p0 = (blockIdx.x - nb * tiles) * a.TH;
  const int Cp = a.Cp, K = a.K, C4 = a.Cp / 4;

  // ---- constants (before the PDL wait) ----
  for (int e = tid; e < K * C4; e += SR_THREADS) {
    const int k = e / C4, c = 4 * (e - k * C4);
    float4 w;
    w.x = c < a.C ? __ldg(a.w_pw + (size_t)c * K + k) : 0.f;
    w.y = c + 1 < a.C ? __ldg(a.w_pw + (size_t)(c + 1) * K + k) : 0.f;
    w.z = c + 2 < a.C ? __ldg(a.w_pw + (size_t)(c + 2) * K + k) : 0.f;
    w.w = c + 3 < a.C ? __ldg(a.w_pw + (size_t)(c + 3) * K + k) : 0.f;
    Wp[e] = w;
  }
  for (int e = tid; e < Cp * KK; e += SR_THREADS) {
    const int c = e / KK, tap = e - c * KK;
    Wd[e] = c < a.C ? __ldg(a.w_dw + tap * a.C + c) : 0.f;
  }
  for (int e = tid; e < Cp; e += SR_THREADS) Bdw[e] = (a.b_dw && e < a.C) ? __ldg(a.b_dw + e) : 0.f;
  for (int e = tid; e < K; e += SR_THREADS) Bpw[e] = a.b_pw ? __ldg(a.b_pw + e) : 0.f;
  pdl_trigger();
  pdl_wait();

  const float* inb = a.in + nb * a.in_sn;
  const int CC = a.CC;      // channels per staged chunk
  const int RL = a.RL;      // staged row length (floats): (iw, c) at iw*CC + c + (iw / PS) * padG
  const int padG = a.padG;  // (PS*CC + padG) % 32 == CC % 32: the lanes of a warp hit distinct banks
  const int bufsz = a.IR * RL;
  const float lo = a.pre_relu ? 0.f : __int_as_float(0xff800000);  // ReLU on the staged input, applied as read
  // stage rows (p0*sh - ph + ir), columns (iw - pw), channels of chunk ch by
  // cp.async (zero-filled outside the image / past C): every copy of the
  // chunk is in flight at once
  auto stage = [&](int ch, int buf) {
    const int c0 = ch * CC;
    float* Xb = X + buf * bufsz;
    // a row's (column, channel) elements are walked with an incremental
    // (iw, cc) pair: no divisions in the copy loop
    const int V = a.in_vec ? 4 : 1;  // 16-B copies of 4 channels (CC % 4 == 0, padG % 4 == 0)
    const int CV = CC / V;
    const int diw = SR_THREADS / CV, dcv = SR_THREADS % CV;
#pragma unroll 1
    for (int ir = 0; ir < a.IR; ++ir) {
      const int ih = p0 * a.sh - a.ph + ir;
      const bool rok = (unsigned)ih < (unsigned)a.H;
      const float* srow = inb + (rok ? ih * a.in_sh : 0);
      float* drow = Xb + ir * RL;
      int iw = tid / CV, cv = tid - (tid / CV) * CV;
#pragma unroll 4
      for (int f = tid; f < a.WP * CV; f += SR_THREADS) {
        const int iwg = iw - a.pw;
        const int c = c0 + cv * V;
        const bool ok = rok && (unsigned)iwg < (unsigned)a.W && c < a.C;
        float* dst = drow + iw * CC + cv * V + (iw / PS) * padG;
        if (V == 4)
          cp_async16(dst, srow + (ok ? iwg * a.in_sw + c : 0), ok);
        else
          cp_async4(dst, srow + (ok ? iwg * a.in_sw + (int64_t)c * a.in_sc : 0), ok);
        cv += dcv;
        iw += diw;
        if (cv >= CV) {
          cv -= CV;
          ++iw;
        }
      }
    }
    cp_async_commit();
  };
  // depthwise thread role: one channel of the chunk (its k x k taps live in
  // registers) x a stream of (output row, PX-pixel group) items
  const int cl = tid % CC;
  const int slot = tid / CC;
  const int nslots = SR_THREADS / CC;
  stage(0, 0);
#pragma unroll 1
  for (int ch = 0; ch < a.nch; ++ch) {
    const int c = ch * CC + cl;
    // the next chunk streams in while this one is convolved
    if (ch + 1 < a.nch) {
      stage(ch + 1, (ch + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (slot < nslots) {
      float w[KK];
#pragma unroll
      for (int i = 0; i < KK; ++i) w[i] = Wd[c * KK + i];
      const float bdw = Bdw[c];
      const float* Xc = X + (ch & 1) * bufsz + cl;
#pragma unroll 1
      for (int it = slot; it < a.TH * a.QG; it += nslots) {
        const int qg = it % a.QG;
        const int tr = it / a.QG;
        float acc[PX];
#pragma unroll
        for (int j = 0; j < PX; ++j) acc[j] = 0.f;
        const float* xb = Xc + tr * a.sh * RL + qg * (PS * CC + padG);
#pragma unroll
        for (int r = 0; r < KS; ++r) {
          float x[NW];
#pragma unroll
          for (int j = 0; j < NW; ++j) x[j] = fmaxf(xb[r * RL + j * CC + (j / PS) * padG], lo);
#pragma unroll
          for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
            for (int j = 0; j < PX; ++j) acc[j] = fmaf(x[j * SW + s2], w[r * KS + s2], acc[j]);
        }
        float* dp = D + (tr * a.Q + qg * PX) * Cp + c;
#pragma unroll
        for (int j = 0; j < PX; ++j)
          if (qg * PX + j < a.Q) dp[j * Cp] = apply_act(acc[j] + bdw, a.dw_act);
      }
    }
    __syncthreads();  // chunk buffer free for the copy two chunks ahead; D complete after the last
  }
  // padded channels of D (Cp > C) hold zero weights in Wp, but must not be NaN
  if (Cp > a.C) {
    for (int e = tid; e < a.TH * a.Q * (Cp - a.C); e += SR_THREADS) {
      const int pc = e % (Cp - a.C), px = e / (Cp - a.C);
      D[px * Cp + a.C + pc] = 0.f;
    }
    __syncthreads();
  }

  // ---- pointwise + epilogue: a thread owns one output pixel: its depthwise
  // row in registers, the weight rows broadcast from shared memory ----
  const int rows = min(a.TH, a.P - p0);
  switch (C4) {  // uniform: the row length is a compile-time constant in each case
    case 1: sep_rows_pw<1>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 2: sep_rows_pw<2>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 3: sep_rows_pw<3>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 4: sep_rows_pw<4>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 5: sep_rows_pw<5>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 6: sep_rows_pw<6>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 8: sep_rows_pw<8>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 11: sep_rows_pw<11>(a, D, Wp, Bpw, nb, p0, rows); break;
    case 12: sep_rows_pw<12>(a, D, Wp, Bpw, nb, p0, rows); break;
    default: sep_rows_pw<16>(a, D, Wp, Bpw, nb, p0, rows); break;  // zero-padded quads past C4
  }
}

namespace {
struct SrCfg {
  int th, px;
};
constexpr SrCfg kSr[] = {{2, 8}, {4, 8}, {8, 8}, {4, 4}};
constexpr int kSrSmemMax = 200 * 1024;
}  // namespace

// shared-memory plan for (TH, PX); false if the op cannot run this variant
static bool sep_rows_geo(SepRowsArgs& a, int ks, int th, int px, size_t* smem) {
  a.TH = th;
  a.Cp = (a.C + 3) / 4 * 4;
  a.QG = (a.Q + px - 1) / px;
  a.IR = (th - 1) * a.sh + ks;
  a.WP = (a.QG * px - 1) * a.sw + ks;
  const int ps = px * a.sw;
  auto r4 = [](int x) { return (x + 3) / 4 * 4; };
  int o = 0;
  a.o_wp = o; o += a.K * a.Cp;
  a.o_wd = o; o += r4(ks * ks * a.Cp);
  a.o_bdw = o; o += a.Cp;
  a.o_bpw = o; o += r4(a.K);
  a.o_d = o; o += th * a.Q * a.Cp;
  a.o_x = o;
  // largest channel chunk whose staged rows fit (whole channel count first,
  // then divisors: multiples of 4 when the 16-B copy path is used)
  for (int cc = a.C; cc >= 1; --cc) {
    if (a.C % cc || (a.in_vec && cc % 4) || cc > SR_THREADS) continue;
    const int pad = ((cc - ps * cc) % 32 + 32) % 32;
    const int rl = r4(a.WP * cc + ((a.WP - 1) / ps) * pad + 1);
    const int bufs = cc == a.C ? 1 : 2;  // chunked: double-buffered staging
    const size_t bytes = 4 * ((size_t)o + (size_t)bufs * a.IR * rl);
    if (bytes <= (size_t)kSrSmemMax) {
      a.CC = cc;
      a.nch = a.C / cc;
      a.padG = pad;
      a.RL = rl;
      *smem = bytes;
      return true;
    }
  }
  return false;
}

template <int KS, int SW>
static int launch_sr_ksw(const SepRowsArgs& a, int px, size_t smem, cudaStream_t st) {
  const dim3 grid((unsigned)(a.N * ((a.P + a.TH - 1) / a.TH)));
  if (px == 4) return (int)launch_k(sep_rows_kernel<KS, SW, 4>, grid, dim3(SR_THREADS), smem, st, 1, a);
  return (int)launch_k(sep_rows_kernel<KS, SW, 8>, grid, dim3(SR_THREADS), smem, st, 1, a);
}

template <int KS>
static int launch_sr_ks(const SepRowsArgs& a, int px, size_t smem, cudaStream_t st) {
  if (a.sw == 1) return launch_sr_ksw<KS, 1>(a, px, smem, st);
  return launch_sr_ksw<KS, 2>(a, px, smem, st);
}

int launch_sep_rows(const sw_op_desc& op, void* stream) {
  const int64_t* p = op.params;
  const int v = op.variant - 20;
  if (v < 0 || v >= (int)(sizeof(kSr) / sizeof(kSr[0]))) return (int)cudaErrorInvalidValue;
  SepRowsArgs a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.w_pw = reinterpret_cast<const float*>(op.ptrs[PT_W]);
  a.b_pw = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.w_dw = reinterpret_cast<const float*>(op.ptrs[PT_WS]);
  a.b_dw = reinterpret_cast<const float*>(op.ptrs[PT_DW_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.dw_act = (int)p[SP_DW_ACT];
  a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.in_sn = p[SP_IN_SN]; a.in_sh = p[SP_IN_SH]; a.in_sw = p[SP_IN_SW]; a.in_sc = p[SP_IN_SC] ? p[SP_IN_SC] : 1;
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  if ((int64_t)a.N * a.P * a.Q == 0 || a.K == 0) return 0;
  const int ks = (int)p[SP_R];
  if (p[SP_R] != p[SP_S] || (ks != 3 && ks != 5 && ks != 7) || a.sh != a.sw || (a.sw != 1 && a.sw != 2) ||
      a.C > 64 || a.K > 64)
    return (int)cudaErrorInvalidValue;
  a.in_vec = a.C % 4 == 0 && a.in_sc == 1 && !((a.in_sn | a.in_sh | a.in_sw) & 3) && !(op.ptrs[PT_IN] & 15);
  size_t smem = 0;
  if (!sep_rows_geo(a, ks, kSr[v].th, kSr[v].px, &smem)) return (int)cudaErrorInvalidValue;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (ks) {
    case 3: return launch_sr_ks<3>(a, kSr[v].px, smem, st);
    case 5: return launch_sr_ks<5>(a, kSr[v].px, smem, st);
    default: return launch_sr_ks<7>(a, kSr[v].px, smem, st);
  }
}

// ---------------------------------------------------------------------------
// Row-staged k x k pooling (K_POOL variant 2) for thin wide maps: the same
// staging as above (input rows once per CTA, a channel-per-thread window
// sliding along the staged row), out-of-range taps staged as -inf (max) or 0
// (avg, divisor from the valid-tap count or torch's count_include_pad clamp).
// The 11 / 22-channel NASNet stem pools ran at 0.9-1.5 TB/s per-pixel (r03l).
namespace {
struct PoolRowsArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, sh, sw, ph, pw, act, pre_relu, has_res, mode, count_pad, pad_b, pad_r;
  float mul;
  int64_t in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  int TH, CC, nch, IR, WP, RL, padG, QG;
};
}  // namespace

template <int KS, int SW, int PX>
__global__ void __launch_bounds__(SR_THREADS) pool_rows_kernel(PoolRowsArgs a) {
  constexpr int NW = (PX - 1) * SW + KS;
  constexpr int PS = PX * SW;
  extern __shared__ __align__(16) float smem[];
  float* X = smem;  // [buf][IR][RL]
  const int tid = threadIdx.x;
  const int tiles = (a.P + a.TH - 1) / a.TH;
  const int nb = blockIdx.x / tiles;
  const int p0 = (blockIdx.x - nb * tiles) * a.TH;
  pdl_trigger();
  pdl_wait();
  const float* inb = a.in + nb * a.in_sn;
  const int CC = a.CC, RL = a.RL, padG = a.padG;
  const int bufsz = a.IR * RL;
  const float fill = a.mode == 0 ? __int_as_float(0xff800000) : 0.f;  // max: -inf, avg: 0 (not counted)
  auto stage = [&](int ch, int buf) {
    const int c0 = ch * CC;
    float* Xb = X + buf * bufsz;
    const int diw = SR_THREADS / CC, dcc = SR_THREADS % CC;
#pragma unroll 1
    for (int ir = 0; ir < a.IR; ++ir) {
      const int ih = p0 * a.sh - a.ph + ir;
      const bool rok = (unsigned)ih < (unsigned)a.H;
      const float* srow = inb + (rok ? ih * a.in_sh : 0);
      float* drow = Xb + ir * RL;
      int iw = tid / CC, cc = tid - (tid / CC) * CC;
#pragma unroll 4
      for (int f = tid; f < a.WP * CC; f += SR_THREADS) {
        const int iwg = iw - a.pw;
        const bool ok = rok && (unsigned)iwg < (unsigned)a.W;
        float* dst = drow + iw * CC + cc + (iw / PS) * padG;
        if (ok)
          cp_async4(dst, srow + iwg * a.in_sw + (int64_t)(c0 + cc) * a.in_sc, true);
        else
          *dst = fill;
        cc += dcc;
        iw += diw;
        if (cc >= CC) {
          cc -= CC;
          ++iw;
        }
      }
    }
    cp_async_commit();
  };
  const int cl = tid % CC;
  const int slot = tid / CC;
  const int nslots = SR_THREADS / CC;
  const float lo = a.pre_relu ? 0.f : __int_as_float(0xff800000);
  stage(0, 0);
#pragma unroll 1
  for (int ch = 0; ch < a.nch; ++ch) {
    const int c = ch * CC + cl;
    if (ch + 1 < a.nch) {
      stage(ch + 1, (ch + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (slot < nslots) {
      const float* Xc = X + (ch & 1) * bufsz + cl;
#pragma unroll 1
      for (int it = slot; it < a.TH * a.QG; it += nslots) {
        const int qg = it % a.QG;
        const int tr = it / a.QG;
        const int p = p0 + tr;
        if (p >= a.P) continue;
        float acc[PX];
#pragma unroll
        for (int j = 0; j < PX; ++j) acc[j] = a.mode == 0 ? __int_as_float(0xff800000) : 0.f;
        const float* xb = Xc + tr * a.sh * RL + qg * (PS * CC + padG);
#pragma unroll
        for (int r = 0; r < KS; ++r) {
          float x[NW];
#pragma unroll
          for (int j = 0; j < NW; ++j) x[j] = xb[r * RL + j * CC + (j / PS) * padG];
          // ReLU before pooling (staged -inf / 0 fills are unchanged by it
          // where they matter: max ignores -inf, avg adds 0)
          if (a.pre_relu) {
#pragma unroll
            for (int j = 0; j < NW; ++j) x[j] = fmaxf(x[j], a.mode == 0 ? lo : 0.f);
          }
#pragma unroll
          for (int s2 = 0; s2 < KS; ++s2)
#pragma unroll
            for (int j = 0; j < PX; ++j)
              acc[j] = a.mode == 0 ? fmaxf(acc[j], x[j * SW + s2]) : acc[j] + x[j * SW + s2];
        }
        const int ih0 = p * a.sh - a.ph;
        const int vr = min(ih0 + KS, a.H) - max(ih0, 0);
        const int hr = min(ih0 + KS, a.H + a.pad_b) - ih0;
        float* op = a.out + nb * a.out_sn + p * a.out_sh + c * a.out_sc;
        const float* rp = a.has_res ? a.res + nb * a.res_sn + p * a.res_sh + c * a.res_sc : nullptr;
#pragma unroll
        for (int j = 0; j < PX; ++j) {
          const int q = qg * PX + j;
          if (q >= a.Q) break;
          float v = acc[j];
          if (a.mode == 1) {
            const int iw0 = q * a.sw - a.pw;
            const int div = a.count_pad ? hr * (min(iw0 + KS, a.W + a.pad_r) - iw0)
                                        : vr * (min(iw0 + KS, a.W) - max(iw0, 0));
            v *= div > 0 ? 1.f / (float)div : 0.f;
          }
          v *= a.mul;
          if (rp) v += rp[q * a.res_sw];
          op[q * a.out_sw] = apply_act(v, a.act);
        }
      }
    }
    __syncthreads();
  }
}

template <int KS, int SW>
static int launch_pr_ksw(const PoolRowsArgs& a, int px, size_t smem, cudaStream_t st) {
  const dim3 grid((unsigned)(a.N * ((a.P + a.TH - 1) / a.TH)));
  if (px == 4) return (int)launch_k(pool_rows_kernel<KS, SW, 4>, grid, dim3(SR_THREADS), smem, st, 1, a);
  return (int)launch_k(pool_rows_kernel<KS, SW, 8>, grid, dim3(SR_THREADS), smem, st, 1, a);
}

int launch_pool_rows(const sw_op_desc& op, void* stream) {
  const int64_t* p = op.params;
  PoolRowsArgs a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.mode = (int)p[SP_POOL_MODE]; a.count_pad = (int)p[SP_COUNT_PAD];
  a.pad_b = (int)p[SP_PAD_BOTTOM]; a.pad_r = (int)p[SP_PAD_RIGHT];
  a.mul = p[SP_POOL_MUL] > 0 ? (float)p[SP_POOL_MUL] : 1.f;
  a.in_sn = p[SP_IN_SN]; a.in_sh = p[SP_IN_SH]; a.in_sw = p[SP_IN_SW]; a.in_sc = p[SP_IN_SC] ? p[SP_IN_SC] : 1;
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  if ((int64_t)a.N * a.P * a.Q * a.C == 0) return 0;
  const int ks = (int)p[SP_R];
  if (p[SP_R] != p[SP_S] || (ks != 3 && ks != 5 && ks != 7) || a.sh != a.sw || (a.sw != 1 && a.sw != 2) ||
      a.C > 256 || (a.mode != 0 && a.mode != 1) || a.ph < 0 || a.pw < 0)
    return (int)cudaErrorInvalidValue;
  const int th = 4, px = a.sw == 1 ? 8 : 4;
  a.TH = th;
  a.QG = (a.Q + px - 1) / px;
  a.IR = (th - 1) * a.sh + ks;
  a.WP = (a.QG * px - 1) * a.sw + ks;
  const int ps = px * a.sw;
  size_t smem = 0;
  bool fit = false;
  for (int cc = std::min(a.C, 64); cc >= 1; --cc) {
    if (a.C % cc) continue;
    const int pad = ((cc - ps * cc) % 32 + 32) % 32;
    const int rl = (a.WP * cc + ((a.WP - 1) / ps) * pad + 4) / 4 * 4;
    const int bufs = cc == a.C ? 1 : 2;
    const size_t bytes = 4 * (size_t)bufs * a.IR * rl;
    if (bytes <= (size_t)kSrSmemMax) {
      a.CC = cc; a.nch = a.C / cc; a.padG = pad; a.RL = rl; smem = bytes; fit = true;
      break;
    }
  }
  if (!fit) return (int)cudaErrorInvalidValue;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (ks) {
    case 3: return a.sw == 1 ? launch_pr_ksw<3, 1>(a, 8, smem, st) : launch_pr_ksw<3, 2>(a, 4, smem, st);
    case 5: return a.sw == 1 ? launch_pr_ksw<5, 1>(a, 8, smem, st) : launch_pr_ksw<5, 2>(a, 4, smem, st);
    default: return a.sw == 1 ? launch_pr_ksw<7, 1>(a, 8, smem, st) : launch_pr_ksw<7, 2>(a, 4, smem, st);
  }
}

template <int KS, int SW>
static void init_sr_ksw() {
  cudaFuncSetAttribute(sep_rows_kernel<KS, SW, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  cudaFuncSetAttribute(sep_rows_kernel<KS, SW, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
}

void init_sep_rows_kernels() {
  cudaFuncSetAttribute(pool_rows_kernel<3, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  cudaFuncSetAttribute(pool_rows_kernel<3, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  cudaFuncSetAttribute(pool_rows_kernel<5, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  cudaFuncSetAttribute(pool_rows_kernel<5, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  cudaFuncSetAttribute(pool_rows_kernel<7, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  cudaFuncSetAttribute(pool_rows_kernel<7, 2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSrSmemMax);
  init_sr_ksw<3, 1>(); init_sr_ksw<3, 2>();
  init_sr_ksw<5, 1>(); init_sr_ksw<5, 2>();
  init_sr_ksw<7, 1>(); init_sr_ksw<7, 2>();
}

}  // namespace sw
