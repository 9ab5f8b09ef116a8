// Bandwidth-bound spatial kernels: depthwise convolution and k x k pooling.
//
// One thread owns one output pixel x VEC channels (VEC = 4 → 128-bit loads
// and stores when channel strides are 1 and addresses/channels align), so a
// warp reads 32*VEC consecutive channels of one input pixel per tap — fully
// coalesced in NHWC; the k*k tap reuse across neighbouring pixels is served
// by L1.  Epilogues fuse bias (folded BN), activation, a residual add (NASNet
// cell combines, pooling branch + identity) and the strided store that makes
// concat zero-copy.  Padding is top/left (may be negative for the NASNet
// "pad-then-slice" shifts); out-of-range taps are zero (conv), skipped (max)
// or excluded/counted per torch's count_include_pad rule (avg).
#include "common.cuh"

namespace sw {

struct SpatialArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w;     // depthwise weights [R][S][C]
  const float* __restrict__ bias;  // [C]
  const float* __restrict__ res;
  int N, H, W, C, P, Q, R, S, sh, sw, ph, pw, act, pre_relu, has_res, mode, count_pad, pad_b, pad_r;
  float mul;  // pool output multiplier (twin pools of one input merged)
  int64_t in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
};

static SpatialArgs spatial_args(const sw_op_desc& op) {
  const int64_t* p = op.params;
  SpatialArgs a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.w = reinterpret_cast<const float*>(op.ptrs[PT_W]);
  a.bias = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q];
  a.R = (int)p[SP_R]; a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.mode = (int)p[SP_POOL_MODE]; a.count_pad = (int)p[SP_COUNT_PAD];
  a.pad_b = (int)p[SP_PAD_BOTTOM]; a.pad_r = (int)p[SP_PAD_RIGHT];
  a.mul = p[SP_POOL_MUL] > 0 ? (float)p[SP_POOL_MUL] : 1.f;
  a.in_sn = p[SP_IN_SN]; a.in_sh = p[SP_IN_SH]; a.in_sw = p[SP_IN_SW]; a.in_sc = p[SP_IN_SC];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  return a;
}

template <int VEC>
struct VecT;
template <>
struct VecT<1> {
  using T = float;
  static __device__ __forceinline__ float ld(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ void st(float* p, float v) { *p = v; }
};
template <>
struct VecT<4> {
  using T = float4;
  static __device__ __forceinline__ float4 ld(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ void st(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
};

__device__ __forceinline__ float relu1(float v) { return fmaxf(v, 0.f); }
__device__ __forceinline__ float4 relu1(float4 v) {
  return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
}
__device__ __forceinline__ void fma_acc(float& acc, float x, float w) { acc = fmaf(x, w, acc); }
__device__ __forceinline__ void fma_acc(float4& acc, float4 x, float4 w) {
  acc.x = fmaf(x.x, w.x, acc.x); acc.y = fmaf(x.y, w.y, acc.y);
  acc.z = fmaf(x.z, w.z, acc.z); acc.w = fmaf(x.w, w.w, acc.w);
}
__device__ __forceinline__ void add_to(float& a, float b) { a += b; }
__device__ __forceinline__ void add_to(float4& a, float4 b) { a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w; }
__device__ __forceinline__ void max_to(float& a, float b) { a = fmaxf(a, b); }
__device__ __forceinline__ void max_to(float4& a, float4 b) {
  a.x = fmaxf(a.x, b.x); a.y = fmaxf(a.y, b.y); a.z = fmaxf(a.z, b.z); a.w = fmaxf(a.w, b.w);
}
__device__ __forceinline__ void scale(float& a, float s) { a *= s; }
__device__ __forceinline__ void scale(float4& a, float s) { a.x *= s; a.y *= s; a.z *= s; a.w *= s; }
__device__ __forceinline__ float splat(float v, float) { return v; }
__device__ __forceinline__ float4 splat(float v, float4) { return make_float4(v, v, v, v); }
__device__ __forceinline__ float actv(float v, int act) { return apply_act(v, act); }
__device__ __forceinline__ float4 actv(float4 v, int act) { return act4(v, act); }

// KIND 0 = depthwise conv, 1 = pool
template <int KIND, int VEC, int KS>
__global__ void __launch_bounds__(256) spatial_kernel(SpatialArgs a, int64_t total) {
  const int RR = KS ? KS : a.R;
  const int SS = KS ? KS : a.S;
  using V = VecT<VEC>;
  using T = typename V::T;
  pdl_trigger();
  pdl_wait();
  // 32-bit index math (the launcher guarantees total < 2^31): the int64
  // div / mod chain was ~500 instructions per thread, most of a bs256 pool
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int64_t)idx >= total) return;
  const uint32_t CG = (uint32_t)(a.C / VEC);
  const int cg = (int)(idx % CG);
  uint32_t t = idx / CG;
  const int q = (int)(t % (uint32_t)a.Q);
  t /= (uint32_t)a.Q;
  const int p = (int)(t % (uint32_t)a.P);
  const int n = (int)(t / (uint32_t)a.P);
  int c = cg * VEC;
  const float* base = a.in + n * a.in_sn + c * a.in_sc;
  const int ih0 = p * a.sh - a.ph, iw0 = q * a.sw - a.pw;
  // Branch-free taps: every load is issued unconditionally from a clamped
  // (always valid) address and out-of-range values are masked with selects,
  // so the unrolled loop keeps all tap loads in flight at once instead of one
  // memory round trip per tap (ncu: 45.8K cycles for a 7x7 with branches).
  T acc = splat(0.f, T{});
  int cnt = 0;
  if (KIND == 1 && a.mode == 0) acc = splat(-INFINITY, T{});
#pragma unroll
  for (int r = 0; r < RR; ++r) {
    const int ih = ih0 + r;
    const bool rok = (unsigned)ih < (unsigned)a.H;
    const int ihc = rok ? ih : 0;
#pragma unroll
    for (int s = 0; s < SS; ++s) {
      const int iw = iw0 + s;
      const bool ok = rok && (unsigned)iw < (unsigned)a.W;
      const int iwc = ok ? iw : 0;
      T x = V::ld(base + ihc * a.in_sh + iwc * a.in_sw);
      if (a.pre_relu) x = relu1(x);
      if (KIND == 0) {
        T wv = V::ld(a.w + (r * SS + s) * a.C + c);
        x = ok ? x : splat(0.f, T{});
        fma_acc(acc, x, wv);
      } else if (a.mode == 0) {
        if (ok) max_to(acc, x);
      } else {
        x = ok ? x : splat(0.f, T{});
        add_to(acc, x);
        cnt += ok ? 1 : 0;
      }
    }
  }
  if (KIND == 0) {
    if (a.bias) add_to(acc, V::ld(a.bias + c));
  } else if (a.mode == 1) {
    int div = cnt;
    if (a.count_pad) {  // torch: window clipped to [-pad, H + pad_bottom)
      int he = min(ih0 + RR, a.H + a.pad_b);
      int we = min(iw0 + SS, a.W + a.pad_r);
      div = (he - ih0) * (we - iw0);
    }
    scale(acc, div > 0 ? 1.f / (float)div : 0.f);
    if (a.mul != 1.f) scale(acc, a.mul);  // power-of-two multiplier: exact, = summing the twins
  } else if (a.mul != 1.f) {
    scale(acc, a.mul);
  }
  if (a.has_res) {
    const float* rp = a.res + n * a.res_sn + p * a.res_sh + q * a.res_sw + c * a.res_sc;
    if (VEC == 1 || a.res_sc == 1) {
      add_to(acc, V::ld(rp));
    } else {
      float* v = reinterpret_cast<float*>(&acc);
      for (int i = 0; i < VEC; ++i) v[i] += __ldg(rp + i * a.res_sc);
    }
  }
  acc = actv(acc, a.act);
  float* dst = a.out + n * a.out_sn + p * a.out_sh + q * a.out_sw + c * a.out_sc;
  if (VEC == 1 || a.out_sc == 1) {
    V::st(dst, acc);
  } else {
    const float* v = reinterpret_cast<const float*>(&acc);
    for (int i = 0; i < VEC; ++i) dst[i * a.out_sc] = v[i];
  }
}

static bool can_vec4(const SpatialArgs& a, const sw_op_desc& op, bool has_w) {
  if (a.C % 4 || a.in_sc != 1 || a.out_sc != 1) return false;
  if (a.in_sn % 4 || a.in_sh % 4 || a.in_sw % 4 || a.out_sn % 4 || a.out_sh % 4 || a.out_sw % 4) return false;
  if (!aligned16(op.ptrs[PT_IN]) || !aligned16(op.ptrs[PT_OUT])) return false;
  if (has_w && (!aligned16(op.ptrs[PT_W]) || (op.ptrs[PT_BIAS] && !aligned16(op.ptrs[PT_BIAS])))) return false;
  if (a.has_res && (!aligned16(op.ptrs[PT_RES]) || a.res_sc != 1 || a.res_sn % 4 || a.res_sh % 4 || a.res_sw % 4)) return false;
  return true;
}

// taps fully unrolled for the kernel sizes the networks use: all k*k loads of
// a thread are in flight together (one memory round trip per output)
template <int KIND, int VEC>
static cudaError_t launch_ks(int ks, int blocks, cudaStream_t st, const SpatialArgs& a, int64_t total) {
  switch (ks) {
    case 1: return launch_k(spatial_kernel<KIND, VEC, 1>, dim3(blocks), dim3(256), 0, st, 1, a, total);
    case 3: return launch_k(spatial_kernel<KIND, VEC, 3>, dim3(blocks), dim3(256), 0, st, 1, a, total);
    case 5: return launch_k(spatial_kernel<KIND, VEC, 5>, dim3(blocks), dim3(256), 0, st, 1, a, total);
    case 7: return launch_k(spatial_kernel<KIND, VEC, 7>, dim3(blocks), dim3(256), 0, st, 1, a, total);
    default: return launch_k(spatial_kernel<KIND, VEC, 0>, dim3(blocks), dim3(256), 0, st, 1, a, total);
  }
}

template <int KIND>
static int launch_spatial(const sw_op_desc& op, void* stream) {
  SpatialArgs a = spatial_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bool v4 = can_vec4(a, op, KIND == 0);
  int64_t total = (int64_t)a.N * a.P * a.Q * (v4 ? a.C / 4 : a.C);
  if (total == 0) return 0;
  if (total >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;  // 32-bit index math in the kernel
  int blocks = (int)cdiv(total, 256);
  const int ks = (a.R == a.S && (a.R == 1 || a.R == 3 || a.R == 5 || a.R == 7)) ? a.R : 0;
  return (int)(v4 ? launch_ks<KIND, 4>(ks, blocks, st, a, total) : launch_ks<KIND, 1>(ks, blocks, st, a, total));
}

// a filter tap load the compiler may not CSE across the unrolled rows (keeping
// all k*k taps live in registers spilled the blocks; each use re-reads L1)
__device__ __forceinline__ float4 ld_tap(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// Variant 1: register-blocked rows (large batches).  A thread owns one
// channel quad x a TH x PX block of output pixels and walks the block's
// (TH-1)*SW + KS input rows once; each row is loaded as one (PX-1)*SW + KS
// float4 window and every tap it feeds is applied from registers (all row /
// tap indices are compile-time).  Input loads per output drop from k*k to
// ((TH-1)s+k)((PX-1)s+k)/(TH PX) (5x5, s 1, 2x4 block: 25 → 6); consecutive threads
// take consecutive channel quads, so every window load is a coalesced
// NHWC row segment.
// ---------------------------------------------------------------------------
template <int KIND, int KS, int SW, int TH, int PX>
__global__ void __launch_bounds__(256, 2) spatial_rows_kernel(SpatialArgs a, int64_t total, int bands, int cols) {
  constexpr int NR = (TH - 1) * SW + KS;  // input rows of the block
  constexpr int WN = (PX - 1) * SW + KS;  // window width
  pdl_trigger();
  pdl_wait();
  const uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x;
  if ((int64_t)idx >= total) return;
  const uint32_t CG = (uint32_t)(a.C / 4);
  const int cg = (int)(idx % CG);
  uint32_t t = idx / CG;
  const int bx = (int)(t % (uint32_t)cols);
  t /= (uint32_t)cols;
  const int by = (int)(t % (uint32_t)bands);
  const int n = (int)(t / (uint32_t)bands);
  const int c = cg * 4;
  const int p0 = by * TH, q0 = bx * PX;
  const int ih0 = p0 * SW - a.ph, iw0 = q0 * SW - a.pw;
  const float* base = a.in + n * a.in_sn + c;
  const bool avg = KIND == 1 && a.mode == 1, mx = KIND == 1 && a.mode == 0;
  float4 acc[TH][PX];
#pragma unroll
  for (int y = 0; y < TH; ++y)
#pragma unroll
    for (int x = 0; x < PX; ++x) acc[y][x] = splat(mx ? -INFINITY : 0.f, float4{});
#pragma unroll
  for (int ir = 0; ir < NR; ++ir) {
    const int ih = ih0 + ir;
    const bool rok = (unsigned)ih < (unsigned)a.H;
    const float* rowp = base + (rok ? ih : 0) * a.in_sh;
    float4 win[WN];
    bool wok[WN];
#pragma unroll
    for (int j = 0; j < WN; ++j) {
      const int iw = iw0 + j;
      wok[j] = rok && (unsigned)iw < (unsigned)a.W;
      float4 v = __ldg(reinterpret_cast<const float4*>(rowp + (wok[j] ? iw : 0) * a.in_sw));
      if (a.pre_relu) v = relu1(v);
      win[j] = (wok[j] || mx) ? v : splat(0.f, float4{});
    }
#pragma unroll
    for (int y = 0; y < TH; ++y) {
      const int r = ir - y * SW;  // tap row of this input row for output row y
      if (r < 0 || r >= KS) continue;
#pragma unroll
      for (int tp = 0; tp < KS; ++tp) {
        if (KIND == 0) {
          const float4 w = ld_tap(a.w + (r * KS + tp) * a.C + c);
#pragma unroll
          for (int x = 0; x < PX; ++x) fma_acc(acc[y][x], win[x * SW + tp], w);
        } else if (mx) {
#pragma unroll
          for (int x = 0; x < PX; ++x)
            if (wok[x * SW + tp]) max_to(acc[y][x], win[x * SW + tp]);
        } else {
#pragma unroll
          for (int x = 0; x < PX; ++x) add_to(acc[y][x], win[x * SW + tp]);
        }
      }
    }
  }
  const float4 bias = (KIND == 0 && a.bias) ? __ldg(reinterpret_cast<const float4*>(a.bias + c)) : splat(0.f, float4{});
#pragma unroll
  for (int y = 0; y < TH; ++y) {
    const int p = p0 + y;
    if (p >= a.P) break;
#pragma unroll
    for (int x = 0; x < PX; ++x) {
      const int q = q0 + x;
      if (q >= a.Q) break;
      float4 v = acc[y][x];
      if (KIND == 0) {
        add_to(v, bias);
      } else if (avg) {
        const int ihs = p * a.sh - a.ph, iws = q * a.sw - a.pw;
        int div;
        if (a.count_pad) {  // torch: window clipped to [-pad, H + pad_bottom)
          const int he = min(ihs + KS, a.H + a.pad_b), we = min(iws + KS, a.W + a.pad_r);
          div = (he - ihs) * (we - iws);
        } else {
          const int hl = max(ihs, 0), hh = min(ihs + KS, a.H), wl = max(iws, 0), wh = min(iws + KS, a.W);
          div = max(hh - hl, 0) * max(wh - wl, 0);
        }
        scale(v, div > 0 ? 1.f / (float)div : 0.f);
        if (a.mul != 1.f) scale(v, a.mul);
      } else if (a.mul != 1.f) {
        scale(v, a.mul);
      }
      if (a.has_res) add_to(v, __ldg(reinterpret_cast<const float4*>(a.res + n * a.res_sn + p * a.res_sh + q * a.res_sw + c)));
      *reinterpret_cast<float4*>(a.out + n * a.out_sn + p * a.out_sh + q * a.out_sw + c) = actv(v, a.act);
    }
  }
}

template <int KIND>
static int launch_rows(const sw_op_desc& op, void* stream) {
  SpatialArgs a = spatial_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (!can_vec4(a, op, KIND == 0) || a.R != a.S || a.sh != a.sw) return (int)cudaErrorInvalidValue;
  const int ks = a.R, s = a.sh;
  // blocks sized to stay within 128 registers (2 CTAs x 256 threads per SM)
  const int TH = (s == 2 && ks == 7) ? 1 : 2;
  const int PX = (s == 1 && ks <= 5) ? 4 : 2;
  const int bands = (a.P + TH - 1) / TH, cols = (a.Q + PX - 1) / PX;
  const int64_t total = (int64_t)a.N * bands * cols * (a.C / 4);
  if (total == 0) return 0;
  if (total >= (int64_t(1) << 31)) return (int)cudaErrorInvalidValue;
  const int blocks = (int)cdiv(total, 256);
#define SW_ROWS(K_, S_, TH_, PX_)                                                                                \
  if (ks == K_ && s == S_)                                                                                      \
    return (int)launch_k(spatial_rows_kernel<KIND, K_, S_, TH_, PX_>, dim3(blocks), dim3(256), 0, st, 1, a, total, \
                         bands, cols);
  SW_ROWS(3, 1, 2, 4) SW_ROWS(5, 1, 2, 4) SW_ROWS(7, 1, 2, 2)
  SW_ROWS(3, 2, 2, 2) SW_ROWS(5, 2, 2, 2) SW_ROWS(7, 2, 1, 2)
#undef SW_ROWS
  return (int)cudaErrorInvalidValue;
}

int launch_dwconv(const sw_op_desc& op, void* stream) {
  return op.variant == 1 ? launch_rows<0>(op, stream) : launch_spatial<0>(op, stream);
}
int launch_pool(const sw_op_desc& op, void* stream) {
  if (op.variant == 2) return launch_pool_rows(op, stream);  // sep_rows.cu: row-staged, thin wide maps
  return op.variant == 1 ? launch_rows<1>(op, stream) : launch_spatial<1>(op, stream);
}

}  // namespace sw
