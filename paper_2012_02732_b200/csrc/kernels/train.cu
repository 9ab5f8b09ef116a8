// Training kernels (sm_100a) for the AoT training step (paper_2012_02732_b200/train.py).
//
// Nimble captures a whole training iteration — forward, loss, backward,
// gradient allreduce, optimizer — as one CUDA graph.  The
// forward convolutions reuse the inference kernels (conv.cu, spatial.cu); this
// file adds what only training needs:
//
//   bn_reduce_kernel     batch statistics / dgamma,dbeta: per-channel sums over
//                        the N*H*W pixels of an NHWC map.  Channel-contiguous
//                        rows are read coalesced; every CTA writes its partial
//                        sums (fp64) to a private workspace and the last CTA to
//                        arrive (atomic ticket) reduces them in a FIXED order —
//                        deterministic, one launch, no second pass.
//   bn_apply_kernel      normalise + affine (+ residual) + activation, float4.
//   bn_bwd_apply_kernel  dx of batch norm (+ accumulate), float4.
//   dw_dgrad_kernel      depthwise transposed conv (gather form), 4 channels/thread.
//   dw_wgrad_kernel      depthwise weight gradient: per-CTA pixel slab, R*S
//                        register accumulators per channel, ticket reduce.
//   gemm_kernel          C = A·B (+bias) (+res) with arbitrary strides or an
//                        implicit-im2col B (dense-conv weight gradient), 64x64
//                        tiles, split-K over gridDim.z with a ticket reduce.
//                        Serves 1x1 dgrad (NN), 1x1 / Linear / stem wgrad (TN).
//   xent_kernel          softmax cross-entropy mean loss + dlogits (one CTA).
//   sgd_kernel           torch.optim.SGD (momentum, weight decay) over the flat
//                        parameter buffer, float4.
//   ew_bwd_kernel        activation backward and broadcast-mul backward
//                        (EfficientNet squeeze-excite).
//
// All kernels follow the engine's PDL protocol (trigger, then wait before the
// first dependent read) so they can sit on programmatic edges.
#include <cuda_runtime.h>

#include <cstring>

#include "common.cuh"

namespace sw {

namespace {

__host__ __device__ __forceinline__ float bits_f(int64_t b) {
  const int32_t i = (int32_t)b;
  float f;
  memcpy(&f, &i, 4);
  return f;
}

__device__ __forceinline__ float act_grad(float z, int act) {
  switch (act) {
    case ACT_RELU: return z > 0.f ? 1.f : 0.f;
    case ACT_RELU6: return (z > 0.f && z < 6.f) ? 1.f : 0.f;
    case ACT_SILU: {
      const float s = 1.f / (1.f + expf(-z));
      return s * (1.f + z * (1.f - s));
    }
    case ACT_SIGMOID: {
      const float s = 1.f / (1.f + expf(-z));
      return s * (1.f - s);
    }
    default: return 1.f;
  }
}

constexpr int kNT = 256;

// Channel tile of the per-channel reductions: one warp spans 32 consecutive
// channels of a row (128-B coalesced), the 8 warps of a CTA are row lanes, and
// channel blocks go to grid.y.  (Wider tiles left one lane per channel and
// made the last-CTA partial reduction serial: 50 µs for a 2048x144 map.)
__host__ __device__ __forceinline__ int chan_tile(int) { return 32; }

// ---------------------------------------------------------------------------
// batch-norm reductions
// ---------------------------------------------------------------------------
struct BnArgs {
  const float* dout;
  const float* y;
  float* stats;         // [mean C | invstd C]
  float* running;       // [mean C | var C]
  const float* gamma;   // [gamma C | beta C]
  float* dgamma;        // [dgamma C | dbeta C]
  const float* res;
  float* out;
  double* ws;           // [grid][2][C] partials, then the ticket
  int64_t M, C, HW, ld, do_sn, do_sp;
  int act, has_res, grid;
  float eps, momentum, do_scale;
};

// MODE 0: batch statistics of y.  MODE 1: dgamma / dbeta from dOut.
// Grid: x = row blocks (a.grid), y = channel blocks of TC channels.  Each
// thread keeps kU independent row loads in flight (a serial dependent row loop
// was latency-bound: 86 µs for 128x576); the last CTA of a channel block
// reduces the row-block partials with all its threads, in a fixed order.
constexpr int kU = 4;

template <int MODE>
__global__ void __launch_bounds__(kNT) bn_reduce_kernel(BnArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[2][kNT];
  __shared__ bool last;
  const int C = (int)a.C;
  const int TC = chan_tile(C);
  const int RL = kNT / TC;
  const int lane_c = threadIdx.x % TC, lane_r = threadIdx.x / TC;
  const int gx = gridDim.x;
  const int64_t rows = (a.M + gx - 1) / gx;
  const int64_t m0 = blockIdx.x * rows, m1 = min(a.M, m0 + rows);
  const int c = blockIdx.y * TC + lane_c;
  float s0 = 0.f, s1 = 0.f;
  if (c < C) {
    float mean = 0.f, istd = 0.f, g = 0.f, b = 0.f;
    if (MODE == 1) {
      mean = a.stats[c];
      istd = a.stats[C + c];
      g = a.gamma[c];
      b = a.gamma[C + c];
    }
    for (int64_t mb = m0 + lane_r; mb < m1; mb += (int64_t)RL * kU) {
      float v[kU], d[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t m = mb + (int64_t)u * RL;
        v[u] = 0.f;
        d[u] = 0.f;
        if (m < m1) {
          v[u] = a.y[m * a.ld + c];
          if (MODE == 1) {
            const int64_t n = m / a.HW, p = m - n * a.HW;
            d[u] = a.dout[n * a.do_sn + p * a.do_sp + c];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (MODE == 0) {
          s0 += v[u];
          s1 += v[u] * v[u];
        } else {
          const float xh = (v[u] - mean) * istd;
          const float dd = d[u] * a.do_scale;
          const float dz = a.act == ACT_NONE ? dd : dd * act_grad(g * xh + b, a.act);
          s0 += dz;
          s1 += dz * xh;  // rows past m1 contribute dz = 0
        }
      }
    }
  }
  red[0][threadIdx.x] = s0;
  red[1][threadIdx.x] = s1;
  __syncthreads();
  if (lane_r == 0 && c < C) {
    double t0 = 0.0, t1 = 0.0;
    for (int r = 0; r < RL; ++r) {
      t0 += red[0][r * TC + lane_c];
      t1 += red[1][r * TC + lane_c];
    }
    double* part = a.ws + (int64_t)blockIdx.x * 2 * C;
    part[c] = t0;
    part[C + c] = t1;
  }
  __threadfence();
  __syncthreads();
  unsigned* ticket = reinterpret_cast<unsigned*>(a.ws + (int64_t)gx * 2 * C) + blockIdx.y;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (unsigned)(gx - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // all threads: lane_r strides over the row-block partials of channel c
  double t0 = 0.0, t1 = 0.0;
  if (c < C) {
    const volatile double* pw = a.ws;
#pragma unroll 4
    for (int g = lane_r; g < gx; g += RL) {
      t0 += pw[(int64_t)g * 2 * C + c];
      t1 += pw[(int64_t)g * 2 * C + C + c];
    }
  }
  __syncthreads();
  red[0][threadIdx.x] = t0;
  red[1][threadIdx.x] = t1;
  __syncthreads();
  if (lane_r == 0 && c < C) {
    t0 = 0.0;
    t1 = 0.0;
    for (int r = 0; r < RL; ++r) {
      t0 += red[0][r * TC + lane_c];
      t1 += red[1][r * TC + lane_c];
    }
    if (MODE == 0) {
      const double mean = t0 / (double)a.M;
      double var = t1 / (double)a.M - mean * mean;
      if (var < 0.0) var = 0.0;
      a.stats[c] = (float)mean;
      a.stats[C + c] = (float)(1.0 / sqrt(var + (double)a.eps));
      if (a.running) {
        const double unb = a.M > 1 ? var * (double)a.M / (double)(a.M - 1) : var;
        a.running[c] = (float)((1.0 - a.momentum) * a.running[c] + a.momentum * mean);
        a.running[C + c] = (float)((1.0 - a.momentum) * a.running[C + c] + a.momentum * unb);
      }
    } else {
      a.dgamma[c] = (float)t1;
      a.dgamma[C + c] = (float)t0;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;  // ready for the next replay
}

// Fused batch norm (MODE 0 forward: statistics + normalise; MODE 1 backward:
// dgamma/dbeta + dx).  Phase 1 is bn_reduce_kernel's partial sums; then the
// gx CTAs of a channel block meet at a barrier (atomic arrive counter, spin
// bounded by a trap so a broken co-residency assumption fails loudly instead
// of hanging), every CTA folds the gx partials of its 32 channels itself
// (fixed order, fp64: no second barrier), CTA 0 of the block publishes the
// statistics / parameter gradients, and phase 3 runs the elementwise pass on
// the CTA's own rows while they are still in L2.  One launch instead of two
// on the training step's critical chain.
__device__ __forceinline__ void block_barrier(unsigned* arrive, unsigned expected) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(arrive, 1u);
    unsigned spins = 0;
    while (atomicAdd(arrive, 0u) < expected) {
      if (++spins > (1u << 28)) __trap();
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <int MODE>
__global__ void __launch_bounds__(kNT) bn_fused_kernel(BnArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[2][kNT];
  __shared__ float fin[4][32];  // mean / istd (fwd) or dgamma / dbeta (bwd) of the block's channels
  const int C = (int)a.C;
  constexpr int TC = 32, RL = kNT / TC;
  const int lane_c = threadIdx.x % TC, lane_r = threadIdx.x / TC;
  const int gx = gridDim.x;
  const int64_t rows = (a.M + gx - 1) / gx;
  const int64_t m0 = blockIdx.x * rows, m1 = min(a.M, m0 + rows);
  const int c = blockIdx.y * TC + lane_c;
  float mean = 0.f, istd = 0.f, g = 0.f, b = 0.f;
  if (c < C) {
    g = a.gamma[c];
    b = a.gamma[C + c];
    if (MODE == 1) {
      mean = a.stats[c];
      istd = a.stats[C + c];
    }
  }
  // ---- phase 1: partial sums of this CTA's rows ----
  float s0 = 0.f, s1 = 0.f;
  if (c < C) {
    for (int64_t mb = m0 + lane_r; mb < m1; mb += (int64_t)RL * kU) {
      float v[kU], d[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t m = mb + (int64_t)u * RL;
        v[u] = 0.f;
        d[u] = 0.f;
        if (m < m1) {
          v[u] = a.y[m * a.ld + c];
          if (MODE == 1) {
            const int64_t n = m / a.HW, p = m - n * a.HW;
            d[u] = a.dout[n * a.do_sn + p * a.do_sp + c];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (MODE == 0) {
          s0 += v[u];
          s1 += v[u] * v[u];
        } else {
          const float xh = (v[u] - mean) * istd;
          const float dd = d[u] * a.do_scale;
          const float dz = a.act == ACT_NONE ? dd : dd * act_grad(g * xh + b, a.act);
          s0 += dz;
          s1 += dz * xh;
        }
      }
    }
  }
  red[0][threadIdx.x] = s0;
  red[1][threadIdx.x] = s1;
  __syncthreads();
  if (lane_r == 0 && c < C) {
    double t0 = 0.0, t1 = 0.0;
    for (int r = 0; r < RL; ++r) {
      t0 += red[0][r * TC + lane_c];
      t1 += red[1][r * TC + lane_c];
    }
    double* part = a.ws + (int64_t)blockIdx.x * 2 * C;
    part[c] = t0;
    part[C + c] = t1;
  }
  // ---- phase 2: barrier of the channel block, every CTA folds the partials ----
  unsigned* arrive = reinterpret_cast<unsigned*>(a.ws + (int64_t)gx * 2 * C) + 2 * blockIdx.y;
  unsigned* leave = arrive + 1;
  block_barrier(arrive, (unsigned)gx);
  double t0 = 0.0, t1 = 0.0;
  if (c < C) {
    const volatile double* pw = a.ws;
#pragma unroll 4
    for (int gi = lane_r; gi < gx; gi += RL) {
      t0 += pw[(int64_t)gi * 2 * C + c];
      t1 += pw[(int64_t)gi * 2 * C + C + c];
    }
  }
  __syncthreads();
  red[0][threadIdx.x] = t0;
  red[1][threadIdx.x] = t1;
  __syncthreads();
  if (lane_r == 0) {
    double u0 = 0.0, u1 = 0.0;
    for (int r = 0; r < RL; ++r) {
      u0 += red[0][r * TC + lane_c];
      u1 += red[1][r * TC + lane_c];
    }
    if (MODE == 0) {
      const double mu = u0 / (double)a.M;
      double var = u1 / (double)a.M - mu * mu;
      if (var < 0.0) var = 0.0;
      fin[0][lane_c] = (float)mu;
      fin[1][lane_c] = (float)(1.0 / sqrt(var + (double)a.eps));
      if (blockIdx.x == 0 && c < C) {
        a.stats[c] = fin[0][lane_c];
        a.stats[C + c] = fin[1][lane_c];
        if (a.running) {
          const double unb = a.M > 1 ? var * (double)a.M / (double)(a.M - 1) : var;
          a.running[c] = (float)((1.0 - a.momentum) * a.running[c] + a.momentum * mu);
          a.running[C + c] = (float)((1.0 - a.momentum) * a.running[C + c] + a.momentum * unb);
        }
      }
    } else {
      fin[2][lane_c] = (float)u1;  // dgamma
      fin[3][lane_c] = (float)u0;  // dbeta
      if (blockIdx.x == 0 && c < C) {
        a.dgamma[c] = (float)u1;
        a.dgamma[C + c] = (float)u0;
      }
    }
  }
  __syncthreads();
  // ---- phase 3: elementwise over this CTA's rows ----
  if (c < C) {
    if (MODE == 0) {
      mean = fin[0][lane_c];
      istd = fin[1][lane_c];
    }
    const float invM = 1.f / (float)a.M;
    const float dg = MODE == 1 ? fin[2][lane_c] * invM : 0.f, db = MODE == 1 ? fin[3][lane_c] * invM : 0.f;
    for (int64_t mb = m0 + lane_r; mb < m1; mb += (int64_t)RL * kU) {
      float yv[kU], dv[kU], rv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // all loads of the kU rows in flight first
        const int64_t m = mb + (int64_t)u * RL;
        yv[u] = dv[u] = rv[u] = 0.f;
        if (m < m1) {
          yv[u] = a.y[m * a.ld + c];
          if (a.has_res) rv[u] = a.res[m * a.ld + c];
          if (MODE == 1) {
            const int64_t n = m / a.HW, p = m - n * a.HW;
            dv[u] = a.dout[n * a.do_sn + p * a.do_sp + c];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t m = mb + (int64_t)u * RL;
        if (m >= m1) break;
        const float xh = (yv[u] - mean) * istd;
        float o;
        if (MODE == 0) {
          o = apply_act(g * xh + b + rv[u], a.act);
        } else {
          const float d = dv[u] * a.do_scale;
          const float dz = a.act == ACT_NONE ? d : d * act_grad(g * xh + b, a.act);
          o = g * istd * (dz - db - xh * dg) + rv[u];
        }
        a.out[m * a.ld + c] = o;
      }
    }
  }
  // the last CTA of the block to leave resets both counters for the next replay
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(leave, 1u) == (unsigned)(gx - 1)) {
      *arrive = 0u;
      *leave = 0u;
      __threadfence();
    }
  }
}

// out = act(gamma * (y - mean) * invstd + beta (+ res))
__global__ void __launch_bounds__(kNT) bn_apply_kernel(BnArgs a) {
  pdl_trigger();
  pdl_wait();
  const int C = (int)a.C;
  const int64_t total = a.M * C;
  const bool v4 = (C & 3) == 0 && (a.ld & 3) == 0;
  if (v4) {
    const int64_t tot4 = total / 4;
    for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < tot4; i += (int64_t)gridDim.x * kNT) {
      const int64_t e = i * 4;
      const int64_t m = e / C;
      const int c = (int)(e - m * C);
      const float4 v = *reinterpret_cast<const float4*>(a.y + m * a.ld + c);
      const float4 mu = *reinterpret_cast<const float4*>(a.stats + c);
      const float4 is = *reinterpret_cast<const float4*>(a.stats + C + c);
      const float4 g = *reinterpret_cast<const float4*>(a.gamma + c);
      const float4 b = *reinterpret_cast<const float4*>(a.gamma + C + c);
      float4 o = make_float4(g.x * (v.x - mu.x) * is.x + b.x, g.y * (v.y - mu.y) * is.y + b.y,
                             g.z * (v.z - mu.z) * is.z + b.z, g.w * (v.w - mu.w) * is.w + b.w);
      if (a.has_res) o = f4add(o, *reinterpret_cast<const float4*>(a.res + m * a.ld + c));
      *reinterpret_cast<float4*>(a.out + m * a.ld + c) = act4(o, a.act);
    }
  } else {
    for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
      const int64_t m = e / C;
      const int c = (int)(e - m * C);
      float o = a.gamma[c] * (a.y[m * a.ld + c] - a.stats[c]) * a.stats[C + c] + a.gamma[C + c];
      if (a.has_res) o += a.res[m * a.ld + c];
      a.out[m * a.ld + c] = apply_act(o, a.act);
    }
  }
}

// dy = gamma*invstd*(dz - dbeta/M - xhat*dgamma/M) (+ res), dz = dOut*act'(z)
__global__ void __launch_bounds__(kNT) bn_bwd_apply_kernel(BnArgs a) {
  pdl_trigger();
  pdl_wait();
  const int C = (int)a.C;
  const int64_t total = a.M * C;
  const float invM = 1.f / (float)a.M;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    const int64_t m = e / C;
    const int c = (int)(e - m * C);
    const float mean = a.stats[c], istd = a.stats[C + c];
    const float g = a.gamma[c], b = a.gamma[C + c];
    const float xh = (a.y[m * a.ld + c] - mean) * istd;
    const int64_t n = m / a.HW, p = m - n * a.HW;
    const float d = a.dout[n * a.do_sn + p * a.do_sp + c] * a.do_scale;
    const float dz = a.act == ACT_NONE ? d : d * act_grad(g * xh + b, a.act);
    float dy = g * istd * (dz - a.dgamma[C + c] * invM - xh * a.dgamma[c] * invM);
    if (a.has_res) dy += a.res[m * a.ld + c];
    a.out[m * a.ld + c] = dy;
  }
}

BnArgs bn_args(const sw_op_desc& d) {
  BnArgs a{};
  const int64_t* p = d.params;
  a.M = p[BN_M];
  a.C = p[BN_C];
  a.HW = p[BN_HW] > 0 ? p[BN_HW] : 1;
  a.act = (int)p[BN_ACT];
  a.has_res = (int)p[BN_HAS_RES];
  a.eps = bits_f(p[BN_EPS]);
  a.momentum = bits_f(p[BN_MOMENTUM]);
  a.grid = (int)(p[BN_GRID] > 0 ? p[BN_GRID] : 1);
  a.do_sn = p[BN_DO_SN];
  a.do_sp = p[BN_DO_SP];
  a.do_scale = p[BN_DO_SCALE] ? bits_f(p[BN_DO_SCALE]) : 1.f;
  a.ld = p[BN_LD] > 0 ? p[BN_LD] : a.C;
  return a;
}

int elementwise_grid(int64_t work) {
  int64_t g = cdiv(work, kNT);
  return (int)(g < 1 ? 1 : (g > 148 * 8 ? 148 * 8 : g));
}

// ---------------------------------------------------------------------------
// depthwise backward
// ---------------------------------------------------------------------------
struct DwArgs {
  const float* dy;
  const float* x;
  const float* w;
  const float* res;
  float* out;
  float* ws;
  int N, H, W, C, P, Q, R, S, sh, sw, ph, pw, has_res, grid;
};

DwArgs dw_args(const sw_op_desc& d) {
  const int64_t* p = d.params;
  DwArgs a{};
  a.N = (int)p[SP_N];
  a.H = (int)p[SP_H];
  a.W = (int)p[SP_W];
  a.C = (int)p[SP_C];
  a.P = (int)p[SP_P];
  a.Q = (int)p[SP_Q];
  a.R = (int)p[SP_R];
  a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H];
  a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H];
  a.pw = (int)p[SP_PAD_W];
  a.has_res = (int)p[SP_HAS_RES];
  a.grid = (int)(p[SP_SPLIT_K] > 0 ? p[SP_SPLIT_K] : 1);
  return a;
}

// dX[n,h,w,c] = sum_{r,s} W[r,s,c] dY[n,(h+ph-r)/sh,(w+pw-s)/sw,c]  (exact division only)
template <int V>
__global__ void __launch_bounds__(kNT) dw_dgrad_kernel(DwArgs a) {
  pdl_trigger();
  pdl_wait();
  const int CG = a.C / V;
  const int64_t total = (int64_t)a.N * a.H * a.W * CG;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < total; i += (int64_t)gridDim.x * kNT) {
    const int c = (int)(i % CG) * V;
    int64_t pix = i / CG;
    const int w = (int)(pix % a.W);
    pix /= a.W;
    const int h = (int)(pix % a.H);
    const int n = (int)(pix / a.H);
    float acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.f;
    for (int r = 0; r < a.R; ++r) {
      const int th = h + a.ph - r;
      if (th < 0 || th % a.sh) continue;
      const int pp = th / a.sh;
      if (pp >= a.P) continue;
      for (int s = 0; s < a.S; ++s) {
        const int tw = w + a.pw - s;
        if (tw < 0 || tw % a.sw) continue;
        const int qq = tw / a.sw;
        if (qq >= a.Q) continue;
        const float* g = a.dy + (((int64_t)n * a.P + pp) * a.Q + qq) * a.C + c;
        const float* wt = a.w + (r * a.S + s) * a.C + c;
        if (V == 4) {
          const float4 gv = *reinterpret_cast<const float4*>(g);
          const float4 wv = *reinterpret_cast<const float4*>(wt);
          acc[0] += gv.x * wv.x;
          acc[1 % V] += gv.y * wv.y;
          acc[2 % V] += gv.z * wv.z;
          acc[3 % V] += gv.w * wv.w;
        } else {
          acc[0] += g[0] * wt[0];
        }
      }
    }
    float* o = a.out + (((int64_t)n * a.H + h) * a.W + w) * a.C + c;
    if (V == 4) {
      float4 v = make_float4(acc[0], acc[1 % V], acc[2 % V], acc[3 % V]);
      if (a.has_res) v = f4add(v, *reinterpret_cast<const float4*>(a.res + (o - a.out)));
      *reinterpret_cast<float4*>(o) = v;
    } else {
      o[0] = acc[0] + (a.has_res ? a.res[o - a.out] : 0.f);
    }
  }
}

// dW[r,s,c] = sum_{n,p,q} dY[n,p,q,c] X[n, p*sh-ph+r, q*sw-pw+s, c]
// Grid: x = output-pixel blocks (a.grid), y = channel blocks of TC.  Each thread
// holds KS*KS accumulators for its channel; the last CTA of a channel block
// reduces the partials [gx][KS*KS][C] in a fixed order with all threads.
template <int KS>
__global__ void __launch_bounds__(kNT) dw_wgrad_kernel(DwArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ bool last;
  extern __shared__ float red[];  // [RL][KS*KS][TC] when RL > 1
  const int C = a.C;
  const int TC = chan_tile(C);
  const int RL = kNT / TC;
  const int lane_c = threadIdx.x % TC, lane_r = threadIdx.x / TC;
  const int gx = gridDim.x;
  const int64_t M = (int64_t)a.N * a.P * a.Q;
  const int64_t rows = (M + gx - 1) / gx;
  const int64_t m0 = blockIdx.x * rows, m1 = min(M, m0 + rows);
  const int c = blockIdx.y * TC + lane_c;
  float* part = a.ws + (int64_t)blockIdx.x * KS * KS * C;
  float acc[KS * KS];
#pragma unroll
  for (int k = 0; k < KS * KS; ++k) acc[k] = 0.f;
  if (c < C) {
    for (int64_t m = m0 + lane_r; m < m1; m += RL) {
      const int q = (int)(m % a.Q);
      const int64_t t = m / a.Q;
      const int p = (int)(t % a.P);
      const int n = (int)(t / a.P);
      const float g = a.dy[m * C + c];
      const int h0 = p * a.sh - a.ph, w0 = q * a.sw - a.pw;
      const float* xb = a.x + (int64_t)n * a.H * a.W * C + c;
#pragma unroll
      for (int r = 0; r < KS; ++r) {
        const int h = h0 + r;
        const bool hv = h >= 0 && h < a.H;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const int w = w0 + s;
          const bool ok = hv && w >= 0 && w < a.W;
          const float xv = ok ? xb[((int64_t)h * a.W + w) * C] : 0.f;
          acc[r * KS + s] += g * xv;
        }
      }
    }
  }
  if (RL > 1) {
#pragma unroll
    for (int k = 0; k < KS * KS; ++k) red[(lane_r * KS * KS + k) * TC + lane_c] = acc[k];
    __syncthreads();
    if (lane_r == 0 && c < C) {
      for (int k = 0; k < KS * KS; ++k) {
        float t = 0.f;
        for (int r = 0; r < RL; ++r) t += red[(r * KS * KS + k) * TC + lane_c];
        part[k * C + c] = t;
      }
    }
  } else if (c < C) {
#pragma unroll
    for (int k = 0; k < KS * KS; ++k) part[k * C + c] = acc[k];
  }
  __threadfence();
  __syncthreads();
  unsigned* ticket = reinterpret_cast<unsigned*>(a.ws + (int64_t)gx * KS * KS * C) + blockIdx.y;
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == (unsigned)(gx - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int c0 = blockIdx.y * TC;
  const int cw = min(TC, C - c0);
  const volatile float* pw = a.ws;
  for (int i = threadIdx.x; i < KS * KS * cw; i += kNT) {
    const int k = i / cw, cc = c0 + i % cw;
    double t = 0.0;
#pragma unroll 4
    for (int g = 0; g < gx; ++g) t += (double)pw[(int64_t)g * KS * KS * C + k * C + cc];
    a.out[k * C + cc] = (float)t;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// ---------------------------------------------------------------------------
// strided / implicit-im2col GEMM with deterministic split-K
// ---------------------------------------------------------------------------
struct GemmArgs {
  const float* A;
  const float* B;
  float* Cp;
  const float* bias;
  const float* res;
  float* ws;
  int64_t M, N, K, a_i, a_r, b_r, b_j, c_i;
  int split, has_res, im2col, partials_only;
  int xN, xH, xW, xC, xP, xQ, xR, xS, xst, xpad;
  int64_t xsn, xsh, xsw, xsc;
};

constexpr int GBM = 64, GBN = 64, GBK = 16;

__device__ __forceinline__ float gemm_b(const GemmArgs& g, int64_t r, int64_t j) {
  if (!g.im2col) return g.B[r * g.b_r + j * g.b_j];
  // r = output pixel (n,p,q); j = (rr, ss, c) of a [K][R][S][C] weight
  const int q = (int)(r % g.xQ);
  const int64_t t = r / g.xQ;
  const int p = (int)(t % g.xP);
  const int n = (int)(t / g.xP);
  const int c = (int)(j % g.xC);
  const int64_t u = j / g.xC;
  const int ss = (int)(u % g.xS), rr = (int)(u / g.xS);
  const int h = p * g.xst - g.xpad + rr, w = q * g.xst - g.xpad + ss;
  if (h < 0 || h >= g.xH || w < 0 || w >= g.xW) return 0.f;
  return g.B[n * g.xsn + h * g.xsh + w * g.xsw + c * g.xsc];
}

__global__ void __launch_bounds__(kNT) gemm_kernel(GemmArgs g) {
  pdl_trigger();
  pdl_wait();
  __shared__ float As[GBK][GBM + 4];
  __shared__ float Bs[GBK][GBN + 4];
  __shared__ bool last;
  const int tid = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.y * GBM, j0 = (int64_t)blockIdx.x * GBN;
  const int64_t kchunk = ((g.K + g.split - 1) / g.split + GBK - 1) / GBK * GBK;
  const int64_t kb = blockIdx.z * kchunk, ke = min(g.K, kb + kchunk);
  const bool a_fast_i = g.a_i <= g.a_r;  // which A index is contiguous
  const bool b_fast_j = g.im2col || g.b_j <= g.b_r;
  const int tx = tid % 16, ty = tid / 16;  // 16 x 16 threads, 4x4 outputs each
  float acc[4][4] = {};
  // register-staged prefetch: the next K tile's global loads are in flight
  // while the current tile is multiplied out of shared memory
  float ra[4], rb[4];
  int ai[4], ak[4], bj[4], bk[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int e = tid + l * kNT;  // 0..1023 over the 64x16 tile
    if (a_fast_i) { ai[l] = e % GBM; ak[l] = e / GBM; } else { ak[l] = e % GBK; ai[l] = e / GBK; }
    if (b_fast_j) { bj[l] = e % GBN; bk[l] = e / GBN; } else { bk[l] = e % GBK; bj[l] = e / GBK; }
  }
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int64_t gi = i0 + ai[l], gk = k0 + ak[l];
      ra[l] = (gi < g.M && gk < ke) ? g.A[gi * g.a_i + gk * g.a_r] : 0.f;
      const int64_t gj = j0 + bj[l], gk2 = k0 + bk[l];
      rb[l] = (gj < g.N && gk2 < ke) ? gemm_b(g, gk2, gj) : 0.f;
    }
  };
  if (kb < ke) fetch(kb);
  for (int64_t k0 = kb; k0 < ke; k0 += GBK) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      As[ak[l]][ai[l]] = ra[l];
      Bs[bk[l]][bj[l]] = rb[l];
    }
    __syncthreads();
    if (k0 + GBK < ke) fetch(k0 + GBK);
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = As[kk][ty + 16 * u];
        bv[u] = Bs[kk][tx + 16 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] += av[u] * bv[v];
    }
    __syncthreads();
  }
  if (g.split > 1) {
    const int tiles = gridDim.x * gridDim.y;
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    float* part = g.ws + ((int64_t)tile * g.split + blockIdx.z) * GBM * GBN;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) part[(ty + 16 * u) * GBN + tx + 16 * v] = acc[u][v];
    if (g.partials_only) return;  // folded by the K_GEMM_REDUCE task that follows
    __threadfence();
    __syncthreads();
    unsigned* ticket = reinterpret_cast<unsigned*>(g.ws + (int64_t)tiles * g.split * GBM * GBN) + tile;
    if (tid == 0) last = atomicAdd(ticket, 1u) == (unsigned)(g.split - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    const volatile float* base = g.ws + (int64_t)tile * g.split * GBM * GBN;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        float t = 0.f;
        for (int z = 0; z < g.split; ++z) t += base[(int64_t)z * GBM * GBN + (ty + 16 * u) * GBN + tx + 16 * v];
        acc[u][v] = t;
      }
    if (tid == 0) *ticket = 0u;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t gi = i0 + ty + 16 * u;
    if (gi >= g.M) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t gj = j0 + tx + 16 * v;
      if (gj >= g.N) continue;
      float o = acc[u][v];
      if (g.bias) o += g.bias[gj];
      if (g.has_res) o += g.res[gi * g.c_i + gj];
      g.Cp[gi * g.c_i + gj] = o;
    }
  }
}

// Folds wide split-K partials: a CTA owns 32 consecutive outputs (lane) and
// 8 partial lanes (warp) that stride over the splits; fixed-order smem tree.
__global__ void __launch_bounds__(kNT) gemm_reduce_kernel(GemmArgs g) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lane;
  const int64_t tiles_n = (g.N + GBN - 1) / GBN;
  float t = 0.f;
  const bool ok = e < g.M * g.N;
  int64_t i = 0, j = 0;
  if (ok) {
    i = e / g.N;
    j = e - i * g.N;
    const int64_t tile = (i / GBM) * tiles_n + j / GBN;
    const float* base = g.ws + tile * g.split * GBM * GBN + (i % GBM) * GBN + j % GBN;
#pragma unroll 4
    for (int z = w; z < g.split; z += 8) t += base[(int64_t)z * GBM * GBN];
  }
  red[w][lane] = t;
  __syncthreads();
  if (w == 0 && ok) {
    float o = 0.f;
#pragma unroll
    for (int r = 0; r < 8; ++r) o += red[r][lane];
    if (g.bias) o += g.bias[j];
    if (g.has_res) o += g.res[i * g.c_i + j];
    g.Cp[i * g.c_i + j] = o;
  }
}

// ---------------------------------------------------------------------------
// loss, optimizer, elementwise backward
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kNT) xent_kernel(const float* logits, const int* labels, float* loss,
                                                   float* dlogits, int N, int K, int64_t ld) {
  pdl_trigger();
  pdl_wait();
  __shared__ float lsum[kNT];
  float mine = 0.f;
  for (int n = threadIdx.x; n < N; n += kNT) {
    const float* z = logits + n * ld;
    float mx = -INFINITY;
    for (int k = 0; k < K; ++k) mx = fmaxf(mx, z[k]);
    float se = 0.f;
    for (int k = 0; k < K; ++k) se += expf(z[k] - mx);
    const int y = labels[n];
    mine += logf(se) + mx - z[y];
    const float inv = 1.f / se, invN = 1.f / (float)N;
    for (int k = 0; k < K; ++k) dlogits[n * K + k] = (expf(z[k] - mx) * inv - (k == y ? 1.f : 0.f)) * invN;
  }
  lsum[threadIdx.x] = mine;
  __syncthreads();
  for (int s = kNT / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) lsum[threadIdx.x] += lsum[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = lsum[0] / (float)N;
}

// torch.optim.SGD (dampening 0, nesterov off): g += wd*p; buf = mu*buf + g; p -= lr*buf
// (a zero-initialised buf reproduces torch's first-step buf = g).
__global__ void __launch_bounds__(kNT) sgd_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                  float* __restrict__ buf, int64_t n, float lr, float mu,
                                                  float wd) {
  pdl_trigger();
  pdl_wait();
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)kNT + threadIdx.x; i < n4; i += (int64_t)gridDim.x * kNT) {
    float4 pv = reinterpret_cast<float4*>(p)[i];
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 bv = reinterpret_cast<float4*>(buf)[i];
    bv.x = mu * bv.x + (gv.x + wd * pv.x);
    bv.y = mu * bv.y + (gv.y + wd * pv.y);
    bv.z = mu * bv.z + (gv.z + wd * pv.z);
    bv.w = mu * bv.w + (gv.w + wd * pv.w);
    pv.x -= lr * bv.x;
    pv.y -= lr * bv.y;
    pv.z -= lr * bv.z;
    pv.w -= lr * bv.w;
    reinterpret_cast<float4*>(buf)[i] = bv;
    reinterpret_cast<float4*>(p)[i] = pv;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
    const float b = mu * buf[i] + (g[i] + wd * p[i]);
    buf[i] = b;
    p[i] -= lr * b;
  }
}

struct EwbArgs {
  const float* dy;
  const float* z;
  const float* s;
  const float* res;
  float* out;
  const float* zs;
  int64_t N, HW, C;
  int mode, act, has_res;
  float scale;
};

__global__ void __launch_bounds__(kNT) ew_bwd_kernel(EwbArgs a) {
  pdl_trigger();
  pdl_wait();
  if (a.mode == 2) {
    // ds[n,c] = act'(zs[n,c]) * sum_hw dy*x ; one warp per (n,c)
    const int64_t warp = (blockIdx.x * (int64_t)kNT + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= a.N * a.C) return;
    const int64_t n = warp / a.C, c = warp % a.C;
    float t = 0.f;
    for (int64_t p = lane; p < a.HW; p += 32) {
      const int64_t e = (n * a.HW + p) * a.C + c;
      t += a.dy[e] * a.z[e];
    }
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) {
      if (a.act != ACT_NONE) t *= act_grad(a.zs[n * a.C + c], a.act);
      a.out[n * a.C + c] = t;
    }
    return;
  }
  const int64_t total = a.N * a.HW * a.C;
  for (int64_t e = blockIdx.x * (int64_t)kNT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kNT) {
    float v;
    if (a.mode == 0) {
      v = a.dy[e] * act_grad(a.z[e], a.act);
    } else if (a.mode == 3) {
      const int64_t c = e % a.C, n = e / (a.HW * a.C);
      v = a.s[n * a.C + c] * a.scale;
    } else {
      const int64_t c = e % a.C, n = e / (a.HW * a.C);
      v = a.dy[e] * a.s[n * a.C + c];
    }
    if (a.has_res) v += a.res[e];
    a.out[e] = v;
  }
}

// 32x32 smem-tiled transpose (rows x cols → cols x rows)
__global__ void __launch_bounds__(kNT) transpose_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                        int rows, int cols) {
  pdl_trigger();
  pdl_wait();
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
  for (int i = ty; i < 32; i += 8)
    if (r0 + i < rows && c0 + tx < cols) t[i][tx] = in[(int64_t)(r0 + i) * cols + c0 + tx];
  __syncthreads();
  for (int i = ty; i < 32; i += 8)
    if (c0 + i < cols && r0 + tx < rows) out[(int64_t)(c0 + i) * rows + r0 + tx] = t[tx][i];
}

}  // namespace

int launch_train(const sw_op_desc& d, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t* p = d.params;
  const uint64_t* q = d.ptrs;
  cudaError_t err = cudaSuccess;  // the launch's own status (never a stale error of an earlier call)
  switch (d.kind) {
    case K_BN_STATS:
    case K_BN_BWD_REDUCE: {
      BnArgs a = bn_args(d);
      if (d.kind == K_BN_STATS) {
        a.y = reinterpret_cast<const float*>(q[0]);
        a.stats = reinterpret_cast<float*>(q[1]);
        a.running = reinterpret_cast<float*>(q[2]);
        a.ws = reinterpret_cast<double*>(q[7]);
        err = launch_k(bn_reduce_kernel<0>, dim3(a.grid, (unsigned)cdiv(a.C, chan_tile((int)a.C))), dim3(kNT), 0, st, 1, a);
      } else {
        a.dout = reinterpret_cast<const float*>(q[0]);
        a.y = reinterpret_cast<const float*>(q[1]);
        a.stats = reinterpret_cast<float*>(q[2]);
        a.gamma = reinterpret_cast<const float*>(q[3]);
        a.dgamma = reinterpret_cast<float*>(q[4]);
        a.ws = reinterpret_cast<double*>(q[7]);
        err = launch_k(bn_reduce_kernel<1>, dim3(a.grid, (unsigned)cdiv(a.C, chan_tile((int)a.C))), dim3(kNT), 0, st, 1, a);
      }
      break;
    }
    case K_BN_FWD:
    case K_BN_BWD: {
      BnArgs a = bn_args(d);
      if (d.kind == K_BN_FWD) {
        a.y = reinterpret_cast<const float*>(q[0]);
        a.stats = reinterpret_cast<float*>(q[1]);
        a.running = reinterpret_cast<float*>(q[2]);
        a.gamma = reinterpret_cast<const float*>(q[3]);
        a.res = reinterpret_cast<const float*>(q[4]);
        a.out = reinterpret_cast<float*>(q[5]);
      } else {
        a.dout = reinterpret_cast<const float*>(q[0]);
        a.y = reinterpret_cast<const float*>(q[1]);
        a.stats = reinterpret_cast<float*>(q[2]);
        a.gamma = reinterpret_cast<const float*>(q[3]);
        a.dgamma = reinterpret_cast<float*>(q[4]);
        a.res = reinterpret_cast<const float*>(q[5]);
        a.out = reinterpret_cast<float*>(q[6]);
      }
      a.ws = reinterpret_cast<double*>(q[7]);
      const dim3 grid(a.grid, (unsigned)cdiv(a.C, 32));
      // every CTA of a channel block must be resident at the barrier: cooperative launch
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = grid;
      cfg.blockDim = dim3(kNT);
      cfg.stream = st;
      cudaLaunchAttribute attr[2];
      unsigned na = 0;
      attr[na].id = cudaLaunchAttributeCooperative;
      attr[na].val.cooperative = 1;
      ++na;
      if (g_launch_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
      }
      cfg.attrs = attr;
      cfg.numAttrs = na;
      if (d.kind == K_BN_FWD)
        return (int)cudaLaunchKernelEx(&cfg, bn_fused_kernel<0>, a);
      return (int)cudaLaunchKernelEx(&cfg, bn_fused_kernel<1>, a);
    }
    case K_BN_APPLY: {
      BnArgs a = bn_args(d);
      a.y = reinterpret_cast<const float*>(q[0]);
      a.stats = reinterpret_cast<float*>(q[1]);
      a.gamma = reinterpret_cast<const float*>(q[2]);
      a.res = reinterpret_cast<const float*>(q[3]);
      a.out = reinterpret_cast<float*>(q[4]);
      err = launch_k(bn_apply_kernel, dim3(elementwise_grid(a.M * a.C / 4)), dim3(kNT), 0, st, 1, a);
      break;
    }
    case K_BN_BWD_APPLY: {
      BnArgs a = bn_args(d);
      a.dout = reinterpret_cast<const float*>(q[0]);
      a.y = reinterpret_cast<const float*>(q[1]);
      a.stats = reinterpret_cast<float*>(q[2]);
      a.gamma = reinterpret_cast<const float*>(q[3]);
      a.dgamma = reinterpret_cast<float*>(q[4]);
      a.res = reinterpret_cast<const float*>(q[5]);
      a.out = reinterpret_cast<float*>(q[6]);
      err = launch_k(bn_bwd_apply_kernel, dim3(elementwise_grid(a.M * a.C)), dim3(kNT), 0, st, 1, a);
      break;
    }
    case K_DW_DGRAD: {
      DwArgs a = dw_args(d);
      a.dy = reinterpret_cast<const float*>(q[0]);
      a.out = reinterpret_cast<float*>(q[1]);
      a.w = reinterpret_cast<const float*>(q[2]);
      a.res = reinterpret_cast<const float*>(q[4]);
      const bool v4 = (a.C & 3) == 0 && aligned16(q[0]) && aligned16(q[1]) && aligned16(q[2]) &&
                      (!a.has_res || aligned16(q[4]));
      const int64_t work = (int64_t)a.N * a.H * a.W * (v4 ? a.C / 4 : a.C);
      if (v4)
        err = launch_k(dw_dgrad_kernel<4>, dim3(elementwise_grid(work)), dim3(kNT), 0, st, 1, a);
      else
        err = launch_k(dw_dgrad_kernel<1>, dim3(elementwise_grid(work)), dim3(kNT), 0, st, 1, a);
      break;
    }
    case K_DW_WGRAD: {
      DwArgs a = dw_args(d);
      a.dy = reinterpret_cast<const float*>(q[0]);
      a.out = reinterpret_cast<float*>(q[1]);
      a.x = reinterpret_cast<const float*>(q[2]);
      a.ws = reinterpret_cast<float*>(q[5]);
      if (a.R != a.S) return (int)cudaErrorInvalidValue;
      const int TC = chan_tile(a.C), RL = kNT / TC;
      const size_t smem = RL > 1 ? (size_t)RL * a.R * a.S * TC * sizeof(float) : 0;
      if (a.R == 3)
        err = launch_k(dw_wgrad_kernel<3>, dim3(a.grid, (unsigned)cdiv(a.C, TC)), dim3(kNT), smem, st, 1, a);
      else if (a.R == 5)
        err = launch_k(dw_wgrad_kernel<5>, dim3(a.grid, (unsigned)cdiv(a.C, TC)), dim3(kNT), smem, st, 1, a);
      else
        return (int)cudaErrorInvalidValue;
      break;
    }
    case K_GEMM:
    case K_GEMM_REDUCE: {
      GemmArgs g{};
      g.A = reinterpret_cast<const float*>(q[0]);
      g.B = reinterpret_cast<const float*>(q[1]);
      g.Cp = reinterpret_cast<float*>(q[2]);
      g.bias = reinterpret_cast<const float*>(q[3]);
      g.res = reinterpret_cast<const float*>(q[4]);
      g.ws = reinterpret_cast<float*>(q[5]);
      g.M = p[GM_M];
      g.N = p[GM_N];
      g.K = p[GM_K];
      g.a_i = p[GM_A_I];
      g.a_r = p[GM_A_R];
      g.b_r = p[GM_B_R];
      g.b_j = p[GM_B_J];
      g.c_i = p[GM_C_I];
      g.split = (int)(p[GM_SPLIT] > 0 ? p[GM_SPLIT] : 1);
      g.has_res = (int)p[GM_HAS_RES];
      g.im2col = (int)p[GM_IM2COL];
      g.xN = (int)p[GM_X_N];
      g.xH = (int)p[GM_X_H];
      g.xW = (int)p[GM_X_W];
      g.xC = (int)p[GM_X_C];
      g.xP = (int)p[GM_X_P];
      g.xQ = (int)p[GM_X_Q];
      g.xR = (int)p[GM_X_R];
      g.xS = (int)p[GM_X_S];
      g.xst = (int)p[GM_X_STRIDE];
      g.xpad = (int)p[GM_X_PAD];
      g.xsn = p[GM_X_SN];
      g.xsh = p[GM_X_SH];
      g.xsw = p[GM_X_SW];
      g.xsc = p[GM_X_SC];
      g.partials_only = (int)p[GM_PARTIALS_ONLY];
      if (g.split > 1 && !g.ws) return (int)cudaErrorInvalidValue;
      if (d.kind == K_GEMM_REDUCE) {
        err = launch_k(gemm_reduce_kernel, dim3((unsigned)cdiv(g.M * g.N, 32)), dim3(kNT), 0, st, 1, g);
        break;
      }
      dim3 grid((unsigned)cdiv(g.N, GBN), (unsigned)cdiv(g.M, GBM), (unsigned)g.split);
      err = launch_k(gemm_kernel, grid, dim3(kNT), 0, st, 1, g);
      break;
    }
    case K_XENT:
      err = launch_k(xent_kernel, dim3(1), dim3(kNT), 0, st, 1, reinterpret_cast<const float*>(q[0]),
               reinterpret_cast<const int*>(q[1]), reinterpret_cast<float*>(q[2]),
               reinterpret_cast<float*>(q[3]), (int)p[0], (int)p[1], (int64_t)p[2]);
      break;
    case K_SGD: {
      if (!aligned16(q[0]) || !aligned16(q[1]) || !aligned16(q[2])) return (int)cudaErrorMisalignedAddress;
      const int64_t n = p[0];
      err = launch_k(sgd_kernel, dim3(elementwise_grid(n / 4 + 1)), dim3(kNT), 0, st, 1, reinterpret_cast<float*>(q[0]),
               reinterpret_cast<const float*>(q[1]), reinterpret_cast<float*>(q[2]), n,
               bits_f((int)p[1]), bits_f((int)p[2]), bits_f((int)p[3]));
      break;
    }
    case K_EW_BWD: {
      EwbArgs a{};
      a.N = p[0];
      a.HW = p[1];
      a.C = p[2];
      a.mode = (int)p[3];
      a.act = (int)p[4];
      a.has_res = (int)p[5];
      a.scale = bits_f(p[6]);
      a.dy = reinterpret_cast<const float*>(q[0]);
      a.z = reinterpret_cast<const float*>(q[1]);
      a.s = reinterpret_cast<const float*>(q[2]);
      a.res = reinterpret_cast<const float*>(q[3]);
      a.out = reinterpret_cast<float*>(q[4]);
      a.zs = reinterpret_cast<const float*>(q[5]);
      const int64_t work = a.mode == 2 ? a.N * a.C * 32 : a.N * a.HW * a.C;
      err = launch_k(ew_bwd_kernel, dim3((unsigned)cdiv(work, kNT)), dim3(kNT), 0, st, 1, a);
      break;
    }
    case K_TRANSPOSE: {
      const int rows = (int)p[0], cols = (int)p[1];
      err = launch_k(transpose_kernel, dim3((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32)), dim3(kNT), 0, st, 1,
               reinterpret_cast<const float*>(q[0]), reinterpret_cast<float*>(q[1]), rows, cols);
      break;
    }
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)err;
}

}  // namespace sw
