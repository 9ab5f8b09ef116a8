// Dense convolution / GEMM on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Implicit GEMM: rows = output pixels (M = N*P*Q), columns = output channels,
// K = R*S*C (weights [K][R][S][C]).  One CTA = 128 threads computes a
// 128 x BN tile: the four warps gather the im2col A tile and the weight B
// tile (128-bit loads, K-contiguous in NHWC), split every fp32 value into a
// TF32 pair (hi = rna(x), lo = x - hi) and store both halves into shared
// memory in the canonical K-major, no-swizzle UMMA layout (8-row x 16-byte
// core matrices).  One elected thread issues, per 8-wide K step,
//     D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi      (tcgen05.mma kind::tf32)
// into a TMEM fp32 accumulator (3xTF32: ~fp32 accuracy, which the fp32
// parity gate of rel 1e-3 needs over 50-300 layers).  Stages are
// double buffered: tcgen05.commit arrives on the stage's mbarrier when the
// tensor core has consumed it, so gathering tile k+1 overlaps the MMAs of
// tile k.  The epilogue reads TMEM with tcgen05.ld (warp w owns TMEM lanes
// 32w..32w+31 = tile rows), applies bias (folded BN) + residual + activation
// and stores NHWC / channel-slice / NCHW output.  Split-K uses a cluster of
// CTAs along z whose partial tiles are reduced through DSMEM, exactly like
// the SIMT kernel (conv.cu).
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace sw {

namespace {

struct TcArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w;
  const float* __restrict__ bias;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, pre_relu, has_res;
  int64_t in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  int M, Kdim, split, vec;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SWIZZLE_NONE, K-major canonical layout: core matrix = 8 rows x 16 B;
// SBO = byte stride between 8-row groups, LBO = byte stride between the two
// 16-byte K chunks of one MMA (mma_sm100_desc.hpp SmemDescriptor bit layout).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  // base_offset = 0, lbo_mode = 0, layout_type (bits 61-63) = 0: SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void store_split(uint8_t* hi_base, uint8_t* lo_base, uint32_t off, float4 v) {
  float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
  float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
  *reinterpret_cast<float4*>(hi_base + off) = h;
  *reinterpret_cast<float4*>(lo_base + off) = l;
}

__device__ __forceinline__ void tc_epilogue_store(const TcArgs& a, int m, int n, float v) {
  int q = m % a.Q;
  int t = m / a.Q;
  int pp = t % a.P;
  int nb = t / a.P;
  v += a.bias ? a.bias[n] : 0.f;
  if (a.has_res) v += a.res[nb * a.res_sn + pp * a.res_sh + q * a.res_sw + n * a.res_sc];
  a.out[nb * a.out_sn + pp * a.out_sh + q * a.out_sw + n * a.out_sc] = apply_act(v, a.act);
}

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;  // fp32 elements per stage (= 8 chunks of 16 B = 4 MMA K-steps)
constexpr int TC_THREADS = 128;

template <int BN>
struct TcSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 4;
  static constexpr int B_BYTES = BN * TC_BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = 2;
  static constexpr int OPER = STAGES * STAGE;
  static constexpr int PART = TC_BM * BN * 4;  // split-K partial tile (reuses operands)
  static constexpr int BODY = OPER > PART ? OPER : PART;
  static constexpr int TOTAL = BODY + 64;      // + mbarriers + tmem slot
  static constexpr int NCOLS = BN < 32 ? 32 : BN;
};

}  // namespace

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1) conv_tc_kernel(TcArgs a) {
  using L = TcSmem<BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::BODY);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::BODY + 32);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int m0 = blockIdx.x * TC_BM;
  const int n0 = blockIdx.y * BN;

  const int ktiles = (a.Kdim + TC_BK - 1) / TC_BK;
  const int per = (ktiles + a.split - 1) / a.split;
  const int kt0 = blockIdx.z * per;
  const int kt1 = min(ktiles, kt0 + per);
  const int iters = max(0, kt1 - kt0);

  if (tid == 0) {
    mbar_init(smem_u32(&mbar[0]), 1);
    mbar_init(smem_u32(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)L::NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  // Loader mapping: thread owns 16-byte K chunk (tid % 8) of rows tid/8 + 16*i.
  const int chunk = tid & 7;
  const int row0 = tid >> 3;
  constexpr int A_ROWS = TC_BM / 16;  // 8 rows per thread
  constexpr int B_ROWS = BN / 16;
  int64_t a_base[A_ROWS];
  int a_ih[A_ROWS], a_iw[A_ROWS];
  bool a_ok[A_ROWS];
#pragma unroll
  for (int i = 0; i < A_ROWS; ++i) {
    int m = m0 + row0 + 16 * i;
    a_ok[i] = m < a.M;
    int mm = a_ok[i] ? m : 0;
    int q = mm % a.Q;
    int t = mm / a.Q;
    int p = t % a.P;
    int nb = t / a.P;
    a_base[i] = nb * a.in_sn;
    a_ih[i] = p * a.sh - a.ph;
    a_iw[i] = q * a.sw - a.pw;
  }

  // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(TC_BM >> 4) << 24);

  float4 ra[A_ROWS], rb[B_ROWS];
  auto gather = [&](int kt) {
    const int k = kt * TC_BK + chunk * 4;
    if (a.vec) {
      // 4 consecutive k share (r, s) because C % 4 == 0
      const bool kin = k < a.Kdim;
      int c = 0, r = 0, s = 0;
      if (kin) {
        c = k % a.C;
        int rs = k / a.C;
        s = rs % a.S;
        r = rs / a.S;
      }
#pragma unroll
      for (int i = 0; i < A_ROWS; ++i) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        int ih = a_ih[i] + r, iw = a_iw[i] + s;
        if (kin && a_ok[i] && ih >= 0 && ih < a.H && iw >= 0 && iw < a.W) {
          v = __ldg(reinterpret_cast<const float4*>(a.in + a_base[i] + ih * a.in_sh + iw * a.in_sw + c));
          if (a.pre_relu) {
            v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
          }
        }
        ra[i] = v;
      }
#pragma unroll
      for (int i = 0; i < B_ROWS; ++i) {
        int n = n0 + row0 + 16 * i;
        rb[i] = (kin && n < a.K) ? __ldg(reinterpret_cast<const float4*>(a.w + (int64_t)n * a.Kdim + k))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      // generic strides / C % 4 != 0 (first layer): rolled to keep code small
#pragma unroll 1
      for (int i = 0; i < A_ROWS; ++i) {
        float e[4];
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          const int kk = k + j;
          const int c = kk % a.C;
          const int rs = kk / a.C;
          const int ih = a_ih[i] + rs / a.S, iw = a_iw[i] + rs % a.S;
          const bool ok = kk < a.Kdim && a_ok[i] && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
          float v = __ldg(a.in + (ok ? a_base[i] + ih * a.in_sh + iw * a.in_sw + c * a.in_sc : 0));
          if (a.pre_relu) v = fmaxf(v, 0.f);
          e[j] = ok ? v : 0.f;
        }
        ra[i] = make_float4(e[0], e[1], e[2], e[3]);
      }
#pragma unroll 1
      for (int i = 0; i < B_ROWS; ++i) {
        const int n = n0 + row0 + 16 * i;
        float e[4];
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          const int kk = k + j;
          const bool ok = kk < a.Kdim && n < a.K;
          const float v = __ldg(a.w + (ok ? (int64_t)n * a.Kdim + kk : 0));
          e[j] = ok ? v : 0.f;
        }
        rb[i] = make_float4(e[0], e[1], e[2], e[3]);
      }
    }
  };
  // canonical offsets: chunk j of row r at j*(ROWS*16) + (r/8)*128 + (r%8)*16
  auto deposit = [&](int stage) {
    uint8_t* st = smem + stage * L::STAGE;
    uint8_t* a_hi = st;
    uint8_t* a_lo = st + L::A_BYTES;
    uint8_t* b_hi = st + 2 * L::A_BYTES;
    uint8_t* b_lo = b_hi + L::B_BYTES;
#pragma unroll
    for (int i = 0; i < A_ROWS; ++i) {
      int r = row0 + 16 * i;
      uint32_t off = chunk * (TC_BM * 16) + (r >> 3) * 128 + (r & 7) * 16;
      store_split(a_hi, a_lo, off, ra[i]);
    }
#pragma unroll
    for (int i = 0; i < B_ROWS; ++i) {
      int r = row0 + 16 * i;
      uint32_t off = chunk * (BN * 16) + (r >> 3) * 128 + (r & 7) * 16;
      store_split(b_hi, b_lo, off, rb[i]);
    }
  };

  for (int it = 0; it < iters; ++it) {
    const int stage = it & 1;
    gather(kt0 + it);
    if (it >= 2) mbar_wait(smem_u32(&mbar[stage]), ((it - 2) >> 1) & 1);
    deposit(stage);
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t st = smem_u32(smem + stage * L::STAGE);
      const uint32_t a_hi = st, a_lo = st + L::A_BYTES;
      const uint32_t b_hi = st + 2 * L::A_BYTES, b_lo = b_hi + L::B_BYTES;
      constexpr uint32_t LBO_A = TC_BM * 16, LBO_B = BN * 16, SBO = 128;
#pragma unroll
      for (int ks = 0; ks < TC_BK / 8; ++ks) {
        const uint64_t ah = make_desc(a_hi + ks * 2 * LBO_A, LBO_A, SBO);
        const uint64_t al = make_desc(a_lo + ks * 2 * LBO_A, LBO_A, SBO);
        const uint64_t bh = make_desc(b_hi + ks * 2 * LBO_B, LBO_B, SBO);
        const uint64_t bl = make_desc(b_lo + ks * 2 * LBO_B, LBO_B, SBO);
        mma_tf32(tmem, ah, bh, idesc, (it | ks) ? 1u : 0u);
        mma_tf32(tmem, ah, bl, idesc, 1u);
        mma_tf32(tmem, al, bh, idesc, 1u);
      }
      mma_commit(smem_u32(&mbar[stage]));
    }
  }
  if (iters > 0) {
    const int last = iters - 1;
    mbar_wait(smem_u32(&mbar[last & 1]), (last >> 1) & 1);
  }
  tc_fence_after();

  const int row = warp * 32 + lane;  // TMEM lane == tile row
  const int m = m0 + row;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);

  // TMEM → smem tile (rows = TMEM lanes) → one rolled epilogue loop, shared
  // with the split-K DSMEM reduction; keeps the kernel's code footprint small
  float* part = reinterpret_cast<float*>(smem);  // [128][BN]; operand smem is free now
  __syncthreads();
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    float v[16];
    if (iters > 0) {
      tmem_ld16(t_row + c0, v);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 16; j += 4)
      *reinterpret_cast<float4*>(&part[row * BN + c0 + j]) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
  }
  (void)m;
  int e0 = 0, e1 = TC_BM * BN, nr = 1;
  cg::cluster_group cluster = cg::this_cluster();
  if (a.split > 1) {
    cluster.sync();
    nr = (int)cluster.num_blocks();
    const int chunk_e = (TC_BM * BN + nr - 1) / nr;
    e0 = (int)cluster.block_rank() * chunk_e;
    e1 = min(TC_BM * BN, e0 + chunk_e);
  } else {
    __syncthreads();
  }
#pragma unroll 1
  for (int e = e0 + tid; e < e1; e += TC_THREADS) {
    const int mm = m0 + e / BN, nn = n0 + e % BN;
    if (mm >= a.M || nn >= a.K) continue;
    float sacc = part[e];
    if (nr > 1) {
      sacc = 0.f;
#pragma unroll 1
      for (int r2 = 0; r2 < nr; ++r2) sacc += cluster.map_shared_rank(part, r2)[e];
    }
    tc_epilogue_store(a, mm, nn, sacc);
  }
  if (a.split > 1) cluster.sync();

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)L::NCOLS)
                 : "memory");
  }
}

static TcArgs tc_args(const sw_op_desc& op) {
  const int64_t* p = op.params;
  TcArgs a;
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
  const bool aligned = ((op.ptrs[PT_IN] & 15) == 0) && ((op.ptrs[PT_W] & 15) == 0);
  a.vec = (a.C % 4 == 0) && a.in_sc == 1 && (a.in_sn % 4 == 0) && (a.in_sh % 4 == 0) && (a.in_sw % 4 == 0) &&
          aligned;
  return a;
}

template <int BN>
static int launch_tc(const TcArgs& a, cudaStream_t st) {
  using L = TcSmem<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL);
    if (e != cudaSuccess) return (int)e;
    configured = true;
  }
  dim3 grid((unsigned)cdiv(a.M, TC_BM), (unsigned)cdiv(a.K, BN), (unsigned)a.split);
  return (int)launch_k(conv_tc_kernel<BN>, grid, dim3(TC_THREADS), (size_t)L::TOTAL, st, (unsigned)a.split, a);
}

// variant = N tile (32, 64, 128, 256); SP_SPLIT_K = cluster split along K.
int launch_conv_tc(const sw_op_desc& op, void* stream) {
  TcArgs a = tc_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  switch (op.variant) {
    case 32: return launch_tc<32>(a, st);
    case 64: return launch_tc<64>(a, st);
    case 128: return launch_tc<128>(a, st);
    case 256: return launch_tc<256>(a, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

// Pre-set the dynamic smem limits outside any stream capture.
void init_tc_kernels() {
  cudaFuncSetAttribute(conv_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<32>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<64>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<128>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<256>::TOTAL);
}

}  // namespace sw
