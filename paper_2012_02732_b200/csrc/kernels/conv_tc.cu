// Dense convolution / GEMM on the 5th-generation tensor cores (tcgen05 + TMEM).
//
// Implicit GEMM: rows = output pixels (M = N*P*Q), columns = output channels,
// K = R*S*C.  One CTA = 128 threads computes a 128 x BN tile over its slice of
// K (split-K across a thread-block cluster along z, reduced through DSMEM).
//
// Latency-first pipeline (batch-1 layers are round-trip bound, not FLOP bound):
//  * every K tile of the CTA's slice is requested at once with cp.async
//    straight into the canonical K-major / no-swizzle UMMA layout (8-row x
//    16-byte core matrices): im2col rows of NHWC activations are 16-byte
//    chunks of 4 consecutive channels; out-of-range taps are zero-filled by
//    cp.async, so a layer costs ~one memory round trip;
//  * fp32 accuracy via 3xTF32: weights arrive pre-split (W_hi = tf32(W),
//    W_lo = W - W_hi, prepared once at plan time, [K][Kpad]); activations are
//    split in shared memory by one pass per stage (hi in place, lo beside it);
//    one elected thread issues, per 8-wide K step,
//        D += A_hi·B_hi + A_hi·B_lo + A_lo·B_hi   (tcgen05.mma.kind::tf32)
//    into an fp32 TMEM accumulator; tcgen05.commit → per-stage mbarrier frees
//    a stage for refill when the slice is longer than the stage ring;
//  * epilogue: tcgen05.ld (warp w owns TMEM lanes 32w..32w+31 = tile rows) →
//    smem tile → one rolled loop: bias (folded BN) + residual + activation,
//    strided NHWC / channel-slice / NCHW store.  Code is kept compact because
//    every CTA of a batch-1 layer starts on a cold SM.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace sw {

namespace {

struct TcArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ w_hi;  // [K][Kpad]
  const float* __restrict__ w_lo;  // [K][Kpad]
  const float* __restrict__ bias;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, pre_relu, has_res;
  int in_sn, in_sh, in_sw, in_sc;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  int M, Kdim, Kpad, split, vec;
  Epi epi;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  uint32_t done = 0;
  do {  // suspended in hardware until the phase completes (tma.cuh mbar_wait_parity)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SWIZZLE_NONE, K-major canonical layout (mma_sm100_desc.hpp SmemDescriptor):
// SBO = byte stride between 8-row groups, LBO = byte stride between the two
// 16-byte K chunks of one MMA, version = 1 (sm_100), layout type 0.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

// K-major SWIZZLE_128B operand (TMA box = 32 fp32 x rows, 1024-B aligned):
// 8-row groups 1024 B apart (SBO), layout type 2 in bits 61-63; a K step of 8
// tf32 advances the start address by 32 B inside the swizzle atom.
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
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

__device__ __forceinline__ void tmem_ld16x2(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr + 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Round-to-nearest TF32 (cvt.rna): the 3xTF32 split x = hi + lo with
// hi = rn(x), lo = rn(x - hi) leaves an unbiased residual <= 2^-22 |x|.
// (A truncating split leaves a residual up to 2^-20 |x| with the sign of x,
// so the dropped parts of every product shrink it the same way and a dot
// product of non-negative activations inherits a coherent ~1e-6 relative
// bias per layer.)
__device__ __forceinline__ float tf32_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void split_tf32(float4 x, float4& h, float4& l) {
  h = make_float4(tf32_rn(x.x), tf32_rn(x.y), tf32_rn(x.z), tf32_rn(x.w));
  l = make_float4(tf32_rn(x.x - h.x), tf32_rn(x.y - h.y), tf32_rn(x.z - h.z), tf32_rn(x.w - h.w));
}

__device__ __forceinline__ void tc_epilogue_store(const TcArgs& a, int m, int n, float v) {
  const int q = m % a.Q;
  const int t = m / a.Q;
  const int pp = t % a.P;
  const int nb = t / a.P;
  v += a.bias ? a.bias[n] : 0.f;
  if (a.has_res) v += a.res[nb * a.res_sn + pp * a.res_sh + q * a.res_sw + n * a.res_sc];
  a.out[nb * a.out_sn + pp * a.out_sh + q * a.out_sw + n * a.out_sc] = apply_act(v, a.act);
}

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;  // fp32 per stage row = 8 chunks of 16 B = 4 MMA K-steps
constexpr int TC_THREADS = 128;

template <int BN, int SOVR = 0, int CPS = (SOVR ? 2 : 1)>  // CPS: CTAs resident per SM
struct TcSmem {
  static constexpr int A_BYTES = TC_BM * TC_BK * 4;  // 16 KB
  static constexpr int B_BYTES = BN * TC_BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // A_hi, A_lo, B_hi, B_lo
  static constexpr int STAGES = SOVR ? SOVR : (BN <= 64) ? 4 : (BN == 128 ? 3 : 2);
  static constexpr int OPER = STAGES * STAGE;
  static constexpr int PS = BN + 4;  // epilogue tile row stride (floats): conflict-free row-per-lane stores
  static constexpr int PART = TC_BM * PS * 4;
  static constexpr int BODY = OPER > PART ? OPER : PART;
  static constexpr int TOTAL = BODY + 128;  // + mbarriers + tmem slot
  // persistent kernel: the epilogue tile sits past the ring (loads stay in flight)
  static constexpr int P_BODY = OPER + PART;
  static constexpr int P_TOTAL = P_BODY + 128;
  // Accumulation precision.  The tensor pipe's fp32 accumulation truncates,
  // so one TMEM accumulator over a long K drifts toward zero
  // (tools/tc_precision.cu: 25x the FFMA rms error at K = 4096).
  //  * PROMO (BN <= 128): every K tile's 3xTF32 products go into a fresh TMEM
  //    accumulator (ping-pong pair); while the tensor pipe works on tile i
  //    the threads add tile i-1's accumulator into fp32 registers
  //    (round-to-nearest), so no TMEM chain is longer than 12 MMAs — more
  //    accurate than a sequential FFMA dot product.
  //  * BN = 256 (no room for 256 register accumulators): ACC accumulators for
  //    the hi·hi products (K tile kt goes to kt % ACC) + one for the hi·lo +
  //    lo·hi corrections, summed in fp32 by the epilogue.
  static constexpr bool PROMO = BN <= 128;
  static constexpr int COLS_CTA = CPS > 1 ? 256 : 512;
  static constexpr int ACC = (COLS_CTA / (BN < 32 ? 32 : BN)) - 1 > 0 ? (COLS_CTA / (BN < 32 ? 32 : BN)) - 1 : 1;
  static constexpr int NCOLS = PROMO ? (2 * BN < 32 ? 32 : 2 * BN) : COLS_CTA;
};

// Issue the 3xTF32 MMAs of one K tile (ksteps of 8): hi·hi into accumulator
// kt % ACC, hi·lo + lo·hi into the correction accumulator (column ACC*BN).
template <int ACC, int BN>
__device__ __forceinline__ void mma_ktile_3xtf32(uint32_t tmem, int kt, const uint64_t (&ah)[4],
                                                 const uint64_t (&al)[4], const uint64_t (&bh)[4],
                                                 const uint64_t (&bl)[4], uint32_t idesc) {
  const uint32_t dh = tmem + (uint32_t)((kt % ACC) * BN);
  const uint32_t dc = tmem + (uint32_t)(ACC * BN);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    mma_tf32(dh, ah[ks], bh[ks], idesc, (kt >= ACC || ks) ? 1u : 0u);
    mma_tf32(dc, ah[ks], bl[ks], idesc, (kt | ks) ? 1u : 0u);
    mma_tf32(dc, al[ks], bh[ks], idesc, 1u);
  }
}

// PROMO: all 12 MMAs of one K tile into one fresh accumulator `d`.
__device__ __forceinline__ void mma_ktile_fresh(uint32_t d, const uint64_t (&ah)[4], const uint64_t (&al)[4],
                                                const uint64_t (&bh)[4], const uint64_t (&bl)[4], uint32_t idesc) {
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    mma_tf32(d, ah[ks], bh[ks], idesc, ks ? 1u : 0u);
    mma_tf32(d, ah[ks], bl[ks], idesc, 1u);
    mma_tf32(d, al[ks], bh[ks], idesc, 1u);
  }
}

template <int ACC, int BN, bool PROMO>
__device__ __forceinline__ void mma_ktile(uint32_t tmem, int kt, const uint64_t (&ah)[4], const uint64_t (&al)[4],
                                          const uint64_t (&bh)[4], const uint64_t (&bl)[4], uint32_t idesc) {
  if constexpr (PROMO)
    mma_ktile_fresh(tmem + (uint32_t)((kt & 1) * BN), ah, al, bh, bl, idesc);
  else
    mma_ktile_3xtf32<ACC, BN>(tmem, kt, ah, al, bh, bl, idesc);
}

// PROMO: racc += this warp's TMEM lanes of the accumulator at column `col`.
template <int BN>
__device__ __forceinline__ void tmem_promote(uint32_t t_row, uint32_t col, float (&racc)[BN]) {
#pragma unroll
  for (int c0 = 0; c0 < BN; c0 += 32) {
    float v[32];
    tmem_ld16x2(t_row + col + (uint32_t)c0, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) racc[c0 + j] += v[j];
  }
}

// 32 accumulator columns [c0, c0 + 32) of this warp's TMEM lanes, summed over
// the nacc used hi·hi accumulators and the correction accumulator.
template <int ACC, int BN>
__device__ __forceinline__ void tmem_sum32(uint32_t t_row, int c0, int nacc, float (&v)[32]) {
  tmem_ld16x2(t_row + (uint32_t)(ACC * BN + c0), v);
#pragma unroll 1
  for (int r = 0; r < nacc; ++r) {
    float w[32];
    tmem_ld16x2(t_row + (uint32_t)(r * BN + c0), w);
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] += w[j];
  }
}


// End of a tile: the fp32 result rows → the smem tile `part` [128][PS]
// (PROMO: the register accumulators; else the TMEM accumulator sum).
template <class L, int BN>
__device__ __forceinline__ void drain_to_part(uint32_t t_row, int row, int iters, const float (&racc)[L::PROMO ? BN : 1],
                                              float* part) {
  if constexpr (L::PROMO) {
#pragma unroll
    for (int j = 0; j < BN; j += 4)
      *reinterpret_cast<float4*>(&part[row * L::PS + j]) = make_float4(racc[j], racc[j + 1], racc[j + 2], racc[j + 3]);
  } else {
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      float v[32];
      if (iters > 0) {
        tmem_sum32<L::ACC, BN>(t_row, c0, min(iters, L::ACC), v);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(&part[row * L::PS + c0 + j]) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    }
  }
}

}  // namespace

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1) conv_tc_kernel(TcArgs a) {
  using L = TcSmem<BN>;
  constexpr int S = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L::BODY);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::BODY + 8 * S);
  const uint32_t sbase = smem_u32(smem);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int m0 = blockIdx.x * TC_BM;
  const int n0 = blockIdx.y * BN;

  const int ktiles = (a.Kdim + TC_BK - 1) / TC_BK;
  const int per = (ktiles + a.split - 1) / a.split;
  const int kt0 = blockIdx.z * per;
  const int iters = max(0, min(ktiles, kt0 + per) - kt0);
  probe_begin();

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&mbar[s]), 1);
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
  const int row = warp * 32 + lane;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
  float racc[L::PROMO ? BN : 1];
#pragma unroll
  for (int j = 0; j < (L::PROMO ? BN : 1); ++j) racc[j] = 0.f;

  // Loader mapping: thread owns 16-byte K chunk (tid % 8) of rows tid/8 + 16*i.
  const int chunk = tid & 7;
  const int row0 = tid >> 3;
  constexpr int A_ROWS = TC_BM / 16;
  constexpr int B_ROWS = BN / 16;
  int a_base[A_ROWS], a_ih[A_ROWS], a_iw[A_ROWS];
#pragma unroll
  for (int i = 0; i < A_ROWS; ++i) {
    const int m = m0 + row0 + 16 * i;
    const int q = m % a.Q;
    const int t = m / a.Q;
    a_base[i] = (t / a.P) * a.in_sn;
    a_ih[i] = m < a.M ? (t % a.P) * a.sh - a.ph : -(1 << 28);
    a_iw[i] = q * a.sw - a.pw;
  }

  // cp.async of K tile `kt` (slice-relative) into stage `st`: A raw → A_hi slot,
  // W_hi / W_lo → B slots
  // part: 1 = activations (A), 2 = weights (B, constants), 3 = both
  auto issue = [&](int kt, int st, int part) {
    const uint32_t stage = sbase + st * L::STAGE;
    const int k = (kt0 + kt) * TC_BK + chunk * 4;
    if (!(part & 1)) {
      // weights only
    } else if (a.vec) {
      const bool kin = k < a.Kdim;
      const int c = k % a.C;
      const int rs = k / a.C;
      const int s = rs % a.S, r = rs / a.S;
#pragma unroll
      for (int i = 0; i < A_ROWS; ++i) {
        const int rr = row0 + 16 * i;
        const int ih = a_ih[i] + r, iw = a_iw[i] + s;
        const bool ok = kin && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
        cp16(stage + chunk * (TC_BM * 16) + (rr >> 3) * 128 + (rr & 7) * 16,
             a.in + (ok ? a_base[i] + ih * a.in_sh + iw * a.in_sw + c : 0), ok);
      }
    } else {
#pragma unroll 1
      for (int i = 0; i < A_ROWS; ++i) {
        const int rr = row0 + 16 * i;
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          const int kk = k + j;
          const int c = kk % a.C;
          const int rs = kk / a.C;
          const int ih = a_ih[i] + rs / a.S, iw = a_iw[i] + rs % a.S;
          const bool ok = kk < a.Kdim && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
          cp4(stage + chunk * (TC_BM * 16) + (rr >> 3) * 128 + (rr & 7) * 16 + 4 * j,
              a.in + (ok ? a_base[i] + ih * a.in_sh + iw * a.in_sw + c * a.in_sc : 0), ok);
        }
      }
    }
    if (!(part & 2)) return;
    const uint32_t b_hi = stage + 2 * L::A_BYTES, b_lo = b_hi + L::B_BYTES;
#pragma unroll
    for (int i = 0; i < B_ROWS; ++i) {
      const int rr = row0 + 16 * i;
      const int n = n0 + rr;
      const bool ok = n < a.K;
      const size_t off = ok ? (size_t)n * a.Kpad + k : 0;
      const uint32_t d = chunk * (BN * 16) + (rr >> 3) * 128 + (rr & 7) * 16;
      cp16(b_hi + d, a.w_hi + off, ok);
      cp16(b_lo + d, a.w_lo + off, ok);
    }
  };

  // instruction descriptor: D f32, A/B tf32, both K-major, N = BN, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(TC_BM >> 4) << 24);

  // the first stages' weights (constants) are requested before the PDL wait,
  // the activations after it; stage s's cp.async group then holds A_s (and
  // group 0 also every prologue B), so the per-stage waits stay correct
#pragma unroll 1
  for (int st = 0; st < S; ++st)
    if (st < iters) issue(st, st, 2);
  probe_pt(1);
  pdl_trigger();
  pdl_wait();
  probe_pt(2);
#pragma unroll 1
  for (int st = 0; st < S; ++st) {
    if (st < iters) issue(st, st, 1);
    cp_commit();
  }
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int st = it % S;
    cp_wait<S - 2>();  // tile `it` landed (refills run one iteration behind)
    __syncthreads();
    if (it == 0) probe_pt(3);
    // split the activation tile: hi = tf32(x) in place, lo = x - hi beside it
    {
      float4* hi = reinterpret_cast<float4*>(smem + st * L::STAGE);
      float4* lo = reinterpret_cast<float4*>(smem + st * L::STAGE + L::A_BYTES);
#pragma unroll 2
      for (int i = tid; i < L::A_BYTES / 16; i += TC_THREADS) {
        float4 x = hi[i];
        if (a.pre_relu) {
          x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
        }
        float4 h, l;
        split_tf32(x, h, l);
        hi[i] = h;
        lo[i] = l;
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_hi = sbase + st * L::STAGE, a_lo = a_hi + L::A_BYTES;
      const uint32_t b_hi = a_hi + 2 * L::A_BYTES, b_lo = b_hi + L::B_BYTES;
      constexpr uint32_t LBO_A = TC_BM * 16, LBO_B = BN * 16, SBO = 128;
      uint64_t ah[4], al[4], bh[4], bl[4];
#pragma unroll
      for (int ks = 0; ks < TC_BK / 8; ++ks) {
        ah[ks] = make_desc(a_hi + ks * 2 * LBO_A, LBO_A, SBO);
        al[ks] = make_desc(a_lo + ks * 2 * LBO_A, LBO_A, SBO);
        bh[ks] = make_desc(b_hi + ks * 2 * LBO_B, LBO_B, SBO);
        bl[ks] = make_desc(b_lo + ks * 2 * LBO_B, LBO_B, SBO);
      }
      mma_ktile<L::ACC, BN, L::PROMO>(tmem, it, ah, al, bh, bl, idesc);
      mma_commit(smem_u32(&mbar[st]));
    }
    // refill the stage of the PREVIOUS tile (its MMAs have had a whole
    // iteration to drain) with tile it-1+S; the tensor pipe stays busy
    if (it >= 1 && it - 1 + S < iters) {
      const int ps = (it - 1) % S;
      mbar_wait(smem_u32(&mbar[ps]), ((it - 1) / S) & 1);
      issue(it - 1 + S, ps, 3);
    }
    cp_commit();
    if constexpr (L::PROMO) {  // tile it-1's accumulator → registers while tile it's MMAs run
      if (it >= 1) {
        mbar_wait(smem_u32(&mbar[(it - 1) % S]), ((it - 1) / S) & 1);
        tc_fence_after();
        tmem_promote<BN>(t_row, (uint32_t)(((it - 1) & 1) * BN), racc);
        tc_fence_before();
      }
    }
  }
  if (iters > 0) {
    const int last = iters - 1;
    mbar_wait(smem_u32(&mbar[last % S]), (last / S) & 1);
    tc_fence_after();
    if constexpr (L::PROMO) tmem_promote<BN>(t_row, (uint32_t)((last & 1) * BN), racc);
  }
  tc_fence_after();
  probe_pt(4);

  // accumulators → smem tile (rows = TMEM lanes) → one rolled epilogue loop,
  // shared with the split-K DSMEM reduction
  float* part = reinterpret_cast<float*>(smem);  // [128][BN]; operands are dead now
  __syncthreads();
  drain_to_part<L, BN>(t_row, row, iters, racc, part);
  probe_pt(5);
  cg::cluster_group cluster = cg::this_cluster();
  tile_epilogue<TC_BM, BN, TC_THREADS, L::PS>(a.epi, part, m0, n0, a.split, cluster);
  probe_pt(6);

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)L::NCOLS)
                 : "memory");
  }
  probe_end();
}

// ---------------------------------------------------------------------------
// TMA-fed variant for 1x1 / stride-1 convolutions (pure GEMMs on NHWC:
// A = activations [M pixels][C], B = pre-split weights [K][Kpad]).
//   * operands arrive by cp.async.bulk.tensor (3-D tensor maps whose box is
//     exactly the canonical no-swizzle K-major UMMA layout [k16-chunk][row][16 B]),
//     completing on a per-stage "full" mbarrier; one thread issues every copy;
//   * the weights of the first stages are requested before the PDL wait
//     (constants), the activations after it;
//   * the 128 threads split the activation stage into tf32 hi / lo (3xTF32),
//     one elected thread issues the 12 MMAs of the stage and commits them to a
//     per-stage "done" mbarrier, and the same thread immediately refills the
//     stage the previous MMAs just released — the other threads never wait on
//     the tensor pipe, only on data.
// ---------------------------------------------------------------------------
struct TcMaps {
  CUtensorMap a, bh, bl;
};

// SOVR > 0: a shallower ring (SOVR stages) so that two CTAs share an SM and
// one CTA's prologue / epilogue overlaps the other's TMA stream (large M).
template <int BN, int SOVR = 0, bool SWZ = false>
__global__ void __launch_bounds__(TC_THREADS, SOVR ? 2 : 1)
    conv_tc_tma_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tbh,
                       const __grid_constant__ CUtensorMap tbl, TcArgs a) {
  using L = TcSmem<BN, SOVR>;
  constexpr int S = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BODY);
  uint64_t* done = full + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + S);
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int m0 = blockIdx.x * TC_BM;
  const int n0 = blockIdx.y * BN;
  const int ktiles = (a.Kdim + TC_BK - 1) / TC_BK;
  const int per = (ktiles + a.split - 1) / a.split;
  const int kt0 = blockIdx.z * per;
  const int iters = max(0, min(ktiles, kt0 + per) - kt0);
  constexpr uint32_t A_TX = L::A_BYTES, B_TX = 2 * L::B_BYTES;

  if (tid == 0) {
    prefetch_tmap(&ta);
    prefetch_tmap(&tbh);
    prefetch_tmap(&tbl);
    for (int st = 0; st < S; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&done[st]), 1);
    }
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
  const int row = warp * 32 + lane;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
  float racc[L::PROMO ? BN : 1];
#pragma unroll
  for (int j = 0; j < (L::PROMO ? BN : 1); ++j) racc[j] = 0.f;

  auto load_b = [&](int kt, int st) {
    const uint32_t stage = sbase + st * L::STAGE;
    const uint32_t bar = smem_u32(&full[st]);
    if constexpr (SWZ) {
      tma_load_2d(stage + 2 * L::A_BYTES, &tbh, (kt0 + kt) * TC_BK, n0, bar);
      tma_load_2d(stage + 2 * L::A_BYTES + L::B_BYTES, &tbl, (kt0 + kt) * TC_BK, n0, bar);
    } else {
      const int kc = (kt0 + kt) * (TC_BK / 4);
      tma_load_3d(stage + 2 * L::A_BYTES, &tbh, 0, n0, kc, bar);
      tma_load_3d(stage + 2 * L::A_BYTES + L::B_BYTES, &tbl, 0, n0, kc, bar);
    }
  };
  auto load_a = [&](int kt, int st) {
    const uint32_t stage = sbase + st * L::STAGE;
    if constexpr (SWZ)
      tma_load_2d(stage, &ta, (kt0 + kt) * TC_BK, m0, smem_u32(&full[st]));
    else
      tma_load_3d(stage, &ta, 0, m0, (kt0 + kt) * (TC_BK / 4), smem_u32(&full[st]));
  };
  if (tid == 0) {
    for (int st = 0; st < S && st < iters; ++st) {
      mbar_expect_tx(smem_u32(&full[st]), A_TX + B_TX);
      load_b(st, st);
    }
  }
  pdl_trigger();
  pdl_wait();
  if (tid == 0)
    for (int st = 0; st < S && st < iters; ++st) load_a(st, st);

  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(TC_BM >> 4) << 24);
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const int st = it % S;
    mbar_wait(smem_u32(&full[st]), (it / S) & 1);
    {
      float4* hi = reinterpret_cast<float4*>(smem + st * L::STAGE);
      float4* lo = reinterpret_cast<float4*>(smem + st * L::STAGE + L::A_BYTES);
#pragma unroll 2
      for (int i = tid; i < L::A_BYTES / 16; i += TC_THREADS) {
        float4 x = hi[i];
        if (a.pre_relu) {
          x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
        }
        float4 h, l;
        split_tf32(x, h, l);
        hi[i] = h;
        lo[i] = l;
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_hi = sbase + st * L::STAGE, a_lo = a_hi + L::A_BYTES;
      const uint32_t b_hi = a_hi + 2 * L::A_BYTES, b_lo = b_hi + L::B_BYTES;
      constexpr uint32_t LBO_A = TC_BM * 16, LBO_B = BN * 16, SBO = 128;
      uint64_t ah[4], al[4], bh[4], bl[4];
#pragma unroll
      for (int ks = 0; ks < TC_BK / 8; ++ks) {
        if constexpr (SWZ) {
          ah[ks] = make_desc_sw128(a_hi + ks * 32);
          al[ks] = make_desc_sw128(a_lo + ks * 32);
          bh[ks] = make_desc_sw128(b_hi + ks * 32);
          bl[ks] = make_desc_sw128(b_lo + ks * 32);
        } else {
          ah[ks] = make_desc(a_hi + ks * 2 * LBO_A, LBO_A, SBO);
          al[ks] = make_desc(a_lo + ks * 2 * LBO_A, LBO_A, SBO);
          bh[ks] = make_desc(b_hi + ks * 2 * LBO_B, LBO_B, SBO);
          bl[ks] = make_desc(b_lo + ks * 2 * LBO_B, LBO_B, SBO);
        }
      }
      mma_ktile<L::ACC, BN, L::PROMO>(tmem, it, ah, al, bh, bl, idesc);
      mma_commit(smem_u32(&done[st]));
      // refill the stage the PREVIOUS tile's MMAs are releasing
      if (it >= 1 && it - 1 + S < iters) {
        const int ps = (it - 1) % S;
        mbar_wait(smem_u32(&done[ps]), ((it - 1) / S) & 1);
        mbar_expect_tx(smem_u32(&full[ps]), A_TX + B_TX);
        load_b(it - 1 + S, ps);
        load_a(it - 1 + S, ps);
      }
    }
    if constexpr (L::PROMO) {  // tile it-1's accumulator → registers while tile it's MMAs run
      if (it >= 1) {
        mbar_wait(smem_u32(&done[(it - 1) % S]), ((it - 1) / S) & 1);
        tc_fence_after();
        tmem_promote<BN>(t_row, (uint32_t)(((it - 1) & 1) * BN), racc);
        tc_fence_before();
      }
    }
  }
  if (iters > 0) {
    const int last = iters - 1;
    mbar_wait(smem_u32(&done[last % S]), (last / S) & 1);
    tc_fence_after();
    if constexpr (L::PROMO) tmem_promote<BN>(t_row, (uint32_t)((last & 1) * BN), racc);
  }
  tc_fence_after();
  float* part = reinterpret_cast<float*>(smem);
  __syncthreads();
  drain_to_part<L, BN>(t_row, row, iters, racc, part);
  cg::cluster_group cluster = cg::this_cluster();
  tile_epilogue<TC_BM, BN, TC_THREADS, L::PS>(a.epi, part, m0, n0, a.split, cluster);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)L::NCOLS)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// Persistent form of the TMA 1x1 kernel (variants 3000 + BN, split 1, large
// M): a CTA walks M tiles blockIdx.x, blockIdx.x + gridDim.x, ... and the
// stage ring runs over the flattened (tile, k-tile) sequence, so the loads of
// the next tile are in flight while this tile's accumulator is drained
// (ncu at bs256: the one-tile kernel spends 32 % of its stalls waiting for
// the first stages of every tile, with nothing else resident to overlap).
// ---------------------------------------------------------------------------
template <int BN, bool SWZ = false>
__global__ void __launch_bounds__(TC_THREADS, 1)
    conv_tc_tma_persistent_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tbh,
                                  const __grid_constant__ CUtensorMap tbl, TcArgs a) {
  using L = TcSmem<BN, BN == 128 ? 2 : 0, 1>;  // 2 x 64 KB ring + 66 KB tile for BN = 128
  constexpr int S = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::P_BODY);
  uint64_t* done = full + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + S);
  const uint32_t sbase = smem_u32(smem);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int n0 = blockIdx.y * BN;
  const int iters = (a.Kdim + TC_BK - 1) / TC_BK;  // k-tiles per M tile
  const int mtiles = (a.M + TC_BM - 1) / TC_BM;
  const int ntl = mtiles > (int)blockIdx.x ? (mtiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const int total = ntl * iters;  // flattened (tile, k-tile) sequence of this CTA
  constexpr uint32_t A_TX = L::A_BYTES, B_TX = 2 * L::B_BYTES;

  if (tid == 0) {
    prefetch_tmap(&ta);
    prefetch_tmap(&tbh);
    prefetch_tmap(&tbl);
    for (int st = 0; st < S; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&done[st]), 1);
    }
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

  auto load_b = [&](int q, int st) {
    const uint32_t stage = sbase + st * L::STAGE;
    const uint32_t bar = smem_u32(&full[st]);
    if constexpr (SWZ) {  // 2-D maps (k, row), 128-B rows swizzled
      tma_load_2d(stage + 2 * L::A_BYTES, &tbh, (q % iters) * TC_BK, n0, bar);
      tma_load_2d(stage + 2 * L::A_BYTES + L::B_BYTES, &tbl, (q % iters) * TC_BK, n0, bar);
    } else {
      const int kc = (q % iters) * (TC_BK / 4);
      tma_load_3d(stage + 2 * L::A_BYTES, &tbh, 0, n0, kc, bar);
      tma_load_3d(stage + 2 * L::A_BYTES + L::B_BYTES, &tbl, 0, n0, kc, bar);
    }
  };
  auto load_a = [&](int q, int st) {
    const uint32_t stage = sbase + st * L::STAGE;
    const int m0 = ((int)blockIdx.x + (q / iters) * (int)gridDim.x) * TC_BM;
    if constexpr (SWZ)
      tma_load_2d(stage, &ta, (q % iters) * TC_BK, m0, smem_u32(&full[st]));
    else
      tma_load_3d(stage, &ta, 0, m0, (q % iters) * (TC_BK / 4), smem_u32(&full[st]));
  };
  if (tid == 0) {
    for (int st = 0; st < S && st < total; ++st) {
      mbar_expect_tx(smem_u32(&full[st]), A_TX + B_TX);
      load_b(st, st);
    }
  }
  pdl_trigger();
  pdl_wait();
  if (tid == 0)
    for (int st = 0; st < S && st < total; ++st) load_a(st, st);

  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                         ((uint32_t)(TC_BM >> 4) << 24);
  const int row = warp * 32 + lane;
  const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
  float* part = reinterpret_cast<float*>(smem + S * L::STAGE);  // past the ring: loads stay in flight
  cg::cluster_group cluster = cg::this_cluster();
  float racc[BN];
#pragma unroll
  for (int j = 0; j < BN; ++j) racc[j] = 0.f;
  auto flush_tile = [&](int qq) {  // registers → part → epilogue; restart the accumulation
    drain_to_part<L, BN>(t_row, row, iters, racc, part);
#pragma unroll
    for (int j = 0; j < BN; ++j) racc[j] = 0.f;
    const int m0 = ((int)blockIdx.x + (qq / iters) * (int)gridDim.x) * TC_BM;
    tile_epilogue<TC_BM, BN, TC_THREADS, L::PS>(a.epi, part, m0, n0, 1, cluster);
    __syncthreads();  // part is rewritten by the next tile
  };
#pragma unroll 1
  for (int q = 0; q < total; ++q) {
    const int st = q % S;
    const int kt = q % iters;
    mbar_wait(smem_u32(&full[st]), (q / S) & 1);
    {
      float4* hi = reinterpret_cast<float4*>(smem + st * L::STAGE);
      float4* lo = reinterpret_cast<float4*>(smem + st * L::STAGE + L::A_BYTES);
#pragma unroll 2
      for (int i = tid; i < L::A_BYTES / 16; i += TC_THREADS) {
        float4 x = hi[i];
        if (a.pre_relu) {
          x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
        }
        float4 h, l;
        split_tf32(x, h, l);
        hi[i] = h;
        lo[i] = l;
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_hi = sbase + st * L::STAGE, a_lo = a_hi + L::A_BYTES;
      const uint32_t b_hi = a_hi + 2 * L::A_BYTES, b_lo = b_hi + L::B_BYTES;
      constexpr uint32_t LBO_A = TC_BM * 16, LBO_B = BN * 16, SBO = 128;
      uint64_t ah[4], al[4], bh[4], bl[4];
#pragma unroll
      for (int ks = 0; ks < TC_BK / 8; ++ks) {
        if constexpr (SWZ) {
          ah[ks] = make_desc_sw128(a_hi + ks * 32);
          al[ks] = make_desc_sw128(a_lo + ks * 32);
          bh[ks] = make_desc_sw128(b_hi + ks * 32);
          bl[ks] = make_desc_sw128(b_lo + ks * 32);
        } else {
          ah[ks] = make_desc(a_hi + ks * 2 * LBO_A, LBO_A, SBO);
          al[ks] = make_desc(a_lo + ks * 2 * LBO_A, LBO_A, SBO);
          bh[ks] = make_desc(b_hi + ks * 2 * LBO_B, LBO_B, SBO);
          bl[ks] = make_desc(b_lo + ks * 2 * LBO_B, LBO_B, SBO);
        }
      }
      mma_ktile<L::ACC, BN, L::PROMO>(tmem, L::PROMO ? q : kt, ah, al, bh, bl, idesc);
      mma_commit(smem_u32(&done[st]));
      if (q >= 1 && q - 1 + S < total) {  // refill the stage the previous MMAs released
        const int ps = (q - 1) % S;
        mbar_wait(smem_u32(&done[ps]), ((q - 1) / S) & 1);
        mbar_expect_tx(smem_u32(&full[ps]), A_TX + B_TX);
        load_b(q - 1 + S, ps);
        load_a(q - 1 + S, ps);
      }
    }
    // PROMO: k-tile q-1's accumulator → registers while k-tile q's MMAs run;
    // a finished tile goes through the epilogue right after its last k-tile
    static_assert(L::PROMO, "persistent kernel: BN <= 128");
    if (q >= 1) {
      mbar_wait(smem_u32(&done[(q - 1) % S]), ((q - 1) / S) & 1);
      tc_fence_after();
      tmem_promote<BN>(t_row, (uint32_t)(((q - 1) & 1) * BN), racc);
      tc_fence_before();
      if ((q - 1) % iters == iters - 1) flush_tile(q - 1);
    }
  }
  if (total > 0) {
    mbar_wait(smem_u32(&done[(total - 1) % S]), ((total - 1) / S) & 1);
    tc_fence_after();
    tmem_promote<BN>(t_row, (uint32_t)(((total - 1) & 1) * BN), racc);
    flush_tile(total - 1);
  }
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
  a.w_hi = reinterpret_cast<const float*>(op.ptrs[PT_W_TC_HI]);
  a.w_lo = reinterpret_cast<const float*>(op.ptrs[PT_W_TC_LO]);
  a.bias = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K];
  a.R = (int)p[SP_R]; a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.in_sn = (int)p[SP_IN_SN]; a.in_sh = (int)p[SP_IN_SH]; a.in_sw = (int)p[SP_IN_SW]; a.in_sc = (int)p[SP_IN_SC];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  a.M = a.N * a.P * a.Q;
  a.Kdim = a.R * a.S * a.C;
  a.Kpad = (int)p[SP_KPAD];
  a.split = p[SP_SPLIT_K] > 1 ? (int)p[SP_SPLIT_K] : 1;
  a.vec = (a.C % 4 == 0) && a.in_sc == 1 && (a.in_sn % 4 == 0) && (a.in_sh % 4 == 0) && (a.in_sw % 4 == 0) &&
          ((op.ptrs[PT_IN] & 15) == 0);
  a.epi = Epi{a.bias, a.res, a.out, a.M, a.K, a.P, a.Q, a.act, a.has_res, 0,
              a.out_sn, a.out_sh, a.out_sw, a.out_sc, a.res_sn, a.res_sh, a.res_sw, a.res_sc};
  a.epi.vec = epi_vec_ok(op.ptrs[PT_OUT], a.out_sn, a.out_sh, a.out_sw, a.out_sc, op.ptrs[PT_BIAS],
                         a.has_res != 0, op.ptrs[PT_RES], a.res_sn, a.res_sh, a.res_sw, a.res_sc) ? 1 : 0;
  return a;
}

// variant = N tile (32, 64, 128, 256); SP_SPLIT_K = cluster split along K.
template <int BN, int SOVR = 0, bool PERSIST = false, bool SWZ = false>
static int launch_tc_tma(const TcArgs& a, const sw_op_desc& op, cudaStream_t st) {
  // 1x1 / stride 1 / no padding on 16-B aligned NHWC rows only
  if (a.R != 1 || a.S != 1 || a.sh != 1 || a.sw != 1 || a.ph != 0 || a.pw != 0 || !a.vec)
    return (int)cudaErrorInvalidValue;
  if (a.in_sn != (int64_t)a.H * a.W * a.in_sw || a.in_sh != (int64_t)a.W * a.in_sw) return (int)cudaErrorInvalidValue;
  CUtensorMap ta, tbh, tbl;
  if constexpr (SWZ) {  // 2-D (k, row) maps, box 32 fp32 x rows, 128-B swizzle
    const uint64_t da[2] = {(uint64_t)a.C, (uint64_t)a.M};
    const uint64_t sa[1] = {(uint64_t)a.in_sw * 4};
    const uint32_t ba[2] = {TC_BK, TC_BM};
    const uint64_t db[2] = {(uint64_t)a.Kpad, (uint64_t)a.K};
    const uint64_t sb[1] = {(uint64_t)a.Kpad * 4};
    const uint32_t bb[2] = {TC_BK, (uint32_t)BN};
    if (!encode_tmap_f32(&ta, a.in, 2, da, sa, ba, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_tmap_f32(&tbh, a.w_hi, 2, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_tmap_f32(&tbl, a.w_lo, 2, db, sb, bb, CU_TENSOR_MAP_SWIZZLE_128B))
      return (int)cudaErrorInvalidValue;
  } else {
  {  // activations: (4 floats, M rows, C/4 chunks)
    const uint64_t dims[3] = {4, (uint64_t)a.M, (uint64_t)(a.C / 4)};
    const uint64_t str[2] = {(uint64_t)a.in_sw * 4, 16};
    const uint32_t box[3] = {4, TC_BM, TC_BK / 4};
    if (!encode_tmap_f32(&ta, a.in, 3, dims, str, box)) return (int)cudaErrorInvalidValue;
  }
  {  // weights hi / lo: (4 floats, K rows, Kpad/4 chunks)
    const uint64_t dims[3] = {4, (uint64_t)a.K, (uint64_t)(a.Kpad / 4)};
    const uint64_t str[2] = {(uint64_t)a.Kpad * 4, 16};
    const uint32_t box[3] = {4, (uint32_t)BN, TC_BK / 4};
    if (!encode_tmap_f32(&tbh, a.w_hi, 3, dims, str, box)) return (int)cudaErrorInvalidValue;
    if (!encode_tmap_f32(&tbl, a.w_lo, 3, dims, str, box)) return (int)cudaErrorInvalidValue;
  }
  }
  if constexpr (PERSIST) {
    if (a.split != 1) return (int)cudaErrorInvalidValue;
    using LP = TcSmem<BN, BN == 128 ? 2 : 0>;
    const int64_t ntn = cdiv(a.K, BN), mt = cdiv(a.M, TC_BM);
    const int64_t gx = std::min<int64_t>(mt, std::max<int64_t>(1, 148 / ntn));
    return (int)launch_k(conv_tc_tma_persistent_kernel<BN, SWZ>, dim3((unsigned)gx, (unsigned)ntn, 1), dim3(TC_THREADS),
                         (size_t)LP::P_TOTAL, st, 1u, ta, tbh, tbl, a);
  }
  dim3 grid((unsigned)cdiv(a.M, TC_BM), (unsigned)cdiv(a.K, BN), (unsigned)a.split);
  return (int)launch_k(conv_tc_tma_kernel<BN, SOVR, SWZ>, grid, dim3(TC_THREADS), (size_t)TcSmem<BN, SOVR>::TOTAL, st,
                       (unsigned)a.split, ta, tbh, tbl, a);
}

int launch_conv_tc(const sw_op_desc& op, void* stream) {
  if (op.variant >= 6000 && op.variant < 8000) return launch_conv_tcs(op, stream);
  if (op.variant >= 8000 && op.variant < 9000) return launch_conv_pw_tc(op, stream);
  TcArgs a = tc_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  if (!a.w_hi || !a.w_lo || a.Kpad < a.Kdim || a.Kpad % TC_BK) return (int)cudaErrorInvalidValue;
  // variants 1000 + BN: the TMA-fed kernel (1x1 convolutions)
  switch (op.variant) {
    case 1032: return launch_tc_tma<32>(a, op, st);
    case 1064: return launch_tc_tma<64>(a, op, st);
    case 1128: return launch_tc_tma<128>(a, op, st);
    case 1256: return launch_tc_tma<256>(a, op, st);
    // 2000 + BN: two stages, two CTAs per SM
    case 2032: return launch_tc_tma<32, 2>(a, op, st);
    case 2064: return launch_tc_tma<64, 2>(a, op, st);
    // 3000 + BN: persistent tile loop (split 1)
    case 3032: return launch_tc_tma<32, 0, true>(a, op, st);
    case 3064: return launch_tc_tma<64, 0, true>(a, op, st);
    case 3128: return launch_tc_tma<128, 0, true>(a, op, st);
    // 5000 + BN: one tile per CTA (split-K clusters), 128-B swizzled operands
    case 5032: return launch_tc_tma<32, 0, false, true>(a, op, st);
    case 5064: return launch_tc_tma<64, 0, false, true>(a, op, st);
    case 5128: return launch_tc_tma<128, 0, false, true>(a, op, st);
    case 5256: return launch_tc_tma<256, 0, false, true>(a, op, st);
    // 4000 + BN: persistent, 128-B swizzled operands (full-row TMA boxes)
    case 4032: return launch_tc_tma<32, 0, true, true>(a, op, st);
    case 4064: return launch_tc_tma<64, 0, true, true>(a, op, st);
    case 4128: return launch_tc_tma<128, 0, true, true>(a, op, st);
    default: break;
  }
  dim3 grid((unsigned)cdiv(a.M, TC_BM), 1, (unsigned)a.split);
  switch (op.variant) {
    case 32:
      grid.y = (unsigned)cdiv(a.K, 32);
      return (int)launch_k(conv_tc_kernel<32>, grid, dim3(TC_THREADS), (size_t)TcSmem<32>::TOTAL, st,
                           (unsigned)a.split, a);
    case 64:
      grid.y = (unsigned)cdiv(a.K, 64);
      return (int)launch_k(conv_tc_kernel<64>, grid, dim3(TC_THREADS), (size_t)TcSmem<64>::TOTAL, st,
                           (unsigned)a.split, a);
    case 128:
      grid.y = (unsigned)cdiv(a.K, 128);
      return (int)launch_k(conv_tc_kernel<128>, grid, dim3(TC_THREADS), (size_t)TcSmem<128>::TOTAL, st,
                           (unsigned)a.split, a);
    case 256:
      grid.y = (unsigned)cdiv(a.K, 256);
      return (int)launch_k(conv_tc_kernel<256>, grid, dim3(TC_THREADS), (size_t)TcSmem<256>::TOTAL, st,
                           (unsigned)a.split, a);
    default:
      return (int)cudaErrorInvalidValue;
  }
}

// Pre-set the dynamic smem limits outside any stream capture.
void init_tc_kernels() {
#define SW_TC_SWZ_ATTR(BN_)                                                                                  \
  cudaFuncSetAttribute(conv_tc_tma_kernel<BN_, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                       TcSmem<BN_>::TOTAL);                                                                  \
  cudaFuncSetAttribute(conv_tc_tma_kernel<BN_, 0, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  SW_TC_SWZ_ATTR(32)
  SW_TC_SWZ_ATTR(64)
  SW_TC_SWZ_ATTR(128)
  SW_TC_SWZ_ATTR(256)
#undef SW_TC_SWZ_ATTR
  cudaFuncSetAttribute(conv_tc_tma_persistent_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TcSmem<32>::P_TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_persistent_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TcSmem<64>::P_TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_persistent_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TcSmem<128, 2>::P_TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_persistent_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TcSmem<32>::P_TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_persistent_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TcSmem<64>::P_TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_persistent_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       TcSmem<128, 2>::P_TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<32, 2>::TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<32, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_tma_kernel<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<64, 2>::TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<64, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<32>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_tma_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<32>::TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<32>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<64>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<64>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_tma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<64>::TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<64>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<128>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_tma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<128>::TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<128>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<256>::TOTAL);
  cudaFuncSetAttribute(conv_tc_kernel<256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(conv_tc_tma_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcSmem<256>::TOTAL);
  cudaFuncSetAttribute(conv_tc_tma_kernel<256>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

}  // namespace sw
