// Weight-streaming convolution on tcgen05 for few output pixels (batch 1).
//
// At batch 1 the deep layers of ResNet-50 / Inception-v3 / NASNet are GEMMs
// with M = P*Q <= a few hundred pixels and megabytes of weights: the layer
// costs one pass over its weights, so every SM must pull weights with many
// bytes in flight.  This kernel swaps the GEMM operands so the weights are
// the 128-row UMMA A operand and the pixels the N dimension:
//
//   D[out channel][pixel] = sum_k W[out channel][k] * X[pixel][k],  k = (r, s, c)
//
// (UMMA M = 128 over a 64-channel tile, see TCS_BM below.)
//
//  * grid = (out-channel tiles of 64) x (pixel tiles of NT) x split, the
//    split-K ranks of one tile form a thread-block cluster (<= 16);
//  * weights (3xTF32 hi / lo) are pre-packed at plan time as the shared-memory
//    images of the K-major no-swizzle UMMA layout, [out tile][K block][hi|lo]
//    (engine.py tcs_pack): a CTA's K slice is one contiguous run of 16-KB
//    blocks that streams by 1-D bulk copies (row-strided 128-B TMA boxes
//    reached 0.67 TB/s of HBM, ncu r02e), requested before the PDL wait
//    (constants), so a CTA has up to ~190 KB of weights in flight;
//  * im2col activation rows (16-B chunks of 4 channels, zero-filled
//    out-of-range taps) arrive by cp.async into a deep raw ring (refilled as
//    soon as a slot is consumed, never gated by the tensor pipe) and are split
//    into tf32 hi / lo (no-swizzle K-major layout) by the 128 threads;
//  * warp specialised: warp 4 streams the weights through a W-deep ring
//    (freed by the MMA commits), warps 0-3 load / split activations through
//    their own SB-deep ring, warp 5 issues D_main += A_hi·B_hi and
//    D_corr += A_hi·B_lo + A_lo·B_hi (two TMEM accumulators of NT columns)
//    per 8-wide K step as soon as both operands of a K block are in;
//  * epilogue: TMEM → smem tile [pixel][channel] → split-K ranks push each
//    peer its pixel rows with bulk DSMEM copies (one cluster barrier once the
//    rings are dead), each rank sums its rows in a fixed order (deterministic)
//    and applies bias (folded BN), residual and activation with coalesced
//    NHWC channel-row stores.
//
// Variants 6000 + NT (NT = 32, 64, 128 pixels per tile).  Variants 7000 + NT
// are the bf16 path (Engine(precision="bf16"), a separately stated
// tolerance): bf16 weight image, activations rounded to bf16 in shared
// memory, one kind::f16 MMA per 16-wide K step into one fp32 accumulator.
#include <cooperative_groups.h>

#include <algorithm>

#include <cuda_bf16.h>

#include "common.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace sw {

namespace {

struct TcsArgs {
  const float* __restrict__ in;
  float* __restrict__ out;
  const float* __restrict__ bias;
  const float* __restrict__ res;
  const float* __restrict__ wimg;  // [out tile][K block][hi | lo][8 chunks][128 rows][4]
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, pre_relu, has_res;
  int64_t in_sn, in_sh, in_sw;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
  int M, Kdim, Kpad, split;
  int ovec;  // output (and residual) pixel rows 16-B aligned with unit channel stride
};

// Out channels per tile = UMMA M = 128.  (A 64-channel tile with the MMA's
// rows 64-127 aliasing the next K chunk doubled the CTAs per layer but
// measured slower: the MMA count per output doubles, r02i.)
constexpr int TCS_BM = 128;
constexpr int TCS_UM = 128;  // UMMA M
constexpr int TCS_BK = 32;   // fp32 per K block = one 128-B swizzle row
constexpr int TCS_THREADS = 192;  // warps 0-3 activations + epilogue, 4 weight TMA, 5 MMA issue

template <int NT, bool BF16 = false>
struct TcsSmem {
  // weights per K block: 3xTF32 hi | lo (2 x 16 KB) or bf16 (8 KB)
  static constexpr int A_BYTES = TCS_BM * TCS_BK * (BF16 ? 2 : 4);
  static constexpr int W_STAGE = BF16 ? A_BYTES : 2 * A_BYTES;
  static constexpr int B_BYTES = NT * TCS_BK * 4;      // one raw fp32 activation K block
  static constexpr int B_OP = NT * TCS_BK * (BF16 ? 2 : 4);  // one activation operand (hi or lo / bf16)
  static constexpr int B_STAGE = BF16 ? B_OP : 2 * B_OP;
  // raw activation ring RB deep (refilled as soon as the split consumed a
  // slot — never gated by the tensor pipe), split ring SB, weight ring W
  // (NT = 64 fp32: 8 raw K blocks in flight and a 2-deep split ring — the
  // im2col gathers, not the tensor pipe, pace a batch-1 layer: 0.77 → 0.48 us
  // per K block on ResNet-50 layer4, probe r03z)
  static constexpr int RB = NT == 32 ? 16 : (NT == 64 && !BF16 ? 8 : 4);
  static constexpr int SB = NT == 128 || (NT == 64 && !BF16) ? 2 : 4;
  static constexpr int W = BF16 ? 8 : (NT == 128 ? 2 : 4);
  static constexpr int RAW_OFF = W * W_STAGE;
  static constexpr int B_OFF = RAW_OFF + RB * B_BYTES;
  static constexpr int RING = B_OFF + SB * B_STAGE;
  static constexpr int ROW = TCS_BM * 4;               // epilogue tile row: 128 channels
  static constexpr int TOTAL = RING + 256;             // + mbarriers + TMEM slot
  // main (+ correction) accumulators
  static constexpr int COLS = (BF16 ? NT : 2 * NT) < 32 ? 32 : (BF16 ? NT : 2 * NT);
  static_assert(NT == 32 || NT == 64 || NT == 128, "pixel tile");
  static_assert(TOTAL <= 227 * 1024, "smem");
  static_assert(NT * ROW * 2 <= RING, "epilogue tiles (part + receive) fit the dead ring");
};

__device__ __forceinline__ void mbar_init_n(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive1(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}


__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);  // .x (low half) = lo
  return *reinterpret_cast<const uint32_t*>(&v);
}

__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, float (&v)[16]) {
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

__device__ __forceinline__ void cp16z(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit_g() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_g() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tc_fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

}  // namespace

template <int NT, bool BF16>
__global__ void __launch_bounds__(TCS_THREADS, 1)
    conv_tcs_kernel(TcsArgs a) {
  using L = TcsSmem<NT, BF16>;
  constexpr int W = L::W, SB = L::SB;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* wfull = reinterpret_cast<uint64_t*>(smem + L::RING);
  uint64_t* wfree = wfull + W;
  uint64_t* bready = wfree + W;
  uint64_t* bfree = bready + SB;
  uint64_t* accfull = bfree + SB;
  uint64_t* recv = accfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv + 1);
  const uint32_t sbase = su32(smem);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int n0 = blockIdx.x * TCS_BM;  // out channels
  const int m0 = blockIdx.y * NT;      // pixels
  const int ktiles = a.Kpad / TCS_BK;
  const int per = (ktiles + a.split - 1) / a.split;
  const int kt0 = blockIdx.z * per;
  const int iters = max(0, min(ktiles, kt0 + per) - kt0);
  probe_begin();

  if (tid == 0) {
    for (int i = 0; i < W; ++i) {
      mbar_init_n(su32(&wfull[i]), 1);
      mbar_init_n(su32(&wfree[i]), 1);
    }
    for (int i = 0; i < SB; ++i) {
      mbar_init_n(su32(&bready[i]), 1);
      mbar_init_n(su32(&bfree[i]), 1);
    }
    mbar_init_n(su32(accfull), 1);
    mbar_init_n(su32(recv), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"((uint32_t)L::COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before_sync();
  __syncthreads();
  tc_fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // folded-BN bias of this thread's 4 epilogue channels: constants, fetched
  // now so their (cold) loads are not on the epilogue's critical path
  float bias[4] = {0.f, 0.f, 0.f, 0.f};
  if (warp < 4 && a.bias) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (n0 + 4 * lane + i < a.K) bias[i] = __ldg(a.bias + n0 + 4 * lane + i);
  }

  if (warp == 4) {
    // ---- weight producer: the whole K slice streams through a W-deep ring,
    // constants, so it runs ahead of the PDL wait
    if (lane == 0) {
      // this CTA's K slice of its out-channel tile is one contiguous run of
      // [hi | lo] (or bf16) images: one bulk copy per K block
      const float* src = a.wimg + ((size_t)blockIdx.x * ktiles + kt0) * (L::W_STAGE / 4);
#pragma unroll 1
      for (int t = 0; t < iters; ++t) {
        const int s = t % W;
        if (t >= W) mbar_wait_parity(su32(&wfree[s]), (uint32_t)(((t / W) - 1) & 1));
        mbar_expect_tx(su32(&wfull[s]), L::W_STAGE);
        bulk_g2s(sbase + s * L::W_STAGE, src + (size_t)t * (L::W_STAGE / 4), L::W_STAGE, su32(&wfull[s]));
      }
    }
  } else if (warp == 5) {
    // ---- MMA issuer: D_main += A_hi B_hi, D_corr += A_hi B_lo + A_lo B_hi.
    // The whole warp runs the loop (uniform control flow) and one elected lane
    // issues.  The loop is unrolled over the W weight stages (SB | W) so every
    // descriptor is a loop-invariant base + an immediate: recomputing them per
    // MMA in registers (R2UR on every issue) held the issue rate to ~135
    // clocks per MMA against 48 for an N = 64 MMA (tools/mma_rate.cu, r02j).
    // D f32; A / B tf32 (2) or bf16 (1), K-major; N = NT pixels, M = 128 channels
    constexpr uint32_t fmt = BF16 ? 1u : 2u;
    constexpr uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(NT >> 3) << 17) |
                               ((uint32_t)(TCS_UM >> 4) << 24);
    // 16-B core-matrix columns: 4 tf32 or 8 bf16; one MMA K step = 32 B = 2 columns
    constexpr uint32_t LBO_B = NT * 16, LBO_A = TCS_BM * 16;
    constexpr int KSTEPS = TCS_BK * (BF16 ? 2 : 4) / 32;
    static_assert(W % SB == 0, "split ring period divides the weight ring");
    const uint64_t a0 = desc_noswz(sbase, LBO_A, 128);
    const uint64_t b0 = desc_noswz(sbase + L::B_OFF, LBO_B, 128);
#pragma unroll 1
    for (int tb = 0; tb < iters; tb += W) {
#pragma unroll
      for (int s = 0; s < W; ++s) {
        const int t = tb + s;
        if (t >= iters) break;
        const int sb = s % SB;
        mbar_wait_parity(su32(&wfull[s]), (uint32_t)((tb / W) & 1));
        if (lane == 0 && t < 24) probe_trace(t);  // weights of K block t in
        mbar_wait_parity(su32(&bready[sb]), (uint32_t)((t / SB) & 1));
        if (lane == 0 && t < 24) probe_trace(24 + t);  // its split activations in
        tc_fence_after_sync();
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < KSTEPS; ++ks) {
            const uint64_t ah = a0 + (uint64_t)((s * L::W_STAGE + ks * 2 * LBO_A) >> 4);
            const uint64_t bh = b0 + (uint64_t)((sb * L::B_STAGE + ks * 2 * LBO_B) >> 4);
            const uint32_t acc = (t | ks) ? 1u : 0u;
            if constexpr (BF16) {
              umma_bf16(tmem, ah, bh, idesc, acc);
            } else {
              const uint64_t al = ah + (uint64_t)(L::A_BYTES >> 4);
              const uint64_t bl = bh + (uint64_t)(L::B_OP >> 4);
              umma_tf32(tmem, ah, bh, idesc, acc);
              umma_tf32(tmem + NT, ah, bl, idesc, acc);
              umma_tf32(tmem + NT, al, bh, idesc, 1u);
            }
          }
          umma_commit(su32(&wfree[s]));
          umma_commit(su32(&bfree[sb]));
        }
        __syncwarp();
      }
    }
    if (elect_one()) umma_commit(su32(accfull));
    __syncwarp();
    if (lane == 0) probe_pt_any(1);  // last MMA issued
  } else {
    // ---- activation warps: im2col rows by cp.async, split into tf32 hi / lo
    const int chunk = tid & 7;
    const int row0 = tid >> 3;  // 0..15
    constexpr int B_ROWS = NT / 16;
    int64_t b_base[B_ROWS];
    int b_ih[B_ROWS], b_iw[B_ROWS];
#pragma unroll
    for (int i = 0; i < B_ROWS; ++i) {
      const int m = m0 + row0 + 16 * i;
      const int q = m % a.Q;
      const int t = m / a.Q;
      b_base[i] = (int64_t)(t / a.P) * a.in_sn;
      b_ih[i] = m < a.M ? (t % a.P) * a.sh - a.ph : -(1 << 28);
      b_iw[i] = q * a.sw - a.pw;
    }
    auto load_b = [&](int t, uint32_t bdst) {
      const int k = (kt0 + t) * TCS_BK + chunk * 4;
      const bool kin = k < a.Kdim;
      const int c = k % a.C;
      const int rs = k / a.C;
      const int s = rs % a.S, r = rs / a.S;
#pragma unroll
      for (int i = 0; i < B_ROWS; ++i) {
        const int rr = row0 + 16 * i;
        const int ih = b_ih[i] + r, iw = b_iw[i] + s;
        const bool ok = kin && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
        cp16z(bdst + chunk * (NT * 16) + (rr >> 3) * 128 + (rr & 7) * 16,
              a.in + (ok ? b_base[i] + ih * a.in_sh + iw * a.in_sw + c : 0), ok);
      }
    };
    pdl_wait();
    probe_pt(2);
    auto raw_slot = [&](int slot) { return sbase + L::RAW_OFF + slot * L::B_BYTES; };
#pragma unroll 1
    for (int t = 0; t < L::RB; ++t) {
      if (t < iters) load_b(t, raw_slot(t));
      cp_commit_g();
    }
#pragma unroll 1
    for (int t = 0; t < iters; ++t) {
      const int sb = t % SB, rb = t % L::RB;
      cp_wait_g<L::RB - 1>();  // raw K block t landed (this thread's part)
      named_bar(1, 128);
      if (t == 0) probe_pt(3);
      if (tid == 0 && t < 8) probe_trace(48 + t);  // raw K block t landed
      // the split slot is free once the MMAs of K block t - SB completed
      if (t >= SB) mbar_wait_parity(su32(&bfree[sb]), (uint32_t)(((t / SB) - 1) & 1));
      const uint8_t* rawb = smem + L::RAW_OFF + rb * L::B_BYTES;
      if constexpr (BF16) {
        // raw 4-float columns 2j, 2j+1 of a row → one 8-bf16 column j
        uint4* ob = reinterpret_cast<uint4*>(smem + L::B_OFF + sb * L::B_STAGE);
#pragma unroll
        for (int i = tid; i < NT * 4; i += 128) {
          const int j = i / NT, row = i - j * NT;
          const int roff = (row >> 3) * 128 + (row & 7) * 16;
          float4 x0 = *reinterpret_cast<const float4*>(rawb + (2 * j) * (NT * 16) + roff);
          float4 x1 = *reinterpret_cast<const float4*>(rawb + (2 * j + 1) * (NT * 16) + roff);
          if (a.pre_relu) {
            x0 = make_float4(fmaxf(x0.x, 0.f), fmaxf(x0.y, 0.f), fmaxf(x0.z, 0.f), fmaxf(x0.w, 0.f));
            x1 = make_float4(fmaxf(x1.x, 0.f), fmaxf(x1.y, 0.f), fmaxf(x1.z, 0.f), fmaxf(x1.w, 0.f));
          }
          ob[(j * (NT * 16) + roff) / 16] = make_uint4(pack_bf16x2(x0.x, x0.y), pack_bf16x2(x0.z, x0.w),
                                                     pack_bf16x2(x1.x, x1.y), pack_bf16x2(x1.z, x1.w));
        }
      } else {
        const float4* raw = reinterpret_cast<const float4*>(rawb);
        float4* hi = reinterpret_cast<float4*>(smem + L::B_OFF + sb * L::B_STAGE);
        float4* lo = reinterpret_cast<float4*>(smem + L::B_OFF + sb * L::B_STAGE + L::B_OP);
#pragma unroll
        for (int i = tid; i < L::B_BYTES / 16; i += 128) {
          float4 x = raw[i];
          if (a.pre_relu) {
            x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
          }
          const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
          hi[i] = h;
          lo[i] = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z), tf32_rna(x.w - h.w));
        }
      }
      fence_proxy_async_cta();
      named_bar(1, 128);  // every thread read raw slot rb and wrote split slot sb
      if (tid == 0) mbar_arrive1(su32(&bready[sb]));
      if (t + L::RB < iters) load_b(t + L::RB, raw_slot(rb));
      cp_commit_g();
    }
  }

  // ---- epilogue (warps 0-3): TMEM (lane = channel, column = pixel) → part[pixel][channel]
  float* part = reinterpret_cast<float*>(smem);
  const int R = NT / a.split;  // pixel rows this rank reduces and stores
  const int me = a.split > 1 ? (int)cluster_rank() : 0;
  if (warp < 4) {
    mbar_wait_parity(su32(accfull), 0);
    tc_fence_after_sync();
    probe_pt(4);
  }
  if (warp < 4) {  // warp w drains TMEM lanes 32w..32w+31 (its sub-partition) = channels
    const int ch = warp * 32 + lane;
    const uint32_t t_row = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < NT; c0 += 16) {
      float v[16], u[16];
      if (iters > 0) {
        tmem_ld_x16(t_row + (uint32_t)c0, v);
        if constexpr (BF16) {
#pragma unroll
          for (int j = 0; j < 16; ++j) u[j] = 0.f;
        } else {
          tmem_ld_x16(t_row + (uint32_t)(NT + c0), u);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = u[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) part[(c0 + j) * TCS_BM + ch] = v[j] + u[j];
    }
    fence_proxy_async_cta();  // part → visible to the bulk-copy proxy
  }
  if (warp < 4) {
    named_bar(1, 128);
    probe_pt(5);
  }
  float* rcv = part + NT * TCS_BM;  // [split - 1][R][64]: peers' rows of my slice
  __syncwarp();
  if (a.split > 1) {
    // every rank's ring is dead (its last MMA completed) before anyone writes into it
    cluster_arrive_relaxed();
    cluster_wait();
    if (tid == 0) probe_trace(56);  // every rank's ring is dead
    if (tid == 0) {
      mbar_expect_tx(su32(recv), (uint32_t)((a.split - 1) * R * L::ROW));
#pragma unroll 1
      for (int r = 0; r < a.split; ++r) {
        if (r == me) continue;
        const int slot = me < r ? me : me - 1;  // my slot in rank r's receive buffer
        bulk_s2peer(mapa_rank(su32(rcv + slot * R * TCS_BM), (uint32_t)r), su32(part + r * R * TCS_BM),
                    (uint32_t)(R * L::ROW), mapa_rank(su32(recv), (uint32_t)r));
      }
      bulk_commit();
    }
    if (warp < 4) mbar_wait_parity(su32(recv), 0);
    if (tid == 0) probe_trace(57);  // peers' rows in
    // once every rank has received its rows every push has read its source:
    // the exit waits on this barrier instead of on the bulk-copy groups
    __syncwarp();
    cluster_arrive_relaxed();
  }
  if (warp < 4) {
    // thread = 4 consecutive output channels (lane) x every 4th pixel row
    // (warp): float4 smem reads, bias, residual and NHWC stores, so a row
    // costs a quarter of the instructions of a channel-per-thread loop (that
    // loop ran ~0.25 us per pixel row, serially, probe r03f)
    const int c4 = 4 * lane;
    const int n = n0 + c4;
    const int rows = min(R, a.M - (m0 + me * R));
    int qq = 0, pp = 0, nb = 0;
    {
      const int m = m0 + me * R + warp;
      qq = m % a.Q;
      const int tt = m / a.Q;
      pp = tt % a.P;
      nb = tt / a.P;
    }
    if (tid == 0) probe_trace(58);
#pragma unroll 2
    for (int j = warp; j < rows; j += 4) {
      const int p = me * R + j;
      float4 v = *reinterpret_cast<const float4*>(part + p * TCS_BM + c4);
      if (a.split > 1) {
        float4 t[15];
#pragma unroll
        for (int r = 0; r < 15; ++r)
          if (r < a.split - 1) t[r] = *reinterpret_cast<const float4*>(rcv + (r * R + j) * TCS_BM + c4);
#pragma unroll
        for (int r = 0; r < 15; ++r)
          if (r < a.split - 1) v = f4add(v, t[r]);
      }
      v = f4add(v, make_float4(bias[0], bias[1], bias[2], bias[3]));
      if (a.ovec && n + 3 < a.K) {
        if (a.has_res)
          v = f4add(v, *reinterpret_cast<const float4*>(a.res + nb * a.res_sn + pp * a.res_sh + qq * a.res_sw + n));
        *reinterpret_cast<float4*>(a.out + nb * a.out_sn + pp * a.out_sh + qq * a.out_sw + n) = act4(v, a.act);
      } else {
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (n + i >= a.K) break;
          float x = vv[i];
          if (a.has_res) x += a.res[nb * a.res_sn + pp * a.res_sh + qq * a.res_sw + (n + i) * a.res_sc];
          a.out[nb * a.out_sn + pp * a.out_sh + qq * a.out_sw + (n + i) * a.out_sc] = apply_act(x, a.act);
        }
      }
#ifdef SW_PROBE
      if (tid == 32 && j < 56) probe_trace(9 + j / 4);  // row j stored (warp 1)
#endif
      qq += 4;
      while (qq >= a.Q) {
        qq -= a.Q;
        if (++pp == a.P) {
          pp = 0;
          ++nb;
        }
      }
    }
    probe_pt(6);
    if (lane == 0) probe_trace(60 + warp);  // warp's stores issued
  }
  if (a.split > 1) cluster_wait();  // every push completed: `part` may be released
  probe_pt(7);
  tc_fence_before_sync();
  __syncthreads();
  probe_pt(8);
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)L::COLS)
                 : "memory");
  }
  probe_end();
}

template <int NT, bool BF16>
static int launch_tcs(const sw_op_desc& op, cudaStream_t st) {
  const int64_t* p = op.params;
  TcsArgs a;
  a.in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.bias = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K];
  a.R = (int)p[SP_R]; a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  a.in_sn = p[SP_IN_SN]; a.in_sh = p[SP_IN_SH]; a.in_sw = p[SP_IN_SW];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.out_sc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1;
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  a.res_sc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  a.M = a.N * a.P * a.Q;
  a.Kdim = a.R * a.S * a.C;
  a.Kpad = (int)p[SP_KPAD];
  a.split = p[SP_SPLIT_K] > 1 ? (int)p[SP_SPLIT_K] : 1;
  if (a.M == 0 || a.K == 0) return 0;
  a.ovec = a.out_sc == 1 && !(op.ptrs[PT_OUT] & 15) && !((a.out_sn | a.out_sh | a.out_sw) & 3) &&
           (!a.has_res || (a.res_sc == 1 && !(op.ptrs[PT_RES] & 15) && !((a.res_sn | a.res_sh | a.res_sw) & 3)));
  a.wimg = reinterpret_cast<const float*>(op.ptrs[PT_WS]);
  // 16-B im2col chunks: 4 consecutive channels of one tap, 16-B aligned rows
  const bool vec = a.C % 4 == 0 && p[SP_IN_SC] == 1 && a.in_sn % 4 == 0 && a.in_sh % 4 == 0 &&
                   a.in_sw % 4 == 0 && (op.ptrs[PT_IN] & 15) == 0;
  // the packed image at PT_WS must be the one this variant reads
  if (p[SP_WS_KIND] != (BF16 ? 1 : 0)) return (int)cudaErrorInvalidValue;
  if (!vec || !a.wimg || (op.ptrs[PT_WS] & 15) || a.Kpad < a.Kdim || a.Kpad % TCS_BK ||
      a.split > 16 || NT % a.split || a.split > a.Kpad / TCS_BK)
    return (int)cudaErrorInvalidValue;
  dim3 grid((unsigned)cdiv(a.K, TCS_BM), (unsigned)cdiv(a.M, NT), (unsigned)a.split);
  return (int)launch_k(conv_tcs_kernel<NT, BF16>, grid, dim3(TCS_THREADS), (size_t)TcsSmem<NT, BF16>::TOTAL, st,
                       (unsigned)a.split, a);
}

int launch_conv_tcs(const sw_op_desc& op, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (op.variant) {
    case 6032: return launch_tcs<32, false>(op, st);
    case 6064: return launch_tcs<64, false>(op, st);
    case 6128: return launch_tcs<128, false>(op, st);
    case 7032: return launch_tcs<32, true>(op, st);
    case 7064: return launch_tcs<64, true>(op, st);
    case 7128: return launch_tcs<128, true>(op, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

void init_tcs_kernels() {
#define SW_TCS_ATTR(NT_, B_)                                                                    \
  cudaFuncSetAttribute(conv_tcs_kernel<NT_, B_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       TcsSmem<NT_, B_>::TOTAL);                                              \
  cudaFuncSetAttribute(conv_tcs_kernel<NT_, B_>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  SW_TCS_ATTR(32, false)
  SW_TCS_ATTR(64, false)
  SW_TCS_ATTR(128, false)
  SW_TCS_ATTR(32, true)
  SW_TCS_ATTR(64, true)
  SW_TCS_ATTR(128, true)
#undef SW_TCS_ATTR
}

}  // namespace sw
