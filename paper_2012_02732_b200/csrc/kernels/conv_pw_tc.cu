// Large-batch pointwise (1x1) convolution on tcgen05: a persistent,
// warp-specialised GEMM with double-buffered TMEM accumulators.
//
//   D[pixel][out channel] = sum_c X[pixel][c] * W[out channel][c]
//
// At NASNet batch 256 the pointwise layers are GEMMs with M = 50k-200k
// pixels, K = 264-1056 input channels and N = 44-176 output channels: they
// stream the activations once and are HBM-bound when the tensor pipe is fed.
// The round-1 persistent kernel (conv_tc.cu) ran every K tile through all of
// its threads (split pass, __syncthreads, one issuing thread, a TMEM → register
// promotion) and reached ~1.1 TB/s.  Here every role runs ahead on its own:
//
//  * warp 4: TMA producer — per (pixel tile, K block of 32 channels) one
//    SW128 box of 128 activation rows and the 3xTF32 weight boxes (hi, lo;
//    BN rows) into an S-deep stage ring, gated only by the stage's "empty"
//    barrier (released by the MMAs' commit);
//  * warps 0-3: split the activation box into tf32 hi (in place) / lo (beside
//    it), then arrive on the stage's "ready" barrier;
//  * warp 5: MMA issuer — D_main += A_hi B_hi, D_corr += A_hi B_lo + A_lo B_hi
//    into one of two TMEM accumulator pairs (tile parity), descriptors as
//    loop-invariant bases + immediates (tools/mma_rate.cu);
//  * warps 6-9: epilogue — as soon as a tile's accumulators are complete they
//    drain them (TMEM lane = pixel) with bias (shared memory) + residual +
//    activation into NHWC, while the next tile's MMAs fill the other pair.
//
// Variants 8000 + BN (BN = 48, 64, 96, 128 output channels per N tile) read
// the prepare-time 3xTF32 weight copies; 8100 + BN (8148, 8164, 8196, 8228)
// read the fp32 weight and split it in the kernel (training steps, whose
// weights change every step).
#include <algorithm>

#include "common.cuh"
#include "tma.cuh"

namespace sw {

namespace {

constexpr int PW_BM = 128;  // pixels per tile (UMMA M)
constexpr int PW_BK = 32;   // channels per K block = one 128-B swizzle row
constexpr int PW_THREADS = 320;  // warps 0-3 split, 4 TMA, 5 MMA, 6-9 epilogue

template <int BN>
struct PwSmem {
  static constexpr int A_BYTES = PW_BM * PW_BK * 4;  // 16 KB raw / hi
  static constexpr int B_BYTES = BN * PW_BK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;  // A hi (raw in place), A lo, B hi, B lo
  static constexpr int S = (200 * 1024) / STAGE;
  static constexpr int RING = S * STAGE;
  static constexpr int TOTAL = RING + 1024 + 512;  // + bias [BN] + mbarriers + TMEM slot
  static_assert(S >= 2, "ring");
  static_assert(STAGE % 1024 == 0, "SW128 operands 1024-B aligned");
};

__device__ __forceinline__ void pw_mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void pw_arrive(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ uint64_t pw_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void pw_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void pw_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void pw_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void pw_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void pw_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void pw_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ bool pw_elect() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ float pw_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

struct PwArgs {
  float* __restrict__ out;
  const float* __restrict__ bias;
  const float* __restrict__ res;
  int M, K, P, Q, act, pre_relu, has_res, kblocks, ovec;  // ovec: float4 output / residual rows
  int64_t out_sn, out_sh, out_sw, res_sn, res_sh, res_sw;
  // implicit GEMM (IM2COL): a tile = RT output rows x CQ columns of one image
  // (RT whole rows when Q <= 128, else one row in nseg column segments);
  // K block kq = 32 channels (zero-filled past C) of tap (kq / CB) of R x S
  int mtiles, RT, CQ, nseg, ptiles, CB, C, S, sh, sw, ph, pw;
  // IM2COL: K blocks per accumulation chunk (see PROMO in the kernel);
  // split > 1: the K blocks split over a (1, 1, split) cluster, one tile per
  // CTA, partial tiles reduced through DSMEM in rank order
  int kchunk, split;
};

}  // namespace

// WSPLIT: the weights arrive as plain fp32 (the conv's [K][C] weight, e.g. a
// training step's current parameters) and the split warps split them into
// tf32 hi / lo beside the activations; otherwise the prepare-time 3xTF32
// copies are loaded as they are.
// IM2COL: k x k / strided convs as an implicit GEMM whose activation operand
// is gathered by TMA: one 4-D box [32 channels][Q columns][RT rows][1 image]
// per (tile, tap, channel block) from the NHWC input, at the tap's shifted
// (and, for stride 2, element-strided) coordinates — the hardware zero-fills
// the padding, and the box lands as the tile's 128-B swizzled K-major rows.
template <int BN, bool WSPLIT, bool IM2COL = false, bool PROMO = IM2COL>
__global__ void __launch_bounds__(PW_THREADS, 1)
    conv_pw_tc_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tbh,
                      const __grid_constant__ CUtensorMap tbl, PwArgs a) {
  using L = PwSmem<BN>;
  constexpr int S = L::S;
  extern __shared__ __align__(1024) uint8_t smem[];
  float* bias_s = reinterpret_cast<float*>(smem + L::RING);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::RING + 1024);
  uint64_t* ready = full + S;
  uint64_t* empty = ready + S;
  uint64_t* acc_full = empty + S;  // [2]
  uint64_t* acc_free = acc_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);
  const uint32_t sbase = su32(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.y * BN;
  const int mtiles = a.mtiles;
  const int ntl = mtiles > (int)blockIdx.x ? (mtiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  const uint32_t a_tx = IM2COL ? (uint32_t)(a.RT * a.CQ * PW_BK * 4) : (uint32_t)L::A_BYTES;
  // split-K (IM2COL, a.split > 1): cluster rank z owns K blocks
  // [kb_lo, kb_lo + kb) of the layer's a.kblocks
  const int zr = (PROMO && a.split > 1) ? (int)blockIdx.z : 0;
  const int kb_lo = PROMO ? (zr * a.kblocks) / a.split : 0;
  const int kb = PROMO ? ((zr + 1) * a.kblocks) / a.split - kb_lo : a.kblocks;
  const int total = ntl * kb;  // (tile, K block) sequence of this CTA

  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      pw_mbar_init(su32(&full[i]), 1);
      pw_mbar_init(su32(&ready[i]), 1);
      pw_mbar_init(su32(&empty[i]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      pw_mbar_init(su32(&acc_full[b]), 1);
      pw_mbar_init(su32(&acc_free[b]), 4);  // the 4 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 5) {  // two (main, correction) accumulator pairs
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"((uint32_t)(4 * BN <= 256 ? 256 : 512))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int c = tid; c < BN; c += PW_THREADS) bias_s[c] = (a.bias && n0 + c < a.K) ? a.bias[n0 + c] : 0.f;
  pw_fence_before();
  __syncthreads();
  pw_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 4) {
    // ---- TMA producer ----
    if (lane == 0) {
      prefetch_tmap(&ta);
      prefetch_tmap(&tbh);
      prefetch_tmap(&tbl);
      pdl_wait();
#pragma unroll 1
      for (int q = 0; q < total; ++q) {
        const int s = q % S;
        if (q >= S) mbar_wait_parity(su32(&empty[s]), (uint32_t)(((q / S) - 1) & 1));
        const int tg = (int)blockIdx.x + (q / kb) * (int)gridDim.x;  // tile
        const int kq = kb_lo + q % kb;
        int k0 = kq * PW_BK;
        const uint32_t st = sbase + s * L::STAGE;
        mbar_expect_tx(su32(&full[s]), a_tx + (WSPLIT ? 1 : 2) * L::B_BYTES);
        if constexpr (IM2COL) {
          const int nb = tg / a.ptiles, rem = tg - nb * a.ptiles;
          const int prow = rem / a.nseg, seg = rem - prow * a.nseg;
          const int p0 = prow * a.RT, q0 = seg * a.CQ;
          const int tap = kq / a.CB, c0 = (kq - tap * a.CB) * PW_BK;
          const int r = tap / a.S, sx = tap - r * a.S;
          k0 = tap * a.C + c0;  // weight columns of (tap, channel block); past C the activations are zero
          tma_load_4d(st, &ta, c0, q0 * a.sw - a.pw + sx, p0 * a.sh - a.ph + r, nb, su32(&full[s]));
        } else {
          tma_load_2d(st, &ta, k0, tg * PW_BM, su32(&full[s]));
        }
        tma_load_2d(st + 2 * L::A_BYTES, &tbh, k0, n0, su32(&full[s]));
        if constexpr (!WSPLIT) tma_load_2d(st + 2 * L::A_BYTES + L::B_BYTES, &tbl, k0, n0, su32(&full[s]));
      }
    }
  } else if (warp < 4) {
    // ---- split: activations → tf32 hi (in place) / lo ----
#pragma unroll 1
    for (int q = 0; q < total; ++q) {
      const int s = q % S;
      mbar_wait_parity(su32(&full[s]), (uint32_t)((q / S) & 1));
      float4* hi = reinterpret_cast<float4*>(smem + s * L::STAGE);
      float4* lo = reinterpret_cast<float4*>(smem + s * L::STAGE + L::A_BYTES);
#pragma unroll 4
      for (int i = tid; i < L::A_BYTES / 16; i += 128) {
        float4 x = hi[i];
        if (a.pre_relu) x = make_float4(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f), fmaxf(x.z, 0.f), fmaxf(x.w, 0.f));
        const float4 h = make_float4(pw_tf32(x.x), pw_tf32(x.y), pw_tf32(x.z), pw_tf32(x.w));
        hi[i] = h;
        lo[i] = make_float4(pw_tf32(x.x - h.x), pw_tf32(x.y - h.y), pw_tf32(x.z - h.z), pw_tf32(x.w - h.w));
      }
      if constexpr (WSPLIT) {
        float4* bhi = reinterpret_cast<float4*>(smem + s * L::STAGE + 2 * L::A_BYTES);
        float4* blo = reinterpret_cast<float4*>(smem + s * L::STAGE + 2 * L::A_BYTES + L::B_BYTES);
#pragma unroll 2
        for (int i = tid; i < L::B_BYTES / 16; i += 128) {
          const float4 x = bhi[i];
          const float4 h = make_float4(pw_tf32(x.x), pw_tf32(x.y), pw_tf32(x.z), pw_tf32(x.w));
          bhi[i] = h;
          blo[i] = make_float4(pw_tf32(x.x - h.x), pw_tf32(x.y - h.y), pw_tf32(x.z - h.z), pw_tf32(x.w - h.w));
        }
      }
      fence_proxy_async_cta();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0) pw_arrive(su32(&ready[s]));
    }
  } else if (warp == 5) {
    // ---- MMA issuer ----
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                               ((uint32_t)(PW_BM >> 4) << 24);
    const uint64_t a0 = pw_desc_sw128(sbase);
    // PROMO (IM2COL): a tile's K blocks run in chunks of a.kchunk, each into a
    // fresh accumulator pair (chunk parity), so no TMEM accumulation chain is
    // longer than one chunk; the epilogue sums the chunks in fp32 registers.
    // (The tensor pipe's fp32 accumulate truncates: over the 27-45 K blocks of
    // an implicit-GEMM 3x3 / 5x5 layer one chain biased outputs by ~-1.3e-6
    // relative, enough to move Inception-v3's logits past the fp32 gate.)
    const int G = PROMO ? a.kchunk : kb;
    int u = 0;  // accumulation unit (tile, or tile chunk) sequence of this CTA
#pragma unroll 1
    for (int t = 0; t < ntl; ++t) {
#pragma unroll 1
      for (int j0 = 0; j0 < kb; j0 += G, ++u) {
        const int b = u & 1;
        const int j1 = min(kb, j0 + G);
        if (u >= 2) mbar_wait_parity(su32(&acc_free[b]), (uint32_t)(((u >> 1) - 1) & 1));
        pw_fence_after();
        const uint32_t dmain = tmem + (uint32_t)(b * 2 * BN), dcorr = dmain + BN;
#pragma unroll 1
        for (int kq = j0; kq < j1; ++kq) {
          const int q = t * kb + kq;
          const int s = q % S;
          mbar_wait_parity(su32(&ready[s]), (uint32_t)((q / S) & 1));
          pw_fence_after();
          if (pw_elect()) {
            const uint64_t st = a0 + (uint64_t)((s * L::STAGE) >> 4);
#pragma unroll
            for (int ks = 0; ks < PW_BK / 8; ++ks) {
              const uint64_t ah = st + (uint64_t)(ks * 2);  // +32 B inside the swizzle atom
              const uint64_t al = ah + (uint64_t)(L::A_BYTES >> 4);
              const uint64_t bh = ah + (uint64_t)((2 * L::A_BYTES) >> 4);
              const uint64_t bl = bh + (uint64_t)(L::B_BYTES >> 4);
              const uint32_t acc = (kq != j0 || ks) ? 1u : 0u;
              pw_mma(dmain, ah, bh, idesc, acc);
              pw_mma(dcorr, ah, bl, idesc, acc);
              pw_mma(dcorr, al, bh, idesc, 1u);
            }
            pw_commit(su32(&empty[s]));
            if (kq == j1 - 1) pw_commit(su32(&acc_full[b]));
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---- epilogue: TMEM lane = pixel row ----
    pdl_wait();  // residual / output buffers of earlier tasks
    const int quad = warp & 3;  // TMEM lanes 32*quad .. +31
    const int row = quad * 32 + lane;
    int u = 0;  // accumulation unit sequence (as the MMA issuer counts it)
#pragma unroll 1
    for (int t = 0; t < ntl; ++t) {
      const int b = t & 1;
      if constexpr (!PROMO) {
        mbar_wait_parity(su32(&acc_full[b]), (uint32_t)((t >> 1) & 1));
        pw_fence_after();
      }
      const int tg = (int)blockIdx.x + t * (int)gridDim.x;
      int qq, pp, nb;
      bool ok;
      if constexpr (IM2COL) {  // tile = RT x CQ output pixels of one image; rows past RT*CQ hold none
        nb = tg / a.ptiles;
        const int rem = tg - nb * a.ptiles;
        const int prow = rem / a.nseg, seg = rem - prow * a.nseg;
        const int rr = row / a.CQ;
        qq = seg * a.CQ + (row - rr * a.CQ);
        pp = prow * a.RT + rr;
        ok = rr < a.RT && pp < a.P && qq < a.Q;
      } else {
        const int m = tg * PW_BM + row;
        ok = m < a.M;
        qq = m % a.Q;
        const int tt = m / a.Q;
        pp = tt % a.P;
        nb = tt / a.P;
      }
      float* o = a.out + (ok ? nb * a.out_sn + pp * a.out_sh + qq * a.out_sw : 0) + n0;
      const float* rp = (a.has_res && ok) ? a.res + nb * a.res_sn + pp * a.res_sh + qq * a.res_sw + n0 : nullptr;
      if constexpr (PROMO) {
        // sum the tile's chunk accumulators (main + correction) in fp32
        // registers, releasing each TMEM pair as soon as it is read
        float racc[BN];
#pragma unroll
        for (int j = 0; j < BN; ++j) racc[j] = 0.f;
#pragma unroll 1
        for (int j0 = 0; j0 < kb; j0 += a.kchunk, ++u) {
          const int bu = u & 1;
          mbar_wait_parity(su32(&acc_full[bu]), (uint32_t)((u >> 1) & 1));
          pw_fence_after();
          const uint32_t tu = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(bu * 2 * BN);
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float v[16], w[16];
            pw_ld16(tu + (uint32_t)c0, v);
            pw_ld16(tu + (uint32_t)(BN + c0), w);
            pw_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) racc[c0 + j] += v[j] + w[j];
          }
          pw_fence_before();
          __syncwarp();
          if (lane == 0) pw_arrive(su32(&acc_free[bu]));
        }
        if (a.split > 1) {
          // one tile per CTA: the ring is quiescent (every MMA has completed);
          // park the partial tile, rows of BN + 4 floats (16-B aligned,
          // conflict-free float4 rows), for the rank-ordered sum
          float4* prow = reinterpret_cast<float4*>(smem) + row * (BN / 4 + 1);
#pragma unroll
          for (int j = 0; j < BN; j += 4) prow[j / 4] = make_float4(racc[j], racc[j + 1], racc[j + 2], racc[j + 3]);
          continue;
        }
        if (ok) {
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            const int nv = min(16, a.K - n0 - c0);
            if (nv <= 0) break;
            if (a.ovec && nv == 16) {
#pragma unroll
              for (int j = 0; j < 16; j += 4) {
                float4 x = make_float4(racc[c0 + j], racc[c0 + j + 1], racc[c0 + j + 2], racc[c0 + j + 3]);
                x = f4add(x, *reinterpret_cast<const float4*>(bias_s + c0 + j));
                if (rp) x = f4add(x, *reinterpret_cast<const float4*>(rp + c0 + j));
                *reinterpret_cast<float4*>(o + c0 + j) = act4(x, a.act);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (j >= nv) break;
                float x = racc[c0 + j] + bias_s[c0 + j];
                if (rp) x += rp[c0 + j];
                o[c0 + j] = apply_act(x, a.act);
              }
            }
          }
        }
        continue;
      }
      const uint32_t tl = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * 2 * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16], w[16];
        pw_ld16(tl + (uint32_t)c0, v);
        pw_ld16(tl + (uint32_t)(BN + c0), w);
        float r[16];
        const int nv = min(16, a.K - n0 - c0);
        if (rp) {
#pragma unroll
          for (int j = 0; j < 16; ++j) r[j] = j < nv ? rp[c0 + j] : 0.f;
        }
        pw_wait_ld();
        if (!ok || nv <= 0) continue;
        if (a.ovec && nv == 16) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 x = make_float4(v[j] + w[j], v[j + 1] + w[j + 1], v[j + 2] + w[j + 2], v[j + 3] + w[j + 3]);
            x = f4add(x, *reinterpret_cast<const float4*>(bias_s + c0 + j));
            if (rp) x = f4add(x, make_float4(r[j], r[j + 1], r[j + 2], r[j + 3]));
            *reinterpret_cast<float4*>(o + c0 + j) = act4(x, a.act);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j >= nv) break;
            float x = v[j] + w[j] + bias_s[c0 + j];
            if (rp) x += r[j];
            o[c0 + j] = apply_act(x, a.act);
          }
        }
      }
      pw_fence_before();
      __syncwarp();
      if (lane == 0) pw_arrive(su32(&acc_free[b]));
    }
  }
  if constexpr (PROMO) {
    if (a.split > 1) {
      // every rank's partial is parked in its smem: each rank's epilogue
      // warps sum their channel slice over ranks 0..split-1 in order (DSMEM
      // loads), add bias / residual / activation and store; the second
      // cluster barrier keeps every CTA's shared memory alive until all those
      // loads are done
      __syncwarp();
      asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
      cluster_wait();
      if (warp >= 6) {
        // rank z owns the 4-channel groups [z*G/split, (z+1)*G/split) of the
        // tile: it sums every rank's partial of those channels in rank order
        // (float4 DSMEM loads, all ranks' loads of a group in flight at once)
        // and applies bias / residual / activation — the same bits whichever
        // rank does it, the reduction spread over the cluster
        const int row = (warp & 3) * 32 + lane;
        const int tg = (int)blockIdx.x;
        const int nb = tg / a.ptiles;
        const int rem = tg - nb * a.ptiles;
        const int prow = rem / a.nseg, seg = rem - prow * a.nseg;
        const int rr = row / a.CQ;
        const int qq = seg * a.CQ + (row - rr * a.CQ), pp = prow * a.RT + rr;
        const bool ok = ntl > 0 && rr < a.RT && pp < a.P && qq < a.Q;
        if (ok) {
          float* o = a.out + nb * a.out_sn + pp * a.out_sh + qq * a.out_sw + n0;
          const float* rp = a.has_res ? a.res + nb * a.res_sn + pp * a.res_sh + qq * a.res_sw + n0 : nullptr;
          const uint32_t rowaddr = sbase + (uint32_t)(row * (BN + 4) * 4);
          const int nv = min(BN, a.K - n0);
          constexpr int G = BN / 4;
          const int g0 = (zr * G) / a.split, g1 = ((zr + 1) * G) / a.split;
#pragma unroll 1
          for (int g = g0; g < g1; ++g) {
            const int j0 = 4 * g;
            if (j0 >= nv) break;
            float4 v[8];
#pragma unroll
            for (int z = 0; z < 8; ++z) {
              if (z < a.split) {
                const uint32_t src = mapa_rank(rowaddr + (uint32_t)(j0 * 4), (uint32_t)z);
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[z].x), "=f"(v[z].y), "=f"(v[z].z), "=f"(v[z].w)
                             : "r"(src));
              }
            }
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int z = 0; z < 8; ++z)
              if (z < a.split) x = f4add(x, v[z]);
            if (a.ovec && j0 + 4 <= nv) {
              float4 y = f4add(x, *reinterpret_cast<const float4*>(bias_s + j0));
              if (rp) y = f4add(y, *reinterpret_cast<const float4*>(rp + j0));
              *reinterpret_cast<float4*>(o + j0) = act4(y, a.act);
            } else {
              const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (j0 + i >= nv) break;
                float y = xs[i] + bias_s[j0 + i];
                if (rp) y += rp[j0 + i];
                o[j0 + i] = apply_act(y, a.act);
              }
            }
          }
        }
      }
      __syncwarp();
      asm volatile("barrier.cluster.arrive.aligned;" ::: "memory");
      cluster_wait();
    }
  }
  pw_fence_before();
  __syncthreads();
  if (warp == 5) {
    pw_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"((uint32_t)(4 * BN <= 256 ? 256 : 512))
                 : "memory");
  }
}

template <int BN, bool WSPLIT, bool IM2COL = false>
static int launch_pw(const sw_op_desc& op, cudaStream_t st) {
  const int64_t* p = op.params;
  const int N = (int)p[SP_N], H = (int)p[SP_H], W = (int)p[SP_W], C = (int)p[SP_C];
  const int P = (int)p[SP_P], Q = (int)p[SP_Q], K = (int)p[SP_K];
  const int64_t in_sn = p[SP_IN_SN], in_sh = p[SP_IN_SH], in_sw = p[SP_IN_SW], in_sc = p[SP_IN_SC];
  const int64_t osc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1, rsc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  const int Kpad = (int)p[SP_KPAD];
  PwArgs a;
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.bias = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.M = N * P * Q;
  a.K = K;
  a.P = P;
  a.Q = Q;
  a.act = (int)p[SP_ACT];
  a.pre_relu = (int)p[SP_PRE_RELU];
  a.has_res = (int)p[SP_HAS_RES];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  if (a.M == 0 || K == 0) return 0;
  // 1x1 / stride 1 / unpadded on dense NHWC pixel rows (a channel slice of a
  // concat is fine), 16-B aligned rows and outputs; NHWC outputs
  const void* in = reinterpret_cast<const void*>(op.ptrs[PT_IN]);
  const void* whi = reinterpret_cast<const void*>(WSPLIT ? op.ptrs[PT_W] : op.ptrs[PT_W_TC_HI]);
  const void* wlo = reinterpret_cast<const void*>(WSPLIT ? op.ptrs[PT_W] : op.ptrs[PT_W_TC_LO]);
  const int R = (int)p[SP_R], S = (int)p[SP_S];
  const int sh = (int)p[SP_STRIDE_H], sw = (int)p[SP_STRIDE_W];
  if (IM2COL) {
    // NHWC input (any pixel / row / image strides that are 16-B multiples),
    // whole 128-B channel blocks per tap, output rows of <= 128 pixels
    if (in_sc != 1 || C % 4 || (in_sw & 3) || (in_sh & 3) || (in_sn & 3) || (op.ptrs[PT_IN] & 15) ||
        (sh != 1 && sh != 2) || (sw != 1 && sw != 2) || osc != 1 || (a.has_res && rsc != 1) || !whi || !wlo ||
        Kpad % PW_BK || Kpad < R * S * C)
      return (int)cudaErrorInvalidValue;
  } else if (R != 1 || S != 1 || sh != 1 || sw != 1 || p[SP_PAD_H] || p[SP_PAD_W] ||
             in_sc != 1 || C % 4 || (in_sw & 3) || (op.ptrs[PT_IN] & 15) || in_sn != (int64_t)H * W * in_sw ||
             in_sh != (int64_t)W * in_sw || osc != 1 || (a.has_res && rsc != 1) || !whi || !wlo ||
             (!WSPLIT && Kpad % PW_BK)) {
    return (int)cudaErrorInvalidValue;
  }
  // float4 epilogue rows when output (and residual) rows are 16-B aligned
  // (e.g. not for an 11-channel NHWC map: scalar stores)
  a.ovec = !((op.ptrs[PT_OUT] & 15) || (a.out_sw & 3) || (a.out_sh & 3) || (a.out_sn & 3) ||
             (a.has_res && ((op.ptrs[PT_RES] & 15) || (a.res_sw & 3) || (a.res_sh & 3) || (a.res_sn & 3))));
  a.kblocks = WSPLIT ? (C + PW_BK - 1) / PW_BK : Kpad / PW_BK;
  CUtensorMap ta, tbh, tbl;
  a.mtiles = (a.M + PW_BM - 1) / PW_BM;
  a.kchunk = a.kblocks;
  a.split = 1;
  if (IM2COL) {
    if (Q <= PW_BM) {
      a.RT = std::min(PW_BM / Q, P);
      if (a.RT * sh > 256) a.RT = 256 / sh;
      a.nseg = 1;
      a.CQ = Q;
    } else {
      a.RT = 1;
      a.nseg = (Q + PW_BM - 1) / PW_BM;
      a.CQ = (Q + a.nseg - 1) / a.nseg;
    }
    a.ptiles = (P + a.RT - 1) / a.RT * a.nseg;
    a.mtiles = N * a.ptiles;
    a.CB = (C + PW_BK - 1) / PW_BK;
    a.C = C;
    a.kblocks = R * S * a.CB;
    // chunks of <= 8 K blocks (256 products), balanced across the tile's K
    a.split = std::max(1, std::min((int)p[SP_SPLIT_K], a.kblocks));
    const int kbr = (a.kblocks + a.split - 1) / a.split;
    const int nch = (kbr + 7) / 8;
    a.kchunk = (kbr + nch - 1) / nch;
    a.S = S;
    a.sh = sh;
    a.sw = sw;
    a.ph = (int)p[SP_PAD_H];
    a.pw = (int)p[SP_PAD_W];
    const uint64_t dims[4] = {(uint64_t)C, (uint64_t)W, (uint64_t)H, (uint64_t)N};
    const uint64_t strides[3] = {(uint64_t)in_sw * 4, (uint64_t)in_sh * 4, (uint64_t)in_sn * 4};
    const uint32_t box[4] = {PW_BK, (uint32_t)(a.CQ * sw), (uint32_t)(a.RT * sh), 1};
    const uint32_t es[4] = {1, (uint32_t)sw, (uint32_t)sh, 1};
    if (!encode_tmap_f32(&ta, in, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, es))
      return (int)cudaErrorInvalidValue;
  } else {
    const uint64_t dims[2] = {(uint64_t)C, (uint64_t)a.M};
    const uint64_t strides[1] = {(uint64_t)in_sw * 4};
    const uint32_t box[2] = {PW_BK, PW_BM};
    if (!encode_tmap_f32(&ta, in, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B)) return (int)cudaErrorInvalidValue;
  }
  {  // pre-split copies [K][Kpad], or the fp32 weight [K][C] (1x1)
    const uint64_t wcols = WSPLIT ? (uint64_t)C : (uint64_t)Kpad;
    const uint64_t dims[2] = {wcols, (uint64_t)K};
    const uint64_t strides[1] = {wcols * 4};
    const uint32_t box[2] = {PW_BK, (uint32_t)BN};
    if (!encode_tmap_f32(&tbh, whi, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode_tmap_f32(&tbl, wlo, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return (int)cudaErrorInvalidValue;
  }
  const int ntn = (K + BN - 1) / BN;
  // split-K: one tile per CTA (the cluster reduces it); else persistent
  const int gx = a.split > 1 ? a.mtiles : std::max(1, std::min(a.mtiles, std::max(1, 148 / ntn)));
  if (a.split > 8) return (int)cudaErrorInvalidValue;
  return (int)launch_k(conv_pw_tc_kernel<BN, WSPLIT, IM2COL>, dim3((unsigned)gx, (unsigned)ntn, (unsigned)a.split),
                       dim3(PW_THREADS), (size_t)PwSmem<BN>::TOTAL, st, (unsigned)a.split, ta, tbh, tbl, a);
}

int launch_conv_pw_tc(const sw_op_desc& op, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (op.variant) {
    case 8048: return launch_pw<48, false>(op, st);
    case 8064: return launch_pw<64, false>(op, st);
    case 8096: return launch_pw<96, false>(op, st);
    case 8128: return launch_pw<128, false>(op, st);
    // 8100 + BN: fp32 weights split in-kernel (no prepare-time copies: training)
    case 8148: return launch_pw<48, true>(op, st);
    case 8164: return launch_pw<64, true>(op, st);
    case 8196: return launch_pw<96, true>(op, st);
    case 8228: return launch_pw<128, true>(op, st);
    // 8400 + BN: k x k / strided implicit GEMM, TMA im2col boxes (pre-split weights)
    case 8448: return launch_pw<48, false, true>(op, st);
    case 8464: return launch_pw<64, false, true>(op, st);
    case 8496: return launch_pw<96, false, true>(op, st);
    case 8528: return launch_pw<128, false, true>(op, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

void init_pw_tc_kernels() {
#define SW_PW_ATTR(BN_, WS_) \
  cudaFuncSetAttribute(conv_pw_tc_kernel<BN_, WS_>, cudaFuncAttributeMaxDynamicSharedMemorySize, PwSmem<BN_>::TOTAL);
  SW_PW_ATTR(48, false) SW_PW_ATTR(64, false) SW_PW_ATTR(96, false) SW_PW_ATTR(128, false)
  SW_PW_ATTR(48, true) SW_PW_ATTR(64, true) SW_PW_ATTR(96, true) SW_PW_ATTR(128, true)
#undef SW_PW_ATTR
#define SW_PW_ATTR_I(BN_)                                                                                \
  cudaFuncSetAttribute(conv_pw_tc_kernel<BN_, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       PwSmem<BN_>::TOTAL);
  SW_PW_ATTR_I(48) SW_PW_ATTR_I(64) SW_PW_ATTR_I(96) SW_PW_ATTR_I(128)
#undef SW_PW_ATTR_I
}

}  // namespace sw
