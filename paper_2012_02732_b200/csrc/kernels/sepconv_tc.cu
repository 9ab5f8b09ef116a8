// Fused separable convolution with the pointwise GEMM on the 5th-generation
// tensor cores: depthwise k x k (CUDA cores, TMA-staged input) →
// tcgen05.mma kind::tf32 (3xTF32, TMEM accumulators) → bias / residual /
// activation epilogue, in one persistent, warp-specialised kernel (K_SEPCONV
// variant SEP_TC_VARIANT).
//
// Work unit ("tile") = TN whole images x a band of TH output rows x all Q
// columns (TN*TH*Q <= 128 pixels = the UMMA M rows, one per TMEM lane) x all
// K <= 256 output channels (UMMA N).  The input channels (UMMA K) are
// processed in chunks of 16; chunk number `seq` (running over the CTA's
// tiles) reads patch ring slot seq % SP and belongs to producer group
// g = seq % G, which owns a stage [pointwise weight chunk | A operand].
//
// Roles (480 threads, one CTA per SM):
//   warp 13    patch loader (one thread), up to SP chunks ahead: one 4-D TMA
//              box of the input patch [TN][IH][IW][16 ch] (halo, padding and
//              channels >= C zero-filled by the tensor map) + a bulk copy of
//              the filter chunk [k*k][16] into a patch ring slot;
//   warp 14    weight loader (one thread): a bulk copy of the chunk's 3xTF32
//              pointwise weights (hi | lo, already in the UMMA smem image)
//              into the group's stage once the group's previous MMAs are done;
//   warps 0-7  depthwise producers, two warps per group: a thread owns a
//              PY x PX block of output pixels and one channel quad, walks the
//              block's (PY-1)*s + k patch rows once as register windows of
//              (PX-1)*s + k pixels and feeds every output row each tap row
//              contributes to (shared-memory loads only, no bounds checks);
//              act(dw + b_dw) is split into TF32 hi / lo (round-to-nearest,
//              conv_tc.cu) and stored into the group's A stage in the
//              canonical K-major UMMA layout.  G groups work on G chunks at
//              once (the per-chunk item count alone cannot fill 8 warps);
//   warp 8     MMA issuer (one thread): chunks in order, 2 K-steps x {hi·hi
//              into the tile's main accumulator, hi·lo + lo·hi into its
//              correction accumulator}; tcgen05.commit releases the stage and,
//              after a tile's last chunk, hands the accumulators over;
//   warps 9-12 epilogue: TMEM lanes = tile pixels; tcgen05.ld main +
//              correction (fp32 add), + bias, + residual, activation, float4
//              NHWC stores; then release the TMEM buffer.
// TMEM holds two tiles (main + correction each) when K <= 128, so the
// epilogue of tile i overlaps the depthwise + MMAs of tile i+1; one tile
// (2 x 256 columns) up to K = 256.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace sw {

namespace {

constexpr int ST_BM = 128;  // UMMA M = TMEM lanes
constexpr int ST_CK = 16;   // channels per K chunk (2 UMMA K-steps of 8)
constexpr int ST_PX = 3;    // output pixels per depthwise thread along a row (register window)
constexpr int ST_DW_WARPS = 8;
constexpr int ST_GROUP_WARPS = 2;
constexpr int ST_MMA_WARP = ST_DW_WARPS;
constexpr int ST_LOAD_WARP = ST_DW_WARPS + 5;   // input patches
constexpr int ST_BLOAD_WARP = ST_DW_WARPS + 6;  // pointwise weight chunks
constexpr int ST_THREADS = (ST_DW_WARPS + 7) * 32;
constexpr int ST_MAX_SP = 8;
constexpr int ST_MAX_G = ST_DW_WARPS / ST_GROUP_WARPS;
// A operand (tile pixels x 16 channels, hi or lo): canonical K-major
// SWIZZLE_NONE core matrices, 8 rows x 16 B, 8-row groups 128 B apart (SBO);
// the four 16-B channel quads (K core-matrix columns) ST_LBO_A apart.  2048
// would be dense; +32 B staggers the quads over the banks so a producer
// phase (2 pixels x 4 quads) stores without conflicts.
constexpr int ST_LBO_A = ST_BM * 16 + 32;
constexpr int ST_AHALF = (3 * ST_LBO_A + 2048 + 127) / 128 * 128;
constexpr int ST_SMEM_MAX = 232448;

struct SepTcArgs {
  float* __restrict__ out;
  const float* __restrict__ w_pw;  // [Cpad/16][hi | lo][4 quads][BN][4] (UMMA smem image per chunk)
  const float* __restrict__ w_dw;  // [Cpad/16][R*S][16] chunk-major depthwise filter, zero padded
  const float* __restrict__ b_pw;
  const float* __restrict__ b_dw;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, dw_act, pre_relu, has_res;
  int64_t out_sn, out_sh, out_sw, res_sn, res_sh, res_sw;
  int Cpad, BN, ntile, TN, TH, IH, IW, bands, G, SP, tbufs, ovec;
  uint32_t patch_bytes, filt_bytes, b_bytes;  // per chunk
  uint32_t pstage, gstage, off_b, off_a;      // patch stage / group stage sizes; B / A inside a group stage
  uint32_t off_g, off_bdw, off_bar;           // smem carve-up (bytes); patch ring from 0
};

__device__ __forceinline__ uint64_t st_desc(uint32_t saddr, uint32_t lbo) {
  // SWIZZLE_NONE, K-major: LBO = bytes between the two 16-B K chunks of a
  // K-step, SBO = 128 B between 8-row groups, version 1 (sm_100)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void st_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void st_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_init(uint32_t bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(n) : "memory");
}
__device__ __forceinline__ float st_rn(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void st_ld16(uint32_t taddr, float (&v)[16]) {
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
__device__ __forceinline__ void st_tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void st_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void st_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ float4 st_relu4(float4 x) {
  return make_float4(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f), fmaxf(x.z, 0.f), fmaxf(x.w, 0.f));
}
__device__ __forceinline__ void st_fma4(float4& acc, float4 x, float4 w) {
  acc.x = fmaf(x.x, w.x, acc.x);
  acc.y = fmaf(x.y, w.y, acc.y);
  acc.z = fmaf(x.z, w.z, acc.z);
  acc.w = fmaf(x.w, w.w, acc.w);
}

}  // namespace

// tile index → (first image, first output row); rows of the band past P and
// images past N are invalid slots (computed from zero-filled patches and
// never stored)
__device__ __forceinline__ void st_tile(const SepTcArgs& a, int tile, int& n0, int& r0) {
  n0 = (tile / a.bands) * a.TN;
  r0 = (tile % a.bands) * a.TH;
}

// ST_PY <= 3: register-blocked items (ST_PY output rows); ST_PY >= 4
// (stride 1, wide maps): sliding-row producers with PXN = ST_PY columns
template <int KS, int SW, int ST_PY>
__global__ void __launch_bounds__(ST_THREADS, 1)
    sepconv_tc_kernel(const __grid_constant__ CUtensorMap tin, SepTcArgs a) {
  constexpr bool SLIDE = SW == 1 && ST_PY >= 4;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = su32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.G;
  const int nchunks = a.Cpad / ST_CK;
  const int BN = a.BN;
  const int t0 = (int)blockIdx.x;
  const int tstride = (int)gridDim.x;
  const int ntiles = t0 < a.ntile ? (a.ntile - 1 - t0) / tstride + 1 : 0;
  const int total = ntiles * nchunks;  // chunk sequence of this CTA
  probe_begin();

  // barriers: p_full[SP], p_empty[SP], b_full[G], a_full[G], a_empty[G], t_full[2], t_empty[2], tmem slot
  const int SP = a.SP;
  const uint32_t bar = sbase + a.off_bar;
  auto p_full = [&](int i) { return bar + 8u * (uint32_t)i; };
  auto p_empty = [&](int i) { return bar + 8u * (uint32_t)(ST_MAX_SP + i); };
  auto b_full = [&](int g) { return bar + 8u * (uint32_t)(2 * ST_MAX_SP + g); };
  auto a_full = [&](int g) { return bar + 8u * (uint32_t)(2 * ST_MAX_SP + ST_MAX_G + g); };
  auto a_empty = [&](int g) { return bar + 8u * (uint32_t)(2 * ST_MAX_SP + 2 * ST_MAX_G + g); };
  auto t_full = [&](int b) { return bar + 8u * (uint32_t)(2 * ST_MAX_SP + 3 * ST_MAX_G + b); };
  auto t_empty = [&](int b) { return bar + 8u * (uint32_t)(2 * ST_MAX_SP + 3 * ST_MAX_G + 2 + b); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + a.off_bar + 8 * (2 * ST_MAX_SP + 3 * ST_MAX_G + 4));
  float* bdw = reinterpret_cast<float*>(smem + a.off_bdw);  // [Cpad] depthwise bias
  float* bpw = bdw + a.Cpad;  // [BN] pointwise bias: the epilogue reads it from smem (a global
                              // __ldg per 4 channels missed the tiny L1 and cost an L2 round
                              // trip per 16 outputs, ~0.8 us per group, probe r02zj)

  if (threadIdx.x == 0) {
    for (int i = 0; i < SP; ++i) {
      st_init(p_full(i), 1);
      st_init(p_empty(i), ST_GROUP_WARPS);
    }
    for (int g = 0; g < G; ++g) {
      st_init(b_full(g), 1);
      st_init(a_full(g), ST_GROUP_WARPS);
      st_init(a_empty(g), 1);
    }
    for (int b = 0; b < 2; ++b) {
      st_init(t_full(b), 1);
      st_init(t_empty(b), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == ST_MMA_WARP) {  // TMEM: tbufs tiles x (main + correction) x BN columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int c = threadIdx.x; c < a.Cpad; c += ST_THREADS) bdw[c] = (a.b_dw && c < a.C) ? a.b_dw[c] : 0.f;
  for (int c = threadIdx.x; c < BN; c += ST_THREADS) bpw[c] = (a.b_pw && c < a.K) ? a.b_pw[c] : 0.f;
  st_fence_before();
  __syncthreads();
  st_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == ST_LOAD_WARP) {
    // ---------------- patch loader: up to SP chunks ahead ----------------
    if (lane == 0) {
      prefetch_tmap(&tin);
      for (int seq = 0; seq < total; ++seq) {
        const int i = seq % SP, use = seq / SP, kc = seq % nchunks;
        int n0, r0;
        st_tile(a, t0 + (seq / nchunks) * tstride, n0, r0);
        const uint32_t dst = sbase + (uint32_t)i * a.pstage;
        if (use >= 1) mbar_wait_parity(p_empty(i), (use & 1) ^ 1);
        mbar_expect_tx(p_full(i), a.patch_bytes + a.filt_bytes);
        tma_load_4d(dst, &tin, kc * ST_CK, -a.pw, r0 * a.sh - a.ph, n0, p_full(i));
        bulk_g2s(dst + a.patch_bytes, a.w_dw + (size_t)kc * KS * KS * ST_CK, a.filt_bytes, p_full(i));
      }
    }
  } else if (warp == ST_BLOAD_WARP) {
    // ---------------- weight loader: a group's chunk once its previous MMAs are done ----------------
    if (lane == 0) {
      for (int seq = 0; seq < total; ++seq) {
        const int g = seq % G, use = seq / G, kc = seq % nchunks;
        if (use >= 1) mbar_wait_parity(a_empty(g), (use & 1) ^ 1);
        mbar_expect_tx(b_full(g), a.b_bytes);
        bulk_g2s(sbase + a.off_g + (uint32_t)g * a.gstage + a.off_b,
                 reinterpret_cast<const char*>(a.w_pw) + (size_t)kc * a.b_bytes, a.b_bytes, b_full(g));
      }
    }
  } else if (SLIDE && warp < G * ST_GROUP_WARPS) {
    // ---------------- depthwise producers (stride 1, wide maps: sliding rows) ----------------
    // thread = (one channel of the 16-channel chunk, a block of PXN output
    // columns of one image); it sweeps the tile's input rows once, each row
    // read as a PXN + k - 1 scalar register window, and keeps the k output
    // rows the row contributes to as rotating register accumulators.  A
    // finished output row is split into TF32 hi / lo and stored into the
    // group's A stage as soon as it completes.  (28x28 NASNet maps at bs256:
    // 84 → 66 us per 44-channel 5x5 layer; narrower maps keep the items,
    // profiles/r02_ab_sepconv_producers.txt)
    constexpr int PXN = SLIDE ? ST_PY : 1;
    constexpr int WN = PXN + KS - 1;
    const int g = warp / ST_GROUP_WARPS;
    const int gt = threadIdx.x - g * ST_GROUP_WARPS * 32;
    const int ch = gt & (ST_CK - 1);
    const int xblocks = (a.Q + PXN - 1) / PXN;
    const int nblk = a.TN * xblocks;
    const int nrows = a.TH + KS - 1;
    for (int seq = g; seq < total; seq += G) {
      const int use = seq / G, kc = seq % nchunks, pi = seq % SP;
      const uint8_t* st = smem + (size_t)pi * a.pstage;
      mbar_wait_parity(p_full(pi), (seq / SP) & 1);
      if (use >= 1) mbar_wait_parity(a_empty(g), (use & 1) ^ 1);  // the group's previous MMAs are done
      const float* patch = reinterpret_cast<const float*>(st);
      const float* filt = reinterpret_cast<const float*>(st + a.patch_bytes) + ch;  // [k*k][16]
      const int c = kc * ST_CK + ch;
      const bool cin = c < a.C;
      const float bias = bdw[c];
      uint8_t* ahi = smem + a.off_g + (size_t)g * a.gstage + a.off_a + (ch >> 2) * ST_LBO_A + (ch & 3) * 4;
      for (int blk = gt >> 4; blk < nblk; blk += (ST_GROUP_WARPS * 32) >> 4) {
        const int img = blk / xblocks;
        const int q0 = (blk - img * xblocks) * PXN;
        const float* prow = patch + ((size_t)img * a.IH * a.IW + q0) * ST_CK + ch;
        float acc[KS][PXN];
#pragma unroll
        for (int j = 0; j < KS; ++j)
#pragma unroll
          for (int x = 0; x < PXN; ++x) acc[j][x] = bias;
#pragma unroll 1
        for (int ir = 0; ir < nrows; ++ir) {
          float win[WN];
#pragma unroll
          for (int j = 0; j < WN; ++j) {
            win[j] = prow[((size_t)ir * a.IW + j) * ST_CK];
            if (a.pre_relu) win[j] = fmaxf(win[j], 0.f);
          }
          // acc[j] = output row ir - (KS-1) + j, tap row KS-1-j
#pragma unroll
          for (int j = 0; j < KS; ++j) {
#pragma unroll
            for (int t = 0; t < KS; ++t) {
              const float w = filt[((KS - 1 - j) * KS + t) * ST_CK];
#pragma unroll
              for (int x = 0; x < PXN; ++x) acc[j][x] = fmaf(win[x + t], w, acc[j][x]);
            }
          }
          const int y = ir - (KS - 1);  // acc[0] is complete
          if (y >= 0) {
            const int rbase = (img * a.TH + y) * a.Q + q0;
#pragma unroll
            for (int x = 0; x < PXN; ++x) {
              if (q0 + x >= a.Q) break;
              const float v = cin ? apply_act(acc[0][x], a.dw_act) : 0.f;
              const float h = st_rn(v);
              const int row = rbase + x;
              const int off = (row >> 3) * 128 + (row & 7) * 16;
              *reinterpret_cast<float*>(ahi + off) = h;
              *reinterpret_cast<float*>(ahi + ST_AHALF + off) = st_rn(v - h);
            }
          }
#pragma unroll
          for (int j = 0; j < KS - 1; ++j)
#pragma unroll
            for (int x = 0; x < PXN; ++x) acc[j][x] = acc[j + 1][x];
#pragma unroll
          for (int x = 0; x < PXN; ++x) acc[KS - 1][x] = bias;
        }
      }
      __syncwarp();
      if (lane == 0) st_arrive(p_empty(pi));  // every patch read of this warp is done
      fence_proxy_async_cta();
      __syncwarp();
      if (lane == 0) st_arrive(a_full(g));
    }
  } else if (!SLIDE && warp < G * ST_GROUP_WARPS) {
    // ---------------- depthwise producers ----------------
    // item = (image, PY x PX block of output pixels, channel quad), quad
    // fastest.  Per output quad ~k*k/PX filter and ((PY-1)*s+k)((PX-1)*s+k)/
    // (PX*PY) patch loads instead of k*k.  PX odd: the two items of an
    // 8-lane phase read 64-B pixel rows an odd multiple of 64 B apart, so
    // the (stride-1) patch loads are bank-conflict free.
    constexpr int WN = (ST_PX - 1) * SW + KS;  // window pixels per patch row
    constexpr int NR = (ST_PY - 1) * SW + KS;  // patch rows per block
    const int g = warp / ST_GROUP_WARPS;
    const int gt = threadIdx.x - g * ST_GROUP_WARPS * 32;
    const int xblocks = (a.Q + ST_PX - 1) / ST_PX;
    const int yblocks = (a.TH + ST_PY - 1) / ST_PY;
    const int items = a.TN * yblocks * xblocks * 4;
    for (int seq = g; seq < total; seq += G) {
      const int use = seq / G, kc = seq % nchunks, pi = seq % SP;
      const uint8_t* st = smem + (size_t)pi * a.pstage;
      mbar_wait_parity(p_full(pi), (seq / SP) & 1);
      const float* patch = reinterpret_cast<const float*>(st);
      const float* filt = reinterpret_cast<const float*>(st + a.patch_bytes);  // [k*k][16]
      // each round: compute a block into registers, (after the last round's
      // loads) release the patch, wait for the A stage (the group's previous
      // chunk's MMAs) and store
      for (int it0 = 0; it0 < items; it0 += ST_GROUP_WARPS * 32) {
        const int it = it0 + gt;
        const bool live = it < items;
        const int quad = it & 3;
        int rest = it >> 2;
        const int bx = rest % xblocks;
        rest /= xblocks;
        const int by = rest % yblocks;
        const int img = live ? rest / yblocks : 0;
        const int q0 = bx * ST_PX, y0 = by * ST_PY;
        const int c = kc * ST_CK + quad * 4;
        const float4 b = *reinterpret_cast<const float4*>(&bdw[c]);
        float4 acc[ST_PY][ST_PX];
#pragma unroll
        for (int y = 0; y < ST_PY; ++y)
#pragma unroll
          for (int x = 0; x < ST_PX; ++x) acc[y][x] = b;
        // patch element (image, row, col) at ((img*IH + row)*IW + col)*16 + quad*4 floats
        const float* pblk = patch + ((size_t)(img * a.IH + y0 * SW) * a.IW + q0 * SW) * ST_CK + quad * 4;
        const float* fq = filt + quad * 4;
#pragma unroll
        for (int ir = 0; ir < NR; ++ir) {
          float4 xw[WN];
#pragma unroll
          for (int j = 0; j < WN; ++j) {
            xw[j] = *reinterpret_cast<const float4*>(pblk + ((size_t)ir * a.IW + j) * ST_CK);
            if (a.pre_relu) xw[j] = st_relu4(xw[j]);
          }
#pragma unroll
          for (int y = 0; y < ST_PY; ++y) {
            const int r = ir - y * SW;  // tap row of this patch row for output row y
            if (r < 0 || r >= KS) continue;
#pragma unroll
            for (int t = 0; t < KS; ++t) {
              const float4 w = *reinterpret_cast<const float4*>(fq + (r * KS + t) * ST_CK);
#pragma unroll
              for (int x = 0; x < ST_PX; ++x) st_fma4(acc[y][x], xw[x * SW + t], w);
            }
          }
        }
        if (it0 + ST_GROUP_WARPS * 32 >= items) {  // last round: the patch is free for the next chunk
          __syncwarp();
          if (lane == 0) st_arrive(p_empty(pi));
        }
        if (it0 == 0 && use >= 1) mbar_wait_parity(a_empty(g), (use & 1) ^ 1);
        if (!live) continue;
        uint8_t* ahi = smem + a.off_g + (size_t)g * a.gstage + a.off_a;
        const bool cin = c < a.C;
#pragma unroll
        for (int y = 0; y < ST_PY; ++y) {
          if (y0 + y >= a.TH) break;
#pragma unroll
          for (int x = 0; x < ST_PX; ++x) {
            if (q0 + x >= a.Q) break;
            const float4 v = cin ? act4(acc[y][x], a.dw_act) : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 h = make_float4(st_rn(v.x), st_rn(v.y), st_rn(v.z), st_rn(v.w));
            const float4 l = make_float4(st_rn(v.x - h.x), st_rn(v.y - h.y), st_rn(v.z - h.z), st_rn(v.w - h.w));
            const int row = (img * a.TH + y0 + y) * a.Q + q0 + x;  // UMMA row = tile pixel slot
            const int off = quad * ST_LBO_A + (row >> 3) * 128 + (row & 7) * 16;
            *reinterpret_cast<float4*>(ahi + off) = h;
            *reinterpret_cast<float4*>(ahi + ST_AHALF + off) = l;
          }
        }
      }
      fence_proxy_async_cta();
      __syncwarp();
      if (lane == 0) st_arrive(a_full(g));
    }
  } else if (warp == ST_MMA_WARP) {
    // ---------------- MMA issuer ----------------
    if (lane == 0 && ntiles > 0) {
      // D f32, A/B tf32, both K-major, N = BN, M = 128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(ST_BM >> 4) << 24);
      const uint32_t LBO_B = (uint32_t)BN * 16;
      const uint32_t bhalf = a.b_bytes / 2;
      // Descriptors are computed once per chunk (no division on the way to
      // an MMA: a per-MMA address chain with `seq % G` held the issue rate
      // to ~135 clocks per MMA, tools/mma_rate.cu r02j); the group index and
      // its phase advance incrementally.
      int g = 0, use = 0;
      for (int ti = 0; ti < ntiles; ++ti) {
        const int b = ti % a.tbufs, tuse = ti / a.tbufs;
        if (tuse >= 1) mbar_wait_parity(t_empty(b), (tuse & 1) ^ 1);
        st_fence_after();
        const uint32_t d_main = tmem + (uint32_t)(b * 2 * BN), d_corr = d_main + (uint32_t)BN;
        for (int kc = 0; kc < nchunks; ++kc) {
          const uint32_t stg = sbase + a.off_g + (uint32_t)g * a.gstage;
          const uint32_t ah = stg + a.off_a, al = ah + ST_AHALF;
          const uint32_t bh = stg + a.off_b, bl = bh + bhalf;
          uint64_t dah[ST_CK / 8], dal[ST_CK / 8], dbh[ST_CK / 8], dbl[ST_CK / 8];
#pragma unroll
          for (int ks = 0; ks < ST_CK / 8; ++ks) {
            dah[ks] = st_desc(ah + ks * 2 * ST_LBO_A, ST_LBO_A);
            dal[ks] = st_desc(al + ks * 2 * ST_LBO_A, ST_LBO_A);
            dbh[ks] = st_desc(bh + ks * 2 * LBO_B, LBO_B);
            dbl[ks] = st_desc(bl + ks * 2 * LBO_B, LBO_B);
          }
          mbar_wait_parity(b_full(g), use & 1);
          mbar_wait_parity(a_full(g), use & 1);
          st_fence_after();
#pragma unroll
          for (int ks = 0; ks < ST_CK / 8; ++ks) {
            const uint32_t first = (kc | ks) ? 1u : 0u;
            st_mma(d_main, dah[ks], dbh[ks], idesc, first);
            st_mma(d_corr, dah[ks], dbl[ks], idesc, first);
            st_mma(d_corr, dal[ks], dbh[ks], idesc, 1u);
          }
          st_commit(a_empty(g));
          if (++g == G) {
            g = 0;
            ++use;
          }
        }
        st_commit(t_full(b));
      }
    }
    __syncwarp();
  } else if (warp > ST_MMA_WARP && warp < ST_MMA_WARP + 5) {
    // ---------------- epilogue ----------------
    const int quad = warp & 3;  // TMEM lanes 32*quad .. +31
    const int row = quad * 32 + lane;
    const int per_img = a.TH * a.Q;
    for (int ti = 0; ti < ntiles; ++ti) {
      const int b = ti % a.tbufs, tuse = ti / a.tbufs;
      int n0, r0;
      st_tile(a, t0 + ti * tstride, n0, r0);
      mbar_wait_parity(t_full(b), tuse & 1);
      if (row == 0 && ti < 4) probe_trace(32 + 8 * ti);  // accumulators of tile ti ready
      st_fence_after();
      const int img = row / per_img, rr = row % per_img;
      const int n = n0 + img, p = r0 + rr / a.Q, q = rr % a.Q;
      const bool ok = img < a.TN && n < a.N && p < a.P;
      float* o = a.out + (ok ? n * a.out_sn + p * a.out_sh + q * a.out_sw : 0);
      const float* rp = (a.has_res && ok) ? a.res + n * a.res_sn + p * a.res_sh + q * a.res_sw : nullptr;
      const uint32_t tl = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * 2 * BN);
      // TMEM → registers is software-pipelined: group k0 + 16's loads are in
      // flight while group k0 is stored (a tcgen05.ld round trip is ~0.5 us
      // while the next tile's MMAs run, probe r02zi; stores are not the cost)
      // residual (global, an L2 round trip) and TMEM groups are prefetched one
      // 16-channel group ahead of the one being stored
      const bool rvec = rp && a.ovec;
      float v[16], w[16];
      float4 r4[4];
      st_ld16(tl, v);
      st_ld16(tl + (uint32_t)BN, w);
      if (rvec && ok && 16 <= a.K) {
#pragma unroll
        for (int j = 0; j < 4; ++j) r4[j] = *reinterpret_cast<const float4*>(rp + 4 * j);
      }
      st_tc_wait_ld();
      for (int k0 = 0; k0 < BN; k0 += 16) {
        float vn[16], wn[16];
        float4 rn[4];
        const bool more = k0 + 16 < BN;
        if (more) {
          st_ld16(tl + (uint32_t)(k0 + 16), vn);
          st_ld16(tl + (uint32_t)(BN + k0 + 16), wn);
          if (rvec && ok && k0 + 32 <= a.K) {
#pragma unroll
            for (int j = 0; j < 4; ++j) rn[j] = *reinterpret_cast<const float4*>(rp + k0 + 16 + 4 * j);
          }
        }
        if (row == 0 && ti < 4 && k0 < 48) probe_trace(33 + 8 * ti + k0 / 16 * 2);  // TMEM group k0 in
        if (ok && k0 < a.K) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += w[j];
          if (a.ovec && k0 + 16 <= a.K) {
#pragma unroll
            for (int j = 0; j < 16; j += 4) {
              float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              x = f4add(x, *reinterpret_cast<const float4*>(bpw + k0 + j));
              if (rp) x = f4add(x, r4[j / 4]);
              *reinterpret_cast<float4*>(o + k0 + j) = act4(x, a.act);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (k0 + j >= a.K) break;
              float x = v[j] + bpw[k0 + j];
              if (rp) x += rp[k0 + j];
              o[k0 + j] = apply_act(x, a.act);
            }
          }
        }
        if (more) {
          st_tc_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            v[j] = vn[j];
            w[j] = wn[j];
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) r4[j] = rn[j];
        }
      }
      st_fence_before();
      __syncwarp();
      if (row == 0 && ti < 4) probe_trace(39 + 8 * ti);  // tile ti stored
      if (lane == 0) st_arrive(t_empty(b));
    }
  }
  st_fence_before();
  __syncthreads();
  if (warp == ST_MMA_WARP) {
    st_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
  probe_end();
}

// Channel padding shared with the host packer (engine.py sep_tc_layout):
// Cpad = C rounded up to 16 (K chunks), BN = K rounded up to 16 (UMMA N).
static void sep_tc_blocking(int C, int K, int& Cpad, int& BN) {
  Cpad = (C + ST_CK - 1) / ST_CK * ST_CK;
  BN = (K + 15) / 16 * 16;
}

int launch_sepconv_tc(const sw_op_desc& op, void* stream) {
  const int64_t* p = op.params;
  SepTcArgs a;
  const float* in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.w_pw = reinterpret_cast<const float*>(op.ptrs[PT_W_TC_LO]);
  a.b_pw = reinterpret_cast<const float*>(op.ptrs[PT_BIAS]);
  a.b_dw = reinterpret_cast<const float*>(op.ptrs[PT_DW_BIAS]);
  a.res = reinterpret_cast<const float*>(op.ptrs[PT_RES]);
  a.N = (int)p[SP_N]; a.H = (int)p[SP_H]; a.W = (int)p[SP_W]; a.C = (int)p[SP_C];
  a.P = (int)p[SP_P]; a.Q = (int)p[SP_Q]; a.K = (int)p[SP_K];
  a.R = (int)p[SP_R]; a.S = (int)p[SP_S];
  a.sh = (int)p[SP_STRIDE_H]; a.sw = (int)p[SP_STRIDE_W];
  a.ph = (int)p[SP_PAD_H]; a.pw = (int)p[SP_PAD_W];
  a.act = (int)p[SP_ACT]; a.dw_act = (int)p[SP_DW_ACT];
  a.pre_relu = (int)p[SP_PRE_RELU]; a.has_res = (int)p[SP_HAS_RES];
  const int64_t in_sn = p[SP_IN_SN], in_sh = p[SP_IN_SH], in_sw = p[SP_IN_SW];
  a.out_sn = p[SP_OUT_SN]; a.out_sh = p[SP_OUT_SH]; a.out_sw = p[SP_OUT_SW];
  a.res_sn = p[SP_RES_SN]; a.res_sh = p[SP_RES_SH]; a.res_sw = p[SP_RES_SW];
  if ((int64_t)a.N * a.P * a.Q == 0 || a.K == 0) return 0;
  const int64_t osc = p[SP_OUT_SC] ? p[SP_OUT_SC] : 1, rsc = p[SP_RES_SC] ? p[SP_RES_SC] : 1;
  // square k in {3,5,7}, equal strides 1/2, K <= 256, NHWC rows of whole
  // channel quads; the autotuner keeps a CUDA-core variant otherwise
  const int ks = a.R == a.S ? a.R : 0;
  if (!a.w_pw || a.C % 4 || a.K > 256 || p[SP_IN_SC] != 1 || osc != 1 || (a.has_res && rsc != 1) ||
      !(ks == 3 || ks == 5 || ks == 7) || a.sh != a.sw || (a.sh != 1 && a.sh != 2) || a.Q > ST_BM)
    return (int)cudaErrorInvalidValue;
  sep_tc_blocking(a.C, a.K, a.Cpad, a.BN);
  a.w_dw = a.w_pw + (size_t)a.Cpad * 2 * a.BN;  // after the pointwise images
  a.tbufs = a.BN <= 128 ? 2 : 1;
  a.ovec = epi_vec_ok(op.ptrs[PT_OUT], a.out_sn, a.out_sh, a.out_sw, 1, op.ptrs[PT_BIAS], a.has_res != 0,
                      op.ptrs[PT_RES], a.res_sn, a.res_sh, a.res_sw, 1)
               ? 1
               : 0;
  // tile geometry: TN whole images when one fits, else bands of whole PY-row
  // blocks (a whole image keeps its ragged last block)
  const int s = a.sh;
  a.TH = std::min(a.P, ST_BM / a.Q);
  a.TN = a.TH == a.P ? std::min(a.N, std::max(1, ST_BM / (a.P * a.Q))) : 1;
  // stride 1 on wide maps (Q >= 21): sliding-row producers, 7 columns per thread
  const bool slide = s == 1 && ks <= 5 && a.Q >= 21;
  constexpr int SLIDE_PXN = 7;
  a.IW = slide ? (a.Q + SLIDE_PXN - 1) / SLIDE_PXN * SLIDE_PXN + ks - 1
               : (((a.Q + ST_PX - 1) / ST_PX) * ST_PX - 1) * s + ks;  // every window column an item reads
  a.filt_bytes = (uint32_t)(ks * ks * ST_CK * 4);
  a.b_bytes = 2u * (uint32_t)a.BN * ST_CK * 4u;
  int PY = 3;
  auto layout = [&](int g, int sp) {
    a.IH = slide ? a.TH + ks - 1
                 : (((a.TH + PY - 1) / PY) * PY - 1) * s + ks;  // rows of the last (ragged) block too
    a.patch_bytes = (uint32_t)(a.TN * a.IH * a.IW * ST_CK * 4);
    a.pstage = (a.patch_bytes + a.filt_bytes + 1023u) / 1024u * 1024u;  // TMA destinations aligned
    a.off_b = 0;
    a.off_a = (a.b_bytes + 127u) / 128u * 128u;
    a.gstage = (a.off_a + 2u * ST_AHALF + 127u) / 128u * 128u;
    a.off_g = (uint32_t)sp * a.pstage;
    a.off_bdw = a.off_g + (uint32_t)g * a.gstage;
    a.off_bar = (a.off_bdw + (uint32_t)(a.Cpad + a.BN) * 4u + 15u) / 16u * 16u;
    return (size_t)a.off_bar + 8 * (2 * ST_MAX_SP + 3 * ST_MAX_G + 4) + 16;
  };
  // output rows per depthwise thread: the block height that wastes least
  // (ragged last block) per patch row loaded
  {
    auto cost = [&](int py) {
      const int rows = (a.TH + py - 1) / py * py;
      return (double)rows / a.TH * (double)((py - 1) * s + ks) / py;
    };
    // (PY = 3 blocks of 7x7 or strided windows exceed the register budget)
    PY = (ks <= 5 && s == 1 && cost(3) <= cost(2)) ? 3 : 2;
  }
  // as many concurrent chunk groups and prefetched patches as fit, then smaller tiles
  int G = ST_MAX_G, SP = ST_MAX_SP;
  size_t smem = layout(G, SP);
  while (smem > (size_t)ST_SMEM_MAX) {
    if (SP > G + 2) --SP;
    else if (G > 2) { --G; SP = std::min(SP, ST_MAX_SP); }
    else if (SP > 2) --SP;
    else if (a.TN > 1) --a.TN;
    else if (a.TH > 1) --a.TH;
    else return (int)cudaErrorInvalidValue;
    smem = layout(G, SP);
  }
  if (a.IW > 256 || a.IH > 256 || a.TN > 256) return (int)cudaErrorInvalidValue;  // TMA box limits
  a.G = G;
  a.SP = SP;
  a.bands = (a.P + a.TH - 1) / a.TH;
  a.ntile = (a.N + a.TN - 1) / a.TN * a.bands;
  CUtensorMap tin;
  {  // input (C, W, H, N), box [16 ch][IW][IH][TN]; out of range → 0 (halo, padding, channels >= C)
    const uint64_t dims[4] = {(uint64_t)a.C, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.N};
    const uint64_t str[3] = {(uint64_t)in_sw * 4, (uint64_t)in_sh * 4, (uint64_t)in_sn * 4};
    const uint32_t box[4] = {ST_CK, (uint32_t)a.IW, (uint32_t)a.IH, (uint32_t)a.TN};
    if (!encode_tmap_f32(&tin, in, 4, dims, str, box)) return (int)cudaErrorInvalidValue;
  }
  if (getenv("SW_DEBUG_LAUNCH"))
    fprintf(stderr, "sepconv_tc: C %d K %d Cpad %d BN %d TN %d TH %d PY %d IH %d IW %d G %d SP %d smem %zu tiles %d\n",
            a.C, a.K, a.Cpad, a.BN, a.TN, a.TH, PY, a.IH, a.IW, G, SP, smem, a.ntile);
  const int grid = std::min(a.ntile, 148);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t rc = cudaErrorInvalidValue;
  if (slide) PY = SLIDE_PXN;
#define SW_SEPTC(K_, S_, PY_)                                                                             \
  if (ks == K_ && s == S_ && PY == PY_)                                                                 \
    rc = launch_k(sepconv_tc_kernel<K_, S_, PY_>, dim3(grid), dim3(ST_THREADS), smem, st, 1u, tin, a);
  SW_SEPTC(3, 1, 7) SW_SEPTC(5, 1, 7)
  SW_SEPTC(3, 1, 3) SW_SEPTC(5, 1, 3)
  SW_SEPTC(3, 1, 2) SW_SEPTC(5, 1, 2) SW_SEPTC(7, 1, 2) SW_SEPTC(3, 2, 2) SW_SEPTC(5, 2, 2) SW_SEPTC(7, 2, 2)
#undef SW_SEPTC
  return (int)rc;
}

void init_sep_tc_kernels() {
#define SW_SEPTC_ATTR(K_, S_, PY_) \
  cudaFuncSetAttribute(sepconv_tc_kernel<K_, S_, PY_>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
  SW_SEPTC_ATTR(3, 1, 7) SW_SEPTC_ATTR(5, 1, 7)
  SW_SEPTC_ATTR(3, 1, 3) SW_SEPTC_ATTR(5, 1, 3)
  SW_SEPTC_ATTR(3, 1, 2) SW_SEPTC_ATTR(5, 1, 2) SW_SEPTC_ATTR(7, 1, 2)
  SW_SEPTC_ATTR(3, 2, 2) SW_SEPTC_ATTR(5, 2, 2) SW_SEPTC_ATTR(7, 2, 2)
#undef SW_SEPTC_ATTR
}

}  // namespace sw
