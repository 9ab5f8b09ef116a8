// Fused separable convolution with the pointwise GEMM on the 5th-generation
// tensor cores: depthwise k x k (CUDA cores, TMA-staged input) →
// tcgen05.mma kind::tf32 (3xTF32, TMEM accumulators) → bias / residual /
// activation epilogue, in one persistent, warp-specialised kernel (K_SEPCONV
// variant SEP_TC_VARIANT).
//
// Work unit ("tile") = TN whole images x a band of TH output rows x all Q
// columns (TN*TH*Q <= 128 pixels = the UMMA M rows, one per TMEM lane) x one
// block of BN <= 128 output channels.  Layers with more than 128 outputs run
// ceil(K/128) channel blocks; each CTA owns one block for its lifetime and
// walks the tiles blockIdx.x / nblk, + gridDim.x / nblk, ...  The K dimension
// (input channels) is processed in chunks of 16.
//
// Roles (448 threads, one CTA per SM):
//   warp 13    loader: per (tile, chunk) one 4-D TMA box of the input patch
//              [TN][IH][IW][16 ch] (halo and padding zero-filled by the
//              tensor map, channels >= C too) + one bulk copy of the chunk's
//              depthwise filter [k*k][16] into a patch ring stage;
//   warps 0-7  depthwise producers: a thread owns PX = 2 adjacent output
//              pixels of one row and one channel quad and slides the k-tap
//              window along the patch row in registers (shared-memory loads
//              only, no bounds checks); act(dw + b_dw) is split into TF32
//              hi / lo (round-to-nearest, conv_tc.cu) and stored straight into
//              an A ring stage in the canonical K-major UMMA layout;
//   warp 8     MMA issuer (one thread): per chunk 2 K-steps x {hi·hi into
//              the tile's main accumulator, hi·lo + lo·hi into its
//              correction accumulator}; tcgen05.commit frees the A stage and,
//              after the last chunk, hands the accumulators to the epilogue;
//   warps 9-12 epilogue: TMEM lanes = tile pixels; tcgen05.ld main +
//              correction (fp32 add), + bias, + residual, activation, float4
//              NHWC stores; then release the TMEM buffer.
// The weights of the CTA's channel block (pre-split hi / lo, packed on the
// host as the UMMA smem image) arrive by bulk copies before the PDL wait and
// stay resident.  TMEM holds two tiles (main + correction each), so the
// epilogue of tile i overlaps the depthwise + MMAs of tile i+1.
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
constexpr int ST_PY = 3;    // output rows per depthwise thread (patch rows shared between them)
// A operand (tile pixels x 16 channels, hi or lo): canonical K-major
// SWIZZLE_NONE core matrices, 8 rows x 16 B, 8-row groups 128 B apart (SBO);
// the four 16-B channel quads (K core-matrix columns) ST_LBO_A apart.  2048
// would be dense; +32 B staggers the quads over the banks so a producer
// phase (2 pixels x 4 quads) stores without conflicts.
constexpr int ST_LBO_A = ST_BM * 16 + 32;
constexpr int ST_DW_WARPS = 8;
constexpr int ST_MMA_WARP = ST_DW_WARPS;
constexpr int ST_EPI_WARP0 = ST_DW_WARPS + 1;
constexpr int ST_LOAD_WARP = ST_DW_WARPS + 5;
constexpr int ST_THREADS = (ST_DW_WARPS + 6) * 32;
constexpr int ST_SMEM_MAX = 232448;

struct SepTcArgs {
  float* __restrict__ out;
  const float* __restrict__ w_img;  // [nblk][hi: Cpad/4][BN][4] [lo: same], then w_dw
  const float* __restrict__ w_dw;   // [Cpad/16][R*S][16] chunk-major depthwise filter, zero padded
  const float* __restrict__ b_pw;
  const float* __restrict__ b_dw;
  const float* __restrict__ res;
  int N, H, W, C, P, Q, K, R, S, sh, sw, ph, pw, act, dw_act, pre_relu, has_res;
  int64_t out_sn, out_sh, out_sw, res_sn, res_sh, res_sw;
  int Cpad, BN, nblk, ntile, TN, TH, IH, IW, bands, qgroups, a_stages, p_stages, ovec;
  uint32_t patch_bytes, filt_bytes, pstage;             // patch stage = patch + filter chunk (pstage bytes)
  uint32_t astage;                                      // A stage: hi + lo (each 3*LBO + 2048 B, 1 KB aligned)
  uint32_t off_a, off_p, off_bdw, off_bar;              // smem carve-up (bytes); B image at 0
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
// images past N are invalid slots (their A rows are never stored / read back)
__device__ __forceinline__ void st_tile(const SepTcArgs& a, int tile, int& n0, int& r0) {
  n0 = (tile / a.bands) * a.TN;
  r0 = (tile % a.bands) * a.TH;
}

template <int KS, int SW>
__global__ void __launch_bounds__(ST_THREADS, 1)
    sepconv_tc_kernel(const __grid_constant__ CUtensorMap tin, SepTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = su32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int SA = a.a_stages, SP = a.p_stages;
  const int nchunks = a.Cpad / ST_CK;
  const int BN = a.BN;
  const int nb = (int)blockIdx.x % a.nblk;
  const int tstride = (int)gridDim.x / a.nblk;
  const int t0 = (int)blockIdx.x / a.nblk;
  const int ntiles = t0 < a.ntile ? (a.ntile - 1 - t0) / tstride + 1 : 0;

  // barriers: a_full[SA], a_empty[SA], p_full[SP], p_empty[SP], t_full[2], t_empty[2], w_full, tmem slot
  const uint32_t bar = sbase + a.off_bar;
  auto a_full = [&](int s) { return bar + 8u * (uint32_t)s; };
  auto a_empty = [&](int s) { return bar + 8u * (uint32_t)(SA + s); };
  auto p_full = [&](int s) { return bar + 8u * (uint32_t)(2 * SA + s); };
  auto p_empty = [&](int s) { return bar + 8u * (uint32_t)(2 * SA + SP + s); };
  auto t_full = [&](int b) { return bar + 8u * (uint32_t)(2 * SA + 2 * SP + b); };
  auto t_empty = [&](int b) { return bar + 8u * (uint32_t)(2 * SA + 2 * SP + 2 + b); };
  const uint32_t w_full = bar + 8u * (uint32_t)(2 * SA + 2 * SP + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + a.off_bar + 8 * (2 * SA + 2 * SP + 5));
  float* bdw = reinterpret_cast<float*>(smem + a.off_bdw);      // [Cpad] depthwise bias
  const uint32_t wbytes = (uint32_t)BN * (uint32_t)a.Cpad * 4u;  // one of hi / lo

  if (threadIdx.x == 0) {
    for (int s = 0; s < SA; ++s) {
      st_init(a_full(s), ST_DW_WARPS);
      st_init(a_empty(s), 1);
    }
    for (int s = 0; s < SP; ++s) {
      st_init(p_full(s), 1);
      st_init(p_empty(s), ST_DW_WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      st_init(t_full(b), 1);
      st_init(t_empty(b), 4);
    }
    st_init(w_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == ST_MMA_WARP) {  // TMEM: 2 tiles x (main + correction) x BN columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int c = threadIdx.x; c < a.Cpad; c += ST_THREADS) bdw[c] = (a.b_dw && c < a.C) ? a.b_dw[c] : 0.f;
  st_fence_before();
  __syncthreads();
  st_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == ST_LOAD_WARP * 32 && ntiles > 0) {  // this CTA's pointwise weight block, hi then lo
    prefetch_tmap(&tin);
    mbar_expect_tx(w_full, 2 * wbytes);
    const char* src = reinterpret_cast<const char*>(a.w_img) + (size_t)nb * 2 * wbytes;
    for (uint32_t off = 0; off < 2 * wbytes; off += 65536u)
      bulk_g2s(sbase + off, src + off, min(65536u, 2 * wbytes - off), w_full);
  }
  pdl_trigger();
  pdl_wait();

  if (warp == ST_LOAD_WARP) {
    // ---------------- loader ----------------
    if (lane == 0) {
      int seq = 0;
      for (int ti = 0; ti < ntiles; ++ti) {
        int n0, r0;
        st_tile(a, t0 + ti * tstride, n0, r0);
        for (int kc = 0; kc < nchunks; ++kc, ++seq) {
          const int s = seq % SP;
          if (seq >= SP) mbar_wait_parity(p_empty(s), ((seq / SP) & 1) ^ 1);
          const uint32_t dst = sbase + a.off_p + (uint32_t)s * a.pstage;
          mbar_expect_tx(p_full(s), a.patch_bytes + a.filt_bytes);
          tma_load_4d(dst, &tin, kc * ST_CK, -a.pw, r0 * a.sh - a.ph, n0, p_full(s));
          bulk_g2s(dst + a.patch_bytes, a.w_dw + (size_t)kc * KS * KS * ST_CK, a.filt_bytes, p_full(s));
        }
      }
    }
  } else if (warp < ST_DW_WARPS) {
    // ---------------- depthwise producers ----------------
    // item = (image, PY x PX block of output pixels, channel quad), quad
    // fastest.  The thread walks the (PY-1)*s + k patch rows its block needs
    // once, each as one register window of (PX-1)*s + k pixels, and feeds
    // every output row that tap row contributes to: per output quad ~k*k/PX
    // filter and ((PY-1)*s+k)((PX-1)*s+k)/(PX*PY) patch loads instead of k*k.
    // PX odd: the two items of an 8-lane phase read 64-B pixel rows an odd
    // multiple of 64 B apart, so the patch loads are bank-conflict free.
    constexpr int WN = (ST_PX - 1) * SW + KS;   // window pixels per patch row
    constexpr int NR = (ST_PY - 1) * SW + KS;   // patch rows per block
    const int xblocks = (a.Q + ST_PX - 1) / ST_PX;
    const int yblocks = (a.TH + ST_PY - 1) / ST_PY;
    const int items = a.TN * yblocks * xblocks * 4;
    int seq = 0;
    for (int ti = 0; ti < ntiles; ++ti) {
      int n0, r0;
      st_tile(a, t0 + ti * tstride, n0, r0);
      for (int kc = 0; kc < nchunks; ++kc, ++seq) {
        const int ps = seq % SP, as = seq % SA;
        mbar_wait_parity(p_full(ps), (seq / SP) & 1);
        if (seq >= SA) mbar_wait_parity(a_empty(as), ((seq / SA) & 1) ^ 1);
        const float* patch = reinterpret_cast<const float*>(smem + a.off_p + (size_t)ps * a.pstage);
        const float* filt = patch + a.patch_bytes / 4;  // [k*k][16]
        uint8_t* stg = smem + a.off_a + (size_t)as * a.astage;
        for (int it = threadIdx.x; it < items; it += ST_DW_WARPS * 32) {
          const int quad = it & 3;
          int rest = it >> 2;
          const int bx = rest % xblocks;
          rest /= xblocks;
          const int by = rest % yblocks;
          const int img = rest / yblocks;
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
          const bool cin = c < a.C;
#pragma unroll
          for (int y = 0; y < ST_PY; ++y) {
            if (y0 + y >= a.TH) break;
#pragma unroll
            for (int x = 0; x < ST_PX; ++x) {
              if (q0 + x >= a.Q) break;
              const float4 v = cin ? act4(acc[y][x], a.dw_act) : make_float4(0.f, 0.f, 0.f, 0.f);
              const float4 h = make_float4(st_rn(v.x), st_rn(v.y), st_rn(v.z), st_rn(v.w));
              const float4 l =
                  make_float4(st_rn(v.x - h.x), st_rn(v.y - h.y), st_rn(v.z - h.z), st_rn(v.w - h.w));
              const int row = (img * a.TH + y0 + y) * a.Q + q0 + x;  // UMMA row = tile pixel slot
              const int off = quad * ST_LBO_A + (row >> 3) * 128 + (row & 7) * 16;
              *reinterpret_cast<float4*>(stg + off) = h;
              *reinterpret_cast<float4*>(stg + a.astage / 2 + off) = l;
            }
          }
        }
        fence_proxy_async_cta();
        __syncwarp();
        if (lane == 0) {
          st_arrive(a_full(as));
          st_arrive(p_empty(ps));
        }
      }
    }
  } else if (warp == ST_MMA_WARP) {
    // ---------------- MMA issuer ----------------
    if (lane == 0 && ntiles > 0) {
      // D f32, A/B tf32, both K-major, N = BN, M = 128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(ST_BM >> 4) << 24);
      const uint32_t LBO_A = ST_LBO_A, LBO_B = (uint32_t)BN * 16;
      mbar_wait_parity(w_full, 0);
      int seq = 0;
      for (int ti = 0; ti < ntiles; ++ti) {
        const int b = ti & 1;
        if (ti >= 2) mbar_wait_parity(t_empty(b), ((ti >> 1) & 1) ^ 1);
        st_fence_after();
        const uint32_t d_main = tmem + (uint32_t)(b * 2 * BN), d_corr = d_main + (uint32_t)BN;
        for (int kc = 0; kc < nchunks; ++kc, ++seq) {
          const int s = seq % SA;
          mbar_wait_parity(a_full(s), (seq / SA) & 1);
          st_fence_after();
          const uint32_t ah = sbase + a.off_a + (uint32_t)s * a.astage, al = ah + a.astage / 2;
#pragma unroll
          for (int ks = 0; ks < ST_CK / 8; ++ks) {
            const uint32_t bofs = (uint32_t)(kc * (ST_CK / 4) + ks * 2) * LBO_B;
            const uint64_t dah = st_desc(ah + ks * 2 * LBO_A, LBO_A), dal = st_desc(al + ks * 2 * LBO_A, LBO_A);
            const uint64_t dbh = st_desc(sbase + bofs, LBO_B), dbl = st_desc(sbase + wbytes + bofs, LBO_B);
            const uint32_t first = (kc | ks) ? 1u : 0u;
            st_mma(d_main, dah, dbh, idesc, first);
            st_mma(d_corr, dah, dbl, idesc, first);
            st_mma(d_corr, dal, dbh, idesc, 1u);
          }
          st_commit(a_empty(s));
        }
        st_commit(t_full(b));
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue ----------------
    const int quad = warp & 3;  // TMEM lanes 32*quad .. +31
    const int row = quad * 32 + lane;
    const int per_img = a.TH * a.Q;
    for (int ti = 0; ti < ntiles; ++ti) {
      const int b = ti & 1;
      int n0, r0;
      st_tile(a, t0 + ti * tstride, n0, r0);
      mbar_wait_parity(t_full(b), (ti >> 1) & 1);
      st_fence_after();
      const int img = row / per_img, rr = row % per_img;
      const int n = n0 + img, p = r0 + rr / a.Q, q = rr % a.Q;
      const bool ok = img < a.TN && n < a.N && p < a.P && rr / a.Q < a.TH;
      float* o = a.out + (ok ? n * a.out_sn + p * a.out_sh + q * a.out_sw : 0);
      const float* rp = (a.has_res && ok) ? a.res + n * a.res_sn + p * a.res_sh + q * a.res_sw : nullptr;
      const uint32_t tl = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * 2 * BN);
      for (int c0 = 0; c0 < BN; c0 += 16) {
        float v[16], w[16];
        st_ld16(tl + (uint32_t)c0, v);
        st_ld16(tl + (uint32_t)(BN + c0), w);
        st_tc_wait_ld();
        const int k0 = nb * BN + c0;
        if (!ok || k0 >= a.K) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += w[j];
        if (a.ovec && k0 + 16 <= a.K) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 x = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            if (a.b_pw) x = f4add(x, __ldg(reinterpret_cast<const float4*>(a.b_pw + k0 + j)));
            if (rp) x = f4add(x, *reinterpret_cast<const float4*>(rp + k0 + j));
            *reinterpret_cast<float4*>(o + k0 + j) = act4(x, a.act);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (k0 + j >= a.K) break;
            float x = v[j] + (a.b_pw ? a.b_pw[k0 + j] : 0.f);
            if (rp) x += rp[k0 + j];
            o[k0 + j] = apply_act(x, a.act);
          }
        }
      }
      st_fence_before();
      __syncwarp();
      if (lane == 0) st_arrive(t_empty(b));
    }
  }
  st_fence_before();
  __syncthreads();
  if (warp == ST_MMA_WARP) {
    st_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
  }
}

// Channel blocking shared with the host packer (engine.py sep_tc_layout):
// Cpad = C rounded up to 16; nblk = ceil(K16 / 128) blocks of BN = ceil(K / nblk)
// rounded up to 16 (K16 = K rounded up to 16).
static void sep_tc_blocking(int C, int K, int& Cpad, int& BN, int& nblk) {
  Cpad = (C + ST_CK - 1) / ST_CK * ST_CK;
  const int k16 = (K + 15) / 16 * 16;
  nblk = (k16 + 127) / 128;
  BN = ((K + nblk - 1) / nblk + 15) / 16 * 16;
}

int launch_sepconv_tc(const sw_op_desc& op, void* stream) {
  const int64_t* p = op.params;
  SepTcArgs a;
  const float* in = reinterpret_cast<const float*>(op.ptrs[PT_IN]);
  a.out = reinterpret_cast<float*>(op.ptrs[PT_OUT]);
  a.w_img = reinterpret_cast<const float*>(op.ptrs[PT_W_TC_LO]);
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
  // square k in {3,5,7}, equal strides 1/2, NHWC rows of whole channel quads
  // (16-B aligned tensor-map strides); the autotuner keeps a CUDA-core variant otherwise
  const int ks = a.R == a.S ? a.R : 0;
  if (!a.w_img || a.C % 4 || p[SP_IN_SC] != 1 || osc != 1 || (a.has_res && rsc != 1) ||
      !(ks == 3 || ks == 5 || ks == 7) || a.sh != a.sw || (a.sh != 1 && a.sh != 2))
    return (int)cudaErrorInvalidValue;
  sep_tc_blocking(a.C, a.K, a.Cpad, a.BN, a.nblk);
  a.w_dw = a.w_img + (size_t)a.nblk * 2 * a.BN * a.Cpad;
  a.ovec = epi_vec_ok(op.ptrs[PT_OUT], a.out_sn, a.out_sh, a.out_sw, 1, op.ptrs[PT_BIAS], a.has_res != 0,
                      op.ptrs[PT_RES], a.res_sn, a.res_sh, a.res_sw, 1)
               ? 1
               : 0;
  // tile geometry: TN whole images when one fits, else bands of TH rows
  const int s = a.sh;
  if (a.Q > ST_BM) return (int)cudaErrorInvalidValue;
  a.TH = std::min(a.P, ST_BM / a.Q);
  // bands of whole PY-row blocks (a whole image keeps its ragged last block)
  if (a.TH < a.P && a.TH > ST_PY) a.TH -= a.TH % ST_PY;
  a.TN = a.TH == a.P ? std::max(1, ST_BM / (a.P * a.Q)) : 1;
  a.TN = std::min(a.TN, a.N);
  a.qgroups = (a.Q + ST_PX - 1) / ST_PX;
  a.IW = (a.qgroups * ST_PX - 1) * s + ks;  // every window column an item may read
  a.astage = 2u * ((3u * ST_LBO_A + 2048u + 1023u) / 1024u * 1024u);
  const uint32_t wbytes = 2u * (uint32_t)a.BN * (uint32_t)a.Cpad * 4u;
  a.filt_bytes = (uint32_t)(ks * ks * ST_CK * 4);
  auto layout = [&](int sa, int sp) {
    a.IH = (((a.TH + ST_PY - 1) / ST_PY) * ST_PY - 1) * s + ks;  // rows of the last (ragged) block too
    a.patch_bytes = (uint32_t)(a.TN * a.IH * a.IW * ST_CK * 4);
    a.pstage = (a.patch_bytes + a.filt_bytes + 1023u) / 1024u * 1024u;  // TMA destinations 1024-B aligned
    a.off_a = (wbytes + 1023u) / 1024u * 1024u;
    a.off_p = a.off_a + (uint32_t)sa * a.astage;
    a.off_bdw = a.off_p + (uint32_t)sp * a.pstage;
    a.off_bar = (a.off_bdw + (uint32_t)a.Cpad * 4u + 15u) / 16u * 16u;
    return (size_t)a.off_bar + 8 * (2 * sa + 2 * sp + 5) + 16;
  };
  // ring depths, then smaller tiles, until the shared memory fits
  int sa = 3, sp = 3;
  size_t smem = layout(sa, sp);
  while (smem > (size_t)ST_SMEM_MAX) {
    if (sp > 2) --sp;
    else if (sa > 2) --sa;
    else if (a.TN > 1) --a.TN;
    else if (a.TH > 1) --a.TH;
    else return (int)cudaErrorInvalidValue;
    smem = layout(sa, sp);
  }
  if (a.IW > 256 || a.IH > 256 || a.TN > 256) return (int)cudaErrorInvalidValue;  // TMA box limits
  a.a_stages = sa;
  a.p_stages = sp;
  a.bands = (a.P + a.TH - 1) / a.TH;
  a.ntile = (a.N + a.TN - 1) / a.TN * a.bands;
  CUtensorMap tin;
  {  // input (C, W, H, N), box [16 ch][IW][IH][TN]; out of range → 0 (halo, padding, channels >= C)
    const uint64_t dims[4] = {(uint64_t)a.C, (uint64_t)a.W, (uint64_t)a.H, (uint64_t)a.N};
    const uint64_t str[3] = {(uint64_t)in_sw * 4, (uint64_t)in_sh * 4, (uint64_t)in_sn * 4};
    const uint32_t box[4] = {ST_CK, (uint32_t)a.IW, (uint32_t)a.IH, (uint32_t)a.TN};
    if (!encode_tmap_f32(&tin, in, 4, dims, str, box)) {
        fprintf(stderr, "sepconv_tc: tensor map refused (C %d W %d H %d N %d strides %lld %lld %lld box %u %u %u %u)\n",
                a.C, a.W, a.H, a.N, (long long)in_sw, (long long)in_sh, (long long)in_sn, box[0], box[1], box[2],
                box[3]);
      return (int)cudaErrorInvalidValue;
    }
  }
  if (getenv("SW_DEBUG_LAUNCH"))
    fprintf(stderr, "sepconv_tc: C %d K %d Cpad %d BN %d nblk %d TN %d TH %d IH %d IW %d stages %d/%d smem %zu tiles %d\n",
            a.C, a.K, a.Cpad, a.BN, a.nblk, a.TN, a.TH, a.IH, a.IW, sa, sp, smem, a.ntile);
  const int per_blk = std::max(1, 148 / a.nblk);
  const int grid = a.nblk * std::min(a.ntile, per_blk);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t rc = cudaErrorInvalidValue;
#define SW_SEPTC(K_, S_) \
  if (ks == K_ && s == S_) rc = launch_k(sepconv_tc_kernel<K_, S_>, dim3(grid), dim3(ST_THREADS), smem, st, 1u, tin, a);
  SW_SEPTC(3, 1) SW_SEPTC(5, 1) SW_SEPTC(7, 1) SW_SEPTC(3, 2) SW_SEPTC(5, 2) SW_SEPTC(7, 2)
#undef SW_SEPTC
  if (rc != cudaSuccess)
    fprintf(stderr, "sepconv_tc launch failed: %s (grid %d smem %zu k %d s %d)\n", cudaGetErrorString(rc), grid, smem,
            ks, s);
  return (int)rc;
}

void init_sep_tc_kernels() {
  cudaFuncSetAttribute(sepconv_tc_kernel<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
  cudaFuncSetAttribute(sepconv_tc_kernel<5, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
  cudaFuncSetAttribute(sepconv_tc_kernel<7, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
  cudaFuncSetAttribute(sepconv_tc_kernel<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
  cudaFuncSetAttribute(sepconv_tc_kernel<5, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
  cudaFuncSetAttribute(sepconv_tc_kernel<7, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM_MAX);
}

}  // namespace sw
