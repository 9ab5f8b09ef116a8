// Pointwise (1x1, stride 1) convolution for latency-bound layers (batch 1):
// the NASNet cell inputs (`prev` / `conv_1x1`, C_in 264..1056 → 44..176) sit on
// the critical path, ~17 of them in a row.
//
// One CTA = BM output pixels x BN output channels x one K slice (Kc input
// channels).  A thread-block cluster of `split` CTAs along z covers C_in and
// reduces through DSMEM.  Operands arrive by TMA on two mbarriers issued by
// one thread: the weight tile [BN][Kc] and the bias slice before the PDL wait
// (constants), the activation tile [BM][Kc] (2-D tensor map over the NHWC
// pixels, so concat channel slices need no address math) and the residual
// tile after it.  The GEMM is split over the 8 warps along Kc: each lane owns
// BN/32 columns for all BM pixels, the A values are warp-broadcast float4
// loads, and Kc/4 is kept odd so the B rows' float4 loads are bank-conflict
// free.  Warp partials → one tile per CTA → cluster reduction + bias +
// residual + activation → float4 stores.
#include <cooperative_groups.h>

#include "common.cuh"
#include "conv_args.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace sw {

struct PwGeo {
  int Kc;
  int o_a, o_b, o_bias, o_res, o_t, o_rcv, o_bar;
  int chunk;  // float4 groups of the tile each cluster rank finishes
  uint32_t bytes_b, bytes_act;
};

template <int BM, int BN>
__global__ void __launch_bounds__(256)
pw_tma_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
              const __grid_constant__ CUtensorMap tr, ConvArgs a, PwGeo g) {
  static_assert(BN % 32 == 0, "tile");
  constexpr int JN = BN / 32;
  constexpr int GPR = BN / 4;
  extern __shared__ __align__(128) float smem[];
  float* As = smem + g.o_a;  // [BM][Kc]
  float* Bs = smem + g.o_b;  // [BN][Kc]
  float* Pt = smem;          // [8][BM][BN] warp partials (reuse A / B after the GEMM)
  float* bias_s = smem + g.o_bias;
  float* Rs = smem + g.o_res;  // [BM][BN]
  float* T = smem + g.o_t;     // [BM][BN] this CTA's K-slice partial
  float* Rcv = smem + g.o_rcv;  // [split][chunk*4] partials pushed by the peers for my slice
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + g.o_bar);
  const uint32_t bar_c = su32(&bars[0]), bar_a = su32(&bars[1]), bar_r = su32(&bars[2]);
  const int split = (int)gridDim.z;
  const int me = split > 1 ? (int)cluster_rank() : 0;
  constexpr int G = BM * GPR;  // float4 groups in the tile
  const int my_g0 = min(G, me * g.chunk), my_g1 = min(G, my_g0 + g.chunk);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int c0 = blockIdx.z * g.Kc;
  const int Kc = g.Kc;
  probe_begin();

  if (tid == 0) {
    prefetch_tmap(&ta);
    prefetch_tmap(&tb);
    mbar_init1(bar_c);
    mbar_init1(bar_a);
    mbar_init1(bar_r);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_proxy_async_cta();
    // the peers push (split-1) partial slices of my_g1-my_g0 groups into Rcv
    if (split > 1) mbar_expect_tx(bar_r, (uint32_t)((split - 1) * (my_g1 - my_g0) * 16));
    const uint32_t bias_bytes = a.bias ? (uint32_t)(min(BN, a.K - n0) * 4) : 0u;
    mbar_expect_tx(bar_c, g.bytes_b + bias_bytes);
    tma_load_2d(su32(Bs), &tb, c0, n0, bar_c);
    if (a.bias) bulk_g2s(su32(bias_s), a.bias + n0, bias_bytes, bar_c);
  }
  if (split > 1) cluster_arrive_relaxed();  // my barriers are initialised (waited on before pushing)
  pdl_trigger();
  probe_pt(1);
  pdl_wait();
  probe_pt(2);
  if (tid == 0) {
    mbar_expect_tx(bar_a, g.bytes_act);
    tma_load_2d(su32(As), &ta, c0, m0, bar_a);
    if (a.has_res) tma_load_2d(su32(Rs), &tr, n0, m0, bar_a);
  }
  __syncthreads();  // barrier inits visible before anyone polls them
  mbar_wait_parity(bar_c, 0);
  mbar_wait_parity(bar_a, 0);
  if (a.pre_relu) {  // shared ReLU once over the A tile, not per use
    float4* a4 = reinterpret_cast<float4*>(As);
#pragma unroll 1
    for (int i = tid; i < BM * Kc / 4; i += 256) {
      float4 v = a4[i];
      v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
      a4[i] = v;
    }
    __syncthreads();
  }
  probe_pt(3);

  float o[BM][JN];
#pragma unroll
  for (int i = 0; i < BM; ++i)
#pragma unroll
    for (int j = 0; j < JN; ++j) o[i][j] = 0.f;
  const int K4 = Kc >> 2;
  const int k0 = warp * K4 / 8, k1 = (warp + 1) * K4 / 8;
#pragma unroll 1
  for (int kg = k0; kg < k1; ++kg) {
    float4 b[JN];
#pragma unroll
    for (int j = 0; j < JN; ++j) b[j] = *reinterpret_cast<const float4*>(Bs + (lane + 32 * j) * Kc + 4 * kg);
#pragma unroll
    for (int i = 0; i < BM; ++i) {
      const float4 av = *reinterpret_cast<const float4*>(As + i * Kc + 4 * kg);
#pragma unroll
      for (int j = 0; j < JN; ++j) {
        o[i][j] = fmaf(av.x, b[j].x, o[i][j]);
        o[i][j] = fmaf(av.y, b[j].y, o[i][j]);
        o[i][j] = fmaf(av.z, b[j].z, o[i][j]);
        o[i][j] = fmaf(av.w, b[j].w, o[i][j]);
      }
    }
  }
  __syncthreads();  // A / B reads done before Pt overwrites them
#pragma unroll
  for (int i = 0; i < BM; ++i)
#pragma unroll
    for (int j = 0; j < JN; ++j) Pt[(warp * BM + i) * BN + lane + 32 * j] = o[i][j];
  __syncthreads();
  probe_pt(4);
#pragma unroll 1
  for (int gi = tid; gi < BM * GPR; gi += 256) {
    float4 t[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) t[w] = reinterpret_cast<const float4*>(Pt + w * BM * BN)[gi];
    float4 v = t[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) v = f4add(v, t[w]);
    reinterpret_cast<float4*>(T)[gi] = v;
  }
  probe_pt(5);

  // split-K reduction: push each peer its slice of my partial tile straight
  // into its shared memory (bulk DSMEM copies completing on its mbarrier) —
  // no cluster-wide barrier (a cg cluster.sync() costs a GPU-scope membar)
  if (split > 1) {
    fence_proxy_async_cta();  // my T writes → visible to the bulk-copy (async) proxy
    __syncthreads();
    cluster_wait();  // every peer initialised its barriers
    if (tid == 0) {
#pragma unroll 1
      for (int r = 0; r < split; ++r) {
        if (r == me) continue;
        const int r0 = min(G, r * g.chunk), r1 = min(G, r0 + g.chunk);
        if (r1 <= r0) continue;
        bulk_s2peer(mapa_rank(su32(Rcv + me * g.chunk * 4), (uint32_t)r), su32(T + r0 * 4), (uint32_t)((r1 - r0) * 16),
                    mapa_rank(bar_r, (uint32_t)r));
      }
      bulk_commit();
    }
    mbar_wait_parity(bar_r, 0);
  } else {
    __syncthreads();
  }
  probe_pt(6);
#pragma unroll 1
  for (int gi = my_g0 + tid; gi < my_g1; gi += 256) {
    const int mm = gi / GPR, nn = (gi % GPR) * 4;
    const int m = m0 + mm, n = n0 + nn;
    if (m >= a.M || n >= a.K) continue;
    float4 v = reinterpret_cast<const float4*>(T)[gi];
    if (split > 1) {
      float4 t[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < split && r != me) t[r] = reinterpret_cast<const float4*>(Rcv + r * g.chunk * 4)[gi - my_g0];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < split && r != me) v = f4add(v, t[r]);
    }
    if (a.bias) v = f4add(v, *reinterpret_cast<const float4*>(bias_s + nn));
    if (a.has_res) v = f4add(v, *reinterpret_cast<const float4*>(Rs + mm * BN + nn));
    const int q = m % a.Q, tt = m / a.Q;
    const int p = tt % a.P, nb = tt / a.P;
    *reinterpret_cast<float4*>(a.out + nb * a.out_sn + p * a.out_sh + q * a.out_sw + n) = act4(v, a.act);
  }
  probe_pt(7);
  if (split > 1 && tid == 0) bulk_wait_read0();  // my pushes have read T before the CTA exits
  probe_end();
}

namespace {
// variants (conv variant 16 + i): (BM, BN) = (8,32) (16,32) (32,32) (16,64) (32,64) (64,32)
constexpr int kPwSmemMax = 227 * 1024;

int r32(int x) { return (x + 31) / 32 * 32; }
}  // namespace

// true if the op can run the TMA pointwise kernel with this tile / split
static bool pw_geo(const ConvArgs& a, const sw_op_desc& op, int bm, int bn, PwGeo* g, size_t* smem) {
  if (a.R != 1 || a.S != 1 || a.sh != 1 || a.sw != 1 || a.ph != 0 || a.pw != 0) return false;
  if (a.in_sc != 1 || a.C % 4 || a.K % 4 || !a.epi.vec) return false;
  // pixels must collapse to one dimension (NHWC buffer, possibly a channel slice)
  if (a.in_sh != (int64_t)a.W * a.in_sw || (a.N > 1 && a.in_sn != (int64_t)a.H * a.in_sh)) return false;
  if (a.has_res && (a.res_sc != 1 || a.res_sh != (int64_t)a.Q * a.res_sw ||
                    (a.N > 1 && a.res_sn != (int64_t)a.P * a.res_sh)))
    return false;
  if (a.bias && (op.ptrs[PT_BIAS] & 15)) return false;
  int kc = (a.C + a.split - 1) / a.split;
  kc = (kc + 3) / 4 * 4;
  if (((kc / 4) & 1) == 0) kc += 4;  // odd float4 pitch: conflict-free B rows
  if (kc > 256) return false;
  g->Kc = kc;
  // TMA destinations 128-B aligned; warp partials reuse the A / B region
  g->o_a = 0;
  g->o_b = r32(bm * kc);
  const int ab = g->o_b + bn * kc;
  const int pt = 8 * bm * bn;
  int o = r32(ab > pt ? ab : pt);
  g->o_bias = o; o += r32(bn);
  g->o_res = o; o += r32(bm * bn);
  g->o_t = o; o += r32(bm * bn);
  const int groups = bm * bn / 4;
  g->chunk = (groups + a.split - 1) / a.split;
  g->o_rcv = o; o += a.split > 1 ? r32(a.split * g->chunk * 4) : 0;
  g->o_bar = o; o += 32;
  *smem = (size_t)o * 4;
  if (*smem > (size_t)kPwSmemMax) return false;
  g->bytes_b = (uint32_t)(bn * kc * 4);
  g->bytes_act = (uint32_t)((bm * kc + (a.has_res ? bm * bn : 0)) * 4);
  return true;
}

template <int BM, int BN>
static cudaError_t launch_pw_t(const ConvArgs& a, const sw_op_desc& op, cudaStream_t st) {
  PwGeo g;
  size_t smem = 0;
  if (!pw_geo(a, op, BM, BN, &g, &smem)) return cudaErrorInvalidValue;
  CUtensorMap ta, tb, tr;
  {
    const uint64_t dims[2] = {(uint64_t)a.C, (uint64_t)a.M};
    const uint64_t str[1] = {(uint64_t)a.in_sw * 4};
    const uint32_t box[2] = {(uint32_t)g.Kc, (uint32_t)BM};
    if (!encode_tmap_f32(&ta, a.in, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[2] = {(uint64_t)a.C, (uint64_t)a.K};
    const uint64_t str[1] = {(uint64_t)a.C * 4};
    const uint32_t box[2] = {(uint32_t)g.Kc, (uint32_t)BN};
    if (!encode_tmap_f32(&tb, a.w, 2, dims, str, box)) return cudaErrorInvalidValue;
  }
  if (a.has_res) {
    const uint64_t dims[2] = {(uint64_t)a.K, (uint64_t)a.M};
    const uint64_t str[1] = {(uint64_t)a.res_sw * 4};
    const uint32_t box[2] = {(uint32_t)BN, (uint32_t)BM};
    if (!encode_tmap_f32(&tr, a.res, 2, dims, str, box)) return cudaErrorInvalidValue;
  } else {
    tr = tb;  // unused
  }
  dim3 grid((unsigned)cdiv(a.M, BM), (unsigned)cdiv(a.K, BN), (unsigned)a.split);
  return launch_k(pw_tma_kernel<BM, BN>, grid, dim3(256), smem, st, (unsigned)a.split, ta, tb, tr, a, g);
}

int launch_conv_pw(const sw_op_desc& op, int v, void* stream) {
  ConvArgs a = conv_args(op);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (a.M == 0 || a.K == 0) return 0;
  if (a.split != 1 && a.split != 2 && a.split != 4 && a.split != 8) return (int)cudaErrorInvalidValue;
  switch (v) {
    case 0: return (int)launch_pw_t<8, 32>(a, op, st);
    case 1: return (int)launch_pw_t<16, 32>(a, op, st);
    case 2: return (int)launch_pw_t<32, 32>(a, op, st);
    case 3: return (int)launch_pw_t<16, 64>(a, op, st);
    case 4: return (int)launch_pw_t<32, 64>(a, op, st);
    case 5: return (int)launch_pw_t<64, 32>(a, op, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

void init_pw_kernels() {
  cudaFuncSetAttribute(pw_tma_kernel<8, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmemMax);
  cudaFuncSetAttribute(pw_tma_kernel<16, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmemMax);
  cudaFuncSetAttribute(pw_tma_kernel<32, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmemMax);
  cudaFuncSetAttribute(pw_tma_kernel<16, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmemMax);
  cudaFuncSetAttribute(pw_tma_kernel<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmemMax);
  cudaFuncSetAttribute(pw_tma_kernel<64, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPwSmemMax);
}

}  // namespace sw
