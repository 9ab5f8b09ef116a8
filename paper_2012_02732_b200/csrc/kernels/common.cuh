// Small device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../runtime/ops.h"
#include "probe.cuh"

namespace sw {

// Transcendental activations live out of line: batch-1 kernels run on cold
// SMs, and every inlined copy of expf grows the code an SM must fetch.
static __device__ __noinline__ float act_slow(float v, int act) {
  if (act == ACT_SILU) return v / (1.f + expf(-v));
  if (act == ACT_SIGMOID) return 1.f / (1.f + expf(-v));
  return v;
}

__device__ __forceinline__ float apply_act(float v, int act) {
  if (act == ACT_NONE) return v;
  if (act == ACT_RELU) return fmaxf(v, 0.f);
  if (act == ACT_RELU6) return fminf(fmaxf(v, 0.f), 6.f);
  return act_slow(v, act);
}

__device__ __forceinline__ float4 act4(float4 v, int act) {
  return make_float4(apply_act(v.x, act), apply_act(v.y, act), apply_act(v.z, act),
                     apply_act(v.w, act));
}

__host__ __device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

__host__ __forceinline__ bool aligned16(uint64_t p) { return (p & 15ull) == 0; }

// Programmatic dependent launch (PDL).  Every kernel lets its dependents be
// scheduled as soon as it starts (launch_dependents) and waits for its
// prerequisite grids before touching activations (wait); both are no-ops
// when the launch carried no programmatic edge.  Constant weights may be
// fetched before pdl_wait().
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Engine-controlled launch flags (set around capture / eager launches).
extern thread_local bool g_launch_pdl;
// Per-task execution priority (cudaLaunchAttributePriority, 0 = default;
// the engine raises the critical-path tasks of the schedule).
extern thread_local int g_launch_priority;

// Single launch path for every kernel: optional cluster (split-K along z)
// and the PDL attribute.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            unsigned cluster_z, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  unsigned n = 0;
  if (g_launch_priority != 0) {
    attr[n].id = cudaLaunchAttributePriority;
    attr[n].val.priority = g_launch_priority;
    ++n;
  }
  if (cluster_z > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 1;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = cluster_z;
    ++n;
  }
  if (g_launch_pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, fn, static_cast<Args&&>(args)...);
}

// ---------------------------------------------------------------------------
// Shared GEMM-tile epilogue.  The CTA's [BM][BN] fp32 tile sits in shared
// memory (rows = output pixels, columns = output channels).  Threads walk it
// in groups of 4 channels: bias / residual / output move as float4 when the
// layout allows (Epi::vec), and a split-K cluster reduces its ranks' tiles
// through DSMEM with every remote load of a group in flight at once (ncu: a
// rank-serial scalar reduction kept a tcgen05 layer at IPC 0.08).
// ---------------------------------------------------------------------------
struct Epi {
  const float* bias;
  const float* res;
  float* out;
  int M, K, P, Q, act, has_res, vec;
  int64_t out_sn, out_sh, out_sw, out_sc;
  int64_t res_sn, res_sh, res_sw, res_sc;
};

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// PS = row stride of the tile in floats (BN, or BN + 4 where the producer
// writes one row per lane: the padding makes those float4 stores conflict-free)
template <int BM, int BN, int NT, int PS = BN, typename Cluster>
__device__ __forceinline__ void tile_epilogue(const Epi& ep, const float* part, int m0, int n0, int split,
                                              Cluster& cluster) {
  static_assert(BN % 4 == 0 && PS % 4 == 0, "channel groups of 4");
  constexpr int GPR = BN / 4;  // groups per row
  constexpr int G = BM * GPR;
  int g0 = 0, g1 = G, nr = 1;
  if (split > 1) {
    cluster.sync();
    nr = (int)cluster.num_blocks();
    const int chunk = (G + nr - 1) / nr;
    g0 = (int)cluster.block_rank() * chunk;
    g1 = min(G, g0 + chunk);
  } else {
    __syncthreads();
  }
#pragma unroll 2
  for (int g = g0 + (int)threadIdx.x; g < g1; g += NT) {
    const int m = m0 + g / GPR, n = n0 + (g % GPR) * 4;
    if (m >= ep.M || n >= ep.K) continue;
    float4 v;
    const int gi = PS == BN ? g : (g / GPR) * (PS / 4) + g % GPR;  // float4 index in the tile
    if (nr == 1) {
      v = reinterpret_cast<const float4*>(part)[gi];
    } else {
      v = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 t[16];  // up to 16 ranks (non-portable cluster size)
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < nr) t[r] = reinterpret_cast<const float4*>(cluster.map_shared_rank(part, r))[gi];
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < nr) v = f4add(v, t[r]);
    }
    const int q = m % ep.Q;
    const int tt = m / ep.Q;
    const int pp = tt % ep.P, nb = tt / ep.P;
    float* o = ep.out + nb * ep.out_sn + pp * ep.out_sh + q * ep.out_sw;
    const float* rp = ep.has_res ? ep.res + nb * ep.res_sn + pp * ep.res_sh + q * ep.res_sw : nullptr;
    if (ep.vec && n + 3 < ep.K) {
      if (ep.bias) v = f4add(v, *reinterpret_cast<const float4*>(ep.bias + n));
      if (rp) v = f4add(v, *reinterpret_cast<const float4*>(rp + n));
      *reinterpret_cast<float4*>(o + n) = act4(v, ep.act);
    } else {
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (n + j >= ep.K) break;
        float x = vv[j] + (ep.bias ? ep.bias[n + j] : 0.f);
        if (rp) x += rp[(n + j) * ep.res_sc];
        o[(n + j) * ep.out_sc] = apply_act(x, ep.act);
      }
    }
  }
  if (split > 1) cluster.sync();
}

// Host-side: can the epilogue move 4 channels at a time?
inline bool epi_vec_ok(uint64_t out, int64_t osn, int64_t osh, int64_t osw, int64_t osc, uint64_t bias,
                       bool has_res, uint64_t res, int64_t rsn, int64_t rsh, int64_t rsw, int64_t rsc) {
  if (osc != 1 || (out & 15) || (osn | osh | osw) & 3) return false;
  if (bias && (bias & 15)) return false;
  if (has_res && (rsc != 1 || (res & 15) || ((rsn | rsh | rsw) & 3))) return false;
  return true;
}

}  // namespace sw
