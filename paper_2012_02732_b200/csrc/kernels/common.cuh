// Small device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../runtime/ops.h"

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
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
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

}  // namespace sw
