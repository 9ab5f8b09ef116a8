// Phase probe: globaltimer stamps inside kernels, compiled only into the
// diagnostic build (libsw_b200_probe.so, -DSW_PROBE; tools/phase_probe.py).
// The product library compiles every probe call to nothing.
//
// Per launch: the first CTA to start stamps start[launch], the last CTA to
// finish stamps end[launch] (launches counted modulo 16); CTA (0,0,0) also
// stamps the phase points pt[i] (clock64) of the kernel it runs (last launch wins).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sw {

#ifdef SW_PROBE
struct ProbeBuf {
  unsigned long long pt[16];
  unsigned long long trace[64];  // free-form clock64 stamps of CTA (0,0,0) (probe_trace)
  unsigned long long start[16];
  unsigned long long end[16];
  unsigned int started, finished;
};

static __device__ ProbeBuf g_probe;

__device__ __forceinline__ unsigned long long probe_time() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// phase points in SM clock cycles (globaltimer ticks in 256 ns steps here)
__device__ __forceinline__ void probe_pt(int i) {
  if (threadIdx.x == 0 && (blockIdx.x | blockIdx.y | blockIdx.z) == 0) g_probe.pt[i] = clock64();
}

// any thread of CTA (0,0,0) (e.g. a specialised producer / MMA warp)
__device__ __forceinline__ void probe_pt_any(int i) {
  if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0) g_probe.pt[i] = clock64();
}

__device__ __forceinline__ void probe_trace(int i) {
  if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0 && i >= 0 && i < 64) g_probe.trace[i] = clock64();
}

__device__ __forceinline__ void probe_begin() {
  if (threadIdx.x == 0) {
    const unsigned n = gridDim.x * gridDim.y * gridDim.z;
    const unsigned s = atomicAdd(&g_probe.started, 1u);
    if (s % n == 0) g_probe.start[(s / n) & 15] = probe_time();
  }
  probe_pt(0);
}

// call where every thread of the CTA passes, after its last store
__device__ __forceinline__ void probe_end() {
  __syncthreads();
  probe_pt(15);
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned n = gridDim.x * gridDim.y * gridDim.z;
    const unsigned f = atomicAdd(&g_probe.finished, 1u);
    if (f % n == n - 1) g_probe.end[(f / n) & 15] = probe_time();
  }
}

// host side: every translation unit registers its own buffer
using ProbeFn = void (*)(ProbeBuf*, bool reset);
int probe_register(ProbeFn fn);

static void probe_tu_access(ProbeBuf* out, bool reset) {
  if (reset) {
    ProbeBuf z = {};
    cudaMemcpyToSymbol(g_probe, &z, sizeof(z));
  } else {
    cudaMemcpyFromSymbol(out, g_probe, sizeof(ProbeBuf));
  }
}
static int g_probe_registered = probe_register(&probe_tu_access);
#else
__device__ __forceinline__ void probe_pt(int) {}
__device__ __forceinline__ void probe_pt_any(int) {}
__device__ __forceinline__ void probe_trace(int) {}
__device__ __forceinline__ void probe_begin() {}
__device__ __forceinline__ void probe_end() {}
#endif

}  // namespace sw
