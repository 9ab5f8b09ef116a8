// Measured fp32 compute peaks of this B200 for the roofline denominators
// (MEASURED_PEAKS.json carries only HBM GB/s and dense bf16): chip-wide FFMA
// TFLOP/s and tcgen05 kind::tf32 TFLOP/s (M = 128, N = 256, one CTA per SM,
// operands resident in shared memory), timed with CUDA events.  The
// fp32-accurate tensor-core path runs 3 tf32 MMAs per product (3xTF32), so
// its effective peak is a third of the tf32 figure.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks_fp32 tools/peaks_fp32.cu
// Run:   ./tools/peaks_fp32 > profiles/peaks_fp32.json
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(512, 2) ffma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.f) out[0] = s;  // keep the chain alive
}

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__global__ void __launch_bounds__(128, 1) tf32_kernel(int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (48 * 1024) / 16; i += 128) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (32u << 17) | (8u << 24);  // N 256, M 128
    uint64_t da[4], db[4];
    for (int ks = 0; ks < 4; ++ks) {
      da[ks] = desc_sw(su(smem) + ks * 32);
      db[ks] = desc_sw(su(smem + 16 * 1024) + ks * 32);
    }
    for (int r = 0; r < reps; r += 4) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(da[ks]), "l"(db[ks]), "r"(idesc), "r"((r | ks) ? 1u : 0u)
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar))
                 : "memory");
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(su(&bar))
          : "memory");
    } while (!done);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

int main() {
  int sms = 0, dev = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // FFMA: 2 CTAs x 512 threads per SM, 16 independent chains per thread
  const int iters = 20000;
  float best_ffma = 0.f;
  for (int w = 0; w < 3; ++w) {
    cudaEventRecord(e0);
    ffma_kernel<<<sms * 2, 512>>>(out, iters, 1.0000001f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * iters * (double)sms * 2 * 512;
    const float tf = (float)(flops / (ms * 1e-3) / 1e12);
    if (tf > best_ffma) best_ffma = tf;
  }
  cudaFuncSetAttribute(tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int reps = 1 << 16;
  float best_tf32 = 0.f;
  for (int w = 0; w < 3; ++w) {
    cudaEventRecord(e0);
    tf32_kernel<<<sms, 128, 64 * 1024>>>(reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 128 * 256 * 8 * (double)reps * sms;
    const float tf = (float)(flops / (ms * 1e-3) / 1e12);
    if (tf > best_tf32) best_tf32 = tf;
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf(
      "{\"ffma_fp32_tflops\": %.1f, \"tcgen05_tf32_tflops\": %.1f, \"tcgen05_3xtf32_effective_tflops\": %.1f, "
      "\"sms\": %d, \"method\": \"tools/peaks_fp32.cu: best of 3 event-timed launches; FFMA 16 independent chains x "
      "1024 threads per SM; tcgen05 kind::tf32 M128 N256 K8 back to back from smem, one CTA per SM\", "
      "\"status\": \"%s\"}\n",
      best_ffma, best_tf32, best_tf32 / 3.f, sms, cudaGetErrorString(err));
  return 0;
}
