// How fast can a subset of SMs pull a weight stream from HBM?  Each CTA
// streams its contiguous slice of a buffer through a ring of 1-D bulk copies
// (the conv_tcs weight producer's pattern) and the time from launch to the
// last CTA's end is measured with CUDA events, L2 flushed before every launch.
// Swept: total bytes, CTAs, cluster size, ring stages x stage bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_rate tools/stream_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(64, 1) stream_kernel(const uint8_t* src, size_t per_cta, int stage_bytes, int stages,
                                                       float* sink, unsigned long long* stamps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[16];
  const int tid = threadIdx.x;
  const size_t off = (size_t)blockIdx.x * per_cta;
  const int iters = (int)(per_cta / stage_bytes);
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float acc = 0.f;
  if (tid == 0) {
    stamps[2 * blockIdx.x] = gtime();
    for (int t = 0; t < iters; ++t) {
      const int s = t % stages;
      if (t >= stages) {
        // consume stage s (the previous fill) before refilling it
        const uint32_t par = (uint32_t)(((t / stages) - 1) & 1);
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, "
              "p;\n\t}"
              : "=r"(done)
              : "r"(su(&full[s])), "r"(par));
        acc += reinterpret_cast<const float*>(smem + s * stage_bytes)[0];
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(stage_bytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su(smem + s * stage_bytes)),
          "l"(src + off + (size_t)t * stage_bytes), "r"(stage_bytes), "r"(su(&full[s]))
          : "memory");
    }
    for (int t = (iters > stages ? iters - stages : 0); t < iters; ++t) {
      const int s = t % stages;
      const uint32_t par = (uint32_t)((t / stages) & 1);
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(su(&full[s])), "r"(par));
      acc += reinterpret_cast<const float*>(smem + s * stage_bytes)[0];
    }
    if (acc == 123.f) sink[0] = acc;
    stamps[2 * blockIdx.x + 1] = gtime();
  }
}

__global__ void flush_kernel(float4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

int main() {
  const size_t maxbytes = 64ull << 20;
  uint8_t* src;
  float* sink;
  float4* fl;
  const size_t fln = (512ull << 20) / 16;
  cudaMalloc(&src, maxbytes);
  cudaMemset(src, 0, maxbytes);
  cudaMalloc(&sink, 4);
  cudaMalloc(&fl, fln * 16);
  unsigned long long* stamps;
  cudaMalloc(&stamps, 2 * 512 * 8);
  unsigned long long hst[1024];
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t totals[] = {4718592, 9437184, 18874368};
  const int grids[] = {16, 32, 64, 96, 128, 144, 148};
  const int clusters[] = {1, 4, 16};
  const int stage_cfg[][2] = {{32768, 4}, {16384, 12}};
  printf("{\"rows\": [\n");
  bool first = true;
  for (size_t total : totals)
    for (int g : grids)
      for (int cs : clusters)
        for (auto& sc : stage_cfg) {
          if (g % cs) continue;
          const int sb = sc[0], st = sc[1];
          size_t per = total / g;
          per = (per / sb) * sb;
          if (per == 0) continue;
          float best = 1e9f, best_span = 1e9f, best_cta = 1e9f;
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(g);
          cfg.blockDim = dim3(64);
          cfg.dynamicSmemBytes = (size_t)sb * st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = cs;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          for (int rep = 0; rep < 6; ++rep) {
            flush_kernel<<<1184, 256>>>(fl, fln);
            cudaEventRecord(e0);
            cudaError_t err = cudaLaunchKernelEx(&cfg, stream_kernel, (const uint8_t*)src, per, sb, st, sink, stamps);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            if (err != cudaSuccess) {
              best = -1.f;
              cudaGetLastError();
              break;
            }
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
            cudaMemcpy(hst, stamps, 2 * g * 8, cudaMemcpyDeviceToHost);
            unsigned long long lo = ~0ull, hi = 0;
            double mean = 0;
            for (int i = 0; i < g; ++i) {
              lo = hst[2 * i] < lo ? hst[2 * i] : lo;
              hi = hst[2 * i + 1] > hi ? hst[2 * i + 1] : hi;
              mean += (double)(hst[2 * i + 1] - hst[2 * i]) / g;
            }
            if (rep > 0 && (hi - lo) * 1e-3f < best_span) best_span = (hi - lo) * 1e-3f;
            if (rep > 0 && mean * 1e-3 < best_cta) best_cta = (float)(mean * 1e-3);
          }
          const double bytes = (double)per * g;
          printf("%s {\"total\": %zu, \"ctas\": %d, \"cluster\": %d, \"stage\": %d, \"stages\": %d, \"us\": %.2f, "
                 "\"span_us\": %.2f, \"cta_us\": %.2f, \"span_GBps\": %.0f, \"per_cta_GBps\": %.1f}",
                 first ? "" : ",\n", (size_t)bytes, g, cs, sb, st, best * 1e3, best_span, best_cta,
                 bytes / (best_span * 1e-6) / 1e9, bytes / g / (best_cta * 1e-6) / 1e9);
          first = false;
        }
  printf("\n], \"status\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
