// tcgen05.mma issue-rate probe (diagnostic, not product).
//
// One CTA per SM; one thread issues `reps` MMAs (kind::tf32 or kind::f16,
// M = 128, N = n, K step = 32 B) on zero-filled shared-memory operands,
// round-robin over `nacc` TMEM accumulators, commits once, and the elapsed
// clock64 → MACs per clock per SM.  Layouts: 0 = K-major no-swizzle canonical,
// 1 = K-major SWIZZLE_128B.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_ns(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (KIND == 0)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) rate_kernel(int n, int reps, int nacc, int layout, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (64 * 1024) / 16; i += 128) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid == 0) {
    // D f32; A/B tf32 (2) or bf16 (1); K-major; N, M = 128
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t a = su(smem), b = su(smem + 32 * 1024);
    uint64_t da[4], db[4];
    for (int ks = 0; ks < 4; ++ks) {
      if (layout == 0) {
        da[ks] = desc_ns(a + ks * 4096, 2048, 128);
        db[ks] = desc_ns(b + ks * 2 * n * 16, n * 16, 128);
      } else {
        da[ks] = desc_sw(a + ks * 32);
        db[ks] = desc_sw(b + ks * 32);
      }
    }
    long long t0 = clock64();
    if (nacc == 1) {
      for (int r = 0; r < reps; r += 4) {
        mma<KIND>(tmem, da[0], db[0], idesc, r ? 1u : 0u);
        mma<KIND>(tmem, da[1], db[1], idesc, 1u);
        mma<KIND>(tmem, da[2], db[2], idesc, 1u);
        mma<KIND>(tmem, da[3], db[3], idesc, 1u);
      }
    } else {
      for (int r = 0; r < reps; ++r) {
        const int ks = r & 3;
        const uint32_t d = tmem + (uint32_t)((r % nacc) * n);
        mma<KIND>(d, da[ks], db[ks], idesc, r >= nacc ? 1u : 0u);
      }
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
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// warp-uniform issue: descriptors recomputed every MMA from the loop counter
// (as a pipelined kernel does from its stage index), one elected lane issues
template <int KIND>
__global__ void __launch_bounds__(128, 1) rate_kernel_warp(int n, int reps, int stages, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (64 * 1024) / 16; i += 128) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid < 32) {
    const uint32_t fmt = KIND == 0 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t a = su(smem), b = su(smem + 32 * 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 4) {
      const int st = (r >> 2) % stages;  // a "stage" of 4 K steps, 8 KB apart
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const uint64_t da = desc_ns(a + (st & 1) * 512 + ks * 4096, 2048, 128);
        const uint64_t db = desc_ns(b + (st & 1) * 512 + ks * 2 * n * 16, n * 16, 128);
        if (elect_one()) mma<KIND>(tmem, da, db, idesc, (r | ks) ? 1u : 0u);
        __syncwarp();
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar))
                   : "memory");
    __syncwarp();
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(su(&bar))
          : "memory");
    } while (!done);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// descriptors precomputed for NS stages (registers), stage walked by an
// unrolled loop: the pattern of a pipelined kernel's issuer after hoisting
template <int NS>
__global__ void __launch_bounds__(128, 1) rate_kernel_table(int n, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < (64 * 1024) / 16; i += 128) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid < 32) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t a = su(smem), b = su(smem + 32 * 1024);
    const uint64_t a0 = desc_ns(a, 2048, 128), b0 = desc_ns(b, n * 16, 128);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 4 * NS) {
#pragma unroll
      for (int st = 0; st < NS; ++st) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint64_t da = a0 + (uint64_t)(((st & 3) * 512 + ks * 4096) >> 4);
          const uint64_t db = b0 + (uint64_t)(((st & 3) * 512 + ks * 2 * n * 16) >> 4);
          if (elect_one()) mma<0>(tmem + (st & 1) * n, da, db, idesc, (r | st | ks) ? 1u : 0u);
          __syncwarp();
        }
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar))
                   : "memory");
    __syncwarp();
    uint32_t done = 0;
    do {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(su(&bar))
          : "memory");
    } while (!done);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(rate_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(rate_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int reps = 4096;
  for (int kind = 0; kind < 2; ++kind)
    for (int layout = 0; layout < 2; ++layout)
      for (int n : {32, 64, 128, 256})
        for (int nacc : {1, 2, 4}) {
          if (n * nacc > 512) continue;
          for (int w = 0; w < 2; ++w) {
            if (kind == 0)
              rate_kernel<0><<<148, 128, 96 * 1024>>>(n, reps, nacc, layout, d);
            else
              rate_kernel<1><<<148, 128, 96 * 1024>>>(n, reps, nacc, layout, d);
          }
          cudaError_t e = cudaDeviceSynchronize();
          long long h[148];
          cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
          double avg = 0;
          for (int i = 0; i < 148; ++i) avg += h[i];
          avg /= 148;
          const double k = kind == 0 ? 8 : 16;  // K per instruction (32 B of operand)
          const double macs = 128.0 * n * k;
          printf("%s layout=%s N=%3d acc=%d: %7.1f clk/MMA  %7.0f MAC/clk/SM  (%s)\n", kind ? "bf16" : "tf32",
                 layout ? "sw128" : "noswz", n, nacc, avg / reps, macs * reps / avg, cudaGetErrorString(e));
        }
  cudaFuncSetAttribute(rate_kernel_warp<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int n : {32, 64, 128, 256}) {
    for (int w = 0; w < 2; ++w) rate_kernel_warp<0><<<148, 128, 96 * 1024>>>(n, reps, 3, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("tf32 warp-uniform elect issue N=%3d: %7.1f clk/MMA  %7.0f MAC/clk/SM  (%s)\n", n, avg / reps,
           128.0 * n * 8 * reps / avg, cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(rate_kernel_table<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(rate_kernel_table<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int ns : {4, 16})
    for (int n : {64, 128, 256}) {
      for (int w = 0; w < 2; ++w) {
        if (ns == 4) rate_kernel_table<4><<<148, 128, 96 * 1024>>>(n, reps, d);
        else rate_kernel_table<16><<<148, 128, 96 * 1024>>>(n, reps, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("tf32 hoisted-table stages=%2d N=%3d: %7.1f clk/MMA  %7.0f MAC/clk/SM  (%s)\n", ns, n, avg / reps,
             128.0 * n * 8 * reps / avg, cudaGetErrorString(e));
    }
  return 0;
}
