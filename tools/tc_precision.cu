// tcgen05 kind::tf32 accumulation-precision probe (diagnostic, not product).
//
// One CTA computes C[128][64] = A[128][K] · B[64][K]^T with fp32 inputs and
// reports the error against an fp64 host product for several 3xTF32 schemes:
//   mode 0: hi = trunc(x), lo = x - hi; hh, hl, lh into ONE TMEM accumulator
//   mode 1: as 0 with hi = rn(x) (cvt.rna.tf32)
//   mode 2: mode 1, hh into acc0, hl + lh into acc1, summed at the end
//   mode 3: mode 2 + promotion: every K tile (32) both accumulators are
//           drained to registers (fp32 RN adds) and restarted
//   mode 4: FFMA (one thread per output, sequential K)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_precision tools/tc_precision.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

constexpr int BM = 128, BN = 64, BK = 16;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ float rn_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar), "r"(par)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tld16(uint32_t t, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// canonical K-major no-swizzle: chunk (4 tf32) major, 8x16B core matrices
__device__ __forceinline__ int off(int r, int k, int R) { return (k >> 2) * (R * 4) + (r >> 3) * 32 + (r & 7) * 4 + (k & 3); }

__global__ void __launch_bounds__(128) tc_kernel(const float* A, const float* B, float* C, int K, int mode) {
  __shared__ __align__(1024) float ahi[BM * BK], alo[BM * BK], bhi[BN * BK], blo[BN * BK];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  float racc[BN];
  for (int j = 0; j < BN; ++j) racc[j] = 0.f;
  uint32_t phase = 0;
  const int tiles = K / BK;
  for (int kt = 0; kt < tiles; ++kt) {
    for (int e = tid; e < BM * BK; e += 128) {
      const int r = e / BK, k = e % BK;
      const float x = A[r * K + kt * BK + k];
      const float h = mode == 0 ? __uint_as_float(__float_as_uint(x) & 0xFFFFE000u) : rn_tf32(x);
      ahi[off(r, k, BM)] = h;
      alo[off(r, k, BM)] = mode == 0 ? x - h : rn_tf32(x - h);
    }
    for (int e = tid; e < BN * BK; e += 128) {
      const int r = e / BK, k = e % BK;
      const float x = B[r * K + kt * BK + k];
      const float h = mode == 0 ? __uint_as_float(__float_as_uint(x) & 0xFFFFE000u) : rn_tf32(x);
      bhi[off(r, k, BN)] = h;
      blo[off(r, k, BN)] = mode == 0 ? x - h : rn_tf32(x - h);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t LA = BM * 16, LB = BN * 16;
      const bool fresh = (mode == 3) || kt == 0;
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint64_t ah = make_desc(su(ahi) + ks * 2 * LA, LA, 128), al = make_desc(su(alo) + ks * 2 * LA, LA, 128);
        const uint64_t bh = make_desc(su(bhi) + ks * 2 * LB, LB, 128), bl = make_desc(su(blo) + ks * 2 * LB, LB, 128);
        const uint32_t first = (fresh && ks == 0) ? 0u : 1u;
        const uint32_t d1 = mode >= 2 ? tmem + BN : tmem;
        mma_tf32(tmem, ah, bh, idesc, first);
        mma_tf32(d1, ah, bl, idesc, mode >= 2 ? first : 1u);
        mma_tf32(d1, al, bh, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
    }
    wait_bar(su(&bar), phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (mode == 3) {
      const uint32_t t = tmem + ((uint32_t)(warp * 32) << 16);
      for (int c = 0; c < BN; c += 16) {
        float v[16], w[16];
        tld16(t + c, v);
        tld16(t + BN + c, w);
        for (int j = 0; j < 16; ++j) racc[c + j] += v[j] + w[j];
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
    }
    __syncthreads();
  }
  const int row = warp * 32 + (tid & 31);
  const uint32_t t = tmem + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < BN; c += 16) {
    float v[16], w[16];
    if (mode == 3) {
      for (int j = 0; j < 16; ++j) C[row * BN + c + j] = racc[c + j];
      continue;
    }
    tld16(t + c, v);
    if (mode >= 2) tld16(t + BN + c, w);
    for (int j = 0; j < 16; ++j) C[row * BN + c + j] = mode >= 2 ? v[j] + w[j] : v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

__global__ void ffma_kernel(const float* A, const float* B, float* C, int K) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= BM * BN) return;
  const int r = i / BN, c = i % BN;
  float s = 0.f;
  for (int k = 0; k < K; ++k) s = fmaf(A[r * K + k], B[c * K + k], s);
  C[i] = s;
}

int main(int argc, char** argv) {
  const int Ks[] = {64, 256, 1024, 4096};
  for (int dist = 0; dist < 2; ++dist) {
    for (int K : Ks) {
      std::mt19937 rng(1234 + K);
      std::normal_distribution<float> nd(0.f, 1.f);
      std::uniform_real_distribution<float> ud(0.f, 1.f);
      std::vector<float> A(BM * K), B(BN * K);
      // dist 0: N(0,1) both; dist 1: post-ReLU activations (>= 0) x N(0,1) weights
      for (auto& v : A) v = dist ? fmaxf(nd(rng), 0.f) : nd(rng);
      for (auto& v : B) v = nd(rng);
      std::vector<double> ref(BM * BN), mag(BM * BN);
      for (int r = 0; r < BM; ++r)
        for (int c = 0; c < BN; ++c) {
          double s = 0, m = 0;
          for (int k = 0; k < K; ++k) {
            s += (double)A[r * K + k] * B[c * K + k];
            m += fabs((double)A[r * K + k] * B[c * K + k]);
          }
          ref[r * BN + c] = s;
          mag[r * BN + c] = m;
        }
      float *dA, *dB, *dC;
      cudaMalloc(&dA, A.size() * 4);
      cudaMalloc(&dB, B.size() * 4);
      cudaMalloc(&dC, BM * BN * 4);
      cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
      std::vector<float> C(BM * BN);
      for (int mode = 0; mode <= 4; ++mode) {
        if (mode < 4)
          tc_kernel<<<1, 128>>>(dA, dB, dC, K, mode);
        else
          ffma_kernel<<<(BM * BN + 127) / 128, 128>>>(dA, dB, dC, K);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("mode %d: %s\n", mode, cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double maxrel = 0, bias = 0, rms = 0, maxabs = 0;
        for (int i = 0; i < BM * BN; ++i) {
          const double d = C[i] - ref[i];
          maxrel = fmax(maxrel, fabs(d) / mag[i]);
          maxabs = fmax(maxabs, fabs(d));
          bias += (ref[i] >= 0 ? d : -d) / mag[i];  // signed toward-|ref| error
          rms += (d / mag[i]) * (d / mag[i]);
        }
        printf("dist %d K %5d mode %d: max|err|/sum|ab| %.3e  rms %.3e  bias(away from 0) %+.3e  max|err| %.3e\n", dist,
               K, mode, maxrel, sqrt(rms / (BM * BN)), bias / (BM * BN), maxabs);
      }
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dC);
    }
  }
  return 0;
}
