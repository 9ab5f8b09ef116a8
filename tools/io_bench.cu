// H2D staging microbenchmark: a kernel reading pinned host memory through its
// UVA mapping (the engine's io_copy node) at several grid shapes vs DMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/io_bench tools/io_bench.cu && /tmp/io_bench
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

template <int U>
__global__ void copy_k(const float4* __restrict__ s, float4* __restrict__ d, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = s[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) d[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) d[i] = s[i];
}

template <int U>
float run(const float4* h, float4* dd, int64_t n, int blocks, int threads, cudaStream_t st) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int r = 0; r < 20; ++r) copy_k<U><<<blocks, threads, 0, st>>>(h, dd, n);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEventRecord(a, st);
  for (int it = 0; it < 20; ++it) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return ms * 1000.f / 400.f;
}

// stem-conv access pattern straight from pinned host memory (UVA): NCHW 3 x 224 x 224,
// 3x3 stride 2, one thread per output pixel summing its 27 taps (reads only)
__global__ void stem_read_k(const float* __restrict__ x, float* __restrict__ y, int H, int W, int P, int Q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P * Q) return;
  const int p = i / Q, q = i % Q;
  float acc = 0.f;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int h = 2 * p + r, w = 2 * q + s;
        if (h < H && w < W) acc += x[(c * H + h) * W + w];
      }
  y[i] = acc;
}

int main() {
  const int64_t bytes = 602112, n = bytes / 16;
  float4 *h, *dd;
  cudaMallocHost(&h, bytes);
  cudaMalloc(&dd, bytes);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int grids[] = {37, 74, 148, 296, 592, 1184};
  const int thr[] = {128, 256, 512};
  for (int t : thr)
    for (int gsz : grids) {
      printf("threads %3d blocks %4d : U1 %6.2f us  U4 %6.2f us  U8 %6.2f us\n", t, gsz,
             run<1>(h, dd, n, gsz, t, st), run<4>(h, dd, n, gsz, t, st), run<8>(h, dd, n, gsz, t, st));
    }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 5; ++w) cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice, st);
  cudaEventRecord(a, st);
  for (int it = 0; it < 100; ++it) cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("DMA cudaMemcpyAsync back-to-back: %.2f us per copy (%.1f GB/s)\n", ms * 10.f, bytes / (ms * 10.f) / 1e3);
  // single-shot latency (one copy, idle GPU before and after)
  for (int gsz : {37, 148, 592}) {
    float tot = 0.f;
    for (int it = 0; it < 50; ++it) {
      cudaStreamSynchronize(st);
      cudaEventRecord(a, st);
      copy_k<1><<<gsz, 256, 0, st>>>(h, dd, n);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float m1;
      cudaEventElapsedTime(&m1, a, b);
      tot += m1;
    }
    printf("single-shot kernel copy, %d blocks: %.2f us\n", gsz, tot * 1000.f / 50);
  }
  {
    float tot = 0.f;
    for (int it = 0; it < 50; ++it) {
      cudaStreamSynchronize(st);
      cudaEventRecord(a, st);
      cudaMemcpyAsync(dd, h, bytes, cudaMemcpyHostToDevice, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float m1;
      cudaEventElapsedTime(&m1, a, b);
      tot += m1;
    }
    printf("single-shot DMA copy: %.2f us\n", tot * 1000.f / 50);
  }
  for (int dev_src = 0; dev_src < 2; ++dev_src) {
    const float* src = dev_src ? reinterpret_cast<const float*>(dd) : reinterpret_cast<const float*>(h);
    float* yo = nullptr;
    cudaMalloc(&yo, 111 * 111 * 4);
    float tot = 0.f;
    for (int it = 0; it < 50; ++it) {
      cudaStreamSynchronize(st);
      cudaEventRecord(a, st);
      stem_read_k<<<(111 * 111 + 255) / 256, 256, 0, st>>>(src, yo, 224, 224, 111, 111);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float m1;
      cudaEventElapsedTime(&m1, a, b);
      tot += m1;
    }
    printf("stem-pattern read from %s: %.2f us\n", dev_src ? "device (HBM/L2)" : "pinned host (UVA)", tot * 1000.f / 50);
    cudaFree(yo);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
