// Calibration of the per-node floor of a captured CUDA graph on this GPU.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mb tools/microbench.cu
// Chains of N dependent kernel nodes: empty, 1-load/1-store per thread
// (L2-resident), with and without programmatic dependent launch; plus a
// k-way fan-out/fan-in on separate streams.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void k_empty() {}

__global__ void k_touch(const float* __restrict__ in, float* __restrict__ out, int n) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] * 1.0001f + 1.f;
}

// dependent chain of 8 loads per thread (serialized latency probe)
__global__ void k_chain(const int* __restrict__ idx, int* __restrict__ out, int steps) {
  int j = threadIdx.x;
  for (int s = 0; s < steps; ++s) j = idx[j];
  out[threadIdx.x] = j;
}

static float time_graph(cudaGraphExec_t ex, cudaStream_t st, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ex, st);
  cudaEventRecord(a, st);
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ex, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const int N = 200;
  float *bufA, *bufB;
  cudaMalloc(&bufA, 1 << 24);
  cudaMalloc(&bufB, 1 << 24);
  cudaMemset(bufA, 0, 1 << 24);
  for (int variant = 0; variant < 6; ++variant) {
    int blocks = (variant % 2 == 0) ? 1 : 100;
    bool touch = variant >= 2;
    bool pdl = variant >= 4;
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) {
      if (!touch) {
        k_empty<<<blocks, 128, 0, st>>>();
      } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(128);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        const float* in = (i % 2) ? bufA : bufB;
        float* out = (i % 2) ? bufB : bufA;
        cudaLaunchKernelEx(&cfg, k_touch, in, out, blocks * 128);
      }
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ex;
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
      printf("instantiate failed %d\n", variant);
      continue;
    }
    float us = time_graph(ex, st, 50);
    printf("chain of %d nodes: blocks=%d touch=%d pdl=%d : %.2f us/node\n", N, blocks, touch, pdl, us / N);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
  }
  // serialized DRAM/L2 latency probe
  {
    int* idx;
    int* out;
    cudaMalloc(&idx, 1 << 20);
    cudaMalloc(&out, 4096);
    std::vector<int> h(1 << 18);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (int)((i * 7919 + 13) % h.size());
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int steps : {1, 65}) {
      k_chain<<<1, 32, 0, st>>>(idx, out, steps);
      cudaEventRecord(a, st);
      k_chain<<<1, 32, 0, st>>>(idx, out, steps);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("dependent-load chain steps=%d: %.2f us\n", steps, ms * 1000.f);
    }
  }
  // fan-out / fan-in across streams inside a graph
  for (int width : {1, 4, 16}) {
    std::vector<cudaStream_t> ss(width);
    std::vector<cudaEvent_t> ev(width);
    for (int i = 0; i < width; ++i) {
      cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking);
      cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    cudaEvent_t fork;
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int layer = 0; layer < 50; ++layer) {
      cudaEventRecord(fork, st);
      for (int i = 0; i < width; ++i) {
        cudaStreamWaitEvent(ss[i], fork, 0);
        k_touch<<<8, 128, 0, ss[i]>>>(bufA + i * 4096, bufB + i * 4096, 1024);
        cudaEventRecord(ev[i], ss[i]);
        cudaStreamWaitEvent(st, ev[i], 0);
      }
    }
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ex;
    cudaGraphInstantiate(&ex, g, 0);
    float us = time_graph(ex, st, 50);
    printf("50 layers x %d parallel nodes: %.2f us/layer\n", width, us / 50);
  }
  return 0;
}
