// Elementwise and reduction kernels (HBM-bound).
//
// K_ELTWISE: out = act(op(a, b, c)) over N x H x W x C with independent
// 4-D strides per operand — stride 0 broadcasts (SE channel scale, per-
// channel affine), channel-slice strides make concat zero-copy, and EW_COPY
// doubles as the strided concat / layout fallback.  128-bit path when every
// operand is channel-contiguous and aligned.
// K_GLOBAL_POOL: mean over H x W per (n, c); one thread per 4 channels,
// consecutive threads on consecutive channels (coalesced NHWC reads).
#include "common.cuh"

namespace sw {

struct EwArgs {
  const float* a;
  const float* b;
  const float* c;
  float* out;
  const float* scale;
  const float* shift;
  int N, H, W, C, op, act, nin, pre_relu;
  int64_t as[4], bs[4], cs[4], os[4];
};

static EwArgs ew_args(const sw_op_desc& d) {
  const int64_t* p = d.params;
  EwArgs e;
  e.a = reinterpret_cast<const float*>(d.ptrs[EP_A]);
  e.b = reinterpret_cast<const float*>(d.ptrs[EP_B]);
  e.c = reinterpret_cast<const float*>(d.ptrs[EP_C]);
  e.out = reinterpret_cast<float*>(d.ptrs[EP_OUT]);
  e.scale = reinterpret_cast<const float*>(d.ptrs[EP_SCALE]);
  e.shift = reinterpret_cast<const float*>(d.ptrs[EP_SHIFT]);
  e.N = (int)p[EW_N]; e.H = (int)p[EW_H]; e.W = (int)p[EW_W]; e.C = (int)p[EW_C];
  e.op = (int)p[EW_OP]; e.act = (int)p[EW_ACT]; e.nin = (int)p[EW_NIN]; e.pre_relu = (int)p[EW_PRE_RELU];
  for (int i = 0; i < 4; ++i) {
    e.as[i] = p[EW_A_SN + i];
    e.bs[i] = p[EW_B_SN + i];
    e.cs[i] = p[EW_C_SN + i];
    e.os[i] = p[EW_O_SN + i];
  }
  return e;
}

__device__ __forceinline__ int64_t off4(const int64_t* s, int n, int h, int w, int c) {
  return n * s[0] + h * s[1] + w * s[2] + c * s[3];
}

__device__ __forceinline__ float ew_combine(const EwArgs& e, float x, float y, float z, int c) {
  float v;
  switch (e.op) {
    case EW_ADD: v = x + (e.nin > 1 ? y : 0.f) + (e.nin > 2 ? z : 0.f); break;
    case EW_MUL: v = x * y; break;
    case EW_AFFINE: v = x * e.scale[c] + e.shift[c]; break;
    default: v = x; break;
  }
  return apply_act(v, e.act);
}

__global__ void __launch_bounds__(256) ew_scalar_kernel(EwArgs e, int64_t total) {
  pdl_trigger();
  pdl_wait();
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int c = (int)(idx % e.C);
  int64_t t = idx / e.C;
  int w = (int)(t % e.W);
  t /= e.W;
  int h = (int)(t % e.H);
  int n = (int)(t / e.H);
  float x = e.a[off4(e.as, n, h, w, c)];
  if (e.pre_relu) x = fmaxf(x, 0.f);
  float y = e.nin > 1 ? e.b[off4(e.bs, n, h, w, c)] : 0.f;
  float z = e.nin > 2 ? e.c[off4(e.cs, n, h, w, c)] : 0.f;
  e.out[off4(e.os, n, h, w, c)] = ew_combine(e, x, y, z, c);
}

__global__ void __launch_bounds__(256) ew_vec4_kernel(EwArgs e, int64_t total) {
  pdl_trigger();
  pdl_wait();
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int CG = e.C / 4;
  int c = (int)(idx % CG) * 4;
  int64_t t = idx / CG;
  int w = (int)(t % e.W);
  t /= e.W;
  int h = (int)(t % e.H);
  int n = (int)(t / e.H);
  float4 x = __ldg(reinterpret_cast<const float4*>(e.a + off4(e.as, n, h, w, c)));
  if (e.pre_relu) {
    x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
  }
  float4 y = make_float4(0.f, 0.f, 0.f, 0.f), z = y;
  if (e.nin > 1) y = __ldg(reinterpret_cast<const float4*>(e.b + off4(e.bs, n, h, w, c)));
  if (e.nin > 2) z = __ldg(reinterpret_cast<const float4*>(e.c + off4(e.cs, n, h, w, c)));
  float4 o;
  o.x = ew_combine(e, x.x, y.x, z.x, c);
  o.y = ew_combine(e, x.y, y.y, z.y, c + 1);
  o.z = ew_combine(e, x.z, y.z, z.z, c + 2);
  o.w = ew_combine(e, x.w, y.w, z.w, c + 3);
  *reinterpret_cast<float4*>(e.out + off4(e.os, n, h, w, c)) = o;
}

static bool ew_vec_ok(const EwArgs& e, const sw_op_desc& d) {
  if (e.C % 4) return false;
  const int64_t* ss[4] = {e.as, e.bs, e.cs, e.os};
  const uint64_t ps[4] = {d.ptrs[EP_A], d.ptrs[EP_B], d.ptrs[EP_C], d.ptrs[EP_OUT]};
  for (int i = 0; i < 4; ++i) {
    if (i >= 1 && i <= 2 && e.nin <= i) continue;
    const int64_t* s = ss[i];
    if (s[3] != 1 || s[0] % 4 || s[1] % 4 || s[2] % 4 || !aligned16(ps[i])) return false;
  }
  return true;
}

int launch_eltwise(const sw_op_desc& d, void* stream) {
  EwArgs e = ew_args(d);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  bool v4 = ew_vec_ok(e, d);
  int64_t total = (int64_t)e.N * e.H * e.W * (v4 ? e.C / 4 : e.C);
  if (total == 0) return 0;
  int blocks = (int)cdiv(total, 256);
  if (v4) return (int)launch_k(ew_vec4_kernel, dim3(blocks), dim3(256), 0, st, 1, e, total);
  return (int)launch_k(ew_scalar_kernel, dim3(blocks), dim3(256), 0, st, 1, e, total);
}

// Global average pool: out[n, c] = mean_hw(relu?(a[n, h, w, c])).
// One warp per (n, 4-channel group): lanes stride over the H*W pixels with
// 128-bit loads (all in flight at once), then a shuffle tree reduces.
__global__ void __launch_bounds__(256) global_pool_vec4_kernel(EwArgs e) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int groups = e.C / 4;
  if (warp >= e.N * groups) return;
  const int n = warp / groups;
  const int c = (warp % groups) * 4;
  const int hw = e.H * e.W;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* base = e.a + n * e.as[0] + c;
#pragma unroll 4
  for (int i = lane; i < hw; i += 32) {
    int h = i / e.W, w = i % e.W;
    float4 x = __ldg(reinterpret_cast<const float4*>(base + h * e.as[1] + w * e.as[2]));
    if (e.pre_relu) {
      x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
    }
    acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    acc.z += __shfl_xor_sync(0xffffffffu, acc.z, o);
    acc.w += __shfl_xor_sync(0xffffffffu, acc.w, o);
  }
  if (lane == 0) {
    const float inv = 1.f / (float)hw;
    float* o = e.out + n * e.os[0];
    o[(c + 0) * e.os[3]] = apply_act(acc.x * inv, e.act);
    o[(c + 1) * e.os[3]] = apply_act(acc.y * inv, e.act);
    o[(c + 2) * e.os[3]] = apply_act(acc.z * inv, e.act);
    o[(c + 3) * e.os[3]] = apply_act(acc.w * inv, e.act);
  }
}

__global__ void __launch_bounds__(128) global_pool_kernel(EwArgs e) {
  pdl_trigger();
  pdl_wait();
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  int n = blockIdx.y;
  if (c >= e.C) return;
  float acc = 0.f;
  const float* base = e.a + n * e.as[0] + c * e.as[3];
  for (int h = 0; h < e.H; ++h)
#pragma unroll 4
    for (int w = 0; w < e.W; ++w) {
      float x = __ldg(base + h * e.as[1] + w * e.as[2]);
      acc += e.pre_relu ? fmaxf(x, 0.f) : x;
    }
  acc /= (float)(e.H * e.W);
  e.out[n * e.os[0] + c * e.os[3]] = apply_act(acc, e.act);
}

int launch_global_pool(const sw_op_desc& d, void* stream) {
  EwArgs e = ew_args(d);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (e.N == 0 || e.C == 0) return 0;
  const bool v4 = e.C % 4 == 0 && e.as[3] == 1 && e.as[0] % 4 == 0 && e.as[1] % 4 == 0 && e.as[2] % 4 == 0 &&
                  aligned16(d.ptrs[EP_A]);
  if (v4) {
    int64_t warps = (int64_t)e.N * (e.C / 4);
    return (int)launch_k(global_pool_vec4_kernel, dim3((unsigned)cdiv(warps * 32, 256)), dim3(256), 0, st, 1, e);
  }
  dim3 grid((unsigned)cdiv(e.C, 128), (unsigned)e.N);
  return (int)launch_k(global_pool_kernel, grid, dim3(128), 0, st, 1, e);
}

}  // namespace sw

namespace sw {

// Unfused concat (fuse=False programs only): one launch copies up to 7 dense
// NHWC inputs into their channel slices of the output.
struct ConcatArgs {
  const float* in[7];
  float* out;
  int c_in[7];
  int c_off[8];
  int N, H, W, nin, ctot;
  int64_t out_sc, out_sp;  // output channel stride, pixel stride
  int64_t hw;
};

__global__ void __launch_bounds__(256) concat_kernel(ConcatArgs a, int64_t total) {
  pdl_trigger();
  pdl_wait();
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int c = (int)(idx % a.ctot);
  int64_t pix = idx / a.ctot;  // n*H*W + h*W + w
  int i = 0;
  while (i + 1 < a.nin && c >= a.c_off[i + 1]) ++i;
  int cl = c - a.c_off[i];
  float v = a.in[i][pix * a.c_in[i] + cl];
  int64_t n = pix / a.hw, hw = pix % a.hw;
  int64_t dst = (a.out_sc == 1) ? pix * a.out_sp + c : n * (int64_t)a.ctot * a.hw + c * a.out_sc + hw;
  a.out[dst] = v;
}

int launch_concat(const sw_op_desc& d, void* stream) {
  const int64_t* p = d.params;
  ConcatArgs a;
  a.N = (int)p[0]; a.H = (int)p[1]; a.W = (int)p[2]; a.nin = (int)p[3]; a.ctot = (int)p[4];
  a.out_sc = p[5] ? p[5] : 1;
  a.out_sp = p[6] ? p[6] : a.ctot;
  a.hw = (int64_t)a.H * a.W;
  if (a.nin < 1 || a.nin > 7) return (int)cudaErrorInvalidValue;
  int off = 0;
  for (int i = 0; i < a.nin; ++i) {
    a.in[i] = reinterpret_cast<const float*>(d.ptrs[i]);
    a.c_in[i] = (int)p[8 + i];
    a.c_off[i] = off;
    off += a.c_in[i];
  }
  a.c_off[a.nin] = off;
  a.out = reinterpret_cast<float*>(d.ptrs[7]);
  int64_t total = (int64_t)a.N * a.hw * a.ctot;
  if (total == 0) return 0;
  return (int)launch_k(concat_kernel, dim3((unsigned)cdiv(total, 256)), dim3(256), 0,
                       reinterpret_cast<cudaStream_t>(stream), 1, a, total);
}

// Diagnostic (SW_ENGINE_NULL_KERNELS): an empty task with the same PDL
// protocol, so a replay of the captured topology measures the graph's own
// issue / dependency floor.
__global__ void null_task_kernel() {
  pdl_trigger();
  pdl_wait();
}

int launch_null(void* stream) {
  return (int)launch_k(null_task_kernel, dim3(1), dim3(32), 0, reinterpret_cast<cudaStream_t>(stream), 1);
}

// Host <-> device staging as a kernel node (SW_ENGINE_KERNEL_IO): the pinned
// host buffer is read / written through its UVA mapping with 16-byte accesses,
// every SM keeping several in flight.  A captured cudaMemcpy node cost ~150 µs
// of graph time for NASNet's 602 KB input + 4 KB output (tools/e2e_breakdown.py).
__global__ void __launch_bounds__(256) io_copy_kernel(const float4* __restrict__ src, float4* __restrict__ dst,
                                                      int64_t n16, const float* __restrict__ src_tail,
                                                      float* __restrict__ dst_tail, int tail) {
  pdl_trigger();
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n16; i += stride) dst[i] = src[i];
  if (blockIdx.x == 0 && (int)threadIdx.x < tail) dst_tail[threadIdx.x] = src_tail[threadIdx.x];
}

static void io_geometry(int64_t bytes, int64_t* n16, int* tail, unsigned* blocks) {
  *n16 = bytes / 16;
  *tail = (int)((bytes % 16) / 4);
  int64_t b = cdiv(*n16, 256);  // one float4 per thread: PCIe reads spread over every SM
  if (b < 1) b = 1;
  if (b > 148 * 4) b = 148 * 4;
  *blocks = (unsigned)b;
}

// Re-point a captured staging-copy node of an instantiated graph (same size,
// other host buffer): a pinned caller buffer is then read / written in place,
// with no host-side memcpy through the engine's staging buffer.
int set_io_copy_node(void* exec, void* node, void* dst, const void* src, int64_t bytes) {
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return (int)cudaErrorMisalignedAddress;
  int64_t n16;
  int tail;
  unsigned blocks;
  io_geometry(bytes, &n16, &tail, &blocks);
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  const float* st = reinterpret_cast<const float*>(src) + n16 * 4;
  float* dt = reinterpret_cast<float*>(dst) + n16 * 4;
  void* args[] = {&s4, &d4, &n16, &st, &dt, &tail};
  cudaKernelNodeParams kp = {};
  kp.func = reinterpret_cast<void*>(io_copy_kernel);
  kp.gridDim = dim3(blocks);
  kp.blockDim = dim3(256);
  kp.sharedMemBytes = 0;
  kp.kernelParams = args;
  kp.extra = nullptr;
  return (int)cudaGraphExecKernelNodeSetParams(reinterpret_cast<cudaGraphExec_t>(exec),
                                               reinterpret_cast<cudaGraphNode_t>(node), &kp);
}

// L2 warm-up of the packed parameters (SW_ENGINE_L2_PREFETCH): a root node of
// the captured graph on its own stream streams every 128-B line of the
// weights into L2 (evict_last) while the first layers run, so later kernels'
// constant fetches (issued before their PDL wait) hit L2 instead of HBM.
__global__ void __launch_bounds__(256) l2_prefetch_kernel(const char* __restrict__ p, int64_t lines) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lines; i += (int64_t)gridDim.x * blockDim.x)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p + i * 128) : "memory");
}

int launch_l2_prefetch(const void* p, int64_t bytes, void* stream) {
  const int64_t lines = (bytes + 127) / 128;
  if (lines <= 0) return 0;
  int64_t blocks = cdiv(lines, 256 * 4);
  if (blocks > 148 * 2) blocks = 148 * 2;
  l2_prefetch_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const char*>(p), lines);
  return (int)cudaPeekAtLastError();
}

int launch_io_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return 0;
  if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) return (int)cudaErrorMisalignedAddress;
  int64_t n16;
  int tail;
  unsigned blocks;
  io_geometry(bytes, &n16, &tail, &blocks);
  const float* st = reinterpret_cast<const float*>(src) + n16 * 4;
  float* dt = reinterpret_cast<float*>(dst) + n16 * 4;
  return (int)launch_k(io_copy_kernel, dim3(blocks), dim3(256), 0, reinterpret_cast<cudaStream_t>(stream), 1,
                       reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), n16, st, dt, tail);
}

}  // namespace sw
