// Device runtime of the AoT engine (include/streamweave_b200.h, group 2).
//
// The pre_run schedule (schedule.py:53-115: per-stream FIFOs of LAUNCH /
// RECORD / WAIT in a global capture order) is realised op for op under CUDA
// stream capture:
//   origin stream:  [H2D input memcpy] → fork event
//   logical stream s (one cudaStream_t each): wait(fork) → its FIFO, where
//       LAUNCH t   = kernel of op t,
//       RECORD e   = cudaEventRecord(event e)      (one event per sync edge),
//       WAIT e     = cudaStreamWaitEvent(event e)
//   → join event per stream → origin waits all → [D2H output memcpy]
// and instantiated once into a cudaGraphExec_t.  Replay is one
// cudaGraphLaunch: no per-op host scheduling remains (the paper's point).
// The captured edge set is exactly MEG edges (stream-order edges for matched
// edges, event edges for sync edges) + memcpy→stream heads + stream
// tails→memcpy; sw_engine_graph_topology exposes it for that check.
#include <cuda_runtime.h>

#include <dlfcn.h>
#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../planner/planner.h"
#include "ops.h"

#ifdef SW_PROBE
#include "../kernels/probe.cuh"

namespace sw {
static std::vector<ProbeFn>& probe_registry() {
  static std::vector<ProbeFn> r;
  return r;
}
int probe_register(ProbeFn fn) {
  probe_registry().push_back(fn);
  return 0;
}
}  // namespace sw

// Diagnostic build only (not in include/): zero every kernel TU's probe
// buffer / read back the one that saw launches as 64 uint64:
// [0,16) phase points, [16,32) first-CTA start per launch, [32,48) last-CTA
// end per launch, [48] CTAs started, [49] CTAs finished.
extern "C" int sw_probe_reset() {
  for (auto fn : sw::probe_registry()) fn(nullptr, true);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
// out: 128 words — pt[16], start[16], end[16], started, finished, ..., trace[64] at 64
extern "C" int sw_probe_read(uint64_t* out) {
  for (int i = 0; i < 128; ++i) out[i] = 0;
  for (auto fn : sw::probe_registry()) {
    sw::ProbeBuf b;
    fn(&b, false);
    if (b.started == 0) continue;
    for (int i = 0; i < 16; ++i) {
      out[i] = b.pt[i];
      out[16 + i] = b.start[i];
      out[32 + i] = b.end[i];
    }
    out[48] = b.started;
    out[49] = b.finished;
    for (int i = 0; i < 64; ++i) out[64 + i] = b.trace[i];
  }
  return 0;
}
#endif

namespace sw {
thread_local bool g_launch_pdl = false;
thread_local int g_launch_priority = 0;
}

namespace {

// SW_SEGV_TRACE=1: print the native stack of a segmentation fault (debugging aid)
void segv_trace(int sig) {
  void* fr[64];
  const int n = backtrace(fr, 64);
  backtrace_symbols_fd(fr, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}
struct SegvTraceInit {
  SegvTraceInit() {
    if (getenv("SW_SEGV_TRACE")) signal(SIGSEGV, segv_trace);
  }
} segv_trace_init;

constexpr int kSlots = 4;

struct Slot {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::unordered_map<cudaGraphNode_t, int64_t> node_task;
  std::unordered_set<cudaGraphNode_t> io_nodes;  // kernel-node staging copies
  cudaGraphNode_t io_in = nullptr, io_out = nullptr;  // the main input / output staging nodes
  bool io_in_custom = false, io_out_custom = false;  // re-pointed at a caller buffer
  const void* io_in_ptr = nullptr;                    // the caller buffer it points at
  bool with_io = false;                               // captured with host staging copies
  int64_t xpdl_edges = 0;                             // task edges re-typed programmatic
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    node_task.clear();
    io_nodes.clear();
    io_in = io_out = nullptr;
    with_io = false;
    io_in_custom = io_out_custom = false;
    io_in_ptr = nullptr;
    xpdl_edges = 0;
  }
};

}  // namespace

struct sw_engine {
  int device = 0;
  cudaStream_t launch = nullptr;
  std::vector<cudaStream_t> streams;  // logical stream pool (capture)
  std::vector<cudaEvent_t> events;    // one per sync edge (schedule.py:71)
  std::vector<cudaEvent_t> joins;
  cudaEvent_t fork = nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  std::vector<sw_op_desc> ops;
  std::vector<int32_t> prio;  // per-task launch priority (sw_engine_set_priorities)
  uint64_t host_in = 0, dev_in = 0, host_out = 0, dev_out = 0;
  // request pipelining (sw_engine_infer_stream): double-buffered device
  // staging of the inputs, filled on a copy stream under the running replay
  void* stage[2] = {nullptr, nullptr};
  cudaStream_t cstream = nullptr;
  cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_done[2] = {nullptr, nullptr};
  int64_t in_bytes = 0, out_bytes = 0;
  uint32_t flags = 0;  // SW_ENGINE_PDL | SW_ENGINE_NULL_KERNELS
  Slot slots[kSlots];
  // extra captured H2D copies (training: labels next to the images)
  std::vector<uint64_t> extra_host, extra_dev;
  std::vector<int64_t> extra_bytes;
  uint64_t prefetch_ptr = 0;  // SW_ENGINE_L2_PREFETCH range
  int64_t prefetch_bytes = 0;
  cudaStream_t pf_stream = nullptr;
  cudaEvent_t pf_join = nullptr;
  void* nccl_comm = nullptr;  // ncclComm_t of the data-parallel group (K_ALLREDUCE)
  // SW_ENGINE_TRACE: timing events around every task (measured Chrome trace)
  std::vector<cudaEvent_t> tr_start, tr_end;
  cudaEvent_t tr0 = nullptr;
  int nccl_ranks = 0;
};

// ---------------------------------------------------------------------------
// NCCL, bound at run time (dlopen) so the library still loads — planner only —
// on hosts without NCCL.  Prototypes restate nccl.h (NCCL 2.28, the copy torch
// bundles under site-packages/nvidia/nccl); enum values from that header.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
  typedef int (*GetUniqueId)(void* id);
  typedef int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*CommDestroy)(void*);
  typedef const char* (*ErrStr)(int);
  void* h = nullptr;
  GetUniqueId get_unique_id = nullptr;
  void* comm_init_rank = nullptr;  // by-value ncclUniqueId: called through a struct wrapper
  AllReduce all_reduce = nullptr;
  CommDestroy comm_destroy = nullptr;
  ErrStr err = nullptr;
};
NcclApi g_nccl;
struct NcclId { char internal[128]; };
typedef int (*CommInitRankV)(void** comm, int nranks, NcclId id, int rank);
constexpr int kNcclFloat32 = 7, kNcclAvg = 4;  // ncclFloat32, ncclAvg
}  // namespace

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  return sw::fail(SW_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

#define CU(expr)                                      \
  do {                                                \
    cudaError_t _e = (expr);                          \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
  } while (0)

int launch_task_impl(sw_engine* e, const sw_op_desc& op, cudaStream_t st);

// priority of the task being launched: set around the kernel launcher
int launch_task(sw_engine* e, const sw_op_desc& op, cudaStream_t st) {
  // `op` may be a caller-owned trial descriptor (sw_engine_time_op): compare
  // addresses as integers (pointer subtraction across objects is undefined
  // and was miscompiled into an unchecked load)
  const uintptr_t base = reinterpret_cast<uintptr_t>(e->ops.data());
  const uintptr_t at = reinterpret_cast<uintptr_t>(&op);
  int prio = 0;
  if (!e->prio.empty() && at >= base) {
    const uintptr_t t = (at - base) / sizeof(sw_op_desc);
    if (t < e->prio.size() && at == base + t * sizeof(sw_op_desc)) prio = e->prio[t];
  }
  sw::g_launch_priority = prio;
  const int rc = launch_task_impl(e, op, st);
  sw::g_launch_priority = 0;
  return rc;
}

int launch_task_impl(sw_engine* e, const sw_op_desc& op, cudaStream_t st) {
  int rc = 0;
  switch (op.kind) {
    case sw::K_BN_STATS:
    case sw::K_BN_APPLY:
    case sw::K_BN_BWD_REDUCE:
    case sw::K_BN_BWD_APPLY:
    case sw::K_DW_DGRAD:
    case sw::K_DW_WGRAD:
    case sw::K_GEMM:
    case sw::K_XENT:
    case sw::K_SGD:
    case sw::K_EW_BWD:
    case sw::K_TRANSPOSE:
    case sw::K_GEMM_REDUCE:
    case sw::K_BN_FWD:
    case sw::K_BN_BWD: rc = sw::launch_train(op, st); break;
    case sw::K_ALLREDUCE: {
      if (!e->nccl_comm || !g_nccl.all_reduce) return sw::fail(SW_CUDA_ERROR, "allreduce task without an NCCL communicator");
      int r = g_nccl.all_reduce(reinterpret_cast<const void*>(op.ptrs[0]), reinterpret_cast<void*>(op.ptrs[0]),
                                (size_t)op.params[0], kNcclFloat32, kNcclAvg, e->nccl_comm, st);
      if (r != 0) return sw::fail(SW_CUDA_ERROR, std::string("ncclAllReduce: ") + (g_nccl.err ? g_nccl.err(r) : "?"));
      return SW_OK;
    }
    case sw::K_CONV: rc = sw::launch_conv(op, st); break;
    case sw::K_CONV_TC: rc = sw::launch_conv_tc(op, st); break;
    case sw::K_DWCONV: rc = sw::launch_dwconv(op, st); break;
    case sw::K_POOL: rc = sw::launch_pool(op, st); break;
    case sw::K_ELTWISE: rc = sw::launch_eltwise(op, st); break;
    case sw::K_GLOBAL_POOL: rc = sw::launch_global_pool(op, st); break;
    case sw::K_CONCAT: rc = sw::launch_concat(op, st); break;
    case sw::K_SEPCONV: rc = sw::launch_sepconv(op, st); break;
    case sw::K_SEP2: rc = sw::launch_sep2(op, st); break;
    default: return sw::fail(SW_VALUE_ERROR, "unknown kernel kind " + std::to_string(op.kind));
  }
  if (rc != 0) return cuda_fail((cudaError_t)rc, "kernel launch");
  return SW_OK;
}

int ensure_streams(sw_engine* e, int64_t n) {
  while ((int64_t)e->streams.size() < n) {
    cudaStream_t s;
    CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    e->streams.push_back(s);
    cudaEvent_t j;
    CU(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
    e->joins.push_back(j);
  }
  return SW_OK;
}

int ensure_events(sw_engine* e, int64_t n) {
  while ((int64_t)e->events.size() < n) {
    cudaEvent_t ev;
    CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    e->events.push_back(ev);
  }
  return SW_OK;
}

}  // namespace

extern "C" {

int sw_engine_create(int32_t device, sw_engine** out) {
  auto* e = new sw_engine();
  e->device = device;
  cudaError_t err = cudaSetDevice(device);
  if (err != cudaSuccess) {
    delete e;
    return cuda_fail(err, "cudaSetDevice");
  }
  CU(cudaStreamCreateWithFlags(&e->launch, cudaStreamNonBlocking));
  sw::init_tc_kernels();
  sw::init_tcs_kernels();
  sw::init_pw_tc_kernels();
  sw::init_simt_kernels();
  sw::init_pw_kernels();
  sw::init_sep_kernels();
  sw::init_sep_tc_kernels();
  sw::init_sep_rows_kernels();
  sw::init_sep2_kernels();
  CU(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
  CU(cudaEventCreate(&e->t0));
  CU(cudaEventCreate(&e->t1));
  *out = e;
  return SW_OK;
}

int sw_engine_destroy(sw_engine* e) {
  if (!e) return SW_OK;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->launch);
  for (auto& s : e->slots) s.reset();
  for (auto s : e->streams) cudaStreamDestroy(s);
  for (auto ev : e->events) cudaEventDestroy(ev);
  for (auto ev : e->joins) cudaEventDestroy(ev);
  if (e->pf_stream) cudaStreamDestroy(e->pf_stream);
  for (int i = 0; i < 2; ++i) {
    if (e->stage[i]) cudaFree(e->stage[i]);
    if (e->ev_h2d[i]) cudaEventDestroy(e->ev_h2d[i]);
    if (e->ev_done[i]) cudaEventDestroy(e->ev_done[i]);
  }
  if (e->cstream) cudaStreamDestroy(e->cstream);
  if (e->pf_join) cudaEventDestroy(e->pf_join);
  for (auto ev : e->tr_start) cudaEventDestroy(ev);
  for (auto ev : e->tr_end) cudaEventDestroy(ev);
  if (e->tr0) cudaEventDestroy(e->tr0);
  cudaEventDestroy(e->fork);
  cudaEventDestroy(e->t0);
  cudaEventDestroy(e->t1);
  cudaStreamDestroy(e->launch);
  if (e->nccl_comm && g_nccl.comm_destroy) g_nccl.comm_destroy(e->nccl_comm);
  delete e;
  return SW_OK;
}

int sw_engine_set_ops(sw_engine* e, int64_t n, const sw_op_desc* ops) {
  e->ops.assign(ops, ops + n);
  return SW_OK;
}

int sw_engine_set_io(sw_engine* e, uint64_t host_in, uint64_t dev_in, int64_t in_bytes, uint64_t host_out,
                     uint64_t dev_out, int64_t out_bytes) {
  e->host_in = host_in;
  e->dev_in = dev_in;
  e->in_bytes = in_bytes;
  e->host_out = host_out;
  e->dev_out = dev_out;
  e->out_bytes = out_bytes;
  return SW_OK;
}

// SW_ENGINE_XSTREAM_PDL: re-type every full task -> task kernel edge of a
// captured graph (the plan's cross-stream sync edges; same-stream edges are
// programmatic already when captured with PDL) as a programmatic edge.  Every
// task kernel is launched by launch_k under the PDL protocol — constants
// before griddepcontrol.wait, every dependent read and every write after it —
// so a successor may be resident before its producers finish, exactly as a
// same-stream successor is; the wait covers all of a node's programmatic
// producers.  Edges touching non-task nodes (staging copies, prefetch,
// fork / join) stay full dependencies.
static int programmatic_task_edges(Slot& sl) {
  size_t n = 0;
  CU(cudaGraphGetEdges_v2(sl.graph, nullptr, nullptr, nullptr, &n));
  if (n == 0) return SW_OK;
  std::vector<cudaGraphNode_t> from(n), to(n);
  std::vector<cudaGraphEdgeData> ed(n);
  CU(cudaGraphGetEdges_v2(sl.graph, from.data(), to.data(), ed.data(), &n));
  std::vector<cudaGraphNode_t> rf, rt;
  std::vector<cudaGraphEdgeData> re;
  for (size_t i = 0; i < n; ++i) {
    if (ed[i].type != cudaGraphDependencyTypeDefault) continue;
    if (!sl.node_task.count(from[i]) || !sl.node_task.count(to[i])) continue;
    cudaGraphNodeType tf, tt;
    CU(cudaGraphNodeGetType(from[i], &tf));
    CU(cudaGraphNodeGetType(to[i], &tt));
    if (tf != cudaGraphNodeTypeKernel || tt != cudaGraphNodeTypeKernel) continue;
    rf.push_back(from[i]);
    rt.push_back(to[i]);
    re.push_back(ed[i]);
  }
  if (rf.empty()) return SW_OK;
  CU(cudaGraphRemoveDependencies_v2(sl.graph, rf.data(), rt.data(), re.data(), rf.size()));
  std::vector<cudaGraphEdgeData> pe(rf.size());
  for (auto& x : pe) {
    x = {};
    x.from_port = cudaGraphKernelNodePortProgrammatic;
    x.type = cudaGraphDependencyTypeProgrammatic;
  }
  CU(cudaGraphAddDependencies_v2(sl.graph, rf.data(), rt.data(), pe.data(), rf.size()));
  sl.xpdl_edges = (int64_t)rf.size();
  return SW_OK;
}

int sw_engine_capture(sw_engine* e, int32_t slot, int64_t n_streams, const int64_t* stream_len,
                      const int32_t* op_kind, const int64_t* op_arg, int64_t n_order, const int64_t* order,
                      int32_t with_io) {
  if (slot < 0 || slot >= kSlots) return sw::fail(SW_VALUE_ERROR, "slot out of range");
  CU(cudaSetDevice(e->device));
  Slot& sl = e->slots[slot];
  sl.reset();
  sl.with_io = with_io != 0;
  int rc = ensure_streams(e, n_streams);
  if (rc) return rc;
  int64_t max_event = -1;
  std::vector<int64_t> base(n_streams + 1, 0);
  for (int64_t s = 0; s < n_streams; ++s) base[s + 1] = base[s] + stream_len[s];
  for (int64_t k = 0; k < base[n_streams]; ++k)
    if (op_kind[k] != SW_OP_LAUNCH) max_event = std::max(max_event, op_arg[k]);
    else if (op_arg[k] < 0 || op_arg[k] >= (int64_t)e->ops.size())
      return sw::fail(SW_GRAPH_ERROR, "schedule launches unknown task " + std::to_string(op_arg[k]));
  rc = ensure_events(e, max_event + 1);
  if (rc) return rc;

  const bool trace = (e->flags & SW_ENGINE_TRACE) != 0;
  if (trace) {
    if (!e->tr0) CU(cudaEventCreate(&e->tr0));
    while (e->tr_start.size() < e->ops.size()) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      e->tr_start.push_back(a);
      e->tr_end.push_back(b);
    }
  }
  cudaStream_t origin = e->launch;
  CU(cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal));
  if (trace) {
    cudaError_t te = cudaEventRecordWithFlags(e->tr0, origin, cudaEventRecordExternal);
    if (te != cudaSuccess) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(origin, &g);
      if (g) cudaGraphDestroy(g);
      return cuda_fail(te, "trace t0 record");
    }
  }
  struct PdlScope {
    explicit PdlScope(bool on) { sw::g_launch_pdl = on; }
    ~PdlScope() { sw::g_launch_pdl = false; }
  } pdl_scope((e->flags & SW_ENGINE_PDL) != 0);
  auto abort_capture = [&](int code) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(origin, &g);
    if (g) cudaGraphDestroy(g);
    return code;
  };
  cudaError_t err;
  const bool kio = (e->flags & SW_ENGINE_KERNEL_IO) != 0;
  auto last_node = [&](cudaStream_t st) {
    cudaStreamCaptureStatus status;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    if (cudaStreamGetCaptureInfo(st, &status, nullptr, nullptr, &deps, &ndeps) == cudaSuccess && ndeps == 1)
      sl.io_nodes.insert(deps[0]);
  };
  auto h2d = [&](uint64_t dev, uint64_t host, int64_t bytes) -> cudaError_t {
    if (kio) {
      cudaError_t r = (cudaError_t)sw::launch_io_copy(reinterpret_cast<void*>(dev), reinterpret_cast<const void*>(host),
                                                      bytes, origin);
      if (r == cudaSuccess) last_node(origin);
      return r;
    }
    return cudaMemcpyAsync(reinterpret_cast<void*>(dev), reinterpret_cast<const void*>(host), (size_t)bytes,
                           cudaMemcpyHostToDevice, origin);
  };
  if (with_io && e->in_bytes > 0) {
    err = h2d(e->dev_in, e->host_in, e->in_bytes);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "capture H2D"));
    if (kio) {
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      if (cudaStreamGetCaptureInfo(origin, &cs, nullptr, nullptr, &deps, &nd) == cudaSuccess && nd == 1)
        sl.io_in = deps[0];
    }
  }
  for (size_t i = 0; with_io && i < e->extra_host.size(); ++i) {
    err = h2d(e->extra_dev[i], e->extra_host[i], e->extra_bytes[i]);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "capture extra H2D"));
  }
  err = cudaEventRecord(e->fork, origin);
  if (err != cudaSuccess) return abort_capture(cuda_fail(err, "fork record"));
  const bool prefetch = (e->flags & SW_ENGINE_L2_PREFETCH) && e->prefetch_bytes > 0 && e->pf_stream;
  if (prefetch) {
    err = cudaStreamWaitEvent(e->pf_stream, e->fork, 0);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "prefetch fork"));
    err = (cudaError_t)sw::launch_l2_prefetch(reinterpret_cast<const void*>(e->prefetch_ptr), e->prefetch_bytes,
                                               e->pf_stream);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "prefetch launch"));
    last_node(e->pf_stream);
  }
  for (int64_t s = 0; s < n_streams; ++s) {
    err = cudaStreamWaitEvent(e->streams[s], e->fork, 0);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "fork wait"));
  }
  std::vector<int64_t> cursor(n_streams, 0);
  for (int64_t i = 0; i < n_order; ++i) {
    int64_t s = order[i];
    if (s < 0 || s >= n_streams || cursor[s] >= stream_len[s])
      return abort_capture(sw::fail(SW_VALUE_ERROR, "capture order does not match the stream FIFOs"));
    int64_t k = base[s] + cursor[s]++;
    cudaStream_t st = e->streams[s];
    if (op_kind[k] == SW_OP_LAUNCH) {
      int64_t t = op_arg[k];
      if (trace && (err = cudaEventRecordWithFlags(e->tr_start[t], st, cudaEventRecordExternal)) != cudaSuccess)
        return abort_capture(cuda_fail(err, "trace record"));
      rc = (e->flags & SW_ENGINE_NULL_KERNELS) ? (sw::launch_null(st) ? SW_CUDA_ERROR : 0) : launch_task(e, e->ops[t], st);
      if (rc) return abort_capture(rc);
      cudaStreamCaptureStatus status;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndeps = 0;
      err = cudaStreamGetCaptureInfo(st, &status, nullptr, nullptr, &deps, &ndeps);
      if (err == cudaSuccess && ndeps == 1) sl.node_task[deps[0]] = t;
      if (trace && (err = cudaEventRecordWithFlags(e->tr_end[t], st, cudaEventRecordExternal)) != cudaSuccess)
        return abort_capture(cuda_fail(err, "trace record"));
    } else if (op_kind[k] == SW_OP_RECORD) {
      err = cudaEventRecord(e->events[op_arg[k]], st);
      if (err != cudaSuccess) return abort_capture(cuda_fail(err, "event record"));
    } else {
      err = cudaStreamWaitEvent(st, e->events[op_arg[k]], 0);
      if (err != cudaSuccess) return abort_capture(cuda_fail(err, "event wait"));
    }
  }
  for (int64_t s = 0; s < n_streams; ++s) {
    err = cudaEventRecord(e->joins[s], e->streams[s]);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "join record"));
    err = cudaStreamWaitEvent(origin, e->joins[s], 0);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "join wait"));
  }
  if (prefetch) {
    err = cudaEventRecord(e->pf_join, e->pf_stream);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(origin, e->pf_join, 0);
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "prefetch join"));
  }
  if (with_io && e->out_bytes > 0) {
    err = kio ? (cudaError_t)sw::launch_io_copy(reinterpret_cast<void*>(e->host_out),
                                               reinterpret_cast<const void*>(e->dev_out), e->out_bytes, origin)
              : cudaMemcpyAsync(reinterpret_cast<void*>(e->host_out), reinterpret_cast<const void*>(e->dev_out),
                                (size_t)e->out_bytes, cudaMemcpyDeviceToHost, origin);
    if (kio && err == cudaSuccess) {
      last_node(origin);
      cudaStreamCaptureStatus cs;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      if (cudaStreamGetCaptureInfo(origin, &cs, nullptr, nullptr, &deps, &nd) == cudaSuccess && nd == 1)
        sl.io_out = deps[0];
    }
    if (err != cudaSuccess) return abort_capture(cuda_fail(err, "capture D2H"));
  }
  CU(cudaStreamEndCapture(origin, &sl.graph));
  if ((e->flags & SW_ENGINE_PDL) && (e->flags & SW_ENGINE_XSTREAM_PDL) && !(e->flags & SW_ENGINE_NULL_KERNELS)) {
    if (int r = programmatic_task_edges(sl)) return r;
  }
  CU(cudaGraphInstantiateWithFlags(&sl.exec, sl.graph, 0));
  CU(cudaGraphUpload(sl.exec, e->launch));
  return SW_OK;
}

static int restore_io(sw_engine* e, Slot& sl) {
  if (!sl.io_in_custom) return SW_OK;
  int r = sw::set_io_copy_node(sl.exec, sl.io_in, reinterpret_cast<void*>(e->dev_in),
                               reinterpret_cast<const void*>(e->host_in), e->in_bytes);
  if (r) return cuda_fail((cudaError_t)r, "restore the input staging node");
  sl.io_in_custom = false;
  sl.io_in_ptr = nullptr;
  return SW_OK;
}

int sw_engine_replay(sw_engine* e, int32_t slot) {
  if (slot < 0 || slot >= kSlots || !e->slots[slot].exec) return sw::fail(SW_VALUE_ERROR, "slot not captured");
  if (int r = restore_io(e, e->slots[slot])) return r;
  CU(cudaGraphLaunch(e->slots[slot].exec, e->launch));
  return SW_OK;
}

int sw_engine_replay_sync(sw_engine* e, int32_t slot, int64_t* out_launch_ns) {
  if (slot < 0 || slot >= kSlots || !e->slots[slot].exec) return sw::fail(SW_VALUE_ERROR, "slot not captured");
  if (int r = restore_io(e, e->slots[slot])) return r;
  auto a = std::chrono::steady_clock::now();
  CU(cudaGraphLaunch(e->slots[slot].exec, e->launch));
  auto b = std::chrono::steady_clock::now();
  CU(cudaStreamSynchronize(e->launch));
  if (out_launch_ns) *out_launch_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count();
  return SW_OK;
}

static bool pinned16(const void* p) {
  if (!p || (reinterpret_cast<uint64_t>(p) & 15)) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

int sw_engine_infer(sw_engine* e, int32_t slot, const void* host_in, void* host_out) {
  if (slot < 0 || slot >= kSlots || !e->slots[slot].exec) return sw::fail(SW_VALUE_ERROR, "slot not captured");
  Slot& sl = e->slots[slot];
  // a pinned caller input is read in place by the captured staging kernel
  // (its node re-pointed), a pageable one goes through the pinned staging buffer
  const bool in_direct = sl.io_in && host_in && pinned16(host_in);
  if (in_direct && reinterpret_cast<uint64_t>(host_in) != e->host_in) {
    if (!sl.io_in_custom || sl.io_in_ptr != host_in) {  // a repeat call with the same buffer skips the update
      int r = sw::set_io_copy_node(sl.exec, sl.io_in, reinterpret_cast<void*>(e->dev_in), host_in, e->in_bytes);
      if (r) return cuda_fail((cudaError_t)r, "re-point the input staging node");
      sl.io_in_custom = true;
      sl.io_in_ptr = host_in;
    }
  } else {
    if (sl.io_in_custom) {
      int r = sw::set_io_copy_node(sl.exec, sl.io_in, reinterpret_cast<void*>(e->dev_in),
                                   reinterpret_cast<const void*>(e->host_in), e->in_bytes);
      if (r) return cuda_fail((cudaError_t)r, "restore the input staging node");
      sl.io_in_custom = false;
      sl.io_in_ptr = nullptr;
    }
    if (host_in && reinterpret_cast<uint64_t>(host_in) != e->host_in)
      std::memcpy(reinterpret_cast<void*>(e->host_in), host_in, (size_t)e->in_bytes);
  }
  CU(cudaGraphLaunch(e->slots[slot].exec, e->launch));
  // spin on the stream instead of a blocking synchronize: the wake-up of a
  // yielding wait costs ~15 µs per call (tools/ab_edges.py, cell: 46 µs e2e
  // around 27 µs of device time)
  cudaError_t q;
  while ((q = cudaStreamQuery(e->launch)) == cudaErrorNotReady) {
  }
  if (q != cudaSuccess) return cuda_fail(q, "cudaStreamQuery");
  if (host_out && reinterpret_cast<uint64_t>(host_out) != e->host_out)
    std::memcpy(host_out, reinterpret_cast<const void*>(e->host_out), (size_t)e->out_bytes);
  return SW_OK;
}

// n requests back to back through a device-resident slot (no staging nodes):
// request i+1's H2D runs on a copy stream into the other staging buffer while
// request i replays; each replay starts with a device-to-device copy of its
// staged input into the arena's input storage and ends with the D2H of its
// output.  Same results as n calls of sw_engine_infer; throughput, not latency.
int sw_engine_infer_stream(sw_engine* e, int32_t slot, int64_t n, const uint64_t* host_in, const uint64_t* host_out) {
  if (slot < 0 || slot >= kSlots || !e->slots[slot].exec) return sw::fail(SW_VALUE_ERROR, "slot not captured");
  if (e->slots[slot].with_io) return sw::fail(SW_VALUE_ERROR, "infer_stream needs a device-resident slot");
  if (n > 0 && (!host_in || !host_out)) return sw::fail(SW_VALUE_ERROR, "infer_stream: null buffer list");
  if (n <= 0) return SW_OK;
  CU(cudaSetDevice(e->device));
  if (!e->cstream) {
    CU(cudaStreamCreateWithFlags(&e->cstream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CU(cudaMalloc(&e->stage[i], (size_t)e->in_bytes));
      CU(cudaEventCreateWithFlags(&e->ev_h2d[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&e->ev_done[i], cudaEventDisableTiming));
    }
  }
  const size_t ib = (size_t)e->in_bytes, ob = (size_t)e->out_bytes;
  CU(cudaMemcpyAsync(e->stage[0], reinterpret_cast<const void*>(host_in[0]), ib, cudaMemcpyHostToDevice, e->cstream));
  CU(cudaEventRecord(e->ev_h2d[0], e->cstream));
  for (int64_t i = 0; i < n; ++i) {
    const int b = (int)(i & 1), nb = b ^ 1;
    if (i + 1 < n) {  // stage the next request into the other buffer (freed by replay i - 1)
      if (i >= 1) CU(cudaStreamWaitEvent(e->cstream, e->ev_done[nb], 0));
      CU(cudaMemcpyAsync(e->stage[nb], reinterpret_cast<const void*>(host_in[i + 1]), ib, cudaMemcpyHostToDevice,
                         e->cstream));
      CU(cudaEventRecord(e->ev_h2d[nb], e->cstream));
    }
    CU(cudaStreamWaitEvent(e->launch, e->ev_h2d[b], 0));
    CU(cudaMemcpyAsync(reinterpret_cast<void*>(e->dev_in), e->stage[b], ib, cudaMemcpyDeviceToDevice, e->launch));
    CU(cudaEventRecord(e->ev_done[b], e->launch));
    CU(cudaGraphLaunch(e->slots[slot].exec, e->launch));
    CU(cudaMemcpyAsync(reinterpret_cast<void*>(host_out[i]), reinterpret_cast<const void*>(e->dev_out), ob,
                       cudaMemcpyDeviceToHost, e->launch));
  }
  cudaError_t q;
  while ((q = cudaStreamQuery(e->launch)) == cudaErrorNotReady) {
  }
  if (q != cudaSuccess) return cuda_fail(q, "cudaStreamQuery");
  return SW_OK;
}

int sw_engine_time_replay(sw_engine* e, int32_t slot, int32_t iters, double* out_gpu_us, double* out_host_us) {
  if (slot < 0 || slot >= kSlots || !e->slots[slot].exec) return sw::fail(SW_VALUE_ERROR, "slot not captured");
  if (int r = restore_io(e, e->slots[slot])) return r;
  if (iters < 1) iters = 1;
  CU(cudaStreamSynchronize(e->launch));
  double host_ns = 0;
  CU(cudaEventRecord(e->t0, e->launch));
  for (int i = 0; i < iters; ++i) {
    auto a = std::chrono::steady_clock::now();
    CU(cudaGraphLaunch(e->slots[slot].exec, e->launch));
    auto b = std::chrono::steady_clock::now();
    host_ns += (double)std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count();
  }
  CU(cudaEventRecord(e->t1, e->launch));
  CU(cudaEventSynchronize(e->t1));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e->t0, e->t1));
  *out_gpu_us = (double)ms * 1000.0 / iters;
  *out_host_us = host_ns / 1000.0 / iters;
  return SW_OK;
}

int sw_engine_launch_op(sw_engine* e, int64_t index) {
  if (index < 0 || index >= (int64_t)e->ops.size()) return sw::fail(SW_VALUE_ERROR, "op index out of range");
  sw::g_launch_pdl = (e->flags & SW_ENGINE_PDL) != 0;
  int rc = launch_task(e, e->ops[index], e->launch);
  sw::g_launch_pdl = false;
  return rc;
}

int sw_engine_set_flags(sw_engine* e, uint32_t flags) {
  e->flags = flags;
  return SW_OK;
}

int sw_engine_run_eager(sw_engine* e, int64_t n, const int64_t* order) {
  for (int64_t i = 0; i < n; ++i) {
    int rc = sw_engine_launch_op(e, order[i]);
    if (rc) return rc;
  }
  return SW_OK;
}

// Framework mode on the device (sim.py:69-80 analogue): the same pre_run
// schedule issued op by op by the host every iteration — LAUNCH on the
// logical stream's CUDA stream, RECORD / WAIT as real cudaEventRecord /
// cudaStreamWaitEvent — with no capture.  Forked from / joined back to the
// launch stream like the captured graph.
int sw_engine_run_schedule(sw_engine* e, int64_t n_streams, const int64_t* stream_len, const int32_t* op_kind,
                           const int64_t* op_arg, int64_t n_order, const int64_t* order) {
  int rc = ensure_streams(e, n_streams);
  if (rc) return rc;
  int64_t max_event = -1;
  std::vector<int64_t> base(n_streams + 1, 0);
  for (int64_t s = 0; s < n_streams; ++s) base[s + 1] = base[s] + stream_len[s];
  for (int64_t k = 0; k < base[n_streams]; ++k)
    if (op_kind[k] != SW_OP_LAUNCH) max_event = std::max(max_event, op_arg[k]);
  rc = ensure_events(e, max_event + 1);
  if (rc) return rc;
  sw::g_launch_pdl = (e->flags & SW_ENGINE_PDL) != 0;
  struct Reset {
    ~Reset() { sw::g_launch_pdl = false; }
  } reset;
  CU(cudaEventRecord(e->fork, e->launch));
  for (int64_t s = 0; s < n_streams; ++s) CU(cudaStreamWaitEvent(e->streams[s], e->fork, 0));
  std::vector<int64_t> cursor(n_streams, 0);
  for (int64_t i = 0; i < n_order; ++i) {
    const int64_t s = order[i];
    if (s < 0 || s >= n_streams || cursor[s] >= stream_len[s])
      return sw::fail(SW_VALUE_ERROR, "order does not match the stream FIFOs");
    const int64_t k = base[s] + cursor[s]++;
    cudaStream_t st = e->streams[s];
    if (op_kind[k] == SW_OP_LAUNCH) {
      if (op_arg[k] < 0 || op_arg[k] >= (int64_t)e->ops.size())
        return sw::fail(SW_GRAPH_ERROR, "schedule launches unknown task " + std::to_string(op_arg[k]));
      rc = launch_task(e, e->ops[op_arg[k]], st);
      if (rc) return rc;
    } else if (op_kind[k] == SW_OP_RECORD) {
      CU(cudaEventRecord(e->events[op_arg[k]], st));
    } else {
      CU(cudaStreamWaitEvent(st, e->events[op_arg[k]], 0));
    }
  }
  for (int64_t s = 0; s < n_streams; ++s) {
    CU(cudaEventRecord(e->joins[s], e->streams[s]));
    CU(cudaStreamWaitEvent(e->launch, e->joins[s], 0));
  }
  return SW_OK;
}

int sw_engine_synchronize(sw_engine* e) {
  CU(cudaStreamSynchronize(e->launch));
  CU(cudaGetLastError());
  return SW_OK;
}

int sw_engine_graph_topology(sw_engine* e, int32_t slot, int64_t cap, int64_t* out_n_nodes, int32_t* out_node_kind,
                             int64_t* out_node_task, int64_t* out_n_edges, int64_t* out_edges) {
  if (slot < 0 || slot >= kSlots || !e->slots[slot].graph) return sw::fail(SW_VALUE_ERROR, "slot not captured");
  Slot& sl = e->slots[slot];
  size_t nn = 0;
  CU(cudaGraphGetNodes(sl.graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CU(cudaGraphGetNodes(sl.graph, nodes.data(), &nn));
  std::unordered_map<cudaGraphNode_t, int64_t> idx;
  for (size_t i = 0; i < nn; ++i) idx[nodes[i]] = (int64_t)i;
  *out_n_nodes = (int64_t)nn;
  if ((int64_t)nn > cap) return sw::fail(SW_VALUE_ERROR, "topology buffer too small");
  for (size_t i = 0; i < nn; ++i) {
    cudaGraphNodeType t;
    CU(cudaGraphNodeGetType(nodes[i], &t));
    out_node_kind[i] = t == cudaGraphNodeTypeKernel ? (sl.io_nodes.count(nodes[i]) ? 3 : 0)
                                                    : (t == cudaGraphNodeTypeMemcpy ? 1 : 2);
    auto it = sl.node_task.find(nodes[i]);
    out_node_task[i] = it == sl.node_task.end() ? -1 : it->second;
  }
  // _v2: programmatic (PDL) edges carry edge data; the v1 query is "lossy"
  size_t ne = 0;
  CU(cudaGraphGetEdges_v2(sl.graph, nullptr, nullptr, nullptr, &ne));
  std::vector<cudaGraphNode_t> from(ne), to(ne);
  std::vector<cudaGraphEdgeData> edata(ne);
  if (ne) CU(cudaGraphGetEdges_v2(sl.graph, from.data(), to.data(), edata.data(), &ne));
  *out_n_edges = (int64_t)ne;
  if ((int64_t)ne > cap) return sw::fail(SW_VALUE_ERROR, "topology buffer too small");
  for (size_t i = 0; i < ne; ++i) {
    out_edges[2 * i] = idx[from[i]];
    out_edges[2 * i + 1] = idx[to[i]];
  }
  return SW_OK;
}

int sw_engine_profile_ops(sw_engine* e, int64_t n, const int64_t* order, int32_t reps, double* out_us) {
  // each task timed as a graph-captured chain (see sw_engine_time_op)
  for (int64_t i = 0; i < n; ++i) {
    int rc = sw_engine_time_op(e, &e->ops[order[i]], reps, &out_us[i]);
    if (rc) return rc;
  }
  return SW_OK;
}

int sw_engine_run_op(sw_engine* e, const sw_op_desc* op) {
  CU(cudaStreamSynchronize(e->launch));
  int rc = launch_task(e, *op, e->launch);
  if (rc) return rc;
  CU(cudaStreamSynchronize(e->launch));
  return SW_OK;
}

// Candidates are timed as a chain of `reps` dependent launches inside a
// captured CUDA graph — the way they will run — so microsecond kernels are not
// masked by the host's stream-launch rate (~4 µs per cudaLaunchKernelEx).
int sw_engine_time_op(sw_engine* e, const sw_op_desc* op, int32_t reps, double* out_us) {
  if (reps < 1) reps = 1;
  CU(cudaStreamSynchronize(e->launch));
  int rc = launch_task(e, *op, e->launch);  // validates the launch outside capture
  if (rc) return rc;
  CU(cudaStreamSynchronize(e->launch));
  cudaGraph_t g = nullptr;
  CU(cudaStreamBeginCapture(e->launch, cudaStreamCaptureModeThreadLocal));
  sw::g_launch_pdl = (e->flags & SW_ENGINE_PDL) != 0;  // same edges as the replayed graph
  for (int r = 0; r < reps && rc == 0; ++r) rc = launch_task(e, *op, e->launch);
  sw::g_launch_pdl = false;
  cudaError_t ce = cudaStreamEndCapture(e->launch, &g);
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "time_op capture");
  cudaGraphExec_t ex = nullptr;
  ce = cudaGraphInstantiateWithFlags(&ex, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return cuda_fail(ce, "time_op instantiate");
  ce = cudaGraphLaunch(ex, e->launch);  // warm (code + data into caches)
  if (ce == cudaSuccess) ce = cudaEventRecord(e->t0, e->launch);
  if (ce == cudaSuccess) ce = cudaGraphLaunch(ex, e->launch);
  if (ce == cudaSuccess) ce = cudaEventRecord(e->t1, e->launch);
  if (ce == cudaSuccess) ce = cudaEventSynchronize(e->t1);
  float ms = 0.f;
  if (ce == cudaSuccess) ce = cudaEventElapsedTime(&ms, e->t0, e->t1);
  cudaGraphExecDestroy(ex);
  if (ce != cudaSuccess) return cuda_fail(ce, "time_op replay");
  *out_us = (double)ms * 1000.0 / reps;
  return SW_OK;
}

int sw_engine_set_prefetch(sw_engine* e, uint64_t dev, int64_t bytes) {
  CU(cudaSetDevice(e->device));
  if (!e->pf_stream) {
    CU(cudaStreamCreateWithFlags(&e->pf_stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&e->pf_join, cudaEventDisableTiming));
  }
  e->prefetch_ptr = dev;
  e->prefetch_bytes = bytes;
  return SW_OK;
}

int sw_engine_set_priorities(sw_engine* e, int64_t n, const int32_t* prio) {
  if (n != (int64_t)e->ops.size() && n != 0) return sw::fail(SW_VALUE_ERROR, "one priority per task");
  int least = 0, greatest = 0;
  CU(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  // level k > 0 → k steps more urgent than the default, clamped to the device range
  e->prio.resize(n);
  for (int64_t i = 0; i < n; ++i) e->prio[i] = prio[i] > 0 ? std::max(greatest, least - prio[i]) : 0;
  return SW_OK;
}

int sw_engine_add_input(sw_engine* e, uint64_t host, uint64_t dev, int64_t bytes) {
  e->extra_host.push_back(host);
  e->extra_dev.push_back(dev);
  e->extra_bytes.push_back(bytes);
  return SW_OK;
}

int sw_nccl_load(const char* path) {
  if (g_nccl.h) return SW_OK;
  void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return sw::fail(SW_CUDA_ERROR, std::string("dlopen NCCL: ") + dlerror());
  g_nccl.get_unique_id = (NcclApi::GetUniqueId)dlsym(h, "ncclGetUniqueId");
  g_nccl.comm_init_rank = dlsym(h, "ncclCommInitRank");
  g_nccl.all_reduce = (NcclApi::AllReduce)dlsym(h, "ncclAllReduce");
  g_nccl.comm_destroy = (NcclApi::CommDestroy)dlsym(h, "ncclCommDestroy");
  g_nccl.err = (NcclApi::ErrStr)dlsym(h, "ncclGetErrorString");
  if (!g_nccl.get_unique_id || !g_nccl.comm_init_rank || !g_nccl.all_reduce || !g_nccl.comm_destroy)
    return sw::fail(SW_CUDA_ERROR, "NCCL library lacks the expected symbols");
  g_nccl.h = h;
  return SW_OK;
}

int sw_nccl_unique_id(char* out128) {
  if (!g_nccl.h) return sw::fail(SW_CUDA_ERROR, "NCCL not loaded (sw_nccl_load)");
  int r = g_nccl.get_unique_id(out128);
  if (r != 0) return sw::fail(SW_CUDA_ERROR, std::string("ncclGetUniqueId: ") + (g_nccl.err ? g_nccl.err(r) : "?"));
  return SW_OK;
}

int sw_engine_nccl_init(sw_engine* e, int32_t nranks, int32_t rank, const char* id128) {
  if (!g_nccl.h) return sw::fail(SW_CUDA_ERROR, "NCCL not loaded (sw_nccl_load)");
  CU(cudaSetDevice(e->device));
  NcclId id;
  memcpy(id.internal, id128, 128);
  void* comm = nullptr;
  int r = reinterpret_cast<CommInitRankV>(g_nccl.comm_init_rank)(&comm, nranks, id, rank);
  if (r != 0) return sw::fail(SW_CUDA_ERROR, std::string("ncclCommInitRank: ") + (g_nccl.err ? g_nccl.err(r) : "?"));
  e->nccl_comm = comm;
  e->nccl_ranks = nranks;
  return SW_OK;
}

int sw_engine_trace_read(sw_engine* e, int64_t n, double* out_start_us, double* out_end_us) {
  if (!e->tr0) return sw::fail(SW_VALUE_ERROR, "no traced capture (SW_ENGINE_TRACE)");
  CU(cudaStreamSynchronize(e->launch));
  for (int64_t t = 0; t < n; ++t) {
    out_start_us[t] = out_end_us[t] = -1.0;
    if (t >= (int64_t)e->tr_start.size()) continue;
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, e->tr0, e->tr_start[t]) == cudaSuccess &&
        cudaEventElapsedTime(&b, e->tr0, e->tr_end[t]) == cudaSuccess) {
      out_start_us[t] = 1000.0 * a;
      out_end_us[t] = 1000.0 * b;
    }
  }
  cudaGetLastError();  // never-recorded events leave a sticky-free error
  return SW_OK;
}

int sw_engine_stream(sw_engine* e, uint64_t* out_stream) {
  *out_stream = reinterpret_cast<uint64_t>(e->launch);
  return SW_OK;
}

}  // extern "C"
