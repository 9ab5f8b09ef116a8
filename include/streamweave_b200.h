/*
 * streamweave_b200.h — C ABI of the B200-native Nimble AoT engine.
 *
 * One shared library, paper_2012_02732_b200/libsw_b200.so, exports two groups:
 *
 *   1. sw_plan_*  : the planning path (graph → MEG → Kuhn matching → streams →
 *                   sync plan → pre_run schedule + arena).  Pure host C++,
 *                   bit-exact with the reference package `streamweave`.
 *   2. sw_engine_*: the device runtime: op table of hand-written sm_100a
 *                   kernels, AoT capture of the pre_run schedule into one CUDA
 *                   graph (kernels + memcpys on their assigned streams with
 *                   cudaEvent dependencies), replay, eager per-op launch.
 *
 * Conventions: plain pointers and sizes only; every call returns an int
 * status (0 = ok, else enum sw_status_code) and leaves a one-line detail in a
 * thread-local buffer read by sw_last_error().  Outputs go to caller-sized
 * buffers whose capacities are derivable from the inputs (documented per
 * call).  The planner is reentrant and thread-safe.  Each engine handle is
 * bound to one device and is not re-entrant.
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/streamweave):
 *   graph.py:111   validate_graph            -> sw_plan_validate
 *   graph.py:200   topological_order         -> sw_plan_topological_order
 *   graph.py:251   transitive_closure        -> sw_plan_transitive_closure
 *   graph.py:275   minimum_equivalent_graph  -> sw_plan_minimum_equivalent_graph
 *   graph.py:291   critical_path_time        -> sw_plan_critical_path_time
 *   assign.py:82   maximum_matching          -> sw_plan_maximum_matching
 *   assign.py:105  validate_matching         -> sw_plan_assignment_from_matching (checks)
 *   assign.py:138  assignment_from_matching  -> sw_plan_assignment_from_matching
 *   assign.py:165  is_max_concurrent         -> sw_plan_is_max_concurrent
 *   assign.py:182  min_sync_plan             -> sw_plan_min_sync_plan
 *   assign.py:212  plan_is_safe              -> sw_plan_plan_is_safe
 *   assign.py:233  assign_streams            -> sw_plan_assign_streams
 *   assign.py:243  fold_streams              -> sw_plan_fold_streams
 *   schedule.py:53 pre_run                  -> sw_plan_pre_run
 *   schedule.py:118 reserve_arena            -> sw_plan_reserve_arena
 *   sim.py:64/69 simulate / run_framework_mode -> sw_plan_simulate
 *   oracle.py:30  oracle_plan_is_safe       -> sw_plan_oracle_plan_is_safe
 *   oracle.py:149 min_syncs_brute           -> sw_plan_min_syncs_brute
 *   oracle.py:219 enumerate_assignments     -> sw_plan_enumerate_assignments
 *   oracle.py:271/296 verify_optimal / verify_given -> sw_plan_verify
 *   (the CUDA Stream Capture / Graph Launch step the
 *    package abstracted into TaskSchedule)   -> sw_engine_capture / sw_engine_replay
 */
#ifndef STREAMWEAVE_B200_H
#define STREAMWEAVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: one per StreamWeaveError subclass (errors.py:10-98). */
enum sw_status_code {
  SW_OK = 0,
  SW_GRAPH_ERROR = 1,
  SW_CYCLE_DETECTED = 2,     /* message: witness "a→b→…→a" */
  SW_SELF_LOOP = 3,
  SW_DANGLING_EDGE = 4,
  SW_DUPLICATE_EDGE = 5,
  SW_DUPLICATE_NODE_ID = 6,
  SW_INVALID_MATCHING = 7,
  SW_NOT_MAX_CONCURRENT = 8,
  SW_TOO_LARGE = 9,
  SW_UNSAFE_PLAN = 10,
  SW_UNKNOWN_STREAM = 11,
  SW_FREE_BEFORE_ALLOC = 12,
  SW_DOUBLE_FREE = 13,
  SW_DEADLOCK_DETECTED = 14,
  SW_CAPACITY_EXCEEDED = 15,
  SW_EMPTY_RUN = 16,
  SW_INVALID_SPEC = 17,
  SW_VALUE_ERROR = 18,       /* Python ValueError in the reference */
  SW_KEY_ERROR = 19,         /* Python KeyError in the reference; message = key */
  SW_CUDA_ERROR = 20
};

enum sw_mem_kind { SW_MEM_ALLOC = 0, SW_MEM_FREE = 1 };
enum sw_op_kind { SW_OP_LAUNCH = 0, SW_OP_RECORD = 1, SW_OP_WAIT = 2 };

/* Thread-local detail text of the last failing call (UTF-8, "→" arrows). */
const char* sw_last_error(void);
/* Library version string. */
const char* sw_version(void);

/* A task graph (graph.py:57-108: CompGraph / TaskNode / MemEvent), in the
 * caller's node order and edge order (the reference semantics depend on both). */
typedef struct sw_graph_view {
  int64_t n_nodes;
  const int64_t* ids;
  const int64_t* durations; /* NULL → every duration 1 */
  const int64_t* demands;   /* NULL → every demand 1 */
  const int64_t* mem_start; /* NULL → no mem events; else n_nodes+1 CSR offsets */
  const int32_t* mem_kind;  /* enum sw_mem_kind; any other value = unknown kind */
  const int64_t* mem_arg;   /* alloc: size in bytes; free: index of the alloc */
  int64_t n_edges;
  const int64_t* edges;     /* n_edges (u, v) pairs, flattened */
} sw_graph_view;

/* A stream assignment (assign.py:47-64): dict task id -> stream id, given as
 * parallel arrays in dict iteration order. */
typedef struct sw_assignment_view {
  int64_t n;
  const int64_t* ids;
  const int64_t* streams;
} sw_assignment_view;

/* ---- graph.py ----------------------------------------------------------- */
int sw_plan_validate(const sw_graph_view* g);
/* out_order: n_nodes ids. */
int sw_plan_topological_order(const sw_graph_view* g, int64_t* out_order);
/* Rows by id rank: out_rows[rank(u) * words + k], words = (n_nodes + 63) / 64. */
int sw_plan_transitive_closure(const sw_graph_view* g, uint64_t* out_rows);
/* out_edges: capacity 2*n_edges; sorted kept edges. */
int sw_plan_minimum_equivalent_graph(const sw_graph_view* g, int64_t* out_edges, int64_t* out_n);
int sw_plan_critical_path_time(const sw_graph_view* g, int64_t* out_time);

/* ---- assign.py ---------------------------------------------------------- */
/* Kuhn with pinned scan order; out_pairs capacity 2*min(left, right). */
int sw_plan_maximum_matching(int64_t left_size, int64_t right_size, int64_t n_edges,
                             const int64_t* edges, int64_t* out_pairs, int64_t* out_n);
/* Validates the matching against the MEG bipartite graph, unions pairs, and
 * writes canonical labels: out_ids / out_streams (n_nodes each) in topo order. */
int sw_plan_assignment_from_matching(const sw_graph_view* base, int64_t n_meg,
                                     const int64_t* meg_edges, int64_t n_pairs,
                                     const int64_t* pairs, int64_t* out_ids,
                                     int64_t* out_streams);
int sw_plan_is_max_concurrent(const sw_graph_view* g, const sw_assignment_view* f,
                              int32_t* out_bool);
/* out_plan capacity 2*n_meg. */
int sw_plan_min_sync_plan(const sw_graph_view* base, int64_t n_meg, const int64_t* meg_edges,
                          const sw_assignment_view* f, int64_t* out_plan, int64_t* out_n);
int sw_plan_plan_is_safe(const sw_graph_view* g, const sw_assignment_view* f, int64_t n_plan,
                         const int64_t* plan, int32_t* out_bool);
/* Full pipeline. out_ids/out_streams: n_nodes (topo order); out_sync and
 * out_meg: capacity 2*n_edges each. */
int sw_plan_assign_streams(const sw_graph_view* g, int64_t* out_ids, int64_t* out_streams,
                           int64_t* out_sync, int64_t* out_n_sync, int64_t* out_meg,
                           int64_t* out_n_meg);
/* out_ids/out_streams: n_nodes (topo order). */
int sw_plan_fold_streams(const sw_graph_view* g, const sw_assignment_view* f,
                         int64_t max_streams, int64_t* out_ids, int64_t* out_streams);

/* ---- oracle.py (exhaustive verifiers; compare.py:85-91 with_oracle) ------ */
/* f == NULL: verify_optimal (checks assign_streams' own plan; plan ignored);
 * else verify_given.  out5 = {optimal, algo_syncs, oracle_min,
 * assignments_checked, plan_safe}.  > 7 nodes or > 20 edges: SW_TOO_LARGE. */
int sw_plan_verify(const sw_graph_view* g, const sw_assignment_view* f, int64_t n_plan,
                   const int64_t* plan, int64_t* out5);
/* Path-walking safety predicate (independent of sw_plan_plan_is_safe). */
int sw_plan_oracle_plan_is_safe(const sw_graph_view* g, const sw_assignment_view* f,
                                int64_t n_plan, const int64_t* plan, int32_t* out_bool);
/* Exact smallest safe plan size for f; bound < 0: no bound. */
int sw_plan_min_syncs_brute(const sw_graph_view* g, const sw_assignment_view* f, int64_t bound,
                            int64_t* out);
/* Max-concurrency set partitions in restricted-growth order: out_order =
 * n_nodes topo-ordered ids; out_streams[a * n_nodes + i] = label of
 * out_order[i] in candidate a, for a < cap; *out_count = all candidates. */
int sw_plan_enumerate_assignments(const sw_graph_view* g, int64_t cap, int64_t* out_order,
                                  int64_t* out_streams, int64_t* out_count);

/* ---- schedule.py -------------------------------------------------------- */
/* Caller capacities: ops_cap >= n_nodes + 2*n_plan, streams_cap >= n_nodes,
 * allocs_cap >= number of alloc events in the graph. */
typedef struct sw_schedule_out {
  int64_t* stream_len;      /* [streams_cap] ops per stream */
  int32_t* op_kind;         /* [ops_cap] enum sw_op_kind, stream 0's FIFO first */
  int64_t* op_arg;          /* [ops_cap] task id or event id */
  int64_t* order;           /* [ops_cap] capture order as stream ids */
  int64_t* block_node;      /* [allocs_cap] arena blocks in placement order */
  int64_t* block_index;
  int64_t* block_offset;
  int64_t* block_size;
  int64_t* walk;            /* [n_nodes] canonical topological walk */
  int64_t* task_args_start; /* [n_nodes+1] CSR over walk positions */
  int64_t* task_args;       /* [allocs_cap] arena offsets of each task's allocs */
  int64_t n_streams, n_ops, event_count, arena_total, n_blocks;
} sw_schedule_out;
int sw_plan_pre_run(const sw_graph_view* g, const sw_assignment_view* f, int64_t n_plan,
                    const int64_t* plan, sw_schedule_out* out);

/* First-fit over a linear trace (schedule.py:118-155). Keys are caller
 * integers; out_offset[i] is written for alloc events; on a key error
 * *out_bad_event is the failing event index (for the caller's message). */
int sw_plan_reserve_arena(int64_t n_events, const int64_t* keys, const int32_t* kinds,
                          const int64_t* sizes, int64_t* out_offset, int64_t* out_total,
                          int64_t* out_bad_event);

/* ---- sim.py: integer-time replay/framework simulator (semantic oracle) --- */
typedef struct sw_sim_config {
  int64_t capacity;           /* <= 0: unbounded (None) */
  int64_t overhead_framework;
  int64_t overhead_replay;
  int32_t framework_mode;     /* 0 = REPLAY (simulate), 1 = FRAMEWORK */
} sw_sim_config;
/* Schedule input as produced by sw_plan_pre_run (stream_len/op_kind/op_arg/order).
 * Outputs: out_start/out_end per graph node (graph order; -1 if never run),
 * out_events (event id, fire time) pairs sorted, capacity 2*n_ops. */
int sw_plan_simulate(const sw_graph_view* g, int64_t n_streams, const int64_t* stream_len,
                     const int32_t* op_kind, const int64_t* op_arg, int64_t n_order,
                     const int64_t* order, const sw_sim_config* cfg, int64_t* out_makespan,
                     int64_t* out_active, int64_t* out_start, int64_t* out_end,
                     int64_t* out_events, int64_t* out_n_events);

/* ======================================================================== */
/* Device engine                                                             */
/* ======================================================================== */

typedef struct sw_engine sw_engine;

/* One kernel task of the op table.  kind = enum sw_kernel_kind (see
 * paper_2012_02732_b200/csrc/runtime/ops.h); params/ptrs meanings per kind are
 * documented there and in DESIGN.md §Kernels. */
#define SW_OP_MAX_PARAMS 56
#define SW_OP_MAX_PTRS 8
typedef struct sw_op_desc {
  int32_t kind;
  int32_t variant;                   /* kernel selection (tile config), chosen at prepare */
  int64_t params[SW_OP_MAX_PARAMS];
  uint64_t ptrs[SW_OP_MAX_PTRS];     /* device addresses */
} sw_op_desc;

int sw_engine_create(int32_t device, sw_engine** out);
int sw_engine_destroy(sw_engine* e);
/* Replace the op table (copied). Task id t of the schedule = op index t. */
int sw_engine_set_ops(sw_engine* e, int64_t n_ops, const sw_op_desc* ops);
/* Input/output staging for the captured memcpy nodes: host pinned pointers
 * and device pointers, byte counts. */
int sw_engine_set_io(sw_engine* e, uint64_t host_in, uint64_t dev_in, int64_t in_bytes,
                     uint64_t host_out, uint64_t dev_out, int64_t out_bytes);
/* AoT capture of a pre_run schedule (streams of LAUNCH/RECORD/WAIT in
 * capture `order`) into one CUDA graph; with_io adds the H2D memcpy node
 * first (forked to every stream head) and the D2H node last (joined from
 * every stream tail).  slot selects one of 4 independent graph slots (e.g.
 * multi-stream vs single-stream). */
int sw_engine_capture(sw_engine* e, int32_t slot, int64_t n_streams, const int64_t* stream_len,
                      const int32_t* op_kind, const int64_t* op_arg, int64_t n_order,
                      const int64_t* order, int32_t with_io);
/* Replay a captured slot on the engine's launch stream (async). */
int sw_engine_replay(sw_engine* e, int32_t slot);
/* One inference from host memory: copy host_in (in_bytes) into the pinned
 * staging buffer, replay a with_io slot, wait, copy the staged output to
 * host_out (out_bytes).  Either pointer may be NULL (staging used as is). */
int sw_engine_infer(sw_engine* e, int32_t slot, const void* host_in, void* host_out);

/* n requests back to back through device-resident slot `slot` (pipelined:
 * request i+1's H2D overlaps request i's replay; staging is double-buffered).
 * host_in[i] / host_out[i]: in_bytes / out_bytes host buffers (pinned for
 * overlap).  Results equal n sw_engine_infer calls. */
int sw_engine_infer_stream(sw_engine* e, int32_t slot, int64_t n, const uint64_t* host_in, const uint64_t* host_out);
/* Replay and wait; returns host wall time of the launch call in ns. */
int sw_engine_replay_sync(sw_engine* e, int32_t slot, int64_t* out_launch_ns);
/* Time `iters` replays with cudaEvents on the launch stream → mean µs,
 * and mean host launch-call time in µs. */
int sw_engine_time_replay(sw_engine* e, int32_t slot, int32_t iters, double* out_gpu_us,
                          double* out_host_us);
/* Eager (non-AoT) execution: launch op `index` on the launch stream now. */
int sw_engine_launch_op(sw_engine* e, int64_t index);
/* Eager run of all ops in the given order on one stream, host loop in C. */
int sw_engine_run_eager(sw_engine* e, int64_t n, const int64_t* order);
/* Framework (non-AoT) mode of a pre_run schedule: every LAUNCH / RECORD / WAIT
 * issued now by the host on the engine's stream pool, no capture (the
 * run-time-scheduling baseline of sim.py:69-80, multi-stream). */
int sw_engine_run_schedule(sw_engine* e, int64_t n_streams, const int64_t* stream_len,
                           const int32_t* op_kind, const int64_t* op_arg, int64_t n_order,
                           const int64_t* order);
int sw_engine_synchronize(sw_engine* e);
/* Captured graph topology of a slot: node count and dependency edge count;
 * out_edges (capacity 2*cap) receives (from, to) node indices where node
 * index = position in cudaGraphGetNodes order; out_node_kind: 0 task kernel,
 * 1 memcpy, 2 other, 3 engine plumbing kernel (staging copy / L2 prefetch);
 * out_node_task: op index for task kernel nodes else -1. */
int sw_engine_graph_topology(sw_engine* e, int32_t slot, int64_t cap, int64_t* out_n_nodes,
                             int32_t* out_node_kind, int64_t* out_node_task,
                             int64_t* out_n_edges, int64_t* out_edges);
/* Per-op device time (µs) of one eager pass, CUDA events around each op. */
int sw_engine_profile_ops(sw_engine* e, int64_t n, const int64_t* order, int32_t reps,
                          double* out_us);
/* Per-task start / end (µs since the traced graph's start) of the last replay
 * of a slot captured with SW_ENGINE_TRACE; -1 for tasks never recorded. */
int sw_engine_trace_read(sw_engine* e, int64_t n, double* out_start_us, double* out_end_us);
/* Launch stream handle (cudaStream_t as integer) for external interop. */
int sw_engine_stream(sw_engine* e, uint64_t* out_stream);
/* Kernel selection support: device time (µs, mean of `reps` back-to-back
 * launches after one warm-up) of an op descriptor that is not in the table. */
int sw_engine_time_op(sw_engine* e, const sw_op_desc* op, int32_t reps, double* out_us);
/* Kernel selection support: launch an op descriptor that is not in the table
 * once on the launch stream and wait for it (the autotuner checks a timed
 * winner's output against a reference candidate's before keeping it). */
int sw_engine_run_op(sw_engine* e, const sw_op_desc* op);
/* Engine flags for subsequent captures / eager launches:
 * SW_ENGINE_PDL = programmatic dependent launch on same-stream kernel edges. */
#define SW_ENGINE_PDL 1u
/* Diagnostic: capture an empty kernel per task (same topology, same PDL
 * protocol) — the replay then measures the graph's issue / dependency floor. */
#define SW_ENGINE_NULL_KERNELS 2u
/* Host staging copies of the with_io slots as kernel nodes that access the
 * pinned host buffers through their UVA mapping (instead of memcpy nodes). */
#define SW_ENGINE_KERNEL_IO 4u
/* Diagnostic: timing events around every task of subsequent captures; after a
 * replay, sw_engine_trace_read returns each task's start / end in µs from the
 * graph's start (the measured timeline behind a Chrome trace). */
#define SW_ENGINE_TRACE 16u
/* A root node on its own stream prefetches the range given to
 * sw_engine_set_prefetch (the packed weights) into L2 at graph start. */
#define SW_ENGINE_L2_PREFETCH 32u
/* With SW_ENGINE_PDL: the captured graph's cross-stream task -> task edges
 * (the sync edges of the plan) become programmatic edges too, so a task on
 * another stream launches as soon as its producers have triggered and waits
 * for their completion in griddepcontrol.wait, as same-stream successors do. */
#define SW_ENGINE_XSTREAM_PDL 64u
int sw_engine_set_flags(sw_engine* e, uint32_t flags);

/* ---- training step (paper_2012_02732_b200/train.py) ---- */
/* One more captured H2D copy in the with_io slots (labels next to images). */
int sw_engine_add_input(sw_engine* e, uint64_t host, uint64_t dev, int64_t bytes);
/* Per-task launch priority for subsequent captures / launches: one int32
 * urgency level per op (0 = default, k > 0 = k steps above the default in the
 * device's stream-priority range, clamped); n = 0 clears. */
int sw_engine_set_priorities(sw_engine* e, int64_t n, const int32_t* prio);
/* Device range warmed into L2 by SW_ENGINE_L2_PREFETCH captures. */
int sw_engine_set_prefetch(sw_engine* e, uint64_t dev, int64_t bytes);
/* Bind NCCL at run time (dlopen of `path`, or "libnccl.so.2" when NULL/empty). */
int sw_nccl_load(const char* path);
/* ncclGetUniqueId into a caller buffer of 128 bytes (rank 0 broadcasts it). */
int sw_nccl_unique_id(char* out128);
/* Data-parallel communicator for the engine's K_ALLREDUCE tasks, which are
 * captured into the training graph as ncclAllReduce(avg) on their stream. */
int sw_engine_nccl_init(sw_engine* e, int32_t nranks, int32_t rank, const char* id128);

#ifdef __cplusplus
}
#endif
#endif /* STREAMWEAVE_B200_H */
