"""ctypes binding of libsw_b200.so (include/streamweave_b200.h).

There is no fallback: if the shared library is missing or does not export
the declared ABI, importing anything that needs it raises ExtensionMissing.
Build it with ``python -m paper_2012_02732_b200.build`` (or
``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import ExtensionMissing, from_status

# SW_B200_LIB selects the diagnostic build (libsw_b200_probe.so) for tools/
LIB_PATH = os.environ.get("SW_B200_LIB") or \
    os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsw_b200.so")

i64 = C.c_int64
i32 = C.c_int32
u64 = C.c_uint64
P64 = C.POINTER(C.c_int64)
P32 = C.POINTER(C.c_int32)
PU64 = C.POINTER(C.c_uint64)


class GraphView(C.Structure):
    _fields_ = [("n_nodes", i64), ("ids", P64), ("durations", P64), ("demands", P64),
                ("mem_start", P64), ("mem_kind", P32), ("mem_arg", P64),
                ("n_edges", i64), ("edges", P64)]


class AssignView(C.Structure):
    _fields_ = [("n", i64), ("ids", P64), ("streams", P64)]


class ScheduleOut(C.Structure):
    _fields_ = [("stream_len", P64), ("op_kind", P32), ("op_arg", P64), ("order", P64),
                ("block_node", P64), ("block_index", P64), ("block_offset", P64),
                ("block_size", P64), ("walk", P64), ("task_args_start", P64),
                ("task_args", P64), ("n_streams", i64), ("n_ops", i64), ("event_count", i64),
                ("arena_total", i64), ("n_blocks", i64)]


class SimConfigC(C.Structure):
    _fields_ = [("capacity", i64), ("overhead_framework", i64), ("overhead_replay", i64),
                ("framework_mode", i32)]


SW_OP_MAX_PARAMS = 56
SW_OP_MAX_PTRS = 8


class OpDesc(C.Structure):
    _fields_ = [("kind", i32), ("variant", i32), ("params", i64 * SW_OP_MAX_PARAMS),
                ("ptrs", u64 * SW_OP_MAX_PTRS)]


# name -> (restype, argtypes); mirrors include/streamweave_b200.h exactly.
PROTOTYPES = {
    "sw_last_error": (C.c_char_p, []),
    "sw_version": (C.c_char_p, []),
    "sw_plan_validate": (C.c_int, [C.POINTER(GraphView)]),
    "sw_plan_topological_order": (C.c_int, [C.POINTER(GraphView), P64]),
    "sw_plan_transitive_closure": (C.c_int, [C.POINTER(GraphView), PU64]),
    "sw_plan_minimum_equivalent_graph": (C.c_int, [C.POINTER(GraphView), P64, P64]),
    "sw_plan_critical_path_time": (C.c_int, [C.POINTER(GraphView), P64]),
    "sw_plan_maximum_matching": (C.c_int, [i64, i64, i64, P64, P64, P64]),
    "sw_plan_assignment_from_matching": (C.c_int, [C.POINTER(GraphView), i64, P64, i64, P64,
                                                   P64, P64]),
    "sw_plan_is_max_concurrent": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), P32]),
    "sw_plan_min_sync_plan": (C.c_int, [C.POINTER(GraphView), i64, P64, C.POINTER(AssignView),
                                        P64, P64]),
    "sw_plan_plan_is_safe": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), i64, P64,
                                       P32]),
    "sw_plan_assign_streams": (C.c_int, [C.POINTER(GraphView), P64, P64, P64, P64, P64, P64]),
    "sw_plan_fold_streams": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), i64, P64,
                                       P64]),
    "sw_plan_verify": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), i64, P64, P64]),
    "sw_plan_oracle_plan_is_safe": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), i64,
                                              P64, P32]),
    "sw_plan_min_syncs_brute": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), i64, P64]),
    "sw_plan_enumerate_assignments": (C.c_int, [C.POINTER(GraphView), i64, P64, P64, P64]),
    "sw_plan_pre_run": (C.c_int, [C.POINTER(GraphView), C.POINTER(AssignView), i64, P64,
                                  C.POINTER(ScheduleOut)]),
    "sw_plan_reserve_arena": (C.c_int, [i64, P64, P32, P64, P64, P64, P64]),
    "sw_plan_simulate": (C.c_int, [C.POINTER(GraphView), i64, P64, P32, P64, i64, P64,
                                   C.POINTER(SimConfigC), P64, P64, P64, P64, P64, P64]),
    # device engine
    "sw_engine_create": (C.c_int, [i32, C.POINTER(C.c_void_p)]),
    "sw_engine_destroy": (C.c_int, [C.c_void_p]),
    "sw_engine_set_ops": (C.c_int, [C.c_void_p, i64, C.POINTER(OpDesc)]),
    "sw_engine_set_io": (C.c_int, [C.c_void_p, u64, u64, i64, u64, u64, i64]),
    "sw_engine_capture": (C.c_int, [C.c_void_p, i32, i64, P64, P32, P64, i64, P64, i32]),
    "sw_engine_replay": (C.c_int, [C.c_void_p, i32]),
    "sw_engine_replay_sync": (C.c_int, [C.c_void_p, i32, P64]),
    "sw_engine_infer": (C.c_int, [C.c_void_p, i32, C.c_void_p, C.c_void_p]),
    "sw_engine_trace_read": (C.c_int, [C.c_void_p, i64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "sw_engine_time_replay": (C.c_int, [C.c_void_p, i32, i32, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]),
    "sw_engine_launch_op": (C.c_int, [C.c_void_p, i64]),
    "sw_engine_run_eager": (C.c_int, [C.c_void_p, i64, P64]),
    "sw_engine_synchronize": (C.c_int, [C.c_void_p]),
    "sw_engine_run_schedule": (C.c_int, [C.c_void_p, i64, P64, P32, P64, i64, P64]),
    "sw_engine_graph_topology": (C.c_int, [C.c_void_p, i32, i64, P64, P32, P64, P64, P64]),
    "sw_engine_profile_ops": (C.c_int, [C.c_void_p, i64, P64, i32, C.POINTER(C.c_double)]),
    "sw_engine_stream": (C.c_int, [C.c_void_p, PU64]),
    "sw_engine_time_op": (C.c_int, [C.c_void_p, C.POINTER(OpDesc), i32, C.POINTER(C.c_double)]),
    "sw_engine_run_op": (C.c_int, [C.c_void_p, C.POINTER(OpDesc)]),
    "sw_engine_set_flags": (C.c_int, [C.c_void_p, C.c_uint32]),
    "sw_engine_add_input": (C.c_int, [C.c_void_p, u64, u64, i64]),
    "sw_engine_set_prefetch": (C.c_int, [C.c_void_p, u64, i64]),
    "sw_engine_set_priorities": (C.c_int, [C.c_void_p, i64, P32]),
    "sw_engine_infer_stream": (C.c_int, [C.c_void_p, C.c_int32, i64, P64, P64]),
    "sw_nccl_load": (C.c_int, [C.c_char_p]),
    "sw_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "sw_engine_nccl_init": (C.c_int, [C.c_void_p, i32, i32, C.c_char_p]),
}

_lib = None


def lib():
    """The loaded native library (raises ExtensionMissing, never falls back)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ExtensionMissing(
            f"{LIB_PATH} is not built; run `python -m paper_2012_02732_b200.build`")
    try:
        h = C.CDLL(LIB_PATH)
    except OSError as e:
        raise ExtensionMissing(f"cannot load {LIB_PATH}: {e}") from None
    missing = []
    for name, (res, args) in PROTOTYPES.items():
        try:
            fn = getattr(h, name)
        except AttributeError:
            missing.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    if missing:
        raise ExtensionMissing(f"{LIB_PATH} does not export {', '.join(missing)}")
    _lib = h
    return h


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().sw_last_error().decode("utf-8", "replace")
        raise from_status(rc, msg)


def ptr64(a: np.ndarray):
    return a.ctypes.data_as(P64)


def ptr32(a: np.ndarray):
    return a.ctypes.data_as(P32)


def arr64(values) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(values, dtype=np.int64).reshape(-1))


def pairs_arr(pairs) -> np.ndarray:
    a = np.asarray(list(pairs), dtype=np.int64).reshape(-1)
    return np.ascontiguousarray(a)


class Marshal:
    """Keeps numpy buffers alive while the view is used."""

    def __init__(self):
        self.keep = []

    def graph(self, g) -> GraphView:
        nodes = g.nodes
        n = len(nodes)
        ids = arr64([t.id for t in nodes])
        dur = arr64([t.duration for t in nodes])
        dem = arr64([t.demand for t in nodes])
        starts = [0]
        kinds, args = [], []
        for t in nodes:
            for ev in t.mem:
                if ev.kind == "alloc":
                    kinds.append(0)
                    args.append(ev.size)
                elif ev.kind == "free":
                    kinds.append(1)
                    args.append(ev.ref)
                else:
                    kinds.append(99)
                    args.append(0)
            starts.append(len(kinds))
        ms = arr64(starts)
        mk = np.ascontiguousarray(np.asarray(kinds if kinds else [0], dtype=np.int32))
        ma = arr64(args if args else [0])
        ed = pairs_arr(g.edges) if g.edges else np.zeros(2, dtype=np.int64)
        self.keep += [ids, dur, dem, ms, mk, ma, ed]
        return GraphView(n, ptr64(ids), ptr64(dur), ptr64(dem), ptr64(ms), ptr32(mk), ptr64(ma),
                         len(g.edges), ptr64(ed))

    def assignment(self, stream_of: dict) -> AssignView:
        ids = arr64(list(stream_of.keys()) or [0])
        ss = arr64(list(stream_of.values()) or [0])
        self.keep += [ids, ss]
        return AssignView(len(stream_of), ptr64(ids), ptr64(ss))

    def pairs(self, pairs):
        pairs = list(pairs)
        a = pairs_arr(pairs) if pairs else np.zeros(2, dtype=np.int64)
        self.keep.append(a)
        return len(pairs), ptr64(a)

    def out64(self, n):
        a = np.zeros(max(1, n), dtype=np.int64)
        self.keep.append(a)
        return a

    def out32(self, n):
        a = np.zeros(max(1, n), dtype=np.int32)
        self.keep.append(a)
        return a
