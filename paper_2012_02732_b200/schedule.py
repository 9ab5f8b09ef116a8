"""AoT schedule capture of the drop-in API (`streamweave/schedule.py:24-215`).

``pre_run`` walks the canonical topological order once and records, per
stream, the FIFO of LAUNCH / RECORD / WAIT operations plus a first-fit arena
layout.  On B200 this list is not simulated: `engine.Engine` realises it op for
op under CUDA stream capture into one CUDA graph.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .assign import StreamAssignment, SyncPlan
from .errors import DoubleFree, FreeBeforeAlloc, from_status
from .graph import ALLOC, FREE, CompGraph, MemEvent

LAUNCH = "launch"
RECORD = "record"
WAIT = "wait"
_KIND_NAMES = (LAUNCH, RECORD, WAIT)
_KIND_CODES = {LAUNCH: 0, RECORD: 1, WAIT: 2}

BlockKey = tuple[int, int]


@dataclass(frozen=True)
class StreamOp:
    kind: str
    arg: int
    position: int


@dataclass(frozen=True)
class ArenaLayout:
    total: int
    blocks: dict[BlockKey, tuple[int, int]]


@dataclass(frozen=True)
class TaskSchedule:
    streams: tuple[tuple[StreamOp, ...], ...]
    event_count: int
    arena: ArenaLayout
    task_args: dict[int, tuple[int, ...]]
    order: tuple[int, ...]


def pre_run(g: CompGraph, f: StreamAssignment, plan: SyncPlan) -> TaskSchedule:
    """Capture the schedule of a safe (assignment, plan) pair (native)."""
    m = N.Marshal()
    v = m.graph(g)
    a = m.assignment(f.stream_of)
    np_, pp = m.pairs(plan.edges)
    n = len(g.nodes)
    ops_cap = n + 2 * len(plan.edges)
    allocs = sum(1 for t in g.nodes for e in t.mem if e.kind == ALLOC)
    out = N.ScheduleOut()
    bufs = {
        "stream_len": m.out64(max(n, 1)), "op_kind": m.out32(ops_cap), "op_arg": m.out64(ops_cap),
        "order": m.out64(ops_cap), "block_node": m.out64(allocs), "block_index": m.out64(allocs),
        "block_offset": m.out64(allocs), "block_size": m.out64(allocs), "walk": m.out64(n),
        "task_args_start": m.out64(n + 1), "task_args": m.out64(allocs),
    }
    for k, b in bufs.items():
        setattr(out, k, N.ptr32(b) if b.dtype == np.int32 else N.ptr64(b))
    N.check(N.lib().sw_plan_pre_run(C.byref(v), C.byref(a), np_, pp, C.byref(out)))
    streams = []
    p = 0
    kinds, args = bufs["op_kind"], bufs["op_arg"]
    for s in range(out.n_streams):
        ln = int(bufs["stream_len"][s])
        streams.append(tuple(StreamOp(_KIND_NAMES[kinds[p + i]], int(args[p + i]), i)
                             for i in range(ln)))
        p += ln
    blocks = {(int(bufs["block_node"][i]), int(bufs["block_index"][i])):
              (int(bufs["block_offset"][i]), int(bufs["block_size"][i]))
              for i in range(out.n_blocks)}
    ta = {}
    st, targs = bufs["task_args_start"], bufs["task_args"]
    for w in range(n):
        ta[int(bufs["walk"][w])] = tuple(int(x) for x in targs[st[w]:st[w + 1]])
    return TaskSchedule(streams=tuple(streams), event_count=int(out.event_count),
                        arena=ArenaLayout(int(out.arena_total), blocks), task_args=ta,
                        order=tuple(int(x) for x in bufs["order"][:out.n_ops]))


def reserve_arena(trace) -> ArenaLayout:
    """First-fit over a linear (key, MemEvent) trace (native)."""
    trace = list(trace)
    key_ids: dict = {}
    keys = []
    kinds = []
    sizes = []
    for key, ev in trace:
        keys.append(key_ids.setdefault(key, len(key_ids)))
        kinds.append(0 if ev.kind == ALLOC else 1 if ev.kind == FREE else 99)
        sizes.append(ev.size if ev.kind == ALLOC else 0)
    n = len(trace)
    m = N.Marshal()
    k = N.arr64(keys or [0])
    kd = np.ascontiguousarray(np.asarray(kinds or [0], dtype=np.int32))
    sz = N.arr64(sizes or [0])
    offs, total, bad = m.out64(n), m.out64(1), m.out64(1)
    rc = N.lib().sw_plan_reserve_arena(n, N.ptr64(k), N.ptr32(kd), N.ptr64(sz), N.ptr64(offs),
                                       N.ptr64(total), N.ptr64(bad))
    if rc != 0:
        i = int(bad[0])
        key, ev = trace[i] if 0 <= i < n else (None, None)
        if rc == 12:
            raise FreeBeforeAlloc(f"free of {key} before its alloc")
        if rc == 13:
            raise DoubleFree(f"block {key} freed twice")
        if ev is not None and ev.kind not in (ALLOC, FREE):
            raise ValueError(f"unknown mem event kind {ev.kind!r}")
        if ev is not None:
            raise ValueError(f"block {key} allocated twice")
        raise from_status(rc, N.lib().sw_last_error().decode())
    placed = {}
    for i, (key, ev) in enumerate(trace):
        if ev.kind == ALLOC:
            placed[key] = (int(offs[i]), ev.size)
    return ArenaLayout(total=int(total[0]), blocks=placed)


def replay_order(ts: TaskSchedule) -> list[tuple[int, StreamOp]]:
    """Flat submission sequence exactly as captured."""
    pos = [0] * len(ts.streams)
    out = []
    for s in ts.order:
        out.append((s, ts.streams[s][pos[s]]))
        pos[s] += 1
    return out


def schedule_arrays(ts: TaskSchedule):
    """(stream_len, op_kind, op_arg, order) int arrays for the native engine/sim."""
    lens = np.asarray([len(s) for s in ts.streams] or [0], dtype=np.int64)
    kinds = np.asarray([_KIND_CODES[o.kind] for s in ts.streams for o in s] or [0], dtype=np.int32)
    args = np.asarray([o.arg for s in ts.streams for o in s] or [0], dtype=np.int64)
    order = np.asarray(list(ts.order) or [0], dtype=np.int64)
    return lens, kinds, args, order


def schedule_to_json(ts: TaskSchedule) -> str:
    doc = {
        "streams": [[{o.kind: o.arg} for o in s] for s in ts.streams],
        "events": ts.event_count,
        "arena": {"total": ts.arena.total,
                  "blocks": {f"{a}:{b}": list(span)
                             for (a, b), span in sorted(ts.arena.blocks.items())}},
        "task_args": {str(t): list(offs) for t, offs in sorted(ts.task_args.items())},
        "order": list(ts.order),
    }
    return json.dumps(doc, separators=(",", ":"))


def schedule_from_json(text: str) -> TaskSchedule:
    doc = json.loads(text)
    streams = []
    for fifo in doc["streams"]:
        ops = []
        for i, item in enumerate(fifo):
            (kind, arg), = item.items()
            if kind not in _KIND_CODES:
                raise ValueError(f"unknown op {item!r}")
            ops.append(StreamOp(kind, int(arg), i))
        streams.append(tuple(ops))
    blocks = {}
    for key, span in doc["arena"]["blocks"].items():
        a, b = key.split(":")
        blocks[(int(a), int(b))] = (int(span[0]), int(span[1]))
    return TaskSchedule(
        streams=tuple(streams), event_count=int(doc.get("events", 0)),
        arena=ArenaLayout(total=int(doc["arena"]["total"]), blocks=blocks),
        task_args={int(t): tuple(int(x) for x in v) for t, v in doc.get("task_args", {}).items()},
        order=tuple(int(s) for s in doc.get("order", [])))
