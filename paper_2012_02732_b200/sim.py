"""Integer-time simulator of the drop-in API (`streamweave/sim.py:38-294`).

The B200 engine replaces this model with a real CUDA-graph replay; the native
simulator (`csrc/planner/sim.cpp`) remains the semantic reference for replay
order (and a predictor when fed measured kernel durations, §8(f) f3).
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from enum import Enum
from fractions import Fraction

from . import _native as N
from .assign import StreamAssignment, SyncPlan
from .errors import EmptyRun
from .graph import CompGraph, critical_path_time
from .schedule import TaskSchedule, pre_run, schedule_arrays


class SubmitMode(Enum):
    FRAMEWORK = "framework"
    REPLAY = "replay"


@dataclass(frozen=True)
class SimConfig:
    capacity: int | None = None
    overhead_framework: int = 0
    overhead_replay: int = 0

    def __post_init__(self) -> None:
        if self.overhead_framework < 0 or self.overhead_replay < 0:
            raise ValueError("overheads must be non-negative")
        if self.capacity is not None and self.capacity < 1:
            raise ValueError("capacity must be at least 1")


@dataclass(frozen=True)
class SimResult:
    makespan: int
    gpu_active_time: int
    intervals: dict[int, tuple[int, int]]
    events_fired: tuple[tuple[int, int], ...]


def _run(ts: TaskSchedule, g: CompGraph, cfg: SimConfig, mode: SubmitMode) -> SimResult:
    m = N.Marshal()
    v = m.graph(g)
    lens, kinds, args, order = schedule_arrays(ts)
    m.keep += [lens, kinds, args, order]
    c = N.SimConfigC(cfg.capacity if cfg.capacity is not None else 0, cfg.overhead_framework,
                     cfg.overhead_replay, 1 if mode is SubmitMode.FRAMEWORK else 0)
    n = len(g.nodes)
    n_ops = sum(len(s) for s in ts.streams)
    ms, act = m.out64(1), m.out64(1)
    st, en = m.out64(n), m.out64(n)
    evs, nev = m.out64(2 * n_ops + 2), m.out64(1)
    N.check(N.lib().sw_plan_simulate(C.byref(v), len(ts.streams), N.ptr64(lens), N.ptr32(kinds),
                                     N.ptr64(args), len(ts.order), N.ptr64(order), C.byref(c),
                                     N.ptr64(ms), N.ptr64(act), N.ptr64(st), N.ptr64(en),
                                     N.ptr64(evs), N.ptr64(nev)))
    iv = {}
    for i, t in enumerate(g.nodes):
        if st[i] >= 0:
            iv[t.id] = (int(st[i]), int(en[i]))
    fired = tuple((int(evs[2 * i]), int(evs[2 * i + 1])) for i in range(int(nev[0])))
    return SimResult(int(ms[0]), int(act[0]), iv, fired)


def simulate(ts: TaskSchedule, g: CompGraph, cfg: SimConfig) -> SimResult:
    """Replay a captured schedule; every op costs ``overhead_replay``."""
    return _run(ts, g, cfg, SubmitMode.REPLAY)


def run_framework_mode(g: CompGraph, f: StreamAssignment, plan: SyncPlan,
                       cfg: SimConfig) -> SimResult:
    """Same ops with run-time scheduling: each launch waits for its preds."""
    return _run(pre_run(g, f, plan), g, cfg, SubmitMode.FRAMEWORK)


@dataclass(frozen=True)
class MetricsReport:
    makespan: int
    gpu_active_time: int
    critical_path: int
    gpu_active_ratio: Fraction
    critical_ratio: Fraction | None


def metrics(r: SimResult, g: CompGraph) -> MetricsReport:
    if r.makespan == 0:
        raise EmptyRun("metrics of a zero-length run")
    cp = critical_path_time(g)
    busy = r.gpu_active_time
    return MetricsReport(r.makespan, busy, cp, Fraction(busy, r.makespan),
                         Fraction(cp, busy) if busy > 0 else None)


def speedup(baseline: SimResult, other: SimResult) -> Fraction:
    if other.makespan == 0:
        raise EmptyRun("speedup against a zero-length run")
    return Fraction(baseline.makespan, other.makespan)


def sim_result_to_json(r: SimResult) -> str:
    return json.dumps({
        "makespan": r.makespan,
        "gpu_active_time": r.gpu_active_time,
        "intervals": {str(t): list(span) for t, span in sorted(r.intervals.items())},
        "events_fired": [list(p) for p in r.events_fired],
    }, separators=(",", ":"))


def chrome_trace(r: SimResult, g: CompGraph, stream_of: dict[int, int]) -> str:
    """Complete-event ("ph":"X") timeline, tid = stream (sim.py:277-294)."""
    rows = []
    for t in g.nodes:
        if t.id in r.intervals:
            a, b = r.intervals[t.id]
            rows.append({"name": t.label if t.label is not None else f"task{t.id}",
                         "ph": "X", "ts": a, "dur": b - a, "tid": stream_of[t.id]})
    rows.sort(key=lambda row: (row["ts"], row["tid"], row["name"]))
    return json.dumps(rows, separators=(",", ":"))
