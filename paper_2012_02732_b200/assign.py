"""Stream assignment of the drop-in API (`streamweave/assign.py:34-299`).

MEG → bipartite → Kuhn maximum matching (pinned scan) → chains as streams →
minimal sync plan (|E'| - |M| event edges).  All computation is native.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

from . import _native as N
from .errors import UnknownStream
from .graph import CompGraph, Edge, Meg, ReachMatrix, minimum_equivalent_graph, topological_order


@dataclass(frozen=True)
class BipartiteGraph:
    left_size: int
    right_size: int
    edges: tuple[tuple[int, int], ...]


@dataclass(frozen=True)
class Matching:
    pairs: tuple[tuple[int, int], ...]


@dataclass(frozen=True)
class StreamAssignment:
    """task id -> dense stream id, labelled by first use along topo order."""

    stream_of: dict[int, int]

    @property
    def num_streams(self) -> int:
        return max(self.stream_of.values(), default=-1) + 1

    def streams(self, order: list[int]) -> list[list[int]]:
        out: list[list[int]] = [[] for _ in range(self.num_streams)]
        for v in order:
            out[self.stream_of[v]].append(v)
        return out


@dataclass(frozen=True)
class SyncPlan:
    edges: tuple[Edge, ...]

    def __len__(self) -> int:
        return len(self.edges)


def _pairs_out(buf, n):
    return tuple((int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(n))


def _assign_out(ids, streams, n):
    return StreamAssignment({int(ids[i]): int(streams[i]) for i in range(n)})


def build_bipartite(meg: Meg) -> BipartiteGraph:
    ranked = sorted(t.id for t in meg.base.nodes)
    pos = {x: i for i, x in enumerate(ranked)}
    return BipartiteGraph(len(ranked), len(ranked),
                          tuple(sorted((pos[a], pos[b]) for a, b in meg.edges)))


def maximum_matching(b: BipartiteGraph) -> Matching:
    m = N.Marshal()
    ne, ep = m.pairs(b.edges)
    out = m.out64(2 * min(b.left_size, b.right_size) + 2)
    cnt = m.out64(1)
    N.check(N.lib().sw_plan_maximum_matching(b.left_size, b.right_size, ne, ep, N.ptr64(out),
                                             N.ptr64(cnt)))
    return Matching(_pairs_out(out, int(cnt[0])))


def validate_matching(b: BipartiteGraph, m: Matching) -> None:
    from .errors import InvalidMatching
    es = set(b.edges)
    xs: set[int] = set()
    ys: set[int] = set()
    for x, y in m.pairs:
        if (x, y) not in es:
            raise InvalidMatching(f"pair ({x},{y}) is not a bipartite edge")
        if x in xs:
            raise InvalidMatching(f"left vertex {x} matched twice")
        if y in ys:
            raise InvalidMatching(f"right vertex {y} matched twice")
        xs.add(x)
        ys.add(y)


def assignment_from_matching(meg: Meg, m: Matching) -> StreamAssignment:
    mm = N.Marshal()
    v = mm.graph(meg.base)
    nm, mp = mm.pairs(meg.edges)
    npairs, pp = mm.pairs(m.pairs)
    n = len(meg.base.nodes)
    ids, ss = mm.out64(n), mm.out64(n)
    N.check(N.lib().sw_plan_assignment_from_matching(C.byref(v), nm, mp, npairs, pp,
                                                     N.ptr64(ids), N.ptr64(ss)))
    return _assign_out(ids, ss, n)


def is_max_concurrent(g: CompGraph, f: StreamAssignment, reach: ReachMatrix | None = None) -> bool:
    m = N.Marshal()
    v = m.graph(g)
    a = m.assignment(f.stream_of)
    out = m.out32(1)
    N.check(N.lib().sw_plan_is_max_concurrent(C.byref(v), C.byref(a), N.ptr32(out)))
    return bool(out[0])


def min_sync_plan(meg: Meg, f: StreamAssignment) -> SyncPlan:
    m = N.Marshal()
    v = m.graph(meg.base)
    nm, mp = m.pairs(meg.edges)
    a = m.assignment(f.stream_of)
    out = m.out64(2 * len(meg.edges))
    cnt = m.out64(1)
    N.check(N.lib().sw_plan_min_sync_plan(C.byref(v), nm, mp, C.byref(a), N.ptr64(out),
                                          N.ptr64(cnt)))
    return SyncPlan(_pairs_out(out, int(cnt[0])))


def plan_is_safe(g: CompGraph, f: StreamAssignment, plan: SyncPlan) -> bool:
    m = N.Marshal()
    v = m.graph(g)
    a = m.assignment(f.stream_of)
    np_, pp = m.pairs(plan.edges)
    out = m.out32(1)
    N.check(N.lib().sw_plan_plan_is_safe(C.byref(v), C.byref(a), np_, pp, N.ptr32(out)))
    return bool(out[0])


def assign_streams_full(g: CompGraph) -> tuple[StreamAssignment, SyncPlan, tuple[Edge, ...]]:
    """assign_streams plus the MEG edges it computed (one native call)."""
    m = N.Marshal()
    v = m.graph(g)
    n, e = len(g.nodes), len(g.edges)
    ids, ss = m.out64(n), m.out64(n)
    sync, nsync = m.out64(2 * e), m.out64(1)
    meg, nmeg = m.out64(2 * e), m.out64(1)
    N.check(N.lib().sw_plan_assign_streams(C.byref(v), N.ptr64(ids), N.ptr64(ss), N.ptr64(sync),
                                           N.ptr64(nsync), N.ptr64(meg), N.ptr64(nmeg)))
    return (_assign_out(ids, ss, n), SyncPlan(_pairs_out(sync, int(nsync[0]))),
            _pairs_out(meg, int(nmeg[0])))


def assign_streams(g: CompGraph) -> tuple[StreamAssignment, SyncPlan]:
    """validate → MEG → match → partition → plan (assign.py:233-240)."""
    f, plan, _ = assign_streams_full(g)
    return f, plan


def fold_streams(g: CompGraph, f: StreamAssignment, plan: SyncPlan,
                 max_streams: int) -> tuple[StreamAssignment, SyncPlan]:
    """Merge logical streams onto a physical budget; the plan is kept whole."""
    if max_streams < 1:
        raise ValueError("max_streams must be >= 1")
    if f.num_streams <= max_streams:
        return f, plan
    m = N.Marshal()
    v = m.graph(g)
    a = m.assignment(f.stream_of)
    n = len(g.nodes)
    ids, ss = m.out64(n), m.out64(n)
    N.check(N.lib().sw_plan_fold_streams(C.byref(v), C.byref(a), max_streams, N.ptr64(ids),
                                         N.ptr64(ss)))
    return _assign_out(ids, ss, n), plan


def assignment_to_json(g: CompGraph, f: StreamAssignment, plan: SyncPlan, meg: Meg) -> str:
    return json.dumps({"streams": f.streams(topological_order(g)),
                       "syncs": [list(e) for e in plan.edges],
                       "meg_edges": [list(e) for e in meg.edges]}, separators=(",", ":"))


def assignment_from_json(text: str, g: CompGraph) -> tuple[StreamAssignment, SyncPlan]:
    doc = json.loads(text)
    declared = {t.id for t in g.nodes}
    stream_of: dict[int, int] = {}
    for sid, members in enumerate(doc["streams"]):
        for x in members:
            x = int(x)
            if x not in declared:
                raise UnknownStream(f"stream {sid} names unknown task {x}")
            stream_of[x] = sid
    for t in g.nodes:
        if t.id not in stream_of:
            raise UnknownStream(f"task {t.id} has no stream")
    syncs = tuple(sorted((int(a), int(b)) for a, b in doc.get("syncs", [])))
    return StreamAssignment(stream_of), SyncPlan(syncs)
