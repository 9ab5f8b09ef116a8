"""Exhaustive sync-optimality verifiers — the reference's ``streamweave.oracle``
API (`/root/reference/pkg/src/streamweave/oracle.py:25-315`), named `verify`
here so it is not confused with this repo's test oracle (`oracle/`).

The searches run natively (`csrc/planner/verify.cpp`, C ABI
``sw_plan_verify`` / ``sw_plan_min_syncs_brute`` /
``sw_plan_enumerate_assignments`` / ``sw_plan_oracle_plan_is_safe``) and are
deliberately independent of the production pipeline: a path-walking safety
DP, raw set partitions, exact set cover.  Same size guards and ``TooLarge``
texts as the reference (7 nodes to verify, 10 to enumerate, 20 edges for the
plan search).
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

from . import _native as N
from .assign import BipartiteGraph, Matching, StreamAssignment
from .graph import CompGraph

MAX_ENUM_NODES = 10
MAX_PLAN_EDGES = 20
MAX_VERIFY_NODES = 7


@dataclass(frozen=True)
class OracleReport:
    optimal: bool
    algo_syncs: int
    oracle_min: int
    assignments_checked: int
    plan_safe: bool

    def to_json(self) -> str:
        doc = {"optimal": self.optimal, "algo_syncs": self.algo_syncs,
               "oracle_min": self.oracle_min, "assignments_checked": self.assignments_checked}
        return json.dumps(doc, separators=(",", ":"))


def _plan_edges(plan):
    return tuple(plan.edges if hasattr(plan, "edges") else plan)


def oracle_plan_is_safe(g: CompGraph, f: StreamAssignment, plan) -> bool:
    """Every cross-stream edge (u, v) has a u..v path through a plan edge
    (oracle.py:30-43), by a forward DP over the topological order."""
    m = N.Marshal()
    v, a = m.graph(g), m.assignment(f.stream_of)
    np_, pp = m.pairs(_plan_edges(plan))
    out = m.out32(1)
    N.check(N.lib().sw_plan_oracle_plan_is_safe(C.byref(v), C.byref(a), np_, pp, N.ptr32(out)))
    return bool(out[0])


def min_syncs_brute(g: CompGraph, f: StreamAssignment, *, bound: int | None = None) -> int:
    """Smallest safe plan size for f by exact search (oracle.py:149-162);
    with ``bound`` the result is min(exact, bound)."""
    m = N.Marshal()
    v, a = m.graph(g), m.assignment(f.stream_of)
    out = m.out64(1)
    N.check(N.lib().sw_plan_min_syncs_brute(C.byref(v), C.byref(a), -1 if bound is None else int(bound),
                                            N.ptr64(out)))
    return int(out[0])


def enumerate_assignments(g: CompGraph) -> list[StreamAssignment]:
    """All maximum-logical-concurrency assignments, canonically labelled, in
    restricted-growth order (oracle.py:219-225)."""
    m = N.Marshal()
    v = m.graph(g)
    n = len(g.nodes)
    order, cnt = m.out64(n), m.out64(1)
    N.check(N.lib().sw_plan_enumerate_assignments(C.byref(v), 0, N.ptr64(order), N.ptr64(m.out64(1)),
                                                  N.ptr64(cnt)))
    k = int(cnt[0])
    labels = m.out64(k * n)
    N.check(N.lib().sw_plan_enumerate_assignments(C.byref(v), k, N.ptr64(order), N.ptr64(labels),
                                                  N.ptr64(cnt)))
    ids = [int(x) for x in order[:n]]
    return [StreamAssignment({ids[i]: int(labels[a * n + i]) for i in range(n)}) for a in range(k)]


def enumerate_matchings(b: BipartiteGraph) -> list[Matching]:
    """Every matching of b, the empty one included, in the include/exclude
    recursion order over sorted edges (oracle.py:228-251)."""
    edges = sorted(b.edges)
    out: list[Matching] = []
    cur: list = []

    def rec(i: int, lx: frozenset, ly: frozenset) -> None:
        if i == len(edges):
            out.append(Matching(tuple(cur)))
            return
        rec(i + 1, lx, ly)
        x, y = edges[i]
        if x not in lx and y not in ly:
            cur.append((x, y))
            rec(i + 1, lx | {x}, ly | {y})
            cur.pop()

    rec(0, frozenset(), frozenset())
    return out


def _report(out) -> OracleReport:
    return OracleReport(optimal=bool(out[0]), algo_syncs=int(out[1]), oracle_min=int(out[2]),
                        assignments_checked=int(out[3]), plan_safe=bool(out[4]))


def verify_optimal(g: CompGraph) -> OracleReport:
    """The pipeline's sync count against the exhaustive minimum over every
    maximum-concurrency assignment (oracle.py:271-293)."""
    m = N.Marshal()
    v = m.graph(g)
    out = m.out64(5)
    N.check(N.lib().sw_plan_verify(C.byref(v), None, 0, None, N.ptr64(out)))
    return _report(out)


def verify_given(g: CompGraph, f: StreamAssignment, plan) -> OracleReport:
    """The same report for a caller-supplied assignment and plan (oracle.py:296-315)."""
    m = N.Marshal()
    v, a = m.graph(g), m.assignment(f.stream_of)
    np_, pp = m.pairs(_plan_edges(plan))
    out = m.out64(5)
    N.check(N.lib().sw_plan_verify(C.byref(v), C.byref(a), np_, pp, N.ptr64(out)))
    return _report(out)
