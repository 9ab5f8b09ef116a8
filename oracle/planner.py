"""CPU restatement of the reference planning path — TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the native planner
(`paper_2012_02732_b200/csrc/planner/planner.cpp`).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s reference/cpu_baseline leg may
import it; the product path never does.

It restates, in plain Python over plain data, the algorithms of the reference
package `streamweave` (`/root/reference/pkg/src/streamweave/`), each function
citing the reference lines it follows.  It is pinned against golden vectors
produced by the reference itself (`tests/golden/make_golden.py` →
`tests/golden/planner_cases.json`, checked by `tests/test_oracle.py`).

Data model (deliberately not the reference's dataclasses):
  graph = (nodes, edges); nodes = list of (id, duration, demand, mem)
  with mem = tuple of ("alloc", size) | ("free", ref); edges = list of (u, v).
Errors are raised as ``OracleError(kind, message)`` where ``kind`` is the
reference exception class name and ``message`` its exact text.
"""

from __future__ import annotations

import heapq
import json


class OracleError(Exception):
    def __init__(self, kind: str, message: str):
        super().__init__(f"{kind}: {message}")
        self.kind = kind
        self.message = message


def build(nodes, edges):
    """CompGraph.build: nodes sorted by id (stable), edges sorted (graph.py:73-77)."""
    nodes = sorted(((int(n[0]), int(n[1]), int(n[2]), tuple(n[3])) for n in nodes),
                   key=lambda t: t[0])
    return nodes, sorted((int(u), int(v)) for u, v in edges)


def graph_from_obj(doc):
    """Plain graph from the reference JSON document shape (graph.py:325-349)."""
    nodes = []
    for it in doc.get("nodes", []):
        mem = []
        for ev in it.get("mem", []):
            if "alloc" in ev:
                mem.append(("alloc", int(ev["alloc"])))
            else:
                mem.append(("free", int(ev["free"])))
        nodes.append((int(it["id"]), int(it.get("duration", 1)),
                      int(it.get("demand", 1)), tuple(mem)))
    return build(nodes, [tuple(e) for e in doc.get("edges", [])])


def _succ(nodes, edges):
    out = {n[0]: [] for n in nodes}
    for u, v in edges:
        out[u].append(v)
    return out


# --- graph.py ---------------------------------------------------------------

def validate(nodes, edges):
    """validate_graph (graph.py:111-136) incl. _validate_mem (:237-252)."""
    ids = set()
    for nid, _d, _q, mem in nodes:
        if nid in ids:
            raise OracleError("DuplicateNodeId", f"node id {nid} declared twice")
        ids.add(nid)
        released = set()
        for i, (kind, arg) in enumerate(mem):
            if kind == "alloc":
                if arg <= 0:
                    raise OracleError("ValueError",
                                      f"node {nid} mem[{i}]: alloc size must be positive")
            elif kind == "free":
                if not (0 <= arg < i) or mem[arg][0] != "alloc":
                    raise OracleError(
                        "FreeBeforeAlloc",
                        f"node {nid} mem[{i}] frees index {arg}, not an earlier alloc")
                if arg in released:
                    raise OracleError("DoubleFree",
                                      f"node {nid} mem[{i}] frees index {arg} again")
                released.add(arg)
            else:
                raise OracleError("ValueError", f"node {nid} mem[{i}]: unknown kind {kind!r}")
    for u, v in edges:
        if u == v:
            raise OracleError("SelfLoop", f"edge {u}→{v}")
        if u not in ids or v not in ids:
            raise OracleError("DanglingEdge", f"edge {u}→{v} references an undeclared node")
    met = set()
    for e in edges:
        if e in met:
            raise OracleError("DuplicateEdge", f"edge {e[0]}→{e[1]} declared twice")
        met.add(e)
    cyc = find_cycle(nodes, edges)
    if cyc is not None:
        raise OracleError("CycleDetected", "→".join(map(str, cyc)))


def find_cycle(nodes, edges):
    """Three-colour DFS, roots ascending, witness [v..v] (graph.py:166-197)."""
    succ = _succ(nodes, edges)
    state = {n[0]: 0 for n in nodes}
    up = {}
    for root in sorted(state):
        if state[root]:
            continue
        state[root] = 1
        stack = [[root, 0]]
        while stack:
            top = stack[-1]
            node, k = top
            if k < len(succ[node]):
                top[1] = k + 1
                nxt = succ[node][k]
                if state[nxt] == 1:
                    walk = [node]
                    while walk[-1] != nxt:
                        walk.append(up[walk[-1]])
                    walk.reverse()
                    return walk + [nxt]
                if state[nxt] == 0:
                    state[nxt] = 1
                    up[nxt] = node
                    stack.append([nxt, 0])
            else:
                state[node] = 2
                stack.pop()
    return None


def topo(nodes, edges):
    """Min-heap Kahn order (graph.py:200-219)."""
    succ = _succ(nodes, edges)
    indeg = {n[0]: 0 for n in nodes}
    for _, v in edges:
        indeg[v] += 1
    heap = sorted(k for k, d in indeg.items() if d == 0)
    out = []
    while heap:
        u = heapq.heappop(heap)
        out.append(u)
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                heapq.heappush(heap, v)
    if len(out) != len(nodes):
        cyc = find_cycle(nodes, edges)
        raise OracleError("CycleDetected", "→".join(map(str, cyc or [])))
    return out


def closure(nodes, edges):
    """Reachability rows by id rank, reverse topo accumulation (graph.py:251-261).

    Returns (rank, rows) where rows[rank[u]] is a Python-int bitmask.
    """
    ids = sorted(n[0] for n in nodes)
    rank = {v: i for i, v in enumerate(ids)}
    succ = _succ(nodes, edges)
    rows = [0] * len(ids)
    for u in reversed(topo(nodes, edges)):
        acc = 0
        for v in succ[u]:
            acc |= rows[rank[v]] | (1 << rank[v])
        rows[rank[u]] = acc
    return rank, rows


def reaches(cl, u, v):
    rank, rows = cl
    return (rows[rank[u]] >> rank[v]) & 1 == 1


def meg(nodes, edges, cl=None):
    """Minimum equivalent graph: keep (u,v) unless a sibling succ reaches v (graph.py:275-288)."""
    cl = cl or closure(nodes, edges)
    succ = _succ(nodes, edges)
    kept = [(u, v) for u, v in edges
            if not any(w != v and reaches(cl, w, v) for w in succ[u])]
    return sorted(kept)


def critical_path(nodes, edges):
    """Longest duration path (graph.py:291-301)."""
    if not nodes:
        return 0
    dur = {n[0]: n[1] for n in nodes}
    preds = {n[0]: [] for n in nodes}
    for u, v in edges:
        preds[v].append(u)
    best = {}
    for v in topo(nodes, edges):
        best[v] = max((best[p] for p in preds[v]), default=0) + dur[v]
    return max(best.values())


# --- assign.py ----------------------------------------------------------------

def bipartite(nodes, meg_edges):
    """Rank-indexed bipartite edges (assign.py:75-79)."""
    rank = {v: i for i, v in enumerate(sorted(n[0] for n in nodes))}
    return len(rank), sorted((rank[u], rank[v]) for u, v in meg_edges)


def kuhn(n_left, bip_edges):
    """Augmenting paths, x ascending, adjacency ascending, one `seen` per x (assign.py:82-102)."""
    adj = [[] for _ in range(n_left)]
    for x, y in sorted(bip_edges):
        adj[x].append(y)
    owner = {}

    def try_x(x, seen):
        for y in adj[x]:
            if y in seen:
                continue
            seen.add(y)
            if y not in owner or try_x(owner[y], seen):
                owner[y] = x
                return True
        return False

    for x in range(n_left):
        try_x(x, set())
    return sorted((x, y) for y, x in owner.items())


def check_matching(bip_edges, pairs):
    """validate_matching (assign.py:105-117)."""
    es = set(bip_edges)
    xs, ys = set(), set()
    for x, y in pairs:
        if (x, y) not in es:
            raise OracleError("InvalidMatching", f"pair ({x},{y}) is not a bipartite edge")
        if x in xs:
            raise OracleError("InvalidMatching", f"left vertex {x} matched twice")
        if y in ys:
            raise OracleError("InvalidMatching", f"right vertex {y} matched twice")
        xs.add(x)
        ys.add(y)


def label_streams(nodes, edges, group_of):
    """First-use labels along canonical topo order (assign.py:154-162).

    Returns stream_of as an insertion-ordered dict (topo order).
    """
    names = {}
    out = {}
    for v in topo(nodes, edges):
        g = group_of[v]
        if g not in names:
            names[g] = len(names)
        out[v] = names[g]
    return out


def partition(nodes, edges, pairs):
    """assignment_from_matching (assign.py:138-151); groups via union-find."""
    ids = sorted(n[0] for n in nodes)
    parent = list(range(len(ids)))

    def find(i):
        while parent[i] != i:
            parent[i] = parent[parent[i]]
            i = parent[i]
        return i

    for x, y in pairs:
        a, b = find(x), find(y)
        if a != b:
            parent[b] = a
    return label_streams(nodes, edges, {v: find(i) for i, v in enumerate(ids)})


def max_concurrent(cl, stream_of):
    """is_max_concurrent (assign.py:165-179)."""
    members = {}
    for v, s in stream_of.items():
        members.setdefault(s, []).append(v)
    for vs in members.values():
        for i, u in enumerate(vs):
            for v in vs[i + 1:]:
                if not (reaches(cl, u, v) or reaches(cl, v, u)):
                    return False
    return True


def sync_plan(nodes, edges, meg_edges, stream_of):
    """min_sync_plan (assign.py:182-209)."""
    for n in nodes:
        if n[0] not in stream_of:
            raise OracleError("UnknownStream", f"task {n[0]} has no stream")
    cl = closure(nodes, edges)
    if not max_concurrent(cl, stream_of):
        raise OracleError("NotMaxConcurrent",
                          "two order-independent tasks share a stream; the unique-parent "
                          "rule does not apply")
    chained = {}
    drop = set()
    for u, v in meg_edges:
        if stream_of[u] == stream_of[v]:
            if v in chained:
                raise OracleError("NotMaxConcurrent",
                                  f"task {v} has two same-stream parents {chained[v]} and {u}")
            chained[v] = u
            drop.add((u, v))
    return [e for e in meg_edges if e not in drop]


def plan_safe(nodes, edges, stream_of, plan):
    """plan_is_safe (assign.py:212-230)."""
    cl = closure(nodes, edges)
    es = set(edges)
    covers = [e for e in plan if e in es]

    def rs(a, b):
        return a == b or reaches(cl, a, b)

    for u, v in edges:
        if stream_of[u] == stream_of[v]:
            continue
        if not any(rs(u, a) and rs(b, v) for a, b in covers):
            return False
    return True


def assign(nodes, edges):
    """assign_streams (assign.py:233-240) → (stream_of, plan, meg_edges)."""
    validate(nodes, edges)
    m = meg(nodes, edges)
    n_left, bip = bipartite(nodes, m)
    pairs = kuhn(n_left, bip)
    check_matching(bip, pairs)
    f = partition(nodes, edges, pairs)
    return f, sync_plan(nodes, edges, m, f), m


def fold(nodes, edges, stream_of, max_streams):
    """fold_streams (assign.py:243-270)."""
    if max_streams < 1:
        raise OracleError("ValueError", "max_streams must be >= 1")
    n_streams = max(stream_of.values(), default=-1) + 1
    if n_streams <= max_streams:
        return stream_of
    dur = {n[0]: n[1] for n in nodes}
    load = {s: 0 for s in range(n_streams)}
    for v, s in stream_of.items():
        load[s] += dur[v]
    heavy = sorted(load, key=lambda s: (-load[s], s))
    keep = sorted(heavy[:max_streams])
    rest = sorted(heavy[max_streams:], key=lambda s: (load[s], s))
    dest = {s: s for s in keep}
    for i, s in enumerate(rest):
        dest[s] = keep[i % len(keep)]
    return label_streams(nodes, edges, {v: dest[s] for v, s in stream_of.items()})


def streams_of(stream_of, order):
    n = max(stream_of.values(), default=-1) + 1
    out = [[] for _ in range(n)]
    for v in order:
        out[stream_of[v]].append(v)
    return out


def assignment_json(nodes, edges, stream_of, plan, meg_edges):
    """assignment_to_json (assign.py:275-282)."""
    doc = {"streams": streams_of(stream_of, topo(nodes, edges)),
           "syncs": [list(e) for e in plan],
           "meg_edges": [list(e) for e in meg_edges]}
    return json.dumps(doc, separators=(",", ":"))


# --- schedule.py ------------------------------------------------------------

def first_fit(live, size):
    """_first_fit (schedule.py:148-155 region: lowest gap among sorted live blocks)."""
    off = 0
    for start, length in sorted(live):
        if off + size <= start:
            break
        off = max(off, start + length)
    return off


def arena(trace):
    """reserve_arena (schedule.py:118-145): trace of (key, kind, arg)."""
    live, placed, total = {}, {}, 0
    for key, kind, arg in trace:
        if kind == "alloc":
            if key in placed:
                raise OracleError("ValueError", f"block {key} allocated twice")
            off = first_fit(live.values(), arg)
            live[key] = placed[key] = (off, arg)
            total = max(total, off + arg)
        elif kind == "free":
            if key not in placed:
                raise OracleError("FreeBeforeAlloc", f"free of {key} before its alloc")
            if key not in live:
                raise OracleError("DoubleFree", f"block {key} freed twice")
            del live[key]
        else:
            raise OracleError("ValueError", f"unknown mem event kind {kind!r}")
    return total, placed


def pre_run(nodes, edges, stream_of, plan):
    """pre_run (schedule.py:53-115).

    Returns dict(streams=[[(kind, arg)]], events, arena_total, blocks,
    task_args, order).
    """
    for n in nodes:
        if n[0] not in stream_of:
            raise OracleError("UnknownStream", f"task {n[0]} has no stream")
    n_streams = max(stream_of.values(), default=-1) + 1
    used = sorted(set(stream_of.values()))
    if used != list(range(n_streams)):
        raise OracleError("UnknownStream", f"stream ids are not dense from 0: {used}")
    es = set(edges)
    for e in plan:
        if e not in es:
            raise OracleError("UnsafePlan", f"sync edge {e[0]}→{e[1]} is not a graph edge")
    if not plan_safe(nodes, edges, stream_of, plan):
        raise OracleError("UnsafePlan", "plan leaves a cross-stream dependency uncovered")
    ordered = sorted(plan)
    ev = {e: i for i, e in enumerate(ordered)}
    rec = {n[0]: [] for n in nodes}
    wai = {n[0]: [] for n in nodes}
    for e in ordered:
        rec[e[0]].append(ev[e])
        wai[e[1]].append(ev[e])
    memof = {}
    for n in nodes:
        memof.setdefault(n[0], n[3])
    fifo = [[] for _ in range(n_streams)]
    order = []
    trace = []
    walk = topo(nodes, edges)
    for v in walk:
        s = stream_of[v]
        for x in wai[v]:
            fifo[s].append(("wait", x))
            order.append(s)
        fifo[s].append(("launch", v))
        order.append(s)
        for x in rec[v]:
            fifo[s].append(("record", x))
            order.append(s)
        for i, (kind, arg) in enumerate(memof[v]):
            trace.append(((v, i) if kind == "alloc" else (v, arg), kind, arg))
    total, blocks = arena(trace)
    targs = {v: tuple(blocks[(v, i)][0] for i, (k, _a) in enumerate(memof[v]) if k == "alloc")
             for v in walk}
    return {"streams": fifo, "events": len(ev), "arena_total": total,
            "blocks": blocks, "task_args": targs, "order": order}


def schedule_json(s):
    """schedule_to_json (schedule.py:174-188)."""
    doc = {
        "streams": [[{k: a} for k, a in fifo] for fifo in s["streams"]],
        "events": s["events"],
        "arena": {"total": s["arena_total"],
                  "blocks": {f"{k[0]}:{k[1]}": list(v) for k, v in sorted(s["blocks"].items())}},
        "task_args": {str(t): list(v) for t, v in sorted(s["task_args"].items())},
        "order": list(s["order"]),
    }
    return json.dumps(doc, separators=(",", ":"))


def graph_json(nodes, edges, labels=None):
    """graph_to_json (graph.py:306-322) for nodes without labels unless given."""
    out = []
    for nid, d, q, mem in nodes:
        item = {"id": nid}
        if labels and nid in labels:
            item["label"] = labels[nid]
        item["duration"] = d
        item["demand"] = q
        if mem:
            item["mem"] = [{k: a} for k, a in mem]
        out.append(item)
    return json.dumps({"nodes": out, "edges": [list(e) for e in edges]}, separators=(",", ":"))


def plan_case(nodes, edges):
    """Everything the golden fixture stores for one graph, or the error."""
    try:
        f, plan, m = assign(nodes, edges)
        sched = pre_run(nodes, edges, f, plan)
        return {"assign": assignment_json(nodes, edges, f, plan, m),
                "sched": schedule_json(sched),
                "critical_path": critical_path(nodes, edges)}
    except OracleError as e:
        return {"error": f"{e.kind}: {e.message}"}
