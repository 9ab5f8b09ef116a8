"""Regenerate tests/golden/verify_cases.json FROM THE REFERENCE ITSELF.

    python tests/golden/make_verify_golden.py

Imports the unmodified reference read-only from /root/reference/pkg/src (and
its seeded corpus helper from /root/reference/pkg/tests) and records, per
graph, the reference `streamweave.oracle` outputs (oracle.py:25-315):

  verify       verify_optimal(g).to_json() + plan_safe, or "<Class>: <detail>"
  given        verify_given for (f, plan) variants: the algorithm's own, the
               plan minus its last edge, everything on one stream, singletons
  brute        min_syncs_brute(g, f) and with bound=1 for the same variants
  safe         oracle_plan_is_safe for the same variants
  enum         enumerate_assignments(g) as label lists over the topo order
  matchings    enumerate_matchings(build_bipartite(g, meg)) pair lists
  compare      compare_modes(g, SimConfig(), with_oracle=True).oracle_status

Consumed by tests/test_verify.py (native verify.cpp through the C ABI).
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")


def err(e):
    return f"{type(e).__name__}: {e}"


def variants(sw, g):
    f, plan = sw.assign_streams(g)
    ids = [t.id for t in g.nodes]
    out = [("algo", f, plan)]
    if len(plan):
        out.append(("drop_last", f, sw.SyncPlan(plan.edges[:-1])))
    out.append(("single", sw.StreamAssignment({i: 0 for i in ids}), sw.SyncPlan(())))
    single_plan = sw.SyncPlan(tuple(e for e in g.edges))
    out.append(("singletons", sw.StreamAssignment({i: k for k, i in enumerate(ids)}), single_plan))
    return out


def case(sw, g, name):
    from streamweave import oracle as O
    c = {"name": name, "graph": sw.graph_to_json(g)}
    try:
        r = O.verify_optimal(g)
        c["verify"] = {"json": r.to_json(), "plan_safe": r.plan_safe, "optimal": r.optimal}
    except Exception as e:  # noqa: BLE001
        c["verify"] = {"error": err(e)}
    try:
        c["compare"] = sw.compare_modes(g, sw.SimConfig(), with_oracle=True).oracle_status
    except Exception as e:  # noqa: BLE001
        c["compare"] = err(e)
    try:
        vs = variants(sw, g)
    except Exception as e:  # noqa: BLE001
        c["variants_error"] = err(e)
        return c
    c["variants"] = []
    for vname, f, plan in vs:
        v = {"name": vname, "stream_of": [[k, s] for k, s in f.stream_of.items()],
             "plan": [list(e) for e in plan.edges]}
        for key, fn in (("given", lambda: O.verify_given(g, f, plan).to_json()),
                        ("brute", lambda: O.min_syncs_brute(g, f)),
                        ("brute_b1", lambda: O.min_syncs_brute(g, f, bound=1)),
                        ("safe", lambda: O.oracle_plan_is_safe(g, f, plan))):
            try:
                v[key] = fn()
            except Exception as e:  # noqa: BLE001
                v[key] = {"error": err(e)}
        c["variants"].append(v)
    try:
        order = sw.topological_order(g)
        c["enum"] = [[a.stream_of[i] for i in order] for a in O.enumerate_assignments(g)]
    except Exception as e:  # noqa: BLE001
        c["enum"] = {"error": err(e)}
    try:
        meg = sw.minimum_equivalent_graph(g)
        b = sw.build_bipartite(g, meg)
        ms = O.enumerate_matchings(b)
        c["matchings"] = {"left": b.left_size, "edges": [list(e) for e in b.edges],
                          "all": [[list(p) for p in m.pairs] for m in ms]} if len(ms) <= 200 else None
    except Exception as e:  # noqa: BLE001
        c["matchings"] = {"error": err(e)}
    return c


def main():
    import streamweave as sw
    from _corpus import random_dag
    T = sw.TaskNode
    cases = []
    for seed in range(120):
        cases.append(case(sw, random_dag(seed, max_nodes=7), f"random7_{seed}"))
    for seed in range(20):
        cases.append(case(sw, random_dag(1000 + seed, max_nodes=10), f"random10_{seed}"))
    # hand-made edge cases: diamond, empty, one node, antichain, the complete
    # 7-node DAG (21 edges > the 20-edge cap), an 8-node chain (node cap),
    # non-contiguous ids
    mk = lambda n, es: sw.CompGraph.build([T(i) for i in n], es)  # noqa: E731
    cases.append(case(sw, mk(range(4), [(0, 1), (0, 2), (1, 3), (2, 3)]), "diamond"))
    cases.append(case(sw, mk([], []), "empty"))
    cases.append(case(sw, mk([5], []), "single"))
    cases.append(case(sw, mk(range(6), []), "antichain6"))
    cases.append(case(sw, mk(range(7), [(u, v) for u in range(7) for v in range(u + 1, 7)]), "complete7"))
    cases.append(case(sw, mk(range(8), [(i, i + 1) for i in range(7)]), "chain8"))
    cases.append(case(sw, mk([3, 10, 42, 7, 99], [(3, 10), (3, 42), (10, 99), (42, 99), (7, 99)]), "sparse_ids"))
    cases.append(case(sw, mk(range(7), [(0, 1), (0, 2), (0, 3), (1, 4), (2, 4), (2, 5), (3, 5), (4, 6), (5, 6)]),
                      "lattice7"))
    with open(os.path.join(HERE, "verify_cases.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_verify_golden.py", "cases": cases}, fh, separators=(",", ":"))
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
