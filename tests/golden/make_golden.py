"""Regenerate the planner golden fixtures FROM THE REFERENCE ITSELF.

Run here (the container that has /root/reference):

    python tests/golden/make_golden.py

It imports the unmodified reference package read-only from
/root/reference/pkg/src (plus the reference test helpers in
/root/reference/pkg/tests for the seeded corpora) and records, for every
case, the reference's own bytes:

  graph      graph_to_json(g)                         (graph.py:306-322)
  assign     assignment_to_json(g, f, plan, meg)      (assign.py:275-282)
  sched      schedule_to_json(pre_run(g, f, plan))    (schedule.py:174-188)
  critical_path, fold[k] (fold_streams, assign.py:243-270),
  sim        sim_result_to_json of replay/framework runs (sim.py:64-80)
  compare    compare_to_json(compare_modes(g, cfg))   (compare.py:50-131)
  error      "<Class>: <detail>" when the reference raises

The fixture is consumed by tests/test_oracle.py (oracle pinned to the
reference) and tests/test_planner_native.py (native C ABI vs fixture).
/root/reference does not exist on the GPU box; nothing there reads it.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"


def _import_reference():
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REF_TESTS)
    sys.setrecursionlimit(100000)
    import streamweave as sw  # noqa: F401
    import _corpus  # noqa: F401
    return sw, _corpus


def reference_case(sw, g, name, sim_cfgs=(), folds=(), compare_cfgs=(), raw=False):
    case = {"name": name, "graph": sw.graph_to_json(g)}
    if raw:
        case["raw"] = True
    try:
        f, plan = sw.assign_streams(g)
        meg = sw.minimum_equivalent_graph(g)
        case["assign"] = sw.assignment_to_json(g, f, plan, meg)
        ts = sw.pre_run(g, f, plan)
        case["sched"] = sw.schedule_to_json(ts)
        case["critical_path"] = sw.critical_path_time(g)
        if folds:
            case["fold"] = {}
            for k in folds:
                f2, p2 = sw.fold_streams(g, f, plan, k)
                case["fold"][str(k)] = sw.assignment_to_json(g, f2, p2, meg)
        if sim_cfgs:
            case["sim"] = []
            for cap, ovf, ovr in sim_cfgs:
                cfg = sw.SimConfig(capacity=cap, overhead_framework=ovf, overhead_replay=ovr)
                item = {"cfg": [cap, ovf, ovr]}
                try:
                    item["replay"] = sw.sim_result_to_json(sw.simulate(ts, g, cfg))
                    item["framework"] = sw.sim_result_to_json(
                        sw.run_framework_mode(g, f, plan, cfg))
                except sw.StreamWeaveError as e:
                    item["error"] = e.diagnostic()
                case["sim"].append(item)
        if compare_cfgs:
            case["compare"] = []
            for cap, ovf, ovr in compare_cfgs:
                cfg = sw.SimConfig(capacity=cap, overhead_framework=ovf, overhead_replay=ovr)
                try:
                    case["compare"].append(
                        {"cfg": [cap, ovf, ovr],
                         "json": sw.compare_to_json(sw.compare_modes(g, cfg))})
                except sw.StreamWeaveError as e:
                    case["compare"].append({"cfg": [cap, ovf, ovr], "error": e.diagnostic()})
    except sw.StreamWeaveError as e:
        case["error"] = e.diagnostic()
    except ValueError as e:
        case["error"] = f"ValueError: {e}"
    return case


def raw_graph(sw, nodes, edges):
    """A CompGraph WITHOUT build()-sorting, for the validation-order cases."""
    return sw.CompGraph(tuple(nodes), tuple(edges))


def planner_cases():
    sw, corpus = _import_reference()
    T = sw.TaskNode
    M = sw.MemEvent
    cases = []
    sims = ((None, 0, 0), (None, 5, 1), (4, 5, 1), (2, 3, 0))

    golden_dir = "/root/reference/pkg/golden"
    for fn in ("diamond.json", "lr.json"):
        with open(os.path.join(golden_dir, fn)) as fh:
            g = sw.graph_from_json(fh.read())
        cases.append(reference_case(sw, g, fn, sim_cfgs=sims, folds=(1, 2),
                                    compare_cfgs=((4, 5, 1), (None, 5, 1))))

    diamond_mem = sw.CompGraph.build(
        [T(0, 1), T(1, 4, 1, None, (M.alloc(100),)),
         T(2, 2, 1, None, (M.alloc(50), M.free(0))), T(3, 1)],
        [(0, 1), (0, 2), (1, 3), (2, 3)])
    cases.append(reference_case(sw, diamond_mem, "diamond_mem", sim_cfgs=sims))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(10), T(20), T(30), T(40)],
                               [(10, 20), (10, 30), (20, 40), (30, 40)]), "diamond_sparse_ids"))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(i) for i in range(5)], [(0, 2), (1, 2), (2, 3), (2, 4)]),
        "hub_width_gap"))
    cases.append(reference_case(sw, sw.CompGraph.build([], []), "empty"))
    cases.append(reference_case(sw, sw.CompGraph.build([T(7, 3)], []), "single"))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(0), T(1)], []), "two_independent", sim_cfgs=sims))

    # error cases, in validation order (graph.py:111-136)
    cases.append(reference_case(sw, sw.CompGraph.build([T(0), T(1)], [(0, 1), (1, 0)]), "cycle2"))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(i) for i in range(5)], [(0, 1), (1, 2), (2, 3), (3, 1), (3, 4)]),
        "cycle3"))
    cases.append(reference_case(sw, sw.CompGraph.build([T(0)], [(0, 0)]), "selfloop"))
    cases.append(reference_case(sw, sw.CompGraph.build([T(0)], [(0, 5)]), "dangling"))
    cases.append(reference_case(sw, sw.CompGraph.build([T(0), T(1)], [(0, 1), (0, 1)]), "dupedge"))
    cases.append(reference_case(sw, sw.CompGraph.build([T(0), T(0)], []), "dupid"))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(0, 1, 1, None, (M.free(0),))], []), "free_before_alloc"))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(0, 1, 1, None, (M.alloc(4), M.free(0), M.free(0)))], []),
        "double_free"))
    cases.append(reference_case(
        sw, sw.CompGraph.build([T(0, 1, 1, None, (M.alloc(0),))], []), "alloc_zero"))
    cases.append(reference_case(
        sw, raw_graph(sw, [T(3), T(1), T(2)], [(3, 1), (1, 2), (2, 3)]), "raw_cycle_unsorted",
        raw=True))

    # seeded corpora exactly as the reference acceptance gates draw them
    for i, g in enumerate(corpus.corpus(500, 7, 1000)):
        cases.append(reference_case(sw, g, f"corpus7_{i}",
                                    sim_cfgs=((None, 3, 1), (2, 3, 1)) if i < 60 else ()))
    for i, g in enumerate(corpus.corpus(200, 6, 2000)):
        cases.append(reference_case(sw, g, f"corpus6_{i}"))
    for i in range(40):
        g = corpus.random_dag(5000 + i, max_nodes=60, max_edges=400)
        cases.append(reference_case(sw, g, f"random60_{i}", folds=(1, 3, 8)))
    for i in range(6):
        g = corpus.random_dag(7000 + i, max_nodes=300, max_edges=1500)
        cases.append(reference_case(sw, g, f"random300_{i}", folds=(4,)))

    # workload generators (workloads.py:118-189)
    W = sw.WorkloadSpec
    C = sw.Constant
    specs = [("chain50", sw.Chain(50)), ("chain400", sw.Chain(400))]
    specs += [(f"forkjoin{k}", sw.ForkJoin(k)) for k in range(1, 9)]
    specs += [("cellstack20x4", sw.CellStack(20, 4)), ("cellstack60x8", sw.CellStack(60, 8))]
    specs += [(f"layered{i}", sw.LayeredRandom(3 + i % 5, 2 + i % 6, 0.3 + 0.03 * i, 40 + i))
              for i in range(20)]
    for name, kind in specs:
        g = sw.generate(W(kind=kind, duration_model=sw.Uniform(1, 9, 3), demand_model=C(1)))
        cases.append(reference_case(sw, g, name, sim_cfgs=((None, 15, 1), (4, 5, 1)),
                                    folds=(1, 2, 4)))
    return cases


def main():
    cases = planner_cases()
    out = os.path.join(HERE, "planner_cases.json")
    with open(out, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "/root/reference/pkg/src/streamweave (v0.1.0)",
                   "cases": cases}, fh, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {out} ({os.path.getsize(out)} bytes)")


if __name__ == "__main__" and "--networks" not in sys.argv:
    main()


def network_cases():
    """The op DAGs our builder emits for the BASELINE networks, planned by the
    reference ("parity of streams is defined on the DAG the
    builder emits: feed that same DAG to the reference")."""
    sw, _ = _import_reference()
    root = os.path.dirname(os.path.dirname(HERE))
    sys.path.insert(0, root)
    from paper_2012_02732_b200.networks import build_model, example_input
    from paper_2012_02732_b200.trace import build_program
    cases = []
    for name in ("cell", "resnet50", "inception_v3", "nasnet_mobile", "mobilenet_v2",
                 "efficientnet_b0"):
        model, shape = build_model(name)
        x = example_input(shape)
        for fuse in (True, False):
            prog = build_program(model, x, fuse=fuse)
            text = graph_text(prog.graph)
            g = sw.graph_from_json(text)
            case = reference_case(sw, g, f"{name}:{'fused' if fuse else 'raw'}")
            cases.append(case)
    return cases


def graph_text(g):
    """graph_to_json of our CompGraph (same canonical format as the reference)."""
    from paper_2012_02732_b200.graph import graph_to_json
    return graph_to_json(g)


def main_networks():
    cases = network_cases()
    out = os.path.join(HERE, "network_dags.json")
    with open(out, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py --networks",
                   "reference": "/root/reference/pkg/src/streamweave (v0.1.0)",
                   "cases": cases}, fh, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {out} ({os.path.getsize(out)} bytes)")


if __name__ == "__main__" and "--networks" in sys.argv:
    main_networks()
