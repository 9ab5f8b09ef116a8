"""Native planner (C ABI via the drop-in API) vs the reference's golden bytes.

Every case of tests/golden/planner_cases.json — produced by the unmodified
reference — must come out byte-identical: assignment JSON (stream ids, sync
edges, MEG edges), schedule JSON (per-stream FIFOs, event ids, arena,
task_args, capture order), critical path, fold_streams, simulator results
and the 4-mode compare matrix, or the identical error diagnostic.
"""

import json
import os
import re

import pytest

import paper_2012_02732_b200 as sw
from paper_2012_02732_b200 import _native

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "planner_cases.json")
with open(GOLDEN) as fh:
    CASES = json.load(fh)["cases"]

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "streamweave_b200.h")


def load_graph(case):
    doc = json.loads(case["graph"])
    nodes = []
    for d in doc["nodes"]:
        mem = tuple(sw.MemEvent.alloc(e["alloc"]) if "alloc" in e else sw.MemEvent.free(e["free"])
                    for e in d.get("mem", []))
        nodes.append(sw.TaskNode(d["id"], d.get("duration", 1), d.get("demand", 1),
                                 d.get("label"), mem))
    edges = [tuple(e) for e in doc["edges"]]
    if case.get("raw"):
        return sw.CompGraph(tuple(nodes), tuple(edges))
    return sw.CompGraph.build(nodes, edges)


def test_library_exports_every_declared_symbol():
    text = open(HEADER).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(sw_\w+)\(", text, re.M))
    assert len(declared) > 25
    lib = _native.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_native.PROTOTYPES) == declared


def run_case(case):
    g = load_graph(case)
    try:
        f, plan = sw.assign_streams(g)
        meg = sw.minimum_equivalent_graph(g)
        ts = sw.pre_run(g, f, plan)
        out = {"assign": sw.assignment_to_json(g, f, plan, meg), "sched": sw.schedule_to_json(ts),
               "critical_path": sw.critical_path_time(g)}
    except sw.StreamWeaveError as e:
        return {"error": e.diagnostic()}, None
    except ValueError as e:
        return {"error": f"ValueError: {e}"}, None
    return out, (g, f, plan, meg, ts)


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_native_matches_reference_bytes(idx):
    case = CASES[idx]
    got, ctx = run_case(case)
    if "error" in case:
        assert got == {"error": case["error"]}
        return
    assert got["assign"] == case["assign"]
    assert got["sched"] == case["sched"]
    assert got["critical_path"] == case["critical_path"]
    g, f, plan, meg, ts = ctx
    assert sw.graph_to_json(g) == case["graph"]
    for k, want in case.get("fold", {}).items():
        f2, p2 = sw.fold_streams(g, f, plan, int(k))
        assert sw.assignment_to_json(g, f2, p2, meg) == want
    for item in case.get("sim", []):
        cap, ovf, ovr = item["cfg"]
        cfg = sw.SimConfig(capacity=cap, overhead_framework=ovf, overhead_replay=ovr)
        try:
            rep = sw.sim_result_to_json(sw.simulate(ts, g, cfg))
            fw = sw.sim_result_to_json(sw.run_framework_mode(g, f, plan, cfg))
        except sw.StreamWeaveError as e:
            assert item.get("error") == e.diagnostic()
            continue
        assert rep == item["replay"]
        assert fw == item["framework"]
    for item in case.get("compare", []):
        cap, ovf, ovr = item["cfg"]
        cfg = sw.SimConfig(capacity=cap, overhead_framework=ovf, overhead_replay=ovr)
        assert sw.compare_to_json(sw.compare_modes(g, cfg)) == item["json"]


def test_diamond_api_surface():
    # reference tests/test_assign.py:51-83 and tests/test_schedule.py:57-64
    g = sw.CompGraph.build([sw.TaskNode(0, 1), sw.TaskNode(1, 4), sw.TaskNode(2, 2),
                            sw.TaskNode(3, 1)], [(0, 1), (0, 2), (1, 3), (2, 3)])
    meg = sw.minimum_equivalent_graph(g)
    assert sw.maximum_matching(sw.build_bipartite(meg)).pairs == ((0, 1), (1, 3))
    f, plan = sw.assign_streams(g)
    assert f.stream_of == {0: 0, 1: 0, 2: 1, 3: 0}
    assert plan.edges == ((0, 2), (2, 3))
    assert sw.is_max_concurrent(g, f)
    assert not sw.is_max_concurrent(g, sw.StreamAssignment({0: 0, 1: 0, 2: 0, 3: 0}))
    assert sw.plan_is_safe(g, f, plan)
    assert not sw.plan_is_safe(g, f, sw.SyncPlan(()))
    ts = sw.pre_run(g, f, plan)
    assert [(s, op.kind, op.arg) for s, op in sw.replay_order(ts)] == [
        (0, "launch", 0), (0, "record", 0), (0, "launch", 1), (1, "wait", 0),
        (1, "launch", 2), (1, "record", 1), (0, "wait", 1), (0, "launch", 3)]
    r = sw.transitive_closure(g)
    assert r.reaches(0, 3) and not r.reaches(1, 2) and r.ordered(3, 0)
    assert sw.topological_order(g) == [0, 1, 2, 3]
    m2 = sw.assignment_from_matching(meg, sw.Matching(((0, 1), (1, 3))))
    assert m2.stream_of == f.stream_of
    assert sw.min_sync_plan(meg, f).edges == plan.edges


def test_errors_and_arena():
    with pytest.raises(sw.UnsafePlan):
        g = sw.CompGraph.build([sw.TaskNode(i) for i in range(4)], [(0, 1), (0, 2), (1, 3), (2, 3)])
        f, _ = sw.assign_streams(g)
        sw.pre_run(g, f, sw.SyncPlan(()))
    with pytest.raises(sw.UnknownStream):
        sw.pre_run(g, sw.StreamAssignment({0: 0, 1: 0, 2: 2, 3: 0}), sw.SyncPlan(((0, 2), (2, 3))))
    with pytest.raises(sw.InvalidMatching):
        sw.assignment_from_matching(sw.minimum_equivalent_graph(g), sw.Matching(((0, 3),)))
    with pytest.raises(sw.NotMaxConcurrent):
        sw.min_sync_plan(sw.minimum_equivalent_graph(g), sw.StreamAssignment({i: 0 for i in range(4)}))
    lay = sw.reserve_arena([(("A", 0), sw.MemEvent.alloc(100)), (("B", 0), sw.MemEvent.alloc(50)),
                            (("A", 0), sw.MemEvent.free(0)), (("C", 0), sw.MemEvent.alloc(100))])
    assert lay.blocks[("C", 0)] == (0, 100) and lay.total == 150
    with pytest.raises(sw.FreeBeforeAlloc):
        sw.reserve_arena([(("x", 0), sw.MemEvent.free(0))])
    with pytest.raises(sw.DoubleFree):
        sw.reserve_arena([(("x", 0), sw.MemEvent.alloc(10)), (("x", 0), sw.MemEvent.free(0)),
                          (("x", 0), sw.MemEvent.free(0))])
    with pytest.raises(sw.CycleDetected) as e:
        sw.validate_graph(sw.CompGraph.build([sw.TaskNode(0), sw.TaskNode(1)], [(0, 1), (1, 0)]))
    assert e.value.cycle == [0, 1, 0]
    assert e.value.diagnostic() == "CycleDetected: 0→1→0"


def test_large_chain_is_fast():
    import time
    n = 5000
    g = sw.CompGraph.build([sw.TaskNode(i) for i in range(n)], [(i, i + 1) for i in range(n - 1)])
    t = time.perf_counter()
    f, plan = sw.assign_streams(g)
    ts = sw.pre_run(g, f, plan)
    dt = time.perf_counter() - t
    assert f.num_streams == 1 and len(plan) == 0 and len(ts.streams[0]) == n
    assert dt < 2.0  # the reference needs ~2.8 s for assign_streams alone


def test_cli_assign_matches_the_reference_bytes(tmp_path):
    """`python -m paper_2012_02732_b200 assign graph.json` prints the
    reference's assignment JSON (diamond golden case)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "tests", "golden", "planner_cases.json")) as fh:
        cases = json.load(fh)["cases"]
    case = next(c for c in cases if c.get("assign") and c.get("graph"))
    gp = tmp_path / "g.json"
    gp.write_text(case["graph"])
    out = subprocess.run([sys.executable, "-m", "paper_2012_02732_b200", "assign", str(gp)], cwd=root,
                         capture_output=True, text=True, check=True).stdout.strip()
    assert out == case["assign"]


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only host behaviour")
def test_engine_without_gpu_raises_cuda_error():
    """No CPU fallback: on a host without a CUDA device the engine's prepare
    and call raise CudaError (the C ABI's SW_CUDA_ERROR class) and nothing
    is computed on the CPU."""
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import InceptionCell, example_input
    model = InceptionCell().eval()
    x = example_input((1, 3, 32, 32))
    with pytest.raises(sw.CudaError):
        Engine(model).prepare(x)
    with pytest.raises(sw.CudaError):
        Engine(model)(x)
    assert sw.CudaError.__mro__[1] is sw.StreamWeaveError
