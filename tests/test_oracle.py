"""Pin the CPU oracle (oracle/planner.py) to the reference's own golden bytes.

The fixture tests/golden/planner_cases.json was produced by running the
unmodified reference (tests/golden/make_golden.py).  If the oracle agrees with
every case here, it is a trustworthy checker for the native planner.
"""

import json
import os

import pytest

from oracle import planner as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "planner_cases.json")


def load_cases():
    with open(GOLDEN) as fh:
        return json.load(fh)["cases"]


CASES = load_cases()


def graph_of(case):
    doc = json.loads(case["graph"])
    if case.get("raw"):
        nodes = [(it["id"], it.get("duration", 1), it.get("demand", 1),
                  tuple(("alloc", e["alloc"]) if "alloc" in e else ("free", e["free"])
                        for e in it.get("mem", []))) for it in doc["nodes"]]
        return nodes, [tuple(e) for e in doc["edges"]]
    return O.graph_from_obj(doc)


def test_fixture_is_large_enough():
    names = {c["name"] for c in CASES}
    assert len(CASES) > 700
    assert {"diamond.json", "lr.json", "corpus7_499", "corpus6_199"} <= names


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_oracle_matches_reference(idx):
    case = CASES[idx]
    nodes, edges = graph_of(case)
    got = O.plan_case(nodes, edges)
    if "error" in case:
        assert got == {"error": case["error"]}
        return
    assert got["assign"] == case["assign"]
    assert got["sched"] == case["sched"]
    assert got["critical_path"] == case["critical_path"]
    assert O.graph_json(nodes, edges) == case["graph"] or case.get("raw")
    for k, want in case.get("fold", {}).items():
        f, plan, m = O.assign(nodes, edges)
        f2 = O.fold(nodes, edges, f, int(k))
        assert O.assignment_json(nodes, edges, f2, plan, m) == want


def test_diamond_known_answers():
    # tests/test_assign.py:51-55, :79-83 and tests/test_schedule.py:57-64 of the reference
    nodes, edges = O.build([(0, 1, 1, ()), (1, 4, 1, ()), (2, 2, 1, ()), (3, 1, 1, ())],
                           [(0, 1), (0, 2), (1, 3), (2, 3)])
    m = O.meg(nodes, edges)
    assert O.kuhn(*O.bipartite(nodes, m)) == [(0, 1), (1, 3)]
    f, plan, _ = O.assign(nodes, edges)
    assert f == {0: 0, 1: 0, 2: 1, 3: 0}
    assert plan == [(0, 2), (2, 3)]
    s = O.pre_run(nodes, edges, f, plan)
    assert s["streams"] == [[("launch", 0), ("record", 0), ("launch", 1), ("wait", 1),
                             ("launch", 3)], [("wait", 0), ("launch", 2), ("record", 1)]]
    assert s["order"] == [0, 0, 0, 1, 1, 1, 0, 0]


def test_arena_first_fit_known_answers():
    # tests/test_schedule.py:176-200 of the reference
    total, blocks = O.arena([(("A", 0), "alloc", 100), (("B", 0), "alloc", 50),
                             (("A", 0), "free", 0), (("C", 0), "alloc", 100)])
    assert blocks[("C", 0)] == (0, 100) and total == 150
    with pytest.raises(O.OracleError) as e:
        O.arena([(("x", 0), "free", 0)])
    assert e.value.kind == "FreeBeforeAlloc"
