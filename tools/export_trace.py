"""Measured Chrome trace of one replay (reference format
sim.py:277-294 / CLI `export-trace`, cli.py:225-240):

    python tools/export_trace.py --config nasnet_mobile --out profiles/r01_trace_nasnet_bs1.json

Open the JSON in chrome://tracing or Perfetto: one row per logical stream.
Also prints makespan, summed task time, average concurrency, and the
reference simulator's makespan for the same DAG fed with the measured
durations (zero overhead) for comparison.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2012_02732_b200.engine import Engine  # noqa: E402
from paper_2012_02732_b200.networks import build_model, example_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--single", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--tuning-cache", default=None)
    a = ap.parse_args()
    import paper_2012_02732_b200 as sw
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model, tuning_cache=a.tuning_cache).prepare(x)
    eng.load_input_device(x)
    iv, js = eng.trace(multi=not a.single)
    lo = min(s for s, _ in iv.values())
    hi = max(e for _, e in iv.values())
    busy = sum(e - s for s, e in iv.values())
    g = eng.graph
    gd = sw.CompGraph.build([sw.TaskNode(n.id, max(1, int(round(1000 * (iv[n.id][1] - iv[n.id][0])))), 1,
                                         n.label, n.mem) for n in g.nodes], g.edges)
    f, plan = sw.assign_streams(gd)
    sim = sw.simulate(sw.pre_run(gd, f, plan), gd, sw.SimConfig()).makespan / 1000
    summary = {"config": a.config, "batch": a.batch, "multi_stream": not a.single, "tasks": len(iv),
               "makespan_us": round(hi - lo, 2), "sum_task_us": round(busy, 2),
               "avg_concurrency": round(busy / (hi - lo), 3),
               "simulated_makespan_us_from_these_durations": round(sim, 2),
               "note": "timing events around every task: same-stream PDL overlap is off in this capture"}
    print(json.dumps(summary))
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(js)
        with open(os.path.splitext(a.out)[0] + ".summary.json", "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
