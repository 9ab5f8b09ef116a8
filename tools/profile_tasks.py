"""Per-task device-time profile of a prepared engine (run on a GPU box).

    python tools/profile_tasks.py --config nasnet_mobile [--batch 1] [--top 40]

Prints: per-family totals, the slowest tasks with their shapes and the kernel
the autotuner picked, the measured multi/single-stream replay latency, and the
reference simulator's prediction when fed the measured per-task durations
(simulator-in-the-loop).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--conv-impl", default="auto")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()

    import paper_2012_02732_b200 as sw
    from paper_2012_02732_b200.engine import Engine, task_cost
    from paper_2012_02732_b200.networks import build_model, example_input

    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model, conv_impl=a.conv_impl).prepare(x)
    per = eng.profile_tasks(reps=20)
    rows = []
    for t in eng.program.tasks:
        d = eng.ops[t.tid]
        p = list(d.params)
        f, b = task_cost(t)
        rows.append({"tid": t.tid, "kind": t.kind, "name": t.name, "us": float(per[t.tid]),
                     "kernel": [int(d.kind), int(d.variant), int(p[30])],
                     "in": [p[0], p[3], p[1], p[2]], "out": [p[4], p[5], p[6]] if t.kind in ("conv", "dwconv", "pool") else None,
                     "rs": [p[7], p[8]], "gflop": f / 1e9, "mb": b / 1e6})
    fam = {}
    for r in rows:
        fam.setdefault(r["kind"], [0.0, 0])
        fam[r["kind"]][0] += r["us"]
        fam[r["kind"]][1] += 1
    print("families:", {k: (round(v[0], 1), v[1]) for k, v in fam.items()})
    print("sum of tasks (serial) us:", round(sum(r["us"] for r in rows), 1))
    for r in sorted(rows, key=lambda r: -r["us"])[: a.top]:
        print(f"{r['tid']:4d} {r['kind']:6s} {r['us']:8.2f}us k={r['kernel']} in={r['in']} "
              f"out={r['out']} rs={r['rs']} {r['gflop']*1e3:.1f}MF {r['mb']:.2f}MB {r['name']}")
    eng.load_input_device(x)
    gm, hm = eng.time_replay(multi=True, iters=100)
    gs, hs = eng.time_replay(multi=False, iters=100)
    print(f"replay multi {gm:.1f} us  single {gs:.1f} us  host launch {hm:.2f} us")
    eng.recapture(null_kernels=True)
    fm, _ = eng.time_replay(multi=True, iters=100)
    fs, _ = eng.time_replay(multi=False, iters=100)
    eng.recapture()
    print(f"graph floor (empty kernel per task, same topology): multi {fm:.1f} us  single {fs:.1f} us")
    # simulator in the loop: measured durations (ns) into the reference replay model
    g = eng.graph
    dur = {t.tid: max(1, int(round(per[t.tid] * 1000))) for t in eng.program.tasks}
    g2 = sw.CompGraph.build([sw.TaskNode(n.id, dur[n.id], 1, n.label, n.mem) for n in g.nodes],
                            g.edges)
    f, plan = sw.assign_streams(g2)
    r_multi = sw.simulate(sw.pre_run(g2, f, plan), g2, sw.SimConfig())
    single = sw.StreamAssignment({n.id: 0 for n in g2.nodes})
    r_single = sw.simulate(sw.pre_run(g2, single, sw.SyncPlan(())), g2, sw.SimConfig())
    print(f"simulated (measured durations, zero overhead): multi {r_multi.makespan/1000:.1f} us "
          f"single {r_single.makespan/1000:.1f} us critical path "
          f"{sw.critical_path_time(g2)/1000:.1f} us")
    print("tuning picks:", {k: v for k, v in list(eng.tuning.items())[:5]}, "...")
    for r in sorted(rows, key=lambda r: -r["us"])[:4]:
        log = eng.tuning_log.get(r["tid"], [])
        print(f"  candidates of task {r['tid']} ({r['name']}):")
        for kind, var, split, us, err in sorted(log, key=lambda c: (c[3] is None, c[3] or 0))[:12]:
            print(f"     kind={kind} variant={var} split={split} " + (f"{us:.2f}us" if us is not None else f"FAILED {err}"))
        fails = [c for c in log if c[3] is None]
        if fails:
            print(f"     ... {len(fails)} failed, e.g. {fails[0]}")
    # the critical path itself (longest measured-duration chain)
    preds = {t.tid: sorted(t.deps) for t in eng.program.tasks}
    best, arg = {}, {}
    for tid in sw.topological_order(g):
        b, a_ = 0.0, None
        for p in preds[tid]:
            if best[p] > b:
                b, a_ = best[p], p
        best[tid] = b + per[tid]
        arg[tid] = a_
    end = max(best, key=best.get)
    chain = []
    while end is not None:
        chain.append(end)
        end = arg[end]
    chain.reverse()
    kinds = {}
    for tid in chain:
        k = eng.program.tasks[tid].kind
        kinds[k] = kinds.get(k, 0) + 1
    print(f"critical path: {len(chain)} tasks {kinds}")
    print("  " + " > ".join(f"{eng.program.tasks[t].kind}{t}({per[t]:.1f})" for t in chain[:60]))
    if a.json:
        with open(a.json, "w") as fh:
            json.dump({"rows": rows, "replay_multi_us": gm, "replay_single_us": gs,
                       "sim_multi_us": r_multi.makespan / 1000, "sim_single_us": r_single.makespan / 1000,
                       "critical_path_us": sw.critical_path_time(g2) / 1000}, fh)


if __name__ == "__main__":
    main()
