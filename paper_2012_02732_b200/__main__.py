"""Command line over the engine (the reference's `compare` and
`export-trace` subcommands, cli.py:178-240, measured on the device instead of
simulated):

    python -m paper_2012_02732_b200 compare --config nasnet_mobile [--batch 1] [--iters 50]
    python -m paper_2012_02732_b200 export-trace --config nasnet_mobile --out trace.json [--single]
    python -m paper_2012_02732_b200 assign graph.json          # planner only (no GPU)
    python -m paper_2012_02732_b200 verify graph.json [--assignment a.json]   # cli.py:189-203

`compare` prints the 4-mode matrix as JSON: (framework | replay) x (single |
multi), where framework = the pre_run schedule issued op by op by the host
each iteration and replay = one launch of the captured CUDA graph.
"""

from __future__ import annotations

import argparse
import json
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2012_02732_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("compare", help="measured 4-mode matrix of a network")
    c.add_argument("--config", default="nasnet_mobile")
    c.add_argument("--batch", type=int, default=1)
    c.add_argument("--iters", type=int, default=50)
    t = sub.add_parser("export-trace", help="measured Chrome trace of one replay")
    t.add_argument("--config", default="nasnet_mobile")
    t.add_argument("--batch", type=int, default=1)
    t.add_argument("--single", action="store_true")
    t.add_argument("--out", required=True)
    a = sub.add_parser("assign", help="stream assignment of a graph JSON (reference format)")
    a.add_argument("graph")
    v = sub.add_parser("verify", help="check sync minimality exhaustively (<= 7 nodes)")
    v.add_argument("graph")
    v.add_argument("--assignment", help="verify this assignment instead")
    args = ap.parse_args(argv)

    import paper_2012_02732_b200 as sw
    if args.cmd == "assign":
        with open(args.graph) as fh:
            g = sw.graph_from_json(fh.read())
        f, plan = sw.assign_streams(g)
        print(sw.assignment_to_json(g, f, plan, sw.minimum_equivalent_graph(g)))
        return 0
    if args.cmd == "verify":
        # exit codes as the reference CLI (cli.py:336-351): 4 too large, 5 violation
        with open(args.graph) as fh:
            g = sw.graph_from_json(fh.read())
        try:
            if args.assignment:
                with open(args.assignment) as fh:
                    f, plan = sw.assignment_from_json(fh.read(), g)
                rep = sw.verify_given(g, f, plan)
            else:
                rep = sw.verify_optimal(g)
        except sw.TooLarge as e:
            print(f"TooLarge: {e}", file=sys.stderr)
            return 4
        print(rep.to_json())
        if not rep.optimal:
            print(f"OptimalityViolation: algo_syncs={rep.algo_syncs} oracle_min={rep.oracle_min}",
                  file=sys.stderr)
            return 5
        return 0
    from .engine import Engine
    from .networks import build_model, example_input
    model, shape = build_model(args.config)
    x = example_input(shape, batch=args.batch)
    eng = Engine(model).prepare(x)
    eng.load_input_device(x)
    try:
        if args.cmd == "compare":
            rep = eng.compare(iters=args.iters)
            rep.update({"config": args.config, "batch": args.batch, "unit": "us per iteration"})
            print(json.dumps(rep))
        else:
            _, js = eng.trace(multi=not args.single)
            with open(args.out, "w") as fh:
                fh.write(js)
            print(f"wrote {args.out}")
    finally:
        eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
