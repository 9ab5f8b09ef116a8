"""Graph-level kernel selection (Engine.refine_graph): replay time per CTA cap.

    python tools/ab_graph_tune.py [--config nasnet_mobile] [--batch 1]
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
    a = ap.parse_args()
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model).prepare(x)
    eng.load_input_device(x)
    y0 = eng(x)
    before, _ = eng.time_replay(True, 200)
    res = eng.refine_graph(caps=(None, 1184, 592, 296, 148, 74))
    after, _ = eng.time_replay(True, 200)
    y1 = eng(x)
    print(json.dumps({"config": a.config, "batch": a.batch, "before_us": round(before, 2),
                      "after_us": round(after, 2), **res,
                      "max_abs_diff": float((y0 - y1).abs().max())}))


if __name__ == "__main__":
    main()
