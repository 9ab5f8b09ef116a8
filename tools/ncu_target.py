"""Small target for ncu: prepare an engine, run one eager pass + one replay.

    ncu --set full -k regex:conv_simt -c 3 python tools/ncu_target.py --config nasnet_mobile
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--conv-impl", default="simt")
    ap.add_argument("--replays", type=int, default=1)
    ap.add_argument("--eager", type=int, default=1)
    ap.add_argument("--tuning-cache", default=None)
    a = ap.parse_args()
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model, conv_impl=a.conv_impl, tuning_cache=a.tuning_cache).prepare(x)
    eng.load_input_device(x)
    for _ in range(a.eager):
        eng.run_eager(python_loop=False)
    for _ in range(a.replays):
        eng.replay(multi=True)
    eng.synchronize()
    print("tasks", len(eng.program.tasks))


if __name__ == "__main__":
    main()
