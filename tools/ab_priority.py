"""A/B: critical-path tasks launched at raised priority vs default.

    python tools/ab_priority.py [--config nasnet_mobile] [--batch 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

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
    for rnd in range(2):
        eng.clear_priorities()
        base, _ = eng.time_replay(True, 300)
        for lv in (1, 3, 5):
            info = eng.critical_path_priorities(levels=lv)
            us, _ = eng.time_replay(True, 300)
            same = torch.equal(eng(x), y0)
            print(f"{a.config} bs{a.batch}: default {base:.1f} us | critical-path priority level {lv}: {us:.1f} us "
                  f"{info} identical {same}")


if __name__ == "__main__":
    main()
