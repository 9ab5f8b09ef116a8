"""A/B of the captured graph's edge types (same topology): PDL on same-stream
edges only vs PDL on every kernel -> kernel edge (SW_ENGINE_PDL_ALL_EDGES).

    python tools/ab_edges.py [--config nasnet_mobile] [--batch 1]
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
    ap.add_argument("--tuning-cache", default=None)
    a = ap.parse_args()
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model, tuning_cache=a.tuning_cache).prepare(x)
    eng.load_input_device(x)
    ref = None
    for rnd in range(2):
        for flag in (False, True):
            eng.pdl_all_edges = flag
            eng.recapture()
            eng.replay(True)
            eng.synchronize()
            y = eng.device_output().clone()
            if ref is None:
                ref = y
            same = torch.equal(y, ref)
            gm, _ = eng.time_replay(True, 300)
            ge, _ = eng.time_replay(True, 300, io=True)
            e2e = []
            import time
            for _ in range(100):
                t = time.perf_counter()
                eng(x)
                e2e.append(time.perf_counter() - t)
            e2e.sort()
            print(f"{a.config} bs{a.batch} all_edges={flag}: replay {gm:.1f} us, with IO {ge:.1f} us, "
                  f"e2e median {1e6 * e2e[50]:.1f} us, output bit-identical {same}")


if __name__ == "__main__":
    main()
