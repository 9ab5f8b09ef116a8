"""A/B: NASNet with the two sepconvs of every separable block as one fused
K_SEP2 cluster kernel vs two K_SEPCONV tasks (same engine otherwise).

    python tools/ab_sep2.py [--batch 1]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle.numerics import cpu_forward  # noqa: E402
from paper_2012_02732_b200.engine import Engine  # noqa: E402
from paper_2012_02732_b200.networks import build_model, example_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--config", default="nasnet_mobile")
    a = ap.parse_args()
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    ref = cpu_forward(model, x) if a.batch <= 8 else None
    for fused in (False, 49, 196, 784):
        eng = Engine(model, fuse_sep_pairs=fused).prepare(x)
        y = eng(x)
        err = (y - ref).abs().max().item() if ref is not None else float("nan")
        eng.load_input_device(x)
        gm, _ = eng.time_replay(True, 300)
        gs, _ = eng.time_replay(False, 100)
        e2e = []
        xp = x.clone().pin_memory()
        for _ in range(200):
            t = time.perf_counter()
            eng(xp)
            e2e.append(time.perf_counter() - t)
        e2e.sort()
        print(f"fuse_sep_pairs={fused}: tasks {len(eng.program.tasks)} streams {eng.assignment.num_streams} "
              f"multi {gm:.1f} us single {gs:.1f} us e2e {1e6 * e2e[100]:.1f} us max|err| {err:.2e}")
        eng.close()


if __name__ == "__main__":
    main()
