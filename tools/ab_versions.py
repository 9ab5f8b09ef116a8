"""A/B two builds of the package on the same box: NASNet bs1 replay time.

    python tools/ab_versions.py --root _ab   (one side; run alternately)
"""
import argparse
import os
import sys


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--root", default=".")
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    sys.path.insert(0, os.path.abspath(a.root))
    import paper_2012_02732_b200.engine as E
    from paper_2012_02732_b200.networks import build_model, example_input
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = E.Engine(model).prepare(x)
    eng.load_input_device(x)
    ts = [eng.time_replay(True, 300)[0] for _ in range(3)]
    print(f"{a.root}: {E.__file__} replay us {' '.join(f'{t:.1f}' for t in ts)}")


if __name__ == "__main__":
    main()
