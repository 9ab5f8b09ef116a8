"""A/B: physical-stream cap (fold_streams, assign.py:243-270) on the
multi-stream replay of a network (B200).

    python tools/ab_fold.py --config nasnet_mobile [--batch 1] [--caps 4,8,16,32,0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--caps", default="4,8,16,24,32,48,0")
    ap.add_argument("--tuning-cache", default="/tmp/sw_ab_fold_tune.json")
    a = ap.parse_args()
    import torch
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for cap in [int(c) for c in a.caps.split(",")]:
        eng = Engine(model, max_streams=cap or None, tuning_cache=a.tuning_cache).prepare(x)
        y = eng(x)
        eng.load_input_device(x)
        times = []
        for _ in range(3):
            eng.replay(multi=True)
        torch.cuda.synchronize()
        for _ in range(100):
            flush.zero_()
            torch.cuda.synchronize()
            gpu, _ = eng.time_replay(multi=True, iters=1)
            times.append(gpu)
        times.sort()
        print(f"cap {cap or 'none':>4}: streams {eng.assignment.num_streams:3d} syncs {len(eng.plan):3d}  "
              f"replay median {times[len(times) // 2]:.1f} us  min {times[0]:.1f} us", flush=True)
        eng.close()


if __name__ == "__main__":
    main()
