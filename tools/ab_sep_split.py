"""A/B: fused sepconv tasks vs separate depthwise + pointwise tasks
(Engine(fuse_separable=False): the pointwise then runs on the large-batch
tcgen05 GEMM) on NASNet-A mobile at a large batch (B200).

    python tools/ab_sep_split.py [--batch 256]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    a = ap.parse_args()
    import torch
    from oracle.numerics import cpu_forward
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input
    model, shape = build_model("nasnet_mobile")
    x = example_input(shape, batch=a.batch)
    ref = cpu_forward(model, x[:4])
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for fs in (True, False):
        eng = Engine(model, fuse_separable=fs).prepare(x)
        y = eng(x)
        err = (y[:4] - ref).abs().max().item()
        eng.load_input_device(x)
        ts = []
        for _ in range(10):
            flush.zero_()
            torch.cuda.synchronize()
            gpu, _ = eng.time_replay(multi=True, iters=1)
            ts.append(gpu)
        ts.sort()
        print(f"fuse_separable={fs}: tasks {len(eng.program.tasks)} replay {ts[len(ts) // 2]:.0f} us "
              f"({a.batch / (ts[len(ts) // 2] * 1e-6):.0f} img/s) max|err| {err:.2e}", flush=True)
        eng.close()


if __name__ == "__main__":
    main()
