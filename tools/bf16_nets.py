"""bf16 path (Engine(precision="bf16")) on the batch-1 configs: latency of the
multi-stream replay and the error of the logits against the fp32 CPU forward
(tools for DESIGN §7's stated bf16 tolerance).

    python tools/bf16_nets.py [--configs resnet50,inception_v3,nasnet_mobile]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="resnet50,inception_v3,nasnet_mobile")
    a = ap.parse_args()
    import torch
    from oracle.numerics import cpu_forward
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for name in a.configs.split(","):
        model, shape = build_model(name)
        x = example_input(shape)
        ref = cpu_forward(model, x)
        for prec in ("fp32", "bf16"):
            eng = Engine(model, precision=prec).prepare(x)
            y = eng(x)
            eng.load_input_device(x)
            ts = []
            for _ in range(30):
                flush.zero_()
                torch.cuda.synchronize()
                gpu, _ = eng.time_replay(multi=True, iters=1)
                ts.append(gpu)
            ts.sort()
            n_bf16 = sum(1 for d in eng.ops[:len(eng.program.tasks)] if 7000 <= d.variant < 8000)
            rel = ((y - ref).norm() / ref.norm()).item()
            print(f"{name} {prec}: replay {ts[len(ts) // 2]:.1f} us  bf16 tasks {n_bf16}  "
                  f"max|err| {(y - ref).abs().max().item():.3e}  rel L2 {rel:.3e}  max|ref| {ref.abs().max().item():.2f}",
                  flush=True)
            eng.close()


if __name__ == "__main__":
    main()
