"""ncu target: one pointwise conv forced onto a tcgen05 variant.

    ncu --set full -k regex:conv_tc -c 1 python tools/tc_target.py --variant 1128 --split 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.nn as nn  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cin", type=int, default=1024)
    ap.add_argument("--cout", type=int, default=1024)
    ap.add_argument("--hw", type=int, default=14)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--variant", type=int, default=1128)
    ap.add_argument("--split", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--kind", type=int, default=6, help="6 = tcgen05, 1 = SIMT")
    ap.add_argument("--tail", action="store_true",
                    help="append a 1x1 conv so the tested conv writes an NHWC activation (not the NCHW output)")
    a = ap.parse_args()
    from paper_2012_02732_b200 import _native as N
    from paper_2012_02732_b200.engine import Engine, K_CONV_TC, SP_SPLIT_K, SLOT_MULTI
    layers = [nn.Conv2d(a.cin, a.cin, 1), nn.ReLU(), nn.Conv2d(a.cin, a.cout, a.k, padding=a.k // 2)]
    if a.tail:
        layers.append(nn.Conv2d(a.cout, 8, 1))
    m = nn.Sequential(*layers).eval()
    x = torch.randn(a.batch, a.cin, a.hw, a.hw)
    eng = Engine(m, conv_impl="tc").prepare(x)
    d = eng.ops[1]
    assert d.kind == K_CONV_TC
    d.kind = a.kind
    d.variant = a.variant
    d.params[SP_SPLIT_K] = a.split
    N.check(N.lib().sw_engine_set_ops(eng._h, len(eng.program.tasks), eng.ops))
    eng._capture(SLOT_MULTI, eng.schedule, False)
    eng.load_input_device(x)
    for _ in range(a.reps):
        eng.replay(True)
    eng.synchronize()
    gpu, _ = eng.time_replay(True, 20)
    flops = 2.0 * a.batch * a.hw * a.hw * a.cin * a.cout * a.k * a.k
    print(f"replay (both convs) {gpu:.1f} us; layer {flops / 1e9:.2f} GFLOP")


if __name__ == "__main__":
    main()
