"""Throughput of the conv kernels on large implicit GEMMs (roofline sanity).

    python tools/gemm_bench.py
Times one conv layer (1x1 and 3x3) at growing batch through the engine with
each kernel family forced, reporting µs and achieved TFLOP/s.
"""

from __future__ import annotations

import os
import sys

import torch
import torch.nn as nn

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2012_02732_b200 import _native as N
    from paper_2012_02732_b200.engine import Engine, K_CONV, K_CONV_TC, SP_SPLIT_K
    import ctypes as C

    cases = [(512, 512, 1, 7, 1), (512, 512, 3, 7, 1), (256, 256, 3, 14, 8), (512, 512, 1, 28, 32),
             (256, 256, 3, 56, 16), (128, 128, 3, 56, 64), (264, 88, 1, 28, 256), (1024, 1024, 1, 14, 64)]
    for cin, cout, k, hw, batch in cases:
        torch.manual_seed(0)
        # a leading 1x1 conv (task 0) so the measured layer (task 1) reads an
        # NHWC activation like every layer inside a network (the input is NCHW)
        m = nn.Sequential(nn.Conv2d(cin, cin, 1), nn.ReLU(), nn.Conv2d(cin, cout, k, padding=k // 2)).eval()
        x = torch.randn(batch, cin, hw, hw)
        flops = 2.0 * batch * hw * hw * cout * cin * k * k
        line = f"conv {cin}->{cout} k{k} {batch}x{hw}x{hw}: {flops / 1e9:.2f} GFLOP"
        eng = Engine(m, conv_impl="auto").prepare(x)
        log = eng.tuning_log.get(1, [])
        best = {}
        for kind, var, split, us, err in log:
            if us is None:
                continue
            if kind == K_CONV_TC and var >= 1000:
                kind = "tma"
            if kind not in best or us < best[kind][0]:
                best[kind] = (us, var, split)
        for kind, name in ((K_CONV, "simt"), (K_CONV_TC, "tcgen05"), ("tma", "tcgen05+TMA")):
            if kind in best:
                us, var, split = best[kind]
                line += f" | {name} {us:.1f}us ({flops / us / 1e6:.1f} TFLOP/s, v{var} s{split})"
        fails = [c for c in log if c[3] is None]
        if fails:
            line += f" | {len(fails)} failed e.g. {fails[0][:3]} {fails[0][4]}"
        print(line, flush=True)
        eng.close()


if __name__ == "__main__":
    main()
