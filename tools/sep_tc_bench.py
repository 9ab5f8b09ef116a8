"""One fused sepconv layer at NASNet bs256 shapes, a forced kernel variant,
timed through the engine's op timer (diagnostic; also the ncu target).

    python tools/sep_tc_bench.py --c 88 --h 14 --k 5 [--variant 100] [--batch 256]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn as nn

ap = argparse.ArgumentParser()
ap.add_argument("--c", type=int, default=88)
ap.add_argument("--h", type=int, default=14)
ap.add_argument("--k", type=int, default=5)
ap.add_argument("--s", type=int, default=1)
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--variant", type=int, default=100)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()

from paper_2012_02732_b200 import _native as N
from paper_2012_02732_b200.engine import K_SEPCONV, Engine, task_cost


class Sep(nn.Module):
    def __init__(self, c, k, s):
        super().__init__()
        self.c0 = nn.Conv2d(c, c, 1)
        self.dw = nn.Conv2d(c, c, k, s, k // 2, groups=c, bias=False)
        self.pw = nn.Conv2d(c, c, 1, bias=False)
        self.pool = nn.AvgPool2d(3, 1, 1)  # the sepconv writes an NHWC intermediate

    def forward(self, x):
        return self.pool(self.pw(self.dw(torch.relu(self.c0(x)))))


m = Sep(a.c, a.k, a.s).eval()
x = torch.randn(a.batch, a.c, a.h, a.h)
eng = Engine(m, conv_impl="simt").prepare(x)
idx = [i for i, d in enumerate(eng.ops) if d.kind == K_SEPCONV][0]
d = eng.ops[idx]
d.variant = a.variant
us = C.c_double()
N.check(N.lib().sw_engine_time_op(eng._h, C.byref(d), a.reps, C.byref(us)))
mb = task_cost(eng.program.tasks[idx])[1] / 1e6
print(f"sepconv C={a.c} h={a.h} k={a.k} s={a.s} batch={a.batch} variant={a.variant}: "
      f"{us.value:.1f} us  {mb / us.value * 1e3:.0f} GB/s ({mb:.1f} MB)")
