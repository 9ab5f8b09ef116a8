"""Autotuner candidate times per fused-sepconv shape class (diagnostic):
the tcgen05 variant (100) against the best CUDA-core variant.

    python tools/sep_candidates.py [--batch 256]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=256)
ap.add_argument("--config", default="nasnet_mobile")
a = ap.parse_args()

from paper_2012_02732_b200.engine import SEP_TC_VARIANT, SP_C, SP_P, SP_R, SP_STRIDE_H, SP_K, Engine, task_cost
from paper_2012_02732_b200.networks import build_model, example_input

model, shape = build_model(a.config)
x = example_input(shape, batch=a.batch)
eng = Engine(model).prepare(x)
cls = {}
for t in eng.program.tasks:
    if t.kind != "sepconv":
        continue
    p = eng.ops[t.tid].params
    key = (p[SP_C], p[SP_K], p[SP_P], p[SP_R], p[SP_STRIDE_H])
    log = eng.tuning_log.get(t.tid, [])
    tc = [c[3] for c in log if c[1] == SEP_TC_VARIANT and c[3] is not None]
    other = [c[3] for c in log if c[1] != SEP_TC_VARIANT and c[3] is not None]
    mb = task_cost(t)[1] / 1e6
    c = cls.setdefault(key, [0, 0.0, 0.0, 0.0, None])
    c[0] += 1
    c[1] += tc[0] if tc else float("nan")
    c[2] += min(other) if other else float("nan")
    c[3] += mb
    c[4] = eng.tuning.get(t.tid)
print("class (C, K, P, k, s): n, tcgen05 us/launch, best CUDA-core us/launch, tcgen05 GB/s, pick")
for k, (n, tc, oth, mb, pick) in sorted(cls.items(), key=lambda kv: -kv[1][2]):
    print(f"{k}: n={n} tc={tc / n:8.1f} cuda={oth / n:8.1f}  tc {mb / tc * 1e3:7.0f} GB/s  pick={pick[1:] if pick else None}")
rej = {k: v for k, v in eng.tuning_rejected.items() if v}
print("rejected candidates:", {k: [(c, f'{e:.2e}') for c, e in v] for k, v in list(rej.items())[:10]})
