"""Per-impl parity diagnostic: max |GPU - CPU fp32| and |GPU - CPU fp64| for
each conv_impl, plus the worst task by comparing every task's output slice
with the fp64 module's intermediate (fx ShapeProp-free: hooks on modules)."""
import copy
import sys

import torch

sys.path.insert(0, ".")
from oracle.numerics import cpu_forward
from paper_2012_02732_b200.engine import Engine
from paper_2012_02732_b200.networks import build_model, example_input

name = sys.argv[1] if len(sys.argv) > 1 else "inception_v3"
m, shape = build_model(name)
x = example_input(shape)
ref = cpu_forward(m, x)
m64 = copy.deepcopy(m).double()
with torch.no_grad():
    r64 = m64(x.double())
for impl in ("simt", "tc", "auto"):
    eng = Engine(m, conv_impl=impl).prepare(x)
    y = eng(x).cpu()
    e32 = (y - ref).abs()
    e64 = (y.double() - r64).abs()
    viol = (e32 > 1e-4 + 1e-3 * ref.abs()).sum().item()
    print(f"{name} {impl}: max|y-ref32| {e32.max():.3e} max|y-ref64| {e64.max():.3e} viol {viol}", flush=True)
    if impl == "auto":
        kinds = {}
        for tid, b in eng.tuning.items():
            kinds[(b[1], b[2], b[3])] = kinds.get((b[1], b[2], b[3]), 0) + 1
        print("picks", kinds)
    eng.close()
