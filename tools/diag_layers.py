"""Per-task kernel agreement: every conv task of a net, each tcgen05
candidate vs the SIMT reference candidate on the same seeded arena, error
relative to max|ref| (diagnostic)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_02732_b200 import _native as N
from paper_2012_02732_b200.engine import (Engine, K_CONV_TC, SP_K, SP_N, SP_P, SP_Q, SP_R, SP_S, SP_C,
                                          SP_SPLIT_K, conv_candidates, SP_PAD_H, SP_PAD_W)
from paper_2012_02732_b200.networks import build_model, example_input

name = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
m, shape = build_model(name)
x = example_input(shape)
eng = Engine(m, conv_impl="simt").prepare(x)
lib = N.lib()
gen = torch.Generator(device=eng.arena.device).manual_seed(1234)
words = eng.arena.numel() // 4
eng.arena[: 4 * words].view(torch.float32).uniform_(0, 1, generator=gen)
rows = []
for t in eng.program.tasks:
    if t.kind != "conv":
        continue
    d = eng.ops[t.tid]
    p = d.params
    M = p[SP_N] * p[SP_P] * p[SP_Q]
    Kdim = p[SP_R] * p[SP_S] * p[SP_C]
    trial = N.OpDesc()
    C.memmove(C.byref(trial), C.byref(d), C.sizeof(N.OpDesc))
    N.check(lib.sw_engine_run_op(eng._h, C.byref(trial)))
    ref = eng._out_tensor(t).double().clone()
    scale = ref.abs().max().item()
    for kind, v, split in conv_candidates(M, p[SP_K], Kdim, p[SP_R], p[SP_S], (p[SP_PAD_H], p[SP_PAD_W])):
        if kind != K_CONV_TC:
            continue
        trial.kind, trial.variant = kind, v
        trial.params[SP_SPLIT_K] = split
        eng._out_tensor(t).fill_(float("nan"))
        if lib.sw_engine_run_op(eng._h, C.byref(trial)) != 0:
            continue
        err = (eng._out_tensor(t).double() - ref).abs().max().item() / max(scale, 1e-30)
        rows.append((err, t.tid, t.name, v, split, M, p[SP_K], Kdim))
rows.sort(reverse=True)
for r in rows[:25]:
    print("err/max %.3e  task %d %s  variant %d split %d  M %d N %d K %d" % r)
print("median", sorted(r[0] for r in rows)[len(rows) // 2])
