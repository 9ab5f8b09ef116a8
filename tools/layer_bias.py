"""Per-layer error of a prepared engine's tcgen05 picks against the SIMT fp32
reference kernel on the same random arena: max and rms relative error, and the
mean signed error (the tensor pipe's truncating fp32 accumulate shows up as a
negative bias that grows with the length of a TMEM accumulation chain;
profiles/r04_tmem_chain_bias.txt).  GPU box:

    python tools/layer_bias.py inception_v3
"""

from __future__ import annotations

import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2012_02732_b200.engine as E
    from paper_2012_02732_b200 import _native as N
    from paper_2012_02732_b200.networks import build_model, example_input

    name = sys.argv[1] if len(sys.argv) > 1 else "inception_v3"
    model, shape = build_model(name)
    x = example_input(shape)
    eng = E.Engine(model).prepare(x)
    lib = N.lib()
    gen = torch.Generator(device=eng.arena.device).manual_seed(7)
    words = eng.arena.numel() // 4
    for t in eng.program.tasks:
        d = eng.ops[t.tid]
        if d.kind != E.K_CONV_TC:
            continue
        rc = eng._reference_candidate(t, d)
        trial = N.OpDesc()
        C.memmove(C.byref(trial), C.byref(d), C.sizeof(N.OpDesc))
        eng.arena[:words * 4].view(torch.float32).normal_(generator=gen)
        trial.kind, trial.variant = rc[0], rc[1]
        trial.params[E.SP_SPLIT_K] = rc[2]
        N.check(lib.sw_engine_run_op(eng._h, C.byref(trial)))
        ref = eng._out_tensor(t).clone().double()
        C.memmove(C.byref(trial), C.byref(d), C.sizeof(N.OpDesc))
        N.check(lib.sw_engine_run_op(eng._h, C.byref(trial)))
        y = eng._out_tensor(t).double()
        e = (y - ref).abs()
        p = d.params
        print(f"{t.name:40s} v{d.variant} split {p[E.SP_SPLIT_K]} M={p[E.SP_N] * p[E.SP_P] * p[E.SP_Q]} "
              f"K={p[E.SP_K]} C={p[E.SP_C]} RS={p[E.SP_R]}x{p[E.SP_S]} s={p[E.SP_STRIDE_H]} "
              f"maxerr/max {e.max().item() / ref.abs().max().item():.2e} "
              f"rms_rel {(e.pow(2).mean() / ref.pow(2).mean()).sqrt().item():.2e} "
              f"bias {((y - ref).mean() / ref.abs().mean()).item():+.2e}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
