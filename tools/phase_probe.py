"""Where does a batch-1 kernel's time go?  Phase stamps from the diagnostic
build (libsw_b200_probe.so, `python -m paper_2012_02732_b200.build --probe`).

    python tools/phase_probe.py --config nasnet_mobile --kinds sepconv,conv --limit 12

Each selected task runs as a graph-captured chain of `--reps` launches (the
way time_op / the autotuner time it).  Printed per task:
  * launch: mean first-CTA-start → last-CTA-end span, and the mean gap from
    one launch's end to the next one's start (negative = PDL overlap);
  * phases of CTA (0,0,0) in the last launch, µs after its start:
    1 constants issued, 2 PDL wait returned, 3 first operands in smem,
    4 main loop / depthwise done, 5 GEMM done, 15 CTA end (clock64 → µs at --sm-mhz).
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SW_B200_LIB", os.path.join(ROOT, "paper_2012_02732_b200", "libsw_b200_probe.so"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--kinds", default="sepconv,conv")
    ap.add_argument("--tasks", default=None, help="comma-separated task ids")
    ap.add_argument("--limit", type=int, default=12)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--tuning-cache", default=None)
    ap.add_argument("--no-pdl", action="store_true", help="time the chains without programmatic dependent launch")
    ap.add_argument("--sm-mhz", type=float, default=1965.0, help="SM clock for the clock64 phase stamps")
    ap.add_argument("--force", default=None, help="kind,variant,split to time instead of the tuned pick")
    a = ap.parse_args()

    import numpy as np

    from paper_2012_02732_b200 import _native as N
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input

    lib = N.lib()
    lib.sw_probe_reset.restype = C.c_int
    lib.sw_probe_read.restype = C.c_int
    lib.sw_probe_read.argtypes = [C.POINTER(C.c_uint64)]

    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model, tuning_cache=a.tuning_cache).prepare(x)
    if a.no_pdl:
        N.check(lib.sw_engine_set_flags(eng._h, 0))
    per = eng.profile_tasks(reps=20)
    if a.tasks:
        tids = [int(t) for t in a.tasks.split(",")]
    else:
        kinds = set(a.kinds.split(","))
        cand = [t for t in eng.program.tasks if t.kind in kinds]
        cand.sort(key=lambda t: -per[t.tid])
        tids = [t.tid for t in cand[: a.limit]]
    buf = (C.c_uint64 * 128)()
    for tid in tids:
        t = eng.program.tasks[tid]
        d = eng.ops[tid]
        if a.force:
            fk, fv, fs = (int(v) for v in a.force.split(","))
            d.kind, d.variant = fk, fv
            d.params[30] = fs  # SP_SPLIT_K
        lib.sw_probe_reset()
        us = C.c_double()
        N.check(lib.sw_engine_time_op(eng._h, C.byref(d), a.reps, C.byref(us)))
        lib.sw_probe_read(buf)
        v = np.array(buf[:], dtype=np.float64)
        nl = 2 * a.reps + 1  # validation launch + warm graph + timed graph
        ctas = int(v[48]) // nl
        starts, ends = v[16:32], v[32:48]
        timed = [i % 16 for i in range(a.reps + 1, nl)]  # the timed graph's launches
        spans = [(ends[i] - starts[i]) / 1e3 for i in timed]
        gaps = [(starts[j] - ends[i]) / 1e3 for i, j in zip(timed[:-1], timed[1:])]
        pts = v[:16]
        ph = {i: (pts[i] - pts[0]) / (a.sm_mhz * 1e-3) / 1e3 for i in range(1, 16) if pts[i]}
        print(f"task {tid:4d} {t.kind:7s} k=({d.kind},{d.variant},split {d.params[30]}) "
              f"time_op {us.value:6.2f}us  span {np.mean(spans) if spans else 0:6.2f}us "
              f"gap {np.mean(gaps) if gaps else 0:+6.2f}us  CTAs {ctas}  "
              f"{t.name}")
        print("        phases(us): " + "  ".join(f"{i}:{p:.2f}" for i, p in sorted(ph.items())))
        tr = v[64:128]
        if tr.any():
            print("        trace(us):  " + "  ".join(f"{i}:{(tr[i] - pts[0]) / (a.sm_mhz * 1e-3) / 1e3:.2f}"
                                                   for i in range(64) if tr[i]))



if __name__ == "__main__":
    main()
