"""Per contraction task of a prepared engine: the fastest tcgen05 candidate vs
the fastest CUDA-core (FFMA) candidate the autotuner timed, and which won
(why the batch-1 NASNet replay runs few tcgen05 kernels).  GPU box:

    python tools/tc_vs_simt_picks.py --config nasnet_mobile [--batch 1]
"""

from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    a = ap.parse_args()
    import paper_2012_02732_b200.engine as E
    from paper_2012_02732_b200.networks import build_model, example_input
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = E.Engine(model).prepare(x)
    tc_fam = (E.K_CONV_TC,)
    rows = []
    for t in eng.program.tasks:
        log = [c for c in eng.tuning_log.get(t.tid, []) if c[3] is not None]
        if not log or t.kind not in ("conv", "sepconv"):
            continue
        tc = [c for c in log if c[0] in tc_fam or (t.kind == "sepconv" and c[1] == E.SEP_TC_VARIANT)]
        cc = [c for c in log if c not in tc]
        bt = min(tc, key=lambda c: c[3]) if tc else None
        bc = min(cc, key=lambda c: c[3]) if cc else None
        d = eng.ops[t.tid]
        rows.append((t.name, t.kind, bt, bc, (d.kind, d.variant, d.params[E.SP_SPLIT_K])))
    n_tc = sum(1 for r in rows if r[4][0] in tc_fam)
    print(f"{a.config} bs{a.batch}: {len(rows)} tuned contraction tasks, {n_tc} picked a tcgen05 kernel")
    print(f"{'task':44s} {'kind':8s} {'best tcgen05 (us)':>18s} {'best FFMA (us)':>15s}  pick")
    for name, kind, bt, bc, pick in rows:
        ft = f"{bt[3]:.2f} v{bt[1]}/{bt[2]}" if bt else "-"
        fc = f"{bc[3]:.2f} v{bc[1]}/{bc[2]}" if bc else "-"
        print(f"{name[:44]:44s} {kind:8s} {ft:>18s} {fc:>15s}  {pick}")
    eng.close()


if __name__ == "__main__":
    main()
