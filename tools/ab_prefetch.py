"""A/B of the L2 weight prefetch root node (SW_ENGINE_L2_PREFETCH), L2 flushed
before every replay like bench.py, and back-to-back.

    python tools/ab_prefetch.py [--config nasnet_mobile] [--batch 1]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2012_02732_b200 import _native as N  # noqa: E402
from paper_2012_02732_b200.engine import Engine  # noqa: E402
from paper_2012_02732_b200.networks import build_model, example_input  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    model, shape = build_model(a.config)
    x = example_input(shape, batch=a.batch)
    eng = Engine(model).prepare(x)
    eng.load_input_device(x)
    sh = C.c_uint64()
    N.check(N.lib().sw_engine_stream(eng._h, C.byref(sh)))
    dev = torch.device("cuda", 0)
    st = torch.cuda.ExternalStream(sh.value, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    ref = None
    for rnd in range(2):
        for on in (False, True):
            eng.l2_prefetch = on
            eng.recapture()
            eng.replay(True)
            eng.synchronize()
            y = eng.device_output().clone()
            ref = y if ref is None else ref
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
            with torch.cuda.stream(st):
                for s0, s1 in ev:
                    flush.zero_()
                    s0.record(st)
                    eng.replay(True)
                    s1.record(st)
            torch.cuda.synchronize()
            flushed = sum(s0.elapsed_time(s1) for s0, s1 in ev) / a.steps * 1e3
            warm, _ = eng.time_replay(True, 200)
            print(f"{a.config} bs{a.batch} l2_prefetch={on}: L2-flushed {flushed:.1f} us, back-to-back {warm:.1f} us, "
                  f"identical {torch.equal(y, ref)}")
    eng.close()


if __name__ == "__main__":
    main()
