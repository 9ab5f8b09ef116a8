"""Where the end-to-end (host tensor in → host tensor out) time goes, NASNet bs1.

    python tools/e2e_breakdown.py [--config nasnet_mobile] [--iters 200]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2012_02732_b200 import _native as N  # noqa: E402
from paper_2012_02732_b200.engine import SLOT_MULTI, SLOT_MULTI_IO, Engine  # noqa: E402
from paper_2012_02732_b200.networks import build_model, example_input  # noqa: E402


def wall(fn, iters):
    ts = []
    for _ in range(iters):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    ts.sort()
    return 1e6 * ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--tuning-cache", default=None)
    a = ap.parse_args()
    model, shape = build_model(a.config)
    x = example_input(shape)
    eng = Engine(model, tuning_cache=a.tuning_cache).prepare(x)
    lib = N.lib()
    xh = x.clone()
    xp = x.clone().pin_memory()
    for _ in range(10):
        eng(xh)
    res = {
        "engine(x) e2e (pageable x)": wall(lambda: eng(xh), a.iters),
        "engine(x) e2e (pinned x)": wall(lambda: eng(xp), a.iters),
        "host copy x -> pinned staging": wall(lambda: eng.h_in.copy_(xh.reshape(eng.h_in.shape)), a.iters),
        "replay_sync slot MULTI_IO": wall(lambda: N.check(lib.sw_engine_replay_sync(eng._h, SLOT_MULTI_IO, None)),
                                          a.iters),
        "replay_sync slot MULTI (no memcpy nodes)": wall(
            lambda: N.check(lib.sw_engine_replay_sync(eng._h, SLOT_MULTI, None)), a.iters),
        "h_out.clone()": wall(lambda: eng.h_out.clone(), a.iters),
    }
    gpu, host = eng.time_replay(True, 200, io=True)
    gpu2, _ = eng.time_replay(True, 200, io=False)
    res["device time per replay, with memcpy nodes (back-to-back)"] = gpu
    res["device time per replay, device-resident (back-to-back)"] = gpu2
    # DMA copies issued around a device-resident replay (outside the graph)
    import ctypes as C
    sh = C.c_uint64()
    N.check(lib.sw_engine_stream(eng._h, C.byref(sh)))
    st = torch.cuda.ExternalStream(sh.value)
    ho = torch.empty(eng.out_shape).pin_memory()

    def dma_step():
        with torch.cuda.stream(st):
            eng.d_in.copy_(xp.reshape(-1), non_blocking=True)
        N.check(lib.sw_engine_replay(eng._h, SLOT_MULTI))
        with torch.cuda.stream(st):
            ho.copy_(eng.device_output(), non_blocking=True)
        st.synchronize()
    res["DMA H2D + device-resident replay + DMA D2H (outside the graph)"] = wall(dma_step, a.iters)

    def h2d_only():
        with torch.cuda.stream(st):
            eng.d_in.copy_(xp.reshape(-1), non_blocking=True)
        st.synchronize()
    res["DMA H2D alone (602 KB)"] = wall(h2d_only, a.iters)
    e2 = Engine(model, tuning_cache=a.tuning_cache, kernel_io=not eng.kernel_io).prepare(x)
    for _ in range(10):
        e2(xh)
    tag = "kernel-node IO" if e2.kernel_io else "memcpy-node IO"
    res[f"[{tag}] engine(x) e2e"] = wall(lambda: e2(xh), a.iters)
    res[f"[{tag}] device time per replay with IO"] = e2.time_replay(True, 200, io=True)[0]
    ok = torch.allclose(e2(xh), eng(xh), rtol=1e-4, atol=1e-5)  # picks may differ (autotune)
    for k, v in res.items():
        print(f"{v:9.1f} us  {k}")
    print("outputs identical across IO modes:", ok)
    torch.cuda.synchronize()
    e2.close()
    eng.close()
    del st


if __name__ == "__main__":
    main()
