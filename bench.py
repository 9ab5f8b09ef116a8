"""Benchmark: Nimble-style AoT engine on B200 vs the reference CPU path.

    python bench.py [--gpus N --steps K --warmup W] [--config nasnet_mobile --batch 1]
    python bench.py --impl reference ...        # the CPU path, same metric

Workload (BASELINE.json north_star target): NASNet-A mobile, batch-1 fp32
inference, multi-stream AoT CUDA-graph replay.  One step = one forward pass
of one batch per GPU.  Multi-GPU = independent replicas (batch-1 latency does
not shard), one process per GPU under torchrun, weak scaling.
At N > 1 the line also carries the configs that do shard: NASNet-A mobile
bs256 batch-sharded 256/N per rank (replicas, max-over-ranks device time)
and MobileNetV2 / EfficientNet-B0 data-parallel training with the captured
NCCL gradient allreduce (bs32 per rank).

Printed JSON (rank 0): value = whole-job images/s with the input already in
HBM (device-resident replay, L2 flushed between steps); e2e = the same metric
through the public API call engine(x_host) (pinned H2D + graph + D2H inside
the timed region).  Extra keys: batch-1 latency, the same engine's
single-stream AoT replay and non-AoT eager launch loop, host launch overhead
per iteration and its fraction of GPU time, Σ per-kernel roofline, roofline
object for the dominant kernel family, CPU baseline, clocks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "batch-1 inference latency (µs) + images/s on 1/2/4/8 B200; vs ref CPU path"
UNIT = "images/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured (MEASURED_PEAKS.json)"
    return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def load_fp32_peaks():
    """fp32 compute peaks measured on a B200 of this pool (tools/peaks_fp32.cu
    → profiles/peaks_fp32.json): FFMA, and the fp32-accurate tensor-core rate
    (tcgen05 kind::tf32 / 3, the 3xTF32 split every contraction here uses)."""
    with open(os.path.join(ROOT, "profiles", "peaks_fp32.json")) as fh:
        d = json.load(fh)
    return float(d["ffma_fp32_tflops"]), float(d["tcgen05_3xtf32_effective_tflops"])


def roofline_sum_fp32(eng, hbm):
    """Σ per task max(flops / P, bytes / BW) at fp32: contractions (dense /
    1x1 conv, the sepconv pointwise) at the 3xTF32 tensor-core peak, the
    depthwise / pool / elementwise flops at the FFMA peak."""
    from paper_2012_02732_b200.engine import task_cost
    ffma, tc3 = load_fp32_peaks()
    total = 0.0
    for t in eng.program.tasks:
        f, b = task_cost(t)
        if t.kind == "sepconv":
            R, S = t.node.attrs["k"]
            pix = t.out.st.n * t.out.st.h * t.out.st.w
            c = t.inputs[0].c
            dwf = 2.0 * pix * c * R * S
            tf = dwf / (ffma * 1e12) + (f - dwf) / (tc3 * 1e12)
        elif t.kind == "conv":
            tf = f / (tc3 * 1e12)
        else:
            tf = f / (ffma * 1e12)
        total += max(tf, b / (hbm * 1e9)) * 1e6
    return total


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/sw_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[5:9]):
                if flag.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if torch.cuda.is_available() and torch.cuda.device_count() > 0:
        # one GPU per rank; more ranks than GPUs (a plumbing check on a 1-GPU
        # box with SW_DIST_BACKEND=gloo) share devices round-robin
        local = local % torch.cuda.device_count()
    if world > 1:
        backend = os.environ.get("SW_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend, init_method="env://")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_max(world, value, device=None):
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = None  # gloo reduces host tensors
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------
# reference arm: the CPU path (oracle restatement) on the host cores
# ----------------------------------------------------------------------------

def cpu_path_run(config, batch, steps, warmup, threads):
    """The reference CPU path for this workload (SURVEY §8(d) mode 4): the
    planner restatement (assign_streams + pre_run, oracle/planner.py, run once
    as the reference does at prepare time) and the fp32 CPU forward of the same
    module (oracle/numerics.py) per step."""
    import torch
    from oracle import planner as O
    from oracle.numerics import cpu_forward
    from paper_2012_02732_b200.networks import build_model, example_input
    from paper_2012_02732_b200.trace import build_program

    torch.set_num_threads(threads)
    model, shape = build_model(config)
    x = example_input(shape, batch=batch)
    prog = build_program(model, x, fuse=True)
    g = prog.graph
    nodes = [(t.id, t.duration, t.demand, tuple((e.kind, e.size) for e in t.mem)) for t in g.nodes]
    t0 = time.perf_counter()
    f, plan, _ = O.assign(nodes, list(g.edges))
    O.pre_run(nodes, list(g.edges), f, plan)
    plan_s = time.perf_counter() - t0
    for _ in range(warmup):
        cpu_forward(model, x)
    times = []
    for _ in range(steps):
        t = time.perf_counter()
        cpu_forward(model, x)
        times.append(time.perf_counter() - t)
    return times, plan_s


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle.numerics import cpu_threads
    threads = cpu_threads()
    times, plan_s = cpu_path_run(args.config, args.batch, args.steps, args.warmup, threads)
    mean = sum(times) / len(times)
    value = args.batch / mean
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(mean * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded randn input, random-init weights)",
        "config": {"workload": f"{args.config} batch-{args.batch} fp32 inference, CPU path",
                   "batch_per_replica": args.batch},
        "latency_us": round(mean * 1e6, 1),
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.steps} forward passes of {args.config} bs{args.batch} "
                                   f"(torch CPU fp32, same module) + one oracle planner pass "
                                   f"({plan_s * 1e3:.1f} ms)"},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "planner_ms": round(plan_s * 1e3, 3),
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

def run_ours(args, world, rank, local):
    import torch
    from paper_2012_02732_b200 import _native as N
    from paper_2012_02732_b200.engine import Engine, task_cost
    from paper_2012_02732_b200.networks import build_model, example_input
    import ctypes as C

    hbm, bf16, peak_src = load_peaks()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    model, shape = build_model(args.config)
    x = example_input(shape, batch=args.batch, seed=1 + rank)
    eng = Engine(model, multi_stream=True, device=local,
                 tuning_cache=args.tuning_cache).prepare(x)
    # correctness gate before timing (cheap at batch 1)
    y = eng(x)
    parity = None
    if rank == 0 and args.batch <= 8:
        from oracle.numerics import cpu_forward
        ref = cpu_forward(model, x)
        err = (y - ref).abs().max().item()
        parity = {"max_abs_err": err, "ok": bool(torch.allclose(y, ref, rtol=1e-3, atol=1e-4))}

    sh = C.c_uint64()
    N.check(N.lib().sw_engine_stream(eng._h, C.byref(sh)))
    stream = torch.cuda.ExternalStream(sh.value, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    eng.load_input_device(x)

    def timed_replays(multi, steps):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        with torch.cuda.stream(stream):
            for a, b in ev:
                flush.zero_()
                a.record(stream)
                eng.replay(multi=multi)
                b.record(stream)
        torch.cuda.synchronize(dev)
        return [a.elapsed_time(b) for a, b in ev]

    for _ in range(args.warmup):
        eng.replay(multi=True)
        eng.replay(multi=False)
    torch.cuda.synchronize(dev)
    barrier(world)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    times = timed_replays(True, args.steps)
    torch.cuda.synchronize(dev)
    barrier(world)
    clock_info = clocks.stop()
    ms = sum(times) / len(times)
    ms_max = reduce_max(world, ms, dev)
    value = world * args.batch / (ms_max / 1e3)

    # same engine, other modes (same flush discipline)
    single = timed_replays(False, args.steps)
    single_ms = sum(single) / len(single)
    # the same multi-stream graph captured without programmatic dependent launch
    eng.recapture(pdl=not eng.pdl)
    for _ in range(3):
        eng.replay(multi=True)
    alt = timed_replays(True, args.steps)
    alt_ms = sum(alt) / len(alt)
    eng.recapture(pdl=not eng.pdl)

    def eager_once():
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        eng.run_eager(python_loop=True)
        eng.synchronize()
        return time.perf_counter() - t

    for _ in range(3):
        eager_once()
    eager = [eager_once() for _ in range(max(5, args.steps // 4))]
    eager_ms = 1e3 * sum(eager) / len(eager)

    def framework_multi_once():
        # framework mode, multi-stream: the schedule issued op by op with real
        # event record / wait on the logical streams (sim.py:69-80 analogue)
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        eng.run_framework(multi=True)
        eng.synchronize()
        return time.perf_counter() - t

    for _ in range(3):
        framework_multi_once()
    fw = [framework_multi_once() for _ in range(max(5, args.steps // 4))]
    fw_multi_ms = 1e3 * sum(fw) / len(fw)

    # e2e through the public API: host tensor in (pinned host memory, as the
    # contract's e2e specifies; copied into the engine's pinned staging buffer
    # inside the call), host tensor out
    xh = x.clone().pin_memory()
    for _ in range(3):
        eng(xh)
    e2e_times = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        eng(xh)
        e2e_times.append(time.perf_counter() - t)
    e2e_ms = 1e3 * sum(e2e_times) / len(e2e_times)
    e2e_ms_max = reduce_max(world, e2e_ms, dev)

    # serving path: K requests through engine.infer_stream (one call; request
    # i+1's H2D under request i's replay, every request's H2D and D2H inside
    # the timed region; weights stay in L2 across requests, as in serving)
    xs_stream = [x.clone().contiguous().pin_memory() for _ in range(args.steps)]
    outs_stream = [torch.empty(eng.out_shape, dtype=torch.float32, pin_memory=True) for _ in xs_stream]
    eng.infer_stream(xs_stream[:3], outs_stream[:3])
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    eng.infer_stream(xs_stream, outs_stream)
    stream_ms = 1e3 * (time.perf_counter() - t) / len(xs_stream)
    stream_ms_max = reduce_max(world, stream_ms, dev)
    assert torch.equal(outs_stream[-1], eng(xh)), "infer_stream result differs from engine(x)"

    # host launch overhead per iteration: (a) the cudaGraphLaunch call timed
    # in C (sw_engine_time_replay), (b) the whole Python → C-ABI call
    # `eng.replay(multi=True)`, back to back so the host never
    # waits on the device
    gpu_us, host_us = eng.time_replay(multi=True, iters=200)
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    for _ in range(200):
        eng.replay(multi=True)
    py_us = (time.perf_counter() - t) / 200 * 1e6
    torch.cuda.synchronize(dev)

    # dominant kernel family, two per-launch durations:
    #  * in_replay: every task bracketed by timing events inside one replay of
    #    the multi-stream graph after the same 512 MB L2 flush as the timed
    #    steps (Engine.trace; the event nodes add per-task overhead, so this
    #    under-states the kernels' own speed);
    #  * warm_isolated: each task as a graph-captured chain of back-to-back
    #    launches of itself (warm L2), the autotuner's measurement.
    per_task = eng.profile_tasks(reps=10)

    def flush_on_stream():
        with torch.cuda.stream(stream):
            flush.zero_()

    iv, _ = eng.trace(multi=True, before_last=flush_on_stream)
    fam = {}
    for t in eng.program.tasks:
        f_, b_ = task_cost(t)
        k = t.kind
        d = fam.setdefault(k, {"us": 0.0, "trace_us": 0.0, "flops": 0.0, "bytes": 0.0, "n": 0})
        d["us"] += per_task[t.tid]
        d["trace_us"] += iv[t.tid][1] - iv[t.tid][0] if t.tid in iv else 0.0
        d["flops"] += f_
        d["bytes"] += b_
        d["n"] += 1
    # simulator in the loop: the reference replay semantics
    # fed with the measured per-task durations (ns), zero submission overhead
    import paper_2012_02732_b200 as swpkg
    g0 = eng.graph
    gd = swpkg.CompGraph.build(
        [swpkg.TaskNode(n.id, max(1, int(round(per_task[n.id] * 1000))), 1, n.label, n.mem)
         for n in g0.nodes], g0.edges)
    fd, pd = swpkg.assign_streams(gd)
    sim_multi = swpkg.simulate(swpkg.pre_run(gd, fd, pd), gd, swpkg.SimConfig()).makespan / 1000
    sim_single = sum(per_task)
    crit = swpkg.critical_path_time(gd) / 1000
    dom = max(fam, key=lambda k: fam[k]["trace_us"])
    dd = fam[dom]
    bytes_per_launch = dd["bytes"] / dd["n"]
    launch_in_replay = dd["trace_us"] / dd["n"]
    launch_warm = dd["us"] / dd["n"]
    achieved = bytes_per_launch / (launch_in_replay * 1e-6) / 1e9
    # DRAM bytes per launch of this family from the committed ncu --set full
    # capture (profiles/traffic.json, written by tools/ncu_summary.py --traffic)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            traffic = json.load(fh).get(dom)
    roof_sum = roofline_sum_fp32(eng, hbm)
    ffma_peak, tc3_peak = load_fp32_peaks()

    extra = None
    if not args.skip_extra:
        if world == 1:
            if rank == 0:
                extra = other_configs(args, dev, hbm, flush, stream)
        else:
            extra = sharded_big_batch(args, dev, hbm, flush, world, rank)
    training = None
    if not args.skip_train:
        try:
            training = train_configs(args, dev, world, rank)
        except Exception as e:  # noqa: BLE001 — report, do not lose the inference line
            training = {"error": f"{type(e).__name__}: {e}"}

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.skip_cpu:
            from oracle.numerics import cpu_threads
            thr = cpu_threads()
            nsteps = max(3, int(args.cpu_seconds / 0.05))
            t0 = time.perf_counter()
            ct, plan_s = cpu_path_run(args.config, args.batch, nsteps, 2, thr)
            cpu_val = args.batch / (sum(ct) / len(ct))
            cpu = {"value": round(cpu_val, 3), "unit": UNIT, "cores": thr, "kind": "port",
                   "cpu_model": cpu_model(),
                   "sample": f"{nsteps} fp32 CPU forwards of {args.config} bs{args.batch} "
                             f"(same module; oracle/numerics.py) + oracle planner "
                             f"{plan_s * 1e3:.1f} ms; {time.perf_counter() - t0:.1f} s total"}
        n_tasks = len(eng.program.tasks)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded randn input, random-init weights, randomized BN stats)",
            "config": {"workload": f"{args.config} batch-{args.batch} fp32 inference, "
                                   f"multi-stream AoT CUDA-graph replay",
                       "batch_per_replica": args.batch, "replicas": world,
                       "parallelism": f"replicas{world}",
                       "l2": "flushed (512 MB write) before every timed step"},
            "latency_us": round(ms_max * 1e3, 2),
            "modes": {
                "multi_stream_aot_us": round(ms * 1e3, 2),
                "single_stream_aot_us": round(single_ms * 1e3, 2),
                "eager_non_aot_us": round(eager_ms * 1e3, 2),
                "framework_multi_stream_non_aot_us": round(fw_multi_ms * 1e3, 2),
                ("multi_stream_aot_no_pdl_us" if eng.pdl else "multi_stream_aot_pdl_us"):
                    round(alt_ms * 1e3, 2),
                "multi_over_single": round(single_ms / ms, 4),
                "aot_over_eager": round(eager_ms / ms, 4),
            },
            "host_overhead": {"launch_us_per_iter": round(host_us, 3),
                              "python_call_us_per_iter": round(py_us, 3),
                              "gpu_us_per_iter": round(gpu_us, 3),
                              "fraction_of_gpu_time": round(host_us / gpu_us, 5),
                              "python_call_fraction_of_gpu_time": round(py_us / gpu_us, 5),
                              "fraction_of_roofline_sum": round(host_us / roof_sum, 5)},
            "simulated_from_measured": {"multi_stream_us": round(sim_multi, 2),
                                        "single_stream_us": round(sim_single, 2),
                                        "critical_path_us": round(crit, 2)},
            "roofline_sum_us": round(roof_sum, 3),
            "roofline_sum_peaks": {"hbm_gbs": hbm, "contraction_tflops": tc3_peak,
                                   "contraction_peak": "tcgen05 kind::tf32 / 3 (3xTF32), profiles/peaks_fp32.json",
                                   "other_tflops": ffma_peak, "other_peak": "FFMA, profiles/peaks_fp32.json"},
            "latency_over_roofline_sum": round(ms * 1e3 / roof_sum, 3),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 5), "traffic": traffic,
                         "algorithmic_bytes_per_launch": round(bytes_per_launch, 1),
                         "launch_us_in_replay": round(launch_in_replay, 3),
                         "launch_us_warm_isolated": round(launch_warm, 3),
                         "family_share_of_replay_task_time": round(
                             dd["trace_us"] / sum(v["trace_us"] for v in fam.values()), 4),
                         "kernel": f"{dom} family: {dd['n']} launches, {launch_in_replay:.2f} µs per launch "
                                   f"inside a flushed-L2 replay (event-bracketed), {launch_warm:.2f} µs per "
                                   f"launch as a warm isolated chain",
                         "method": "achieved = algorithmic bytes per launch / per-launch time inside the replay",
                         "peak_source": peak_src},
            "e2e": {"value": round(world * args.batch / (e2e_ms_max / 1e3), 3), "unit": UNIT,
                    "ms_per_step": round(e2e_ms_max, 5),
                    "h2d_bytes_per_step": int(eng.h_in.numel() * 4),
                    "d2h_bytes_per_step": int(eng.out_bytes)},
            "e2e_pipelined": {"value": round(world * args.batch / (stream_ms_max / 1e3), 3), "unit": UNIT,
                              "ms_per_step": round(stream_ms_max, 5), "api": "Engine.infer_stream",
                              "h2d_bytes_per_step": int(eng.h_in.numel() * 4),
                              "d2h_bytes_per_step": int(eng.out_bytes),
                              "note": "requests back to back, next H2D overlapped with the current replay; "
                                      "L2 not flushed between requests"},
            "gpu_launches": n_tasks * args.steps,
            "tcgen05_tasks": sum(1 for d in eng.ops[:n_tasks] if d.kind == 6 or (d.kind == 8 and d.variant == 100)),
            "tasks": n_tasks, "streams": eng.assignment.num_streams, "syncs": len(eng.plan),
            "arena": {"mode": eng.arena_mode, "bytes": int(eng.arena.numel()),
                      "never_free_bytes": int(eng.arena_layout.reference_total) if eng.arena_layout else None},
            "clocks": clock_info,
            "parity": parity,
            "prepare_s": {k: round(v, 3) for k, v in eng.plan_seconds.items()},
            "kernel_families_us": {k: round(v["us"], 2) for k, v in fam.items()},
            "kernel_families_in_replay_us": {k: round(v["trace_us"], 2) for k, v in fam.items()},
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        if extra is not None:
            line["other_configs"] = extra
        if training is not None:
            line["training"] = training
        print(json.dumps(line))
    eng.close()
    return line


def _timed_replays(eng, dev, flush, steps, multi):
    """Mean device time (µs) of `steps` replays on the engine's launch stream,
    the 512 MB L2 flush before each (same discipline as the headline)."""
    import ctypes as C
    import torch
    from paper_2012_02732_b200 import _native as N
    sh = C.c_uint64()
    N.check(N.lib().sw_engine_stream(eng._h, C.byref(sh)))
    stream = torch.cuda.ExternalStream(sh.value, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    with torch.cuda.stream(stream):
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            eng.replay(multi=multi)
            b.record(stream)
    torch.cuda.synchronize(dev)
    return sum(a.elapsed_time(b) for a, b in ev) / steps * 1e3


def _parity(model, x, y, n=8):
    """fp32 gate on the first n images (images are independent, so a slice of
    a large batch checks the kernels the autotuner picked for that batch)."""
    import torch
    from oracle.numerics import cpu_forward
    k = min(n, x.shape[0])
    ref = cpu_forward(model, x[:k])
    yy = y[:k].cpu()
    return {"images_checked": k, "max_abs_err": float((yy - ref).abs().max()),
            "ok": bool(torch.allclose(yy, ref, rtol=1e-3, atol=1e-4))}


def _family_roofline(eng, hbm, reps=3):
    from paper_2012_02732_b200.engine import task_cost
    per = eng.profile_tasks(reps=reps)
    fams = {}
    for t in eng.program.tasks:
        f_, b_ = task_cost(t)
        d = fams.setdefault(t.kind, [0.0, 0.0, 0.0, 0])
        d[0] += per[t.tid]
        d[1] += b_
        d[2] += f_
        d[3] += 1
    dom = max(fams, key=lambda k: fams[k][0])
    us_, b_, f_, n_ = fams[dom]
    return {"kernel": f"{dom} family ({n_} launches, {us_ / n_:.1f} µs per launch, warm isolated)",
            "bound": "hbm", "achieved": round(b_ / (us_ * 1e-6) / 1e9, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(b_ / (us_ * 1e-6) / 1e9 / hbm, 4),
            "achieved_tflops_fp32": round(f_ / (us_ * 1e-6) / 1e12, 2),
            "family_share_of_task_time": round(us_ / sum(v[0] for v in fams.values()), 3)}


def other_configs(args, dev, hbm, flush, stream):
    """The remaining BASELINE configs, same engine and timing discipline:
    latency (µs) of multi-stream AoT replay, single-stream AoT replay and the
    eager launch loop for the 8-op cell / ResNet-50 / Inception-v3 at batch 1,
    and NASNet-A mobile images/s at batch 256 (one replica); every config
    carries its fp32 parity against the CPU forward."""
    import torch
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input

    out = {}
    plan = [("cell", 1), ("resnet50", 1), ("inception_v3", 1), ("nasnet_mobile", args.big_batch)]
    # the bf16 path (precision="bf16": batch-1 weight-streaming contractions in
    # bf16 with fp32 accumulation), its own stated tolerance
    plan += [("resnet50", 1, "bf16"), ("inception_v3", 1, "bf16")]
    steps = max(10, min(args.steps, 50))
    for entry in plan:
        name, batch = entry[0], entry[1]
        prec = entry[2] if len(entry) > 2 else "fp32"
        t0 = time.perf_counter()
        model, shape = build_model(name)
        x = example_input(shape, batch=batch)
        eng = Engine(model, device=dev.index or 0, precision=prec).prepare(x)
        y = eng(x)
        if prec == "bf16":
            import torch as _t
            from oracle.numerics import cpu_forward
            ref = cpu_forward(model, x)
            err, rel = (y - ref).abs().max().item(), ((y - ref).norm() / ref.norm()).item()
            parity = {"max_abs_err": err, "rel_l2": rel, "tolerance": "bf16: max abs 1e-1, rel L2 5e-2",
                      "ok": bool(err <= 1e-1 and rel <= 5e-2)}
        else:
            parity = _parity(model, x, y)
        eng.load_input_device(x)
        for _ in range(3):
            eng.replay(multi=True)
            eng.replay(multi=False)
        torch.cuda.synchronize(dev)
        multi_us = _timed_replays(eng, dev, flush, steps, True)
        single_us = _timed_replays(eng, dev, flush, steps, False)
        t = time.perf_counter()
        for _ in range(3):
            eng.run_eager()
        eng.synchronize()
        eager_us = (time.perf_counter() - t) / 3 * 1e6
        roof = roofline_sum_fp32(eng, hbm)
        fam_roof = _family_roofline(eng, hbm) if batch > 1 else None
        out[f"{name}_bs{batch}" + ("_bf16" if prec == "bf16" else "")] = {
            "multi_stream_aot_us": round(multi_us, 2), "single_stream_aot_us": round(single_us, 2),
            "eager_non_aot_us": round(eager_us, 2),
            "images_per_s": round(batch / (multi_us * 1e-6), 2),
            "multi_over_single": round(single_us / multi_us, 4),
            "tasks": len(eng.program.tasks), "streams": eng.assignment.num_streams,
            "syncs": len(eng.plan), "roofline_sum_us": round(roof, 3),
            "latency_over_roofline_sum": round(multi_us / roof, 3),
            "arena_mb": round(eng.arena.numel() / 1e6, 2),
            "roofline_dominant_family": fam_roof, "parity": parity,
            "tcgen05_tasks": sum(1 for d in eng.ops[:len(eng.program.tasks)]
                                 if d.kind == 6 or (d.kind == 8 and d.variant == 100)),
            "precision": prec,
            "prepare_s": round(time.perf_counter() - t0, 2)}
        eng.close()
    return out


def sharded_big_batch(args, dev, hbm, flush, world, rank):
    """BASELINE config 4 at N > 1 GPUs: NASNet-A mobile bs256 batch-sharded,
    256/N images per rank, each rank an independent captured replica (no
    data-path collective).  images/s = 256 / the slowest
    rank's mean device time per step (barrier before the timed steps)."""
    import torch
    from paper_2012_02732_b200.engine import Engine
    from paper_2012_02732_b200.networks import build_model, example_input

    per_rank = max(1, args.big_batch // world)
    model, shape = build_model("nasnet_mobile")
    x = example_input(shape, batch=per_rank, seed=1 + rank)
    t0 = time.perf_counter()
    eng = Engine(model, device=dev.index or 0).prepare(x)
    y = eng(x)
    parity = _parity(model, x, y)
    eng.load_input_device(x)
    for _ in range(3):
        eng.replay(multi=True)
    torch.cuda.synchronize(dev)
    barrier(world)
    steps = max(10, min(args.steps, 50))
    us = _timed_replays(eng, dev, flush, steps, True)
    us_max = reduce_max(world, us, dev)
    ok = reduce_max(world, 0.0 if parity["ok"] else 1.0, dev) == 0.0
    rec = {f"nasnet_mobile_bs{per_rank * world}_sharded": {
        "images_per_rank": per_rank, "ranks": world, "ms_per_step_max_over_ranks": round(us_max / 1e3, 4),
        "images_per_s": round(per_rank * world / (us_max * 1e-6), 2),
        "parity_all_ranks_ok": ok, "parity_rank0": parity,
        "roofline_sum_us": round(roofline_sum_fp32(eng, hbm), 3),
        "prepare_s": round(time.perf_counter() - t0, 2)}}
    eng.close()
    return rec


def train_configs(args, dev, world=1, rank=0):
    """BASELINE config 5: MobileNetV2 / EfficientNet-B0 CIFAR-10 training,
    bs=32 per GPU.  One step = forward + cross-entropy + backward (+ NCCL
    allreduce when world > 1) + SGD, captured as ONE graph.
    Reported per net: multi-stream AoT step, single-stream AoT step, the eager
    launch loop, images/s, e2e step() from host tensors, and the torch CPU
    autograd step on the host cores (the CPU path)."""
    import copy
    import torch
    from paper_2012_02732_b200.networks import build_train_model, train_batch
    from paper_2012_02732_b200.train import TrainEngine
    from oracle.numerics import cpu_threads

    out = {}
    steps = max(10, min(args.steps, 50))
    for name in ("mobilenet_v2", "efficientnet_b0"):
        t0 = time.perf_counter()
        model = build_train_model(name)
        x, y = train_batch(32, rank=rank)
        eng = TrainEngine(copy.deepcopy(model), device=dev.index or 0, world=world, rank=rank).prepare(x, y)
        eng.load_batch_device(x, y)
        st = eng.stream()

        def timed(multi):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(steps)]
            with torch.cuda.stream(st):
                for a, b in ev:
                    a.record(st)
                    eng.replay(multi=multi)
                    b.record(st)
            torch.cuda.synchronize(dev)
            return sum(a.elapsed_time(b) for a, b in ev) / steps * 1e3

        for _ in range(3):
            eng.replay(multi=True)
            eng.replay(multi=False)
        torch.cuda.synchronize(dev)
        barrier(world)
        multi_us = reduce_max(world, timed(True), dev)
        single_us = reduce_max(world, timed(False), dev)
        t = time.perf_counter()
        for _ in range(3):
            eng.run_eager()
        eng.synchronize()
        eager_us = (time.perf_counter() - t) / 3 * 1e6
        eng.run_framework(True)
        eng.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            eng.run_framework(True)
        eng.synchronize()
        fw_us = (time.perf_counter() - t) / 5 * 1e6
        for _ in range(2):
            eng.step(x, y)
        t = time.perf_counter()
        for _ in range(steps):
            eng.step(x, y)
        e2e_us = reduce_max(world, (time.perf_counter() - t) / steps * 1e6, dev)
        rec = {"batch_per_gpu": 32, "gpus": world,
               "multi_stream_aot_us": round(multi_us, 2), "single_stream_aot_us": round(single_us, 2),
               "eager_non_aot_us": round(eager_us, 2),
               "framework_multi_stream_non_aot_us": round(fw_us, 2),
               "images_per_s": round(world * 32 / (multi_us * 1e-6), 1),
               "e2e_images_per_s": round(world * 32 / (e2e_us * 1e-6), 1),
               "multi_over_single": round(single_us / multi_us, 4),
               "aot_over_eager": round(eager_us / multi_us, 4),
               "tasks": len(eng.prog.tasks), "streams": eng.assignment.num_streams,
               "syncs": len(eng.plan), "allreduce": eng.allreduce,
               "tcgen05_tasks": sum(1 for t in eng.prog.tasks if eng.ops[t.tid].kind == 6),
               "params": eng.builder.param_count, "prepare_s": round(time.perf_counter() - t0, 2)}
        eng.close()
        if rank == 0 and world == 1 and not args.skip_cpu:
            # the CPU path: torch fp32 autograd + SGD of the same module on the host cores
            thr = cpu_threads()
            torch.set_num_threads(thr)
            m = copy.deepcopy(model)
            opt = torch.optim.SGD(m.parameters(), lr=0.05, momentum=0.9, weight_decay=4e-5)
            ct = []
            for i in range(5):
                t = time.perf_counter()
                opt.zero_grad(set_to_none=True)
                torch.nn.functional.cross_entropy(m(x), y).backward()
                opt.step()
                if i >= 1:
                    ct.append(time.perf_counter() - t)
            cpu_s = sum(ct) / len(ct)
            rec["cpu_baseline"] = {"value": round(32 / cpu_s, 2), "unit": "images/s", "cores": thr,
                                   "kind": "port", "sample": "4 torch CPU fp32 training steps, bs32"}
        out[f"{name}_train_bs32"] = rec
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="nasnet_mobile")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-extra", action="store_true", help="skip the other BASELINE configs")
    ap.add_argument("--big-batch", type=int, default=256, help="NASNet images/s batch (one replica)")
    ap.add_argument("--skip-train", action="store_true", help="skip the training configs")
    ap.add_argument("--train-dp", action="store_true",
                    help="(default now) under torchrun the training configs run data-parallel with the "
                         "captured NCCL allreduce")
    ap.add_argument("--tuning-cache", default=None,
                    help="reuse kernel picks (e.g. for an ncu launch list of this command)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_setup(args.gpus)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
