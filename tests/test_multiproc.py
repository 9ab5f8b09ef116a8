"""Multi-process (world_size 2, gloo, CPU) coverage of the replica path.

Batch-1 inference does not shard, so N GPUs run N independent replicas
(DESIGN.md §6): each rank plans and captures its own graph, and the only
cross-rank traffic is the barrier and the max-over-ranks timing reduction.
These tests run that plumbing here on CPU: every rank must derive the
identical task DAG / stream assignment / schedule bytes from the same model
(deterministic planning = replicas are interchangeable), and bench.py's
reduce_max must return the slowest rank's time on every rank.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    import paper_2012_02732_b200 as sw
    from paper_2012_02732_b200.networks import build_model, example_input
    from paper_2012_02732_b200.trace import build_program

    w, r, local = bench.dist_setup(world)
    assert (w, r, local) == (world, rank, rank)
    model, shape = build_model("cell")
    prog = build_program(model, example_input(shape, seed=1 + rank))
    g = prog.graph
    f, plan = sw.assign_streams(g)
    sched = sw.schedule_to_json(sw.pre_run(g, f, plan))
    gathered = [None] * world
    dist.all_gather_object(gathered, sched)
    # slowest rank wins the timing reduction
    t = bench.reduce_max(world, float(10 + rank))
    bench.barrier(world)
    q.put((rank, all(s == gathered[0] for s in gathered), t))
    dist.destroy_process_group()


def test_replicas_plan_identically_and_reduce_max():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, t in results:
        assert same, "replicas derived different schedules"
        assert t == 11.0
