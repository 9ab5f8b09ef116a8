"""World-2 replica path on the B200 (two gloo processes sharing cuda:0).

bench.py's multi-GPU inference config (BASELINE config 4: NASNet-A mobile
batch-sharded over N GPUs) runs one captured replica per rank
with no data-path collective.  On this one-GPU box two ranks share the
device (SW_DIST_BACKEND=gloo for the barrier / max-over-ranks reduction);
each rank plans, captures and replays its own shard and checks it against
the fp32 CPU forward, and the slowest rank's time is what every rank sees.
"""

import os
import socket
import types

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank), "SW_DIST_BACKEND": "gloo"})
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import bench
    try:
        w, r, local = bench.dist_setup(world)
        dev = torch.device("cuda", local)
        flush = torch.empty(64 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        args = types.SimpleNamespace(big_batch=8, steps=10)
        rec = bench.sharded_big_batch(args, dev, 6500.0, flush, w, r)
        q.put((rank, rec, None))
    except Exception as e:  # noqa: BLE001
        q.put((rank, None, f"{type(e).__name__}: {e}"))
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


def test_world2_sharded_replicas_with_parity():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, rec, err in results:
        assert err is None, f"rank {rank}: {err}"
        (key, r), = rec.items()
        assert key == "nasnet_mobile_bs8_sharded"
        assert r["images_per_rank"] == 4 and r["ranks"] == 2
        assert r["parity_rank0"]["ok"] and r["parity_all_ranks_ok"]
    # the max-over-ranks reduction gives every rank the same step time
    assert len({r[1]["nasnet_mobile_bs8_sharded"]["ms_per_step_max_over_ranks"] for r in results}) == 1
