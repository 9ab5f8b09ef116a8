"""Training step builder on CPU, through the host emulator
of the training op table (tests/train_emulator.py), against torch autograd.

Gates (one SGD step, momentum 0.9, weight decay 4e-5):
* EfficientNet-B0 (SiLU everywhere: no activation kinks) vs torch float64:
  every parameter gradient within rel-L2 1e-4 — the builder's gradient
  routing, accumulation, squeeze-excite backward and layouts are exact up to
  fp32 storage rounding;
* MobileNetV2 (ReLU6) vs torch float32: rel-L2 3e-2.  ReLU6 kinks make fp32
  gradients chaotic: torch fp32 itself differs from torch fp64 by 0.9 % median
  / 1.2 % max rel-L2 on this step, so a tighter gate would test rounding luck;
* gradients that are exactly zero in exact arithmetic (BN beta feeding a
  batch-normalised consumer) are compared with an absolute floor;
* loss within 1e-4 relative (fp32 forward), BN running statistics within 1e-5 / 1e-4.
"""

import copy
import os
import socket

import numpy as np
import torch

from oracle.numerics import cpu_train_steps
from paper_2012_02732_b200 import train as T
from paper_2012_02732_b200.networks import build_train_model, train_batch
from train_emulator import TrainEmulator

LR, MOM, WD = 0.05, 0.9, 4e-5


def grad_errors(eg: dict, ref_grads: dict, atol=1e-5):
    """(name, rel-L2 error) per torch parameter; zero-valued references use an
    absolute floor scaled by sqrt(numel)."""
    out = []
    for name, v in eg.items():
        if name.endswith(".gamma_beta"):
            base = name[: -len(".gamma_beta")]
            pairs = [(base + ".weight", v[0]), (base + ".bias", v[1])]
        else:
            pairs = [(name, v)]
        for pn, a in pairs:
            r = ref_grads[pn].double().reshape(a.shape)
            d = (a.double() - r).norm().item()
            floor = atol * np.sqrt(r.numel())
            out.append((pn, d / max(r.norm().item(), floor / 1e-4 if r.norm().item() < floor else 0)))
    return out


def _check(model_name, batch, ref_double, tol):
    model = build_train_model(model_name)
    ref = copy.deepcopy(model)
    before = {n: q.detach().double().clone() for n, q in model.named_parameters()}
    x, y = train_batch(batch)
    em = TrainEmulator(model, x.shape, LR, MOM, WD)
    loss = em.step(x, y)
    if ref_double:
        ref = ref.double()
        x_r = x.double()
    else:
        x_r = x
    losses, grads = cpu_train_steps(ref, [(x_r, y)], LR, MOM, WD)
    assert abs(loss - losses[0]) <= 1e-4 * abs(losses[0])
    errs = grad_errors(em.gradients(), grads)
    worst = max(errs, key=lambda e: e[1])
    assert worst[1] <= tol, worst
    # updated parameters (torch layout) and running statistics
    rp = dict(ref.named_parameters())
    for name, v in em.parameters().items():
        if name.endswith(".gamma_beta"):
            base = name[: -len(".gamma_beta")]
            pairs = [(base + ".weight", v[0]), (base + ".bias", v[1])]
        else:
            pairs = [(name, v)]
        for pn, a in pairs:
            # the SGD update (p_new - p_old) agrees like the gradients do
            du = a.double().reshape(before[pn].shape) - before[pn]
            dr = rp[pn].detach().double() - before[pn]
            assert (du - dr).norm() <= tol * dr.norm() + 1e-6 * np.sqrt(dr.numel()), pn
    names = {id(m): n for n, m in model.named_modules()}
    rmods = dict(ref.named_modules())
    for m, rm, rv in em.running_stats():
        ref_m = rmods[names[id(m)]]
        torch.testing.assert_close(rm.double(), ref_m.running_mean.double(), rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(rv.double(), ref_m.running_var.double(), rtol=1e-4, atol=1e-4)
    return em


def test_efficientnet_b0_step_matches_fp64_autograd():
    _check("efficientnet_b0", 8, True, 1e-3)


def test_mobilenet_v2_step_matches_fp32_autograd():
    em = _check("mobilenet_v2", 8, False, 3e-2)
    # the backward DAG branches (wgrad / dgamma off the dgrad chain): multi-stream
    assert em.assignment.num_streams > 1


def test_training_dag_structure():
    model = build_train_model("mobilenet_v2")
    b = T.build_train_program(model, (2, 3, 32, 32), allreduce=True)
    tasks = b.prog.tasks
    kinds = [t.kind for t in tasks]
    ar = kinds.index("allreduce")
    sgd = kinds.index("sgd")
    assert sgd == len(tasks) - 1 and ar == sgd - 1
    # every task that writes a gradient slice precedes the allreduce; the
    # optimizer waits for every reader of a parameter (no WAR race on weights)
    grad_ids = {g.bid for g in b.gbuf}
    pids = {p.bid for p in b.pbuf}
    anc = _ancestors(tasks, ar)
    for t in tasks[:ar]:
        if any(w.bid in grad_ids for w in t.writes):
            assert t.tid in anc
    anc_sgd = _ancestors(tasks, sgd)
    for t in tasks[:sgd]:
        if any(r.bid in pids for r in t.reads):
            assert t.tid in anc_sgd
    # one parameter slice per trainable tensor, 16-B aligned, inside the flat buffer
    n_torch = sum(1 for _ in model.parameters())
    n_slices = sum(2 if isinstance(p.tensor, tuple) else 1 for p in b.prog.params)
    assert n_slices == n_torch
    assert all(p.buf.sub_offset % 16 == 0 for p in b.prog.params)
    assert b.param_count == sum(p.numel() for p in model.parameters())


def _ancestors(tasks, tid):
    seen = set()
    stack = [tid]
    while stack:
        t = stack.pop()
        for d in tasks[t].deps:
            if d not in seen:
                seen.add(d)
                stack.append(d)
    return seen


def test_single_and_multi_stream_schedules_agree():
    model = build_train_model("efficientnet_b0")
    x, y = train_batch(2)
    a = TrainEmulator(copy.deepcopy(model), x.shape, LR, MOM, WD, multi_stream=True)
    b = TrainEmulator(copy.deepcopy(model), x.shape, LR, MOM, WD, multi_stream=False)
    assert a.step(x, y) == b.step(x, y)
    ga, gb = a.gradients(), b.gradients()
    for k in ga:
        va, vb = (ga[k], gb[k]) if not isinstance(ga[k], tuple) else (torch.cat(ga[k]), torch.cat(gb[k]))
        assert torch.equal(va, vb), k


# -- data parallel: world 2 over gloo, the allreduce task averaging gradients --

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _dp_worker(rank, world, port, q):
    import sys
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    from oracle.numerics import cpu_train_steps as oracle_steps
    from paper_2012_02732_b200.networks import build_train_model as btm, train_batch as tb
    from train_emulator import TrainEmulator as TE
    torch.set_num_threads(2)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = btm("efficientnet_b0")
        ref = copy.deepcopy(model).double()
        x, y = tb(8, rank=rank)

        def allreduce(g):
            t = g.clone()
            dist.all_reduce(t)
            return t / world
        em = TE(model, x.shape, LR, MOM, WD, allreduce=allreduce)
        em.step(x, y)
        _, grads = oracle_steps(ref, [(x.double(), y)], LR, MOM, WD)
        for k in grads:
            dist.all_reduce(grads[k])
            grads[k] /= world
        errs = grad_errors(em.gradients(), grads)
        q.put((rank, max(e[1] for e in errs)))
    finally:
        dist.destroy_process_group()


def test_data_parallel_allreduce_world2_gloo():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert len(res) == 2
    for rank, worst in res:
        assert worst <= 1e-3, (rank, worst)
