"""GPU parity of the AoT training step (runs under `pytest -m gpu`).

One captured graph per step: forward (inference conv kernels + batch-norm
training kernels), softmax cross-entropy, backward (csrc/kernels/train.cu),
optional NCCL allreduce, SGD.  Oracle: torch CPU autograd + torch.optim.SGD on
the same module (oracle/numerics.py:cpu_train_steps), gates as in
tests/test_train_builder.py (EfficientNet-B0 vs float64 within rel-L2 1e-3;
MobileNetV2 vs float32 within rel-L2 3e-2 — ReLU6 kinks make fp32 gradients
chaotic, torch fp32 vs fp64 differ by ~1 %).
"""

import copy

import numpy as np
import pytest
import torch

from oracle.numerics import cpu_train_steps
from paper_2012_02732_b200 import train as T
from paper_2012_02732_b200.networks import build_train_model, train_batch
from test_train_builder import grad_errors

pytestmark = pytest.mark.gpu

LR, MOM, WD = 0.05, 0.9, 4e-5


def _engine(name, batch, **kw):
    model = build_train_model(name)
    x, y = train_batch(batch)
    eng = T.TrainEngine(copy.deepcopy(model), LR, MOM, WD, **kw).prepare(x, y)
    return model, eng, x, y


@pytest.mark.parametrize("name,batch,double,tol", [
    ("efficientnet_b0", 32, True, 1e-3),
    ("mobilenet_v2", 32, False, 3e-2),
])
def test_train_step_parity(name, batch, double, tol):
    model, eng, x, y = _engine(name, batch)
    before = {n: p.detach().double().clone() for n, p in model.named_parameters()}
    loss = eng.step(x, y)
    ref = copy.deepcopy(model)
    if double:
        ref = ref.double()
    losses, grads = cpu_train_steps(ref, [(x.double() if double else x, y)], LR, MOM, WD)
    assert abs(loss - losses[0]) <= 1e-4 * abs(losses[0]), (loss, losses[0])
    errs = grad_errors(eng.gradients(), grads)
    worst = max(errs, key=lambda e: e[1])
    assert worst[1] <= tol, worst
    rp = dict(ref.named_parameters())
    for pname, v in eng.parameters().items():
        pairs = [(pname[:-11] + ".weight", v[0]), (pname[:-11] + ".bias", v[1])] \
            if pname.endswith(".gamma_beta") else [(pname, v)]
        for pn, a in pairs:
            du = a.double().reshape(before[pn].shape) - before[pn]
            dr = rp[pn].detach().double() - before[pn]
            assert (du - dr).norm() <= tol * dr.norm() + 1e-6 * np.sqrt(dr.numel()), pn
    names = {id(m): n for n, m in eng.model.named_modules()}
    rmods = dict(ref.named_modules())
    for m, rm, rv in eng.running_stats():
        r = rmods[names[id(m)]]
        torch.testing.assert_close(rm.double(), r.running_mean.double(), rtol=1e-4, atol=1e-4)
        torch.testing.assert_close(rv.double(), r.running_var.double(), rtol=1e-3, atol=1e-3)
    eng.close()


def test_multi_and_single_stream_steps_are_bitwise_equal():
    """Every training kernel reduces in a fixed order, so the multi-stream
    replay must reproduce the single-stream one bit for bit."""
    model = build_train_model("mobilenet_v2")
    x, y = train_batch(32)
    # same kernel picks in both (autotune timing noise would pick differently)
    a = T.TrainEngine(copy.deepcopy(model), LR, MOM, WD, multi_stream=True, autotune=False).prepare(x, y)
    b = T.TrainEngine(copy.deepcopy(model), LR, MOM, WD, multi_stream=False, autotune=False).prepare(x, y)
    for _ in range(3):
        la, lb = a.step(x, y), b.step(x, y)
        assert la == lb
    pa, pb = a.parameters(), b.parameters()
    for k in pa:
        va = torch.cat(pa[k]) if isinstance(pa[k], tuple) else pa[k]
        vb = torch.cat(pb[k]) if isinstance(pb[k], tuple) else pb[k]
        assert torch.equal(va, vb), k
    a.close()
    b.close()


def test_nccl_allreduce_captured_world1():
    """The NCCL allreduce task inside the captured graph (world 1: average of
    one rank = identity) leaves the step unchanged and really runs NCCL."""
    model = build_train_model("mobilenet_v2")
    x, y = train_batch(32)
    a = T.TrainEngine(copy.deepcopy(model), LR, MOM, WD, allreduce=True, autotune=False).prepare(x, y)
    b = T.TrainEngine(copy.deepcopy(model), LR, MOM, WD, allreduce=False, autotune=False).prepare(x, y)
    assert "allreduce" in [t.kind for t in a.prog.tasks]
    for _ in range(2):
        assert a.step(x, y) == b.step(x, y)
    a.close()
    b.close()


def test_training_loss_decreases_and_eager_matches_replay():
    model, eng, x, y = _engine("mobilenet_v2", 32)
    losses = [eng.step(x, y) for _ in range(8)]
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
    # eager (non-AoT) launch loop = the same op table one launch at a time
    model2 = build_train_model("mobilenet_v2")
    e2 = T.TrainEngine(model2, LR, MOM, WD, autotune=False).prepare(x, y)
    e2.load_batch_device(x, y)
    e2.run_eager()
    e2.synchronize()
    e3 = T.TrainEngine(build_train_model("mobilenet_v2"), LR, MOM, WD, autotune=False).prepare(x, y)
    l3 = e3.step(x, y)
    assert e2.device_loss() == l3
    for e in (eng, e2, e3):
        e.close()


@pytest.mark.parametrize("M,N,K,split,mode", [
    (96, 16, 8192, 32, "tn"),     # 1x1 wgrad shape (reduction over pixels, split-K)
    (8192, 16, 96, 1, "nn"),      # 1x1 dgrad shape
    (10, 1280, 32, 1, "tn"),      # Linear wgrad
    (33, 70, 1000, 4, "nn"),      # ragged tiles + split
])
def test_gemm_kernel(M, N, K, split, mode):
    """K_GEMM against torch (strided NN / TN operands, deterministic split-K)."""
    from paper_2012_02732_b200 import _native as NAT
    import ctypes as C
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(0)
    if mode == "tn":       # C = A^T B with A stored [K][M]
        A = torch.randn(K, M, generator=g)
        a_i, a_r = 1, M
    else:                  # A stored [M][K]
        A = torch.randn(M, K, generator=g)
        a_i, a_r = K, 1
    B = torch.randn(K, N, generator=g)
    Am = (A.t() if mode == "tn" else A).double()
    res = torch.randn(M, N, generator=g)
    ref = Am @ B.double() + res.double()
    Ad, Bd, Cd = A.to(dev), B.to(dev), res.to(dev)
    tiles = -(-M // 64) * -(-N // 64)
    ws = torch.zeros(split * tiles * 4096 + tiles + 4, device=dev)
    d = NAT.OpDesc()
    d.kind = T.K_GEMM
    for k, v in {T.GM_M: M, T.GM_N: N, T.GM_K: K, T.GM_A_I: a_i, T.GM_A_R: a_r, T.GM_B_R: N,
                 T.GM_B_J: 1, T.GM_C_I: N, T.GM_SPLIT: split, T.GM_HAS_RES: 1}.items():
        d.params[k] = v
    d.ptrs[0], d.ptrs[1], d.ptrs[2], d.ptrs[4], d.ptrs[5] = (Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr(),
                                                             Cd.data_ptr(), ws.data_ptr())
    lib = NAT.lib()
    h = C.c_void_p()
    NAT.check(lib.sw_engine_create(0, C.byref(h)))
    NAT.check(lib.sw_engine_set_ops(h, 1, d))
    NAT.check(lib.sw_engine_launch_op(h, 0))
    NAT.check(lib.sw_engine_synchronize(h))
    out = Cd.cpu().double()
    torch.testing.assert_close(out, ref, rtol=1e-4, atol=1e-3 * ref.abs().max().item() / 100)
    lib.sw_engine_destroy(h)
