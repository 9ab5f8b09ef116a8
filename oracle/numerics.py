"""CPU numerics oracle — TEST INFRASTRUCTURE ONLY.

The reference ships no network numerics, so the
numeric oracle is the CPU restatement SURVEY §8(c) prescribes: the same
``nn.Module`` (eval mode), fp32, on the host CPU with deterministic
algorithms, on the same seeded weights and inputs.  Parity is therefore
"unpinned by the reference" for numerics (stated in DESIGN.md); the planner
oracle (oracle/planner.py) is pinned to the reference's golden bytes.

Also used by bench.py's reference arm as the CPU path being timed.
"""

from __future__ import annotations

import os

import torch


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_forward(model: torch.nn.Module, x: torch.Tensor) -> torch.Tensor:
    prev = torch.are_deterministic_algorithms_enabled()
    torch.use_deterministic_algorithms(True)
    try:
        with torch.no_grad():
            return model.eval().float()(x.detach().float().cpu())
    finally:
        torch.use_deterministic_algorithms(prev)


def cpu_train_steps(model: torch.nn.Module, batches, lr: float, momentum: float,
                    weight_decay: float):
    """Training oracle: the same module in train mode, fp32
    torch CPU autograd + torch.optim.SGD, one step per (x, y) batch.  Returns
    (losses, grads of the last step by parameter name); the module is updated
    in place (parameters and BN running statistics)."""
    prev = torch.are_deterministic_algorithms_enabled()
    torch.use_deterministic_algorithms(True)
    try:
        model.train()
        opt = torch.optim.SGD(model.parameters(), lr=lr, momentum=momentum, weight_decay=weight_decay)
        losses = []
        grads = {}
        for x, y in batches:
            opt.zero_grad(set_to_none=True)
            loss = torch.nn.functional.cross_entropy(model(x), y.long())
            loss.backward()
            grads = {n: p.grad.detach().clone() for n, p in model.named_parameters()}
            opt.step()
            losses.append(float(loss.detach()))
        return losses, grads
    finally:
        torch.use_deterministic_algorithms(prev)
