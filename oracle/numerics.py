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
