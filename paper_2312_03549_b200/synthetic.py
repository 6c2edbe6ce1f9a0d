"""Seeded synthetic parameters and gradients (SURVEY.md §8d conventions).

theta0 ~ N(0, 0.02^2) from seed 42; per-rank gradients
g ~ N(0, 1e-3^2) from seed 1234 + 1000*step + global_rank, generated tensor
by tensor in registration order.  Generation happens on the target device
with a torch.Generator of that device; CPU tests copy the very same tensors
to the host, so the oracle and the GPU always see identical inputs.
"""

from __future__ import annotations

import torch

from .gradsets import GradSet

PARAM_SEED = 42
PARAM_STD = 0.02
GRAD_STD = 1e-3


def grad_seed(step: int, global_rank: int) -> int:
    return 1234 + 1000 * step + global_rank


def init_params(gs: GradSet, device, dtype=torch.float32, seed: int = PARAM_SEED):
    gen = torch.Generator(device=device).manual_seed(seed)
    out = []
    for t in gs.tensors:
        x = torch.randn(t.shape, generator=gen, device=device, dtype=torch.float32)
        out.append(x.mul_(PARAM_STD).to(dtype))
    return out


def make_grads(gs: GradSet, step: int, global_rank: int, device, dtype=torch.bfloat16):
    gen = torch.Generator(device=device).manual_seed(grad_seed(step, global_rank))
    out = []
    for t in gs.tensors:
        x = torch.randn(t.shape, generator=gen, device=device, dtype=torch.float32)
        out.append(x.mul_(GRAD_STD).to(dtype))
    return out
