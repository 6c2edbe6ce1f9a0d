"""Golden vectors for the optimizer data path from torch.optim.AdamW on CPU.

    python tests/golden/make_adamw_golden.py

The reference has no optimizer; the paper imports Megatron's
(PAPER.md:371), whose update is torch.optim.AdamW algebra.  These vectors pin
oracle/hod_oracle.c against an independent implementation: torch.optim.AdamW
(foreach=False, fused=False) for 1 and 100 steps, with and without
torch.nn.utils.clip_grad_norm_.  Gradients are bf16-rounded N(0, 1e-3^2)
draws from numpy PCG64 (seed 1000 + step), regenerated identically by the test.
"""

from pathlib import Path

import numpy as np
import torch

N = 4099
LR, BETAS, EPS, WD = 1e-4, (0.9, 0.95), 1e-8, 0.1


def grad(step: int) -> np.ndarray:
    g = np.random.default_rng(1000 + step).standard_normal(N).astype(np.float32) * np.float32(1e-3)
    return torch.from_numpy(g).to(torch.bfloat16).float().numpy()


def init() -> np.ndarray:
    return (np.random.default_rng(42).standard_normal(N).astype(np.float32) * np.float32(0.02))


def run(steps: int, clip):
    p = torch.nn.Parameter(torch.from_numpy(init().copy()))
    opt = torch.optim.AdamW([p], lr=LR, betas=BETAS, eps=EPS, weight_decay=WD, foreach=False, fused=False)
    norms = []
    for s in range(1, steps + 1):
        p.grad = torch.from_numpy(grad(s).copy())
        if clip is not None:
            norms.append(float(torch.nn.utils.clip_grad_norm_([p], clip)))
        opt.step()
    st = opt.state[p]
    return p.detach().numpy().copy(), st["exp_avg"].numpy().copy(), st["exp_avg_sq"].numpy().copy(), norms


def main():
    out = {}
    for steps in (1, 100):
        for clip in (None, 0.01):
            tag = f"s{steps}_{'clip' if clip else 'noclip'}"
            p, m, v, norms = run(steps, clip)
            out[f"{tag}_master"], out[f"{tag}_m"], out[f"{tag}_v"] = p, m, v
            out[f"{tag}_norms"] = np.array(norms, dtype=np.float64)
    path = Path(__file__).parent / "adamw_torch.npz"
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
