"""One rank of the multi-GPU parity check (launched by tests/test_multigpu_gpu.py
under torch.distributed.run).  Each rank runs a few DistributedOptimizer steps
and dumps its state; rank 0 then checks every rank against the oracle.

Checks:
  * bucket layout identical on all ranks;
  * reduce-scatter: device-reduced shard within (d-1) bf16 roundings of the
    fp64 sum (NCCL ring order is not the oracle's order) — bit-exact for the
    deterministic p2p backend;
  * AdamW: the oracle fed with the device's own reduced shard reproduces
    master / m / v / bf16 params bit-exactly;
  * all-gather: param buffer bit-identical on every rank and equal to the
    concatenation of the owners' shards.
"""

import argparse
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2312_03549_b200 import DistributedOptimizer  # noqa: E402
from paper_2312_03549_b200.comm import DPGroup  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="toy")
    ap.add_argument("--grad-dtype", default="f32")
    ap.add_argument("--bucket", type=int, default=4_000_000)
    ap.add_argument("--clip", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--out", required=True)
    ap.add_argument("--final-only", type=int, default=0, help="dump only the state after the last step")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    gs = config_gradset(a.config)
    gdt = torch.float32 if a.grad_dtype == "f32" else torch.bfloat16
    clip = a.clip if a.clip > 0 else None
    opt = DistributedOptimizer(init_params(gs, dev), bucket_size=a.bucket, clip=clip,
                               dp_group=DPGroup(tuple(range(world)), rank), backend=a.backend,
                               keep_reduced=True, barrier_timeout_s=30.0)
    L = opt.layout
    out = Path(a.out)
    for step in range(1, a.steps + 1):
        if a.final_only and step < a.steps:
            opt.step(make_grads(gs, step, rank, dev, dtype=gdt))
            continue
        # state BEFORE the step (so the oracle can replay it exactly)
        pre = dict(master=opt.master.cpu().numpy().copy(), m=opt.exp_avg.cpu().numpy().copy(),
                   v=opt.exp_avg_sq.cpu().numpy().copy())
        grads = make_grads(gs, step, rank, dev, dtype=gdt)
        rep = opt.step(grads)
        torch.cuda.synchronize()
        reduced = np.concatenate([u16(opt.grad_buffer[slice(*b.shard_range(opt.shard_index, opt.dp))])
                                  for b in L.buckets])
        np.savez(out / f"r{rank}_s{step}.npz", reduced=reduced, params=u16(opt.param_buffer),
                 master=opt.master.cpu().numpy(), m=opt.exp_avg.cpu().numpy(),
                 v=opt.exp_avg_sq.cpu().numpy(), pre_master=pre["master"], pre_m=pre["m"],
                 pre_v=pre["v"],
                 coef=np.float32(rep.clip_coef.item()) if rep.clip_coef is not None else np.float32(-1),
                 norm=np.float32(rep.grad_norm.item()) if rep.grad_norm is not None else np.float32(-1))
    opt.check_health()
    (out / f"layout_r{rank}.json").write_text(L.to_json())
    opt.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
