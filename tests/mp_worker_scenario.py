"""One rank of the PP x DP scenario parity check (tests/test_multigpu_gpu.py).

The scenario document is planned with the reference-compatible planner; each
rank runs the optimizer of its stage's DP row with the clip norm taken over
the whole world, and dumps its state for the oracle check on rank 0's host.
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2312_03549_b200 as hp  # noqa: E402
from paper_2312_03549_b200.scenario_run import make_optimizer, setup_rank  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--clip", type=float, default=0.0)
    ap.add_argument("--bucket", type=int, default=300_000)
    ap.add_argument("--backend", default="auto")
    ap.add_argument("--steps", type=int, default=2)
    a = ap.parse_args()
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    scenario = hp.load_scenario(a.scenario)
    sr = setup_rank(scenario, rank)
    gs = sr.gradset
    opt = make_optimizer(sr, init_params(gs, dev), bucket_size=a.bucket,
                         clip=a.clip if a.clip > 0 else None, backend=a.backend, keep_reduced=True,
                         barrier_timeout_s=30.0)
    out = Path(a.out)
    for step in range(1, a.steps + 1):
        pre = dict(master=opt.master.cpu().numpy().copy(), m=opt.exp_avg.cpu().numpy().copy(),
                   v=opt.exp_avg_sq.cpu().numpy().copy())
        rep = opt.step(make_grads(gs, step, rank, dev))
        torch.cuda.synchronize()
        reduced = np.concatenate([u16(opt.grad_buffer[slice(*b.shard_range(opt.shard_index, opt.dp))])
                                  for b in opt.layout.buckets])
        np.savez(out / f"r{rank}_s{step}.npz", reduced=reduced, params=u16(opt.param_buffer),
                 master=opt.master.cpu().numpy(), m=opt.exp_avg.cpu().numpy(), v=opt.exp_avg_sq.cpu().numpy(),
                 pre_master=pre["master"], pre_m=pre["m"], pre_v=pre["v"],
                 coef=np.float32(rep.clip_coef.item()) if rep.clip_coef is not None else np.float32(-1),
                 norm=np.float32(rep.grad_norm.item()) if rep.grad_norm is not None else np.float32(-1))
    opt.check_health()
    meta = dict(sr.placement.to_json_dict(), gradset=[[t.name, list(t.shape)] for t in gs.tensors],
                backend=opt.backend, layout=opt.layout.to_json_dict())
    (out / f"meta_r{rank}.json").write_text(json.dumps(meta))
    opt.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
