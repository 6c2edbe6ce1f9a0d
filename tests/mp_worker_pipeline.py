"""One rank of the PP x DP pipeline check (tests/test_multigpu_gpu.py): a 1F1B
iteration over peer-memory stage hand-offs around the DP optimizer."""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2312_03549_b200 as hp  # noqa: E402
from paper_2312_03549_b200.pipeline import PipelineRunner  # noqa: E402
from paper_2312_03549_b200.scenario_run import make_optimizer, setup_rank  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--micro", type=int, default=4)
    ap.add_argument("--compute", type=int, default=0)
    ap.add_argument("--iters", type=int, default=2)
    a = ap.parse_args()
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    s = hp.load_scenario(a.scenario)
    sr = setup_rank(s, rank)
    opt = make_optimizer(sr, init_params(sr.gradset, dev), clip=1.0, barrier_timeout_s=30.0)
    pr = PipelineRunner(s, sr, opt, micro_batches=a.micro, compute=bool(a.compute))
    if not a.compute:
        pr.x.fill_(1.0)
    grads = make_grads(sr.gradset, 1, rank, dev)
    doc = {"rank": rank, "stage": pr.stage}
    if a.compute:
        for with_opt in (False, True):
            for _ in range(2):
                pr.run_iteration(grads, with_optimizer=with_opt)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                pr.run_iteration(grads, with_optimizer=with_opt)
            e1.record()
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1) / a.iters], device=dev, dtype=torch.float64)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            doc["iter_ms_with_opt" if with_opt else "iter_ms_no_opt"] = float(ms.item())
            del t0
    else:
        for _ in range(a.iters):
            pr.run_iteration(grads, with_optimizer=True)
        torch.cuda.synchronize()
        doc["trace"] = [[op, k, float(t.float().mean()), float(t.float().std())] for op, k, t in pr.trace]
    pr.check()
    opt.check_health()
    (Path(a.out) / f"pipe_r{rank}.json").write_text(json.dumps(doc))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
