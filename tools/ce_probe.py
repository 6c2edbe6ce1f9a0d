"""Copy-engine vs SM peer traffic over NVLink (one process per GPU).

    torchrun --nproc-per-node N tools/ce_probe.py [--mb 256]

Each rank owns a symmetric buffer of d chunks (chunk = --mb MB).  Patterns,
all ranks at once, CUDA events, max over ranks:
  ce_pull   rank r copies chunk r of every peer q into local staging (d-1
            cudaMemcpyAsync from peer-mapped addresses, one stream per peer)
  ce_push   rank r copies its chunk q into peer q's staging slot r
  ce_both   pull and push concurrently (RS + AG directions at once)
Bytes per GPU per direction = (d-1) * chunk.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.symm import SymmetricTensor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=256)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    nat.load()
    d = world
    chunk = a.mb << 20
    src = SymmetricTensor(d * chunk, torch.uint8, dev, None, zero=True)
    stage = SymmetricTensor(d * chunk, torch.uint8, dev, None, zero=True)
    streams = [torch.cuda.Stream(dev) for _ in range(2 * d)]
    peers = [q for q in range(d) if q != rank]

    def pull():
        for k, q in enumerate(peers):
            nat.call("hod_ce_copy", stage.tensor.data_ptr() + q * chunk, src.peer(q, rank * chunk), chunk,
                     nat.stream_ptr(streams[k]))

    def push():
        for k, q in enumerate(peers):
            nat.call("hod_ce_copy", stage.peer(q, rank * chunk), src.tensor.data_ptr() + q * chunk, chunk,
                     nat.stream_ptr(streams[d + k]))

    def both():
        pull()
        push()

    def timed(fn):
        cur = torch.cuda.current_stream(dev)
        for _ in range(2):
            for s in streams:
                s.wait_stream(cur)
            fn()
            for s in streams:
                cur.wait_stream(s)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(a.iters):
            for s in streams:
                s.wait_stream(cur)
            fn()
            for s in streams:
                cur.wait_stream(s)
        e1.record(cur)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    out = {"world": d, "chunk_MB": a.mb}
    for name, fn in (("ce_pull", pull), ("ce_push", push), ("ce_both", both)):
        ms = timed(fn)
        out[name] = {"ms": round(ms, 4), "GBps_per_dir": round((d - 1) * chunk / ms / 1e6, 1)}
    if rank == 0:
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
