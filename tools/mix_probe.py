"""Does mixing SM-issued and copy-engine peer reads beat either alone?

    torchrun --nproc-per-node N tools/mix_probe.py [--mb 256]

Every rank pulls one chunk from every peer (the reduce-scatter direction),
all ranks at once: by SM copy kernels only (torch copy from the peer-mapped
view), by the copy engines only (hod_ce_copy), and mixed — the chunk of each
peer split between an SM copy and a copy-engine copy in the ratio --ce-frac.
Incoming GB/s per GPU (= per direction), CUDA events, max over ranks.
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
    stage = torch.empty(d * chunk, dtype=torch.uint8, device=dev)
    peers = [q for q in range(d) if q != rank]
    streams = [torch.cuda.Stream(dev) for _ in range(2 * len(peers))]
    views = {q: src.handle.get_buffer(q, (d * chunk,), torch.uint8) for q in peers}

    def pull(ce_frac):
        for k, q in enumerate(peers):
            cut = int(chunk * ce_frac) // 4096 * 4096
            lo = rank * chunk
            if cut < chunk:      # SM part
                with torch.cuda.stream(streams[2 * k]):
                    stage[q * chunk + cut:(q + 1) * chunk].copy_(views[q][lo + cut:lo + chunk])
            if cut > 0:          # copy-engine part
                nat.call("hod_ce_copy", stage.data_ptr() + q * chunk, src.peer(q, lo), cut,
                         nat.stream_ptr(streams[2 * k + 1]))

    def timed(fn):
        cur = torch.cuda.current_stream(dev)

        def once():
            for s in streams:
                s.wait_stream(cur)
            fn()
            for s in streams:
                cur.wait_stream(s)
        for _ in range(2):
            once()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(a.iters):
            once()
        e1.record(cur)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / a.iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    for frac in (0.0, 1.0, 0.25, 0.5, 0.75):
        ms = timed(lambda: pull(frac))
        if rank == 0:
            print(json.dumps({"world": d, "chunk_MB": a.mb, "ce_frac": frac, "ms": round(ms, 4),
                              "GBps_in_per_gpu": round(len(peers) * chunk / ms / 1e6, 1)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
