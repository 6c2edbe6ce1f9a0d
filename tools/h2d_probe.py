"""Host->device bandwidth of pinned gradient uploads with all ranks at once (tool).

    torchrun --nproc-per-node N tools/h2d_probe.py [--mb 2048]

The e2e arm of bench.py uploads every rank's gradient replica from pinned host
memory each step.  This probe times that upload with every rank copying at
once, first from a pinned buffer allocated with the process's default CPU
affinity, then after binding the process to the CPUs of its GPU's NUMA node
(sysfs local_cpulist) and allocating a fresh buffer there (first touch places
the pages on that node).  Prints one JSON line per variant from rank 0.
"""

import argparse
import json
import os

import torch
import torch.distributed as dist


def gpu_cpus(dev_index: int):
    p = torch.cuda.get_device_properties(dev_index)
    bus = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    path = f"/sys/bus/pci/devices/{bus}"
    cpus = set()
    try:
        txt = open(f"{path}/local_cpulist").read().strip()
        for part in txt.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        node = int(open(f"{path}/numa_node").read())
    except OSError:
        node = -1
    return bus, node, sorted(cpus)


def timed_upload(host, dev_buf, iters):
    s = torch.cuda.current_stream()
    dev_buf.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(iters):
        dev_buf.copy_(host, non_blocking=True)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    t = torch.tensor([ms], device=dev_buf.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    nbytes = a.mb << 20
    dev_buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    bus, node, cpus = gpu_cpus(local)
    info = [None] * world
    dist.all_gather_object(info, {"rank": rank, "bus": bus, "numa": node, "ncpus": len(cpus),
                                  "affinity_before": len(os.sched_getaffinity(0))})
    out = []
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    host.fill_(1)
    out.append(("default", timed_upload(host, dev_buf, a.iters)))
    del host
    if cpus:
        os.sched_setaffinity(0, cpus)
        torch.set_num_threads(max(1, min(8, len(cpus))))
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    host.fill_(1)
    out.append(("numa_bound", timed_upload(host, dev_buf, a.iters)))
    if rank == 0:
        for name, ms in out:
            print(json.dumps({"variant": name, "world": world, "MB_per_rank": a.mb, "ms": round(ms, 3),
                              "GBps_per_rank": round(nbytes / ms / 1e6, 1),
                              "GBps_aggregate": round(world * nbytes / ms / 1e6, 1), "ranks": info}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
