"""Micro-benchmark of the fused peer-memory collectives vs NCCL on one bucket.

    torchrun --nproc-per-node N tools/p2p_microbench.py [--numel 100000000]

Per rank, for a bucket of ``numel`` bf16 elements (shard n = numel/N):
  fused_p2p / fused_nvls : barrier + RS + AdamW + AG in one kernel
  rs_p2p / rs_nvls       : barrier + RS only (reduced shard + sumsq partials)
  adamw_ag_p2p / _nvls   : AdamW + AG from the local reduced shard
  nccl_rs+ag             : ncclReduceScatter + ncclAllGather (bf16, in place)
  adamw_local            : K2 on the shard (HBM only)
Times are CUDA-event device times (max over ranks), after warm-up.
NVLink bytes per GPU per direction for RS+AG = 4 n (N-1) (bf16).
"""

import argparse
import ctypes
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.comm import NcclComm  # noqa: E402
from paper_2312_03549_b200.symm import SymmetricTensor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--numel", type=int, default=104_857_600)
    ap.add_argument("--sweep", action="store_true",
                    help="BASELINE config 5: bucket sizes 1 MB .. 1 GB (0.5M .. 512M bf16 elements)")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    nat.load()
    comm = NcclComm(tuple(range(world)), rank, "bench")
    sizes = [(1 << 20) // 2 * (1 << k) for k in range(11)] if a.sweep else [a.numel]
    for numel in sizes:
        iters = max(5, min(50, int(2e9 // (numel * 2)))) if a.sweep else a.iters
        doc = measure_bucket(numel, iters, world, rank, dev, comm)
        if rank == 0:
            print(json.dumps(doc, indent=None if a.sweep else 1), flush=True)
    comm.close()
    dist.destroy_process_group()


def measure_bucket(numel, iters, world, rank, dev, comm, cases=None) -> dict:
    """Time the fused kernels and NCCL RS+AG on one bucket of ``numel`` bf16
    elements (CUDA events, max over ranks); ``cases`` limits the set."""
    N = numel - numel % (16 * world)
    n = N // world
    pg = dist.group.WORLD
    g = SymmetricTensor(N, torch.bfloat16, dev, pg)
    p = SymmetricTensor(N, torch.bfloat16, dev, pg, zero=True)
    fl = SymmetricTensor(64 * 8, torch.int64, dev, pg, zero=True)
    g.tensor.normal_(0, 1e-3)
    master = torch.randn(n, device=dev) * 0.02
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    red = torch.empty(n, dtype=torch.bfloat16, device=dev)
    parts = torch.empty(nat.HOD_SUMSQ_PARTIALS, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    coef = torch.ones(1, device=dev)
    torch.cuda.synchronize()
    dist.barrier()
    s = torch.cuda.current_stream()
    epoch = [0]

    def bucket(nvls):
        sp = nat.P2PSpan()
        if nvls:
            sp.grad[0], sp.param[0] = g.multicast(), p.multicast()
        else:
            for q in range(world):
                sp.grad[q], sp.param[q] = g.peer(q), p.peer(q)
        for q in range(world):
            sp.flags[q] = fl.peer(q)
        sp.local_grad = g.tensor.data_ptr()
        sp.master, sp.exp_avg, sp.exp_avg_sq = master.data_ptr(), m.data_ptr(), v.data_ptr()
        sp.err = err.data_ptr()
        sp.bucket_start[0], sp.shard_numel[0], sp.n_buckets = 0, n, 1
        sp.d, sp.rank, sp.nvls = world, rank, int(nvls)
        sp.slot, sp.timeout_ns = 0, 10_000_000_000
        return sp

    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)

    def run_mode(mode, nvls):
        sp = bucket(nvls)
        epoch[0] += 1
        sp.epoch = epoch[0]
        if mode == nat.HOD_P2P_RS:
            sp.partials = parts.data_ptr()
        if mode == nat.HOD_P2P_ADAMW_AG:
            sp.clip_coef = coef.data_ptr()
        nat.call("hod_p2p_step", ctypes.byref(sp), mode, ctypes.byref(hp), s.cuda_stream)

    def nccl_rs_ag():
        base = g.tensor.data_ptr()
        comm.reduce_scatter_bf16(base, base + 2 * rank * n, n, s)
        comm.all_gather_bf16(p.tensor.data_ptr() + 2 * rank * n, p.tensor.data_ptr(), n, s)

    def adamw_local():
        nat.call("hod_adamw_bf16", master.data_ptr(), m.data_ptr(), v.data_ptr(), red.data_ptr(),
                 p.tensor.data_ptr() + 2 * rank * n, n, ctypes.byref(hp), None, s.cuda_stream)

    all_cases = {
        "fused_p2p": lambda: run_mode(nat.HOD_P2P_FUSED, False),
        "rs_p2p": lambda: run_mode(nat.HOD_P2P_RS, False),
        "adamw_ag_p2p": lambda: run_mode(nat.HOD_P2P_ADAMW_AG, False),
        "fused_nvls": lambda: run_mode(nat.HOD_P2P_FUSED, True),
        "rs_nvls": lambda: run_mode(nat.HOD_P2P_RS, True),
        "adamw_ag_nvls": lambda: run_mode(nat.HOD_P2P_ADAMW_AG, True),
        "nccl_rs+ag": nccl_rs_ag,
        "adamw_local": adamw_local,
    }
    out = {}
    for name, fn in all_cases.items():
        if (cases is not None and name not in cases) or ("nvls" in name and not (g.mc and p.mc)):
            continue
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nvl = 4 * n * (world - 1) if "fused" in name or "nccl" in name else 2 * n * (world - 1)
        if name == "adamw_local":
            nvl = 0
        # nccl-tests convention for RS+AG over a bucket of N bf16 elements:
        # busBW = (2 N bytes / t) * (d-1)/d per collective, two collectives
        bus = (2 * 2 * N / (ms / 1e3)) * (world - 1) / world / 1e9 if ("fused" in name or "nccl" in name) else None
        out[name] = {"ms": round(ms, 4), "nvlink_GBps_per_dir": round(nvl / ms / 1e6, 1),
                     "hbm_state_GBps": round(28 * n / ms / 1e6, 1),
                     "busBW_GBps": round(bus, 1) if bus else None}
    if int(err.item()):
        out["error"] = int(err.item())
    doc = {"world": world, "numel": N, "bucket_MB": round(2 * N / 2**20, 2), "shard": n, "results": out}
    del g, p, fl
    torch.cuda.empty_cache()
    return doc


if __name__ == "__main__":
    main()
