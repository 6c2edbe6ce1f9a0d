"""SM-issued NVLink bandwidth ceiling over peer-mapped memory (tool).

    torchrun --nproc-per-node N tools/peer_bw.py [--mb 256]

Builds tools/peer_bw.cu into tools/_peer_bw.so (nvcc, sm_100a) on first use.
read : every rank pulls its shard region (chunk bytes) from all d copies at
       once (the reduce-scatter access pattern; own copy local)
write: every rank stores its chunk into all d copies (the all-gather pattern)
NVLink bytes per GPU per direction = (d-1) * chunk.  Sweeps bytes per lane
(8 / 16), loads in flight per thread (unroll) and grid size.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.symm import SymmetricTensor  # noqa: E402


def lib():
    so = os.path.join(HERE, "_peer_bw.so")
    src = os.path.join(HERE, "peer_bw.cu")
    if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", so, src])
    L = ctypes.CDLL(so)
    L.peer_bw_run.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p]
    L.tma_bw_run.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    L.nvls_bw_run.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                              ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=256)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--ops", default="read,write",
                    help="comma list of read, write, both (p2p), tma_read, tma_both (bulk-copy engine) "
                         "and nvls_rs, nvls_ag, nvls_both (multicast)")
    a = ap.parse_args()
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        lib()
    dist.barrier()
    L = lib()
    nat.load()
    d = world
    chunk = a.mb << 20
    ops = a.ops.split(",")
    buf = SymmetricTensor(2 * d * chunk, torch.uint8, dev, None, zero=True)
    out = torch.zeros(16, dtype=torch.uint8, device=dev)
    ptrs = (ctypes.c_void_p * d)(*[buf.peer(q) for q in range(d)])
    s = torch.cuda.current_stream(dev)

    modes = {"read": 0, "write": 1, "nvls_rs": 2, "nvls_ag": 3, "nvls_both": 4, "both": 5,
             "tma_read": 6, "tma_both": 7}

    def run(mode, vec, unroll, grid):
        if mode in (6, 7):
            rc = L.tma_bw_run(ptrs, d, rank * chunk, chunk, out.data_ptr(), mode, vec, unroll, grid,
                              s.cuda_stream)
        elif mode in (2, 3, 4):
            rc = L.nvls_bw_run(buf.multicast(), rank * chunk, (d + rank) * chunk, chunk, out.data_ptr(), mode, vec,
                               unroll, grid, s.cuda_stream)
        else:
            rc = L.peer_bw_run(ptrs, d, rank * chunk, chunk, out.data_ptr(), mode, vec, unroll, grid,
                               s.cuda_stream)
        assert rc == 0, rc

    results = []
    def grid_sweep(mode, vec, unroll):
        if mode not in (6, 7):
            return [(vec, unroll, g) for g in (148, 296, 592, 1184)]
        # TMA: vec = tile bytes per peer, unroll = ring stages; grid = CTAs that fit
        smem = unroll * d * vec + (unroll * vec if mode == 7 else 0) + 64
        per_sm = min(4, (227 * 1024) // smem)
        return [(vec, unroll, 148 * k) for k in range(1, per_sm + 1)] if smem <= 227 * 1024 else []

    for op in ops:
        mode = modes[op]
        if mode in (6, 7):
            combos = [c for t in (4096, 8192, 16384) for st in (2, 3, 4) for c in grid_sweep(mode, t, st)]
        else:
            combos = [c for vec in (8, 16) for unroll in ((1, 2, 4) if mode not in (1, 5) else (1,))
                      for c in grid_sweep(mode, vec, unroll)]
        for vec, unroll, grid in combos:
            for _ in range(2):
                run(mode, vec, unroll, grid)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.iters):
                run(mode, vec, unroll, grid)
            e1.record(s)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.iters], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t)
            r = {"op": op, "bytes_per_lane": vec, "unroll": unroll, "grid": grid, "ms": round(ms, 4),
                 "nvlink_GBps_per_dir": round((d - 1) * chunk / ms / 1e6, 1)}
            if mode in (6, 7):
                r["tile_bytes"], r["stages"] = r.pop("bytes_per_lane"), r.pop("unroll")
            if mode in (5, 7):
                # RS in + AG in from the peers' stores, per direction
                r["nvlink_GBps_per_dir"] = round(2 * (d - 1) * chunk / ms / 1e6, 1)
            if mode in (2, 3, 4):
                # physical bytes per GPU: the switch reads every copy (rs: egress d*chunk,
                # ingress chunk), replicates every store (ag: egress chunk, ingress d*chunk)
                eg = {2: d, 3: 1, 4: d + 1}[mode] * chunk
                ig = {2: 1, 3: d, 4: d + 1}[mode] * chunk
                r.update({"egress_GBps": round(eg / ms / 1e6, 1), "ingress_GBps": round(ig / ms / 1e6, 1)})
                del r["nvlink_GBps_per_dir"]
            results.append(r)
    if rank == 0:
        for r in results:
            print(json.dumps({"world": d, "chunk_MB": a.mb, **r}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
