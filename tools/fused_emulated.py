"""The fused span kernel of ONE rank on ONE GPU (peers emulated; for ncu).

    python tools/fused_emulated.py [--d 2] [--numel 268435456] [--mode fused|rs|adamw_ag]

All d ranks' buffers live on this device and every barrier flag is pre-set,
so the launch runs straight through with the exact d-way code path (peer
loads become local loads).  Prints the device time per launch (CUDA events,
warm) and the per-owned-element algorithmic HBM bytes; run it under
`ncu --set full -k regex:p2p_step_kernel -c 1` for the compute profile
(issue utilisation, stall reasons) that a multi-rank run cannot give.
"""

import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03549_b200 import _native as nat  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--numel", type=int, default=1 << 28)
    ap.add_argument("--mode", default="fused", choices=["fused", "rs", "adamw_ag"])
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    nat.load()
    dev = "cuda"
    d, N = a.d, a.numel
    n = N // d
    grads = [torch.randn(N, device=dev).mul_(1e-3).to(torch.bfloat16) for _ in range(d)]
    params = [torch.zeros(N, dtype=torch.bfloat16, device=dev) for _ in range(d)]
    flags = [torch.full((8 * 8,), 1 << 32, dtype=torch.int64, device=dev) for _ in range(d)]
    st = [torch.randn(n, device=dev) * 0.02, torch.zeros(n, device=dev), torch.zeros(n, device=dev)]
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    parts = torch.zeros(nat.HOD_SUMSQ_PARTIALS, device=dev)
    coef = torch.ones(1, device=dev)
    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)
    sp = nat.P2PSpan()
    for q in range(d):
        sp.grad[q], sp.param[q], sp.flags[q] = grads[q].data_ptr(), params[q].data_ptr(), flags[q].data_ptr()
    sp.local_grad = grads[0].data_ptr()
    sp.master, sp.exp_avg, sp.exp_avg_sq = (x.data_ptr() for x in st)
    sp.err = err.data_ptr()
    sp.bucket_start[0], sp.shard_numel[0] = 0, n
    sp.n_buckets, sp.d, sp.rank, sp.nvls, sp.keep_reduced = 1, d, 0, 0, 0
    sp.slot, sp.epoch, sp.timeout_ns = 0, 1, 5_000_000_000
    mode = {"fused": nat.HOD_P2P_FUSED, "rs": nat.HOD_P2P_RS, "adamw_ag": nat.HOD_P2P_ADAMW_AG}[a.mode]
    if mode == nat.HOD_P2P_RS:
        sp.partials = parts.data_ptr()
    if mode == nat.HOD_P2P_ADAMW_AG:
        sp.clip_coef = coef.data_ptr()

    def run():
        nat.call("hod_p2p_step", ctypes.byref(sp), mode, ctypes.byref(hp), 0)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    ms = e0.elapsed_time(e1) / a.iters
    # local HBM bytes per owned element: d grad reads + (fused/adamw_ag) 24 B state + d param writes
    per = {"fused": 2 * d + 24 + 2 * d, "rs": 2 * d + 2, "adamw_ag": 2 + 24 + 2 * d}[a.mode]
    print(json.dumps({"d": d, "mode": a.mode, "owned_elems": n, "ms": round(ms, 4),
                      "Gelem_per_s": round(n / ms / 1e6, 1), "bytes_per_owned_elem": per,
                      "hbm_GBps": round(per * n / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
