"""Can a memory-bound optimizer kernel co-reside with backward GEMMs?

    python tools/corun_probe.py [--tokens 8192] [--hidden 2048]

Runs a loop of cuBLAS bf16 GEMMs of the GPT-3 1.3B backward shapes on stream A
and the sm_100a AdamW kernel (hod_adamw_bf16, exact and fast) over a 1.3B/2
shard on stream B: alone, and together (GEMMs launched first, the update
second, and the reverse), with the update's grid capped at 148 / 296 / 592
CTAs.  Prints one JSON line per case: t_gemm, t_mem, t_both (CUDA events,
both streams joined) and hidden = (t_gemm + t_mem - t_both) / t_mem (1 = the
update fully hidden behind the GEMMs, 0 = serialised).
"""

import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03549_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=8192)
    ap.add_argument("--hidden", type=int, default=2048)
    ap.add_argument("--numel", type=int, default=1 << 28)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kernel", default="adamw", choices=["adamw", "fused_d2", "pack"])
    ap.add_argument("--grids", default="0,148,296,592")
    ap.add_argument("--green", type=int, default=0,
                    help="run the optimizer kernel on a CUDA green context of this many SMs (the GEMMs keep "
                         "the primary context)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    h, T = a.hidden, a.tokens
    shapes = [(3 * h, h), (h, h), (4 * h, h), (h, 4 * h)] * 4
    acts = {d: torch.randn(T, d, device=dev, dtype=torch.bfloat16) for d in (h, 3 * h, 4 * h)}
    ws = [torch.randn(o, i, device=dev, dtype=torch.bfloat16) * 0.02 for o, i in shapes]
    outs = [torch.empty(o, i, device=dev, dtype=torch.bfloat16) for o, i in shapes]

    def gemms():
        for (o, i), w, out in zip(shapes, ws, outs):
            torch.matmul(acts[o], w)
            torch.matmul(acts[o].t(), acts[i], out=out)

    n = a.numel
    master = torch.randn(n, device=dev) * 0.02
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    g = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
    p = torch.empty(n, device=dev, dtype=torch.bfloat16)
    L = _native.load()

    # fused_d2: the d = 2 span kernel (RS + AdamW + AG) of rank 0 with the
    # peer emulated on this GPU (flags pre-set, as tools/fused_emulated.py)
    g2 = [g, (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)] if a.kernel == "fused_d2" else None
    if g2:
        pp = [p, torch.empty(n, device=dev, dtype=torch.bfloat16)]
        flags = [torch.full((64,), 1 << 32, dtype=torch.int64, device=dev) for _ in range(2)]
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        sp = _native.P2PSpan()
        for q in range(2):
            sp.grad[q], sp.param[q], sp.flags[q] = g2[q].data_ptr(), pp[q].data_ptr(), flags[q].data_ptr()
        sp.local_grad = g.data_ptr()
        sp.master, sp.exp_avg, sp.exp_avg_sq = master.data_ptr(), m.data_ptr(), v.data_ptr()
        sp.err = err.data_ptr()
        sp.bucket_start[0], sp.shard_numel[0] = 0, n // 2
        sp.n_buckets, sp.d, sp.rank, sp.nvls, sp.keep_reduced = 1, 2, 0, 0, 0
        sp.slot, sp.epoch, sp.timeout_ns = 0, 1, 5_000_000_000
    if a.kernel == "pack":
        src = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16)
        ent = (_native.PackEntry * 1)()
        ent[0].src, ent[0].numel, ent[0].dst_offset = src.data_ptr(), n, 0
    # algorithmic HBM bytes per launch
    nbytes = {"adamw": 28 * n, "fused_d2": 32 * (n // 2), "pack": 4 * n}[a.kernel]

    def update(stream, mode):
        hp = _native.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1, mode, 0)
        if a.kernel == "adamw":
            rc = L.hod_adamw_bf16(master.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                                  p.data_ptr(), n, ctypes.byref(hp), None, _native.stream_ptr(stream))
        elif a.kernel == "fused_d2":
            rc = L.hod_p2p_step(ctypes.byref(sp), _native.HOD_P2P_FUSED, ctypes.byref(hp), _native.stream_ptr(stream))
        else:
            rc = L.hod_pack_bf16(ent, 1, g.data_ptr(), n, ctypes.c_float(0.5), 0, _native.stream_ptr(stream))
        _native.check(rc, a.kernel)

    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    if a.green:
        gctx = torch.cuda.green_contexts.GreenContext.create(a.green, 0)
        gs_ = gctx.Stream()
        sb = torch.cuda.Stream(stream_id=gs_.stream_id, device_index=gs_.device_index, device_type=gs_.device_type)

    def timed(fn):
        best = None
        for _ in range(a.reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            sa.wait_event(e0)
            sb.wait_event(e0)
            fn()
            ea, eb = torch.cuda.Event(), torch.cuda.Event()
            ea.record(sa)
            eb.record(sb)
            torch.cuda.current_stream().wait_event(ea)
            torch.cuda.current_stream().wait_event(eb)
            e1.record(torch.cuda.current_stream())
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return best

    for _ in range(2):
        with torch.cuda.stream(sa):
            gemms()
        update(sb, 0)
    torch.cuda.synchronize()

    def g_only():
        with torch.cuda.stream(sa):
            gemms()

    t_g = timed(g_only)
    print(json.dumps({"case": "gemm_alone", "ms": round(t_g, 3), "gemms": 2 * len(shapes)}), flush=True)
    for grid in [int(x) for x in a.grids.split(",")]:
        _native.set_grid_base(grid)
        for mode in ((0, 1) if a.kernel != "pack" else (0,)):
            t_m = timed(lambda: update(sb, mode))
            res = {"kernel": a.kernel, "carveout": os.environ.get("HOD_CARVEOUT", "1"), "grid_cap": grid,
                   "green_sms": a.green,
                   "adamw": "fast" if mode else "exact", "numel": n, "t_gemm": round(t_g, 3),
                   "t_mem": round(t_m, 3), "mem_GBps": round(nbytes / t_m / 1e6, 1)}
            for order in ("gemm_first", "mem_first"):
                def both():
                    if order == "gemm_first":
                        with torch.cuda.stream(sa):
                            gemms()
                        update(sb, mode)
                    else:
                        update(sb, mode)
                        with torch.cuda.stream(sa):
                            gemms()
                t_b = timed(both)
                res[order] = {"t_both": round(t_b, 3), "hidden": round((t_g + t_m - t_b) / t_m, 3)}
            print(json.dumps(res), flush=True)
    _native.set_grid_base(0)


if __name__ == "__main__":
    main()
