"""Launch every hot-path kernel of libhod.so exactly once, at bucket size (for ncu).

    ncu --set full --clock-control none --import-source on -k regex:'_kernel' \
        -o gpurun_out/prof_each python tools/ncu_each.py

One GPU.  Kernels whose peers live on other GPUs (both span kernels in
FUSED / RS / ADAMW_AG modes) run with all d ranks' buffers on this
device and every barrier flag pre-set — the exact d-way code path with peer
loads/stores turned into local ones (tools/fused_emulated.py) — so their DRAM
traffic includes what the peers' NVLink traffic would put on HBM.  Prints the
launch order and each launch's algorithmic bytes (JSON) for
tools/ncu_summary.py.
"""

import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03549_b200 import _native as nat  # noqa: E402

DEV = "cuda"
NB = 33_554_432          # one LLaMA-7B / GPT-3 1.3B bucket (smallest, 2 tensors)
HP = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)


def entries(srcs):
    e = (nat.PackEntry * len(srcs))()
    off = 0
    for k, t in enumerate(srcs):
        e[k].src, e[k].numel, e[k].dst_offset = t.data_ptr(), t.numel(), off
        off += t.numel()
    return e


def span_kernel(d, mode, n_bucket=NB * 4, tma=1):
    """One emulated rank-0 launch of a span kernel over one bucket (tma=1:
    span_tma_kernel, the full-GPU default; 0: p2p_step_kernel, the
    co-resident / NVLS one, here at full grid)."""
    nat.call("hod_set_span_tma", tma)
    n = n_bucket // d
    grads = [torch.randn(n_bucket, device=DEV).mul_(1e-3).to(torch.bfloat16) for _ in range(d)]
    params = [torch.zeros(n_bucket, dtype=torch.bfloat16, device=DEV) for _ in range(d)]
    flags = [torch.full((8 * 8,), 1 << 32, dtype=torch.int64, device=DEV) for _ in range(d)]
    st = [torch.randn(n, device=DEV) * 0.02, torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)]
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    parts = torch.zeros(nat.HOD_SUMSQ_PARTIALS, device=DEV)
    coef = torch.ones(1, device=DEV)
    sp = nat.P2PSpan()
    for q in range(d):
        sp.grad[q], sp.param[q], sp.flags[q] = grads[q].data_ptr(), params[q].data_ptr(), flags[q].data_ptr()
    sp.local_grad = grads[0].data_ptr()
    sp.master, sp.exp_avg, sp.exp_avg_sq = (x.data_ptr() for x in st)
    sp.err = err.data_ptr()
    sp.bucket_start[0], sp.shard_numel[0] = 0, n
    sp.n_buckets, sp.d, sp.rank, sp.nvls, sp.keep_reduced = 1, d, 0, 0, 0
    sp.slot, sp.epoch, sp.timeout_ns = 0, 1, 5_000_000_000
    m = {"fused": nat.HOD_P2P_FUSED, "rs": nat.HOD_P2P_RS, "adamw_ag": nat.HOD_P2P_ADAMW_AG}[mode]
    if m == nat.HOD_P2P_RS:
        sp.partials = parts.data_ptr()
    if m == nat.HOD_P2P_ADAMW_AG:
        sp.clip_coef = coef.data_ptr()
    torch.cuda.synchronize()
    nat.call("hod_p2p_step", ctypes.byref(sp), m, ctypes.byref(HP), 0)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    # HBM bytes per owned element with the peers' copies local (see fused_emulated.py)
    per = {"fused": 2 * d + 24 + 2 * d, "rs": 2 * d + 2, "adamw_ag": 2 + 24 + 2 * d}[mode]
    nat.call("hod_set_span_tma", 1)
    return {"name": f"span_{'tma' if tma else 'reg'}_{mode}_d{d}", "owned_elems": n, "algorithmic_bytes": per * n}


def main():
    nat.load()
    torch.manual_seed(0)
    out = []
    half = [torch.randn(NB // 2, device=DEV).to(torch.bfloat16) for _ in range(2)]
    half32 = [torch.randn(NB // 2, device=DEV) for _ in range(2)]
    bucket = torch.empty(NB, dtype=torch.bfloat16, device=DEV)
    p = torch.randn(NB, device=DEV) * 0.02
    m = torch.zeros(NB, device=DEV)
    v = torch.zeros(NB, device=DEV)
    parts = torch.zeros(nat.HOD_SUMSQ_PARTIALS, device=DEV)
    torch.cuda.synchronize()

    def k(name, nbytes, fn):
        fn()
        torch.cuda.synchronize()
        out.append({"name": name, "elems": NB, "algorithmic_bytes": nbytes})

    k("pack_bf16", 4 * NB, lambda: nat.call("hod_pack_bf16", entries(half), 2, bucket.data_ptr(), NB,
                                           ctypes.c_float(0.5), 0, 0))
    k("pack_f32", 6 * NB, lambda: nat.call("hod_pack_bf16", entries(half32), 2, bucket.data_ptr(), NB,
                                          ctypes.c_float(0.5), 1, 0))
    k("sumsq", 2 * NB, lambda: nat.call("hod_sumsq_bf16", bucket.data_ptr(), NB, parts.data_ptr(), 0))
    k("adamw", 28 * NB, lambda: nat.call("hod_adamw_bf16", p.data_ptr(), m.data_ptr(), v.data_ptr(),
                                        bucket.data_ptr(), bucket.data_ptr(), NB, ctypes.byref(HP), None, 0))
    k("pack_adamw", 28 * NB, lambda: nat.call("hod_pack_adamw", entries(half), 2, NB, ctypes.c_float(1.0), 0,
                                             p.data_ptr(), m.data_ptr(), v.data_ptr(), bucket.data_ptr(),
                                             ctypes.byref(HP), None, 0))
    k("pack_sumsq", 2 * NB, lambda: nat.call("hod_pack_sumsq", entries(half), 2, NB, ctypes.c_float(1.0), 0,
                                            parts.data_ptr(), 0))
    for tma in (1, 0):
        for d in (2, 4, 8):
            out.append(span_kernel(d, "fused", tma=tma))
        for mode in ("rs", "adamw_ag"):
            for d in (2, 4, 8):
                out.append(span_kernel(d, mode, tma=tma))
    # the CO-RESIDENT variants that run beside the backward GEMMs (grid cap 148:
    # one CTA per SM, register span kernel with one item per thread, the
    # unroll-2 pack, max shared-memory carveout) — measured here alone
    nat.set_grid_base(148)
    try:
        k("pack_bf16_coresident", 4 * NB, lambda: nat.call("hod_pack_bf16", entries(half), 2, bucket.data_ptr(), NB,
                                                           ctypes.c_float(0.5), 0, 0))
        for d in (2, 4):
            doc = span_kernel(d, "fused", tma=1)
            doc["name"] = f"span_coresident_fused_d{d}"
            out.append(doc)
        doc = span_kernel(2, "rs", tma=1)
        doc["name"] = "span_coresident_rs_d2"
        out.append(doc)
    finally:
        nat.set_grid_base(0)
    print(json.dumps({"launch_order": out}))


if __name__ == "__main__":
    main()
