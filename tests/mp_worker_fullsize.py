"""One rank of the FULL-SIZE parity check (tests/test_fullsize_gpu.py).

Runs one DistributedOptimizer step over a whole BASELINE gradient set
(GPT-3 1.3B or LLaMA-7B, bf16 grads, backend auto) at d = WORLD_SIZE and
checks, in this process, the properties that hold at any size:

  * all-gather: a device checksum of the full bf16 param buffer is identical
    on every rank;
  * clip: the device grad norm equals an independent fp64 torch norm of the
    device-reduced shards (all-reduced) within 1e-5 relative;
  * sampled buckets (first, middle, last): this rank's shard against the
    oracle — every rank's gradients of the bucket regenerated from their
    seeds, packed and reduce-scattered by the oracle (bit-exact for the
    rank-ordered p2p sum; within d/2 bf16 ulp of sum|x| for NVLS), then the
    oracle AdamW from the pre-step state with the device's reduced shard and
    clip coefficient: master / m / v / the gathered bf16 params bit-exact.

Writes result_r{rank}.json; exits non-zero on any mismatch.
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

from oracle import oracle  # noqa: E402  (test infrastructure: the checker)
from paper_2312_03549_b200 import DistributedOptimizer  # noqa: E402
from paper_2312_03549_b200.comm import DPGroup  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def ulp_bf16(x):
    x = np.maximum(np.abs(x), np.finfo(np.float32).tiny)
    return np.exp2(np.floor(np.log2(x)) - 7)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt1.3b")
    ap.add_argument("--clip", type=float, default=0.0)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    oracle.set_threads(max(1, len(os.sched_getaffinity(0)) // world))
    gs = config_gradset(a.config)
    clip = a.clip if a.clip > 0 else None
    p0 = init_params(gs, dev)
    # d = 1 runs the fused pack+AdamW (the bench path: no bucket is written);
    # d > 1 keeps the reduced shard in place for the check
    opt = DistributedOptimizer(p0, bucket_size=25_000_000, clip=clip,
                               dp_group=DPGroup(tuple(range(world)), rank), keep_reduced=world > 1,
                               barrier_timeout_s=60.0)
    del p0
    torch.cuda.empty_cache()
    L = opt.layout
    nb = len(L.buckets)
    sample = sorted({0, nb // 2, nb - 1})
    offs = L.shard_offsets()
    pre = {}
    for bi in sample:
        n = L.buckets[bi].numel // world
        o = offs[bi]
        pre[bi] = tuple(x[o:o + n].cpu().numpy().copy() for x in (opt.master, opt.exp_avg, opt.exp_avg_sq))

    grads = make_grads(gs, 1, rank, dev)
    rep = opt.step(grads)
    torch.cuda.synchronize()
    opt.check_health()
    ss1 = sum(g.double().pow(2).sum() for g in grads) if world == 1 else None
    del grads
    torch.cuda.empty_cache()
    res = {"rank": rank, "world": world, "config": a.config, "backend": opt.backend, "buckets": nb,
           "sampled": sample, "params": L.param_numel}

    # all-gather: identical full param buffer everywhere (device checksum)
    ck = torch.zeros(2, dtype=torch.int64, device=dev)
    flat = opt.param_buffer.view(torch.int16)
    step_ = 1 << 26
    for lo in range(0, flat.numel(), step_):
        pb = flat[lo:lo + step_].to(torch.int64)
        idx = torch.arange(lo, lo + pb.numel(), device=dev, dtype=torch.int64)
        ck += torch.stack([pb.sum(), (pb * (idx % 65521 + 1)).sum()])
    del pb, idx
    cks = [torch.zeros_like(ck) for _ in range(world)]
    dist.all_gather(cks, ck)
    assert all(torch.equal(c, cks[0]) for c in cks), "param buffers differ between ranks"
    res["param_checksum"] = [int(x) for x in ck.tolist()]

    # clip: device norm vs an fp64 torch norm of the device-reduced shards
    if clip is not None:
        if world == 1:
            ss = ss1.reshape(1)
        else:
            ss = torch.zeros(1, dtype=torch.float64, device=dev)
            for b in L.buckets:
                lo, hi = b.shard_range(opt.shard_index, opt.dp)
                ss += opt.grad_buffer[lo:hi].double().pow(2).sum()
            dist.all_reduce(ss)
        ref = float(ss.sqrt())
        got = float(rep.grad_norm)
        assert abs(got - ref) <= 1e-5 * ref, (got, ref)
        res["grad_norm"], res["grad_norm_fp64"] = got, ref
        coef = float(rep.clip_coef)
    else:
        coef = None

    # sampled buckets against the oracle, streamed rank by rank so a process
    # holds only its own shard of every rank's packed bucket (host memory
    # stays ~1 GB per rank at d = 8 on the LLaMA-7B set)
    scale = 1.0 / world
    slices = {bi: [] for bi in sample}
    for q in range(world):
        gq = make_grads(gs, 1, q, dev)
        for bi in sample:
            b = L.buckets[bi]
            full = oracle.pack([u16(gq[s.index]).reshape(-1) for s in b.slots], [s.offset for s in b.slots],
                               b.numel, scale)
            sh = b.numel // world
            slices[bi].append(full[rank * sh:(rank + 1) * sh].copy())
            del full
        del gq
        torch.cuda.empty_cache()
    exact = opt.backend in ("p2p", "none")
    for bi in sample:
        b = L.buckets[bi]
        lo, hi = b.shard_range(opt.shard_index, opt.dp)
        dev_red = u16(opt.grad_buffer[lo:hi]) if world > 1 else slices[bi][0]
        if exact:
            want = oracle.sum_slices(slices[bi])
            assert np.array_equal(dev_red, want), f"bucket {bi}: reduced shard differs"
        else:
            f64 = oracle.sum_slices_f64(slices[bi])
            absum = sum(np.abs(oracle.bf16_to_f32(p).astype(np.float64)) for p in slices[bi])
            err = np.abs(oracle.bf16_to_f32(dev_red).astype(np.float64) - f64)
            assert np.all(err <= world * 0.5 * ulp_bf16(absum) + 1e-30), float(err.max())
        master, m, v = (x.copy() for x in pre[bi])
        p_bf16 = oracle.adamw(master, m, v, dev_red, 1, opt.lr, opt.betas, opt.eps, opt.weight_decay, coef=coef)
        o, n = offs[bi], hi - lo
        for name, want, got in (("master", master, opt.master), ("m", m, opt.exp_avg), ("v", v, opt.exp_avg_sq)):
            g = got[o:o + n].cpu().numpy()
            assert np.array_equal(g.view(np.uint32), want.view(np.uint32)), f"bucket {bi}: {name} differs"
        assert np.array_equal(u16(opt.param_buffer[lo:hi]), p_bf16), f"bucket {bi}: gathered params differ"
    res["ok"] = True
    Path(a.out, f"result_r{rank}.json").write_text(json.dumps(res))
    opt.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
