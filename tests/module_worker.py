"""Real-module integration at d > 1, checked against the oracle.

Every DP rank trains its own replica of a LLaMA-style block stack
(tests/llama_blocks.py) bound to its DistributedOptimizer with ``attach``:
the parameters are views of the flat bf16 buffer, post-accumulate-grad hooks
launch the buckets during backward, forward pre-hooks ``wait_params`` on
each submodule's buckets, and ``finish_step(wait=False)`` leaves the last
spans' all-gather to overlap the next forward.  Each rank sees different
tokens.  After every step the gradients every rank delivered are packed,
reduce-scattered and stepped by the oracle: reduced shards, master / m / v
and the params the NEXT forward reads are bit-exact (clip coefficient = the
device's, identical on every rank; norm within 1e-5 of the oracle's).

  --mode emulated : d ranks on one GPU (emulation.EmulatedRow; run with
                    emulation.child_env()), the driver-visible case;
  --mode dist     : one process per GPU under torch.distributed.run (real
                    NVLink peer memory), also reports the optimizer's exposed
                    time in the training iteration.
"""

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import llama_blocks  # noqa: E402
from emu_worker import check  # noqa: E402
from paper_2312_03549_b200 import DistributedOptimizer  # noqa: E402
from paper_2312_03549_b200.comm import DPGroup  # noqa: E402


def make_opt(model, a, r, d, **kw):
    init = [p.detach().float().clone() for p in model.parameters()]
    return DistributedOptimizer(init, bucket_size=a.bucket, clip=a.clip if a.clip > 0 else None,
                                dp_group=DPGroup(tuple(range(d)), r), backend="p2p",
                                keep_reduced=True, barrier_timeout_s=a.timeout, **kw)


def train_step(model, opt, step, rank, a, dev):
    """forward (pre-hooks wait for the previous step's params) + backward
    (hooks launch buckets) + finish_step(wait=False); returns the delivered grads."""
    inp, tgt = llama_blocks.batch(a.vocab, a.tokens, a.seq, step, rank, dev)
    opt.begin_step()
    loss = llama_blocks.loss_fn(model, inp, tgt)
    loss.backward()
    grads = [p.grad.detach().clone() for p in model.parameters()]
    rep = opt.finish_step(wait=False)
    for p in model.parameters():
        p.grad = None
    return rep, grads, loss


def model_kw(a):
    return dict(vocab=a.vocab, dim=a.dim, layers=a.layers, heads=a.heads, ffn=a.ffn)


def run_emulated(a):
    from paper_2312_03549_b200.emulation import EmulatedRow, connections_ok

    if not connections_ok():
        raise SystemExit("start with emulation.child_env()")
    dev = torch.device("cuda", 0)
    d = a.d
    out = {"mode": "emulated", "d": d, "clip": a.clip}
    with EmulatedRow(d, dev) as row:
        streams = row.streams()
        models, opts = [], []
        for r in range(d):
            with torch.cuda.stream(streams[r]):
                m = llama_blocks.build(dev, seed=0, **model_kw(a))      # same init on every rank
                o = make_opt(m, a, r, d, symmetric=row.factory(r))
                o.attach(m)
            models.append(m)
            opts.append(o)
        torch.cuda.synchronize()
        state = [[x.cpu().numpy().copy() for x in (o.master, o.exp_avg, o.exp_avg_sq)] for o in opts]
        for step in range(1, a.steps + 1):
            reps, grads = [None] * d, [None] * d
            for r in range(d):
                with torch.cuda.stream(streams[r]):
                    reps[r], grads[r], _ = train_step(models[r], opts[r], step, r, a, dev)
            for rp in reps:
                rp.resolve()
            torch.cuda.synchronize()
            check(argparse.Namespace(d=d, clip=a.clip, keep_reduced=1), opts, None, step, grads, state, reps)
            # the model reads the gathered params: its parameters ARE the buffer
            for m, o in zip(models, opts):
                for p, v in zip(m.parameters(), o.params):
                    assert p.data_ptr() == v.data_ptr()
        out["buckets"] = len(opts[0].layout.buckets)
        out["params"] = opts[0].layout.param_numel
        out["ok"] = True
        for o in opts:
            o.close()
    print(json.dumps(out), flush=True)


def run_dist(a):
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    model = llama_blocks.build(dev, seed=0, **model_kw(a))
    opt = make_opt(model, a, rank, world)
    opt.attach(model)
    out = {"mode": "dist", "d": world, "clip": a.clip, "buckets": len(opt.layout.buckets),
           "params": opt.layout.param_numel}
    if a.check:
        state = [[x.cpu().numpy().copy() for x in (opt.master, opt.exp_avg, opt.exp_avg_sq)]]
        for step in range(1, a.steps + 1):
            rep, grads, _ = train_step(model, opt, step, rank, a, dev)
            rep.resolve()
            torch.cuda.synchronize()
            # every rank's delivered gradients, for the oracle on every rank
            allg = []
            for g in grads:
                parts = [torch.empty_like(g) for _ in range(world)]
                dist.all_gather(parts, g.contiguous())
                allg.append(parts)
            per_rank = [[allg[i][q] for i in range(len(grads))] for q in range(world)]
            check_dist(a, opt, step, per_rank, state, rep, world, rank)
        out["ok"] = True
    if a.time_iters:
        # exposure: training iterations with the optimizer vs the same
        # forward/backward without it (grads dropped)
        def iteration(with_opt, step):
            inp, tgt = llama_blocks.batch(a.vocab, a.tokens, a.seq, step, rank, dev)
            if with_opt:
                opt.begin_step()
                llama_blocks.loss_fn(model, inp, tgt).backward()
                opt.finish_step(wait=False)
            else:
                with opt.no_sync():
                    llama_blocks.loss_fn(model, inp, tgt).backward()
            for p in model.parameters():
                p.grad = None

        res = {}
        for with_opt in (False, True, False, True):
            for i in range(3):
                iteration(with_opt, 1000 + i)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for i in range(a.time_iters):
                iteration(with_opt, 2000 + i)
            for b in range(len(opt.layout.buckets)):
                opt.wait_params(b)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.time_iters], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res.setdefault("with" if with_opt else "without", []).append(float(t))
        t_w, t_wo = min(res["with"]), min(res["without"])
        # the optimizer alone (resident grads, step())
        grads = [torch.randn_like(p) * 1e-3 for p in model.parameters()]
        for _ in range(3):
            opt.step(grads)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            opt.step(grads)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 5], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_opt = float(t)
        out["timing"] = {"tokens_per_gpu": a.tokens, "t_iter_without_opt_ms": t_wo, "t_iter_with_opt_ms": t_w,
                         "t_optimizer_alone_ms": t_opt,
                         "exposed_frac_iteration": (t_w - t_wo) / t_w,
                         "hidden_frac_of_optimizer": 1.0 - (t_w - t_wo) / t_opt}
    opt.check_health()
    if rank == 0:
        print(json.dumps(out), flush=True)
    opt.close()
    dist.barrier()
    dist.destroy_process_group()


def check_dist(a, opt, step, per_rank, state, rep, world, rank):
    """This rank's shard of every bucket against the oracle (all ranks' grads)."""
    from oracle import oracle

    def u16(t):
        return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)

    L = opt.layout
    offs = L.shard_offsets()
    hg = [[u16(g) for g in per_rank[q]] for q in range(world)]
    coef = float(rep.clip_coef.item()) if rep.clip_coef is not None else None
    gbuf, pbuf = u16(opt.grad_buffer), u16(opt.param_buffer)
    dev_state = [x.cpu().numpy() for x in (opt.master, opt.exp_avg, opt.exp_avg_sq)]
    for bi, b in enumerate(L.buckets):
        packs = [oracle.pack([hg[q][s.index] for s in b.slots], [s.offset for s in b.slots], b.numel, 1.0 / world)
                 for q in range(world)]
        red = oracle.reduce_scatter(packs, rank, world)
        n = b.numel // world
        lo = b.start + rank * n
        assert np.array_equal(gbuf[lo:lo + n], red), f"step {step} bucket {bi}: RS"
        master, m, v = (x[offs[bi]:offs[bi] + n] for x in state[0])
        want = oracle.adamw(master, m, v, red, step, coef=coef)
        assert np.array_equal(pbuf[lo:lo + n], want), f"step {step} bucket {bi}: params"
        for name, dv, ov in zip(("master", "m", "v"), dev_state, (master, m, v)):
            assert np.array_equal(dv[offs[bi]:offs[bi] + n].view(np.uint32), ov.view(np.uint32)), name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="emulated", choices=["emulated", "dist"])
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--clip", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--bucket", type=int, default=300_000)
    ap.add_argument("--vocab", type=int, default=1000)
    ap.add_argument("--dim", type=int, default=256)
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--ffn", type=int, default=688)
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--seq", type=int, default=128)
    ap.add_argument("--timeout", type=float, default=20.0)
    ap.add_argument("--check", type=int, default=1)
    ap.add_argument("--time-iters", type=int, default=0)
    a = ap.parse_args()
    if a.mode == "emulated":
        run_emulated(a)
    else:
        run_dist(a)


if __name__ == "__main__":
    main()
