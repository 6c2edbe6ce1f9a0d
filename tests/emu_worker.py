"""d DistributedOptimizer ranks of one DP row, concurrently on ONE GPU.

Launched by tests/test_emulated_optimizer_gpu.py in a fresh process with
CUDA_DEVICE_MAX_CONNECTIONS=32 CUDA_MODULE_LOADING=EAGER (emulation.child_env).  Every
rank owns its optimizer, streams and buffers; peer pointers resolve to the
other ranks' allocations, so arrival barriers, span tags, params-ready
barriers and the peer-memory norm exchange all run for real, each flag raised
by a peer kernel running at the same time.  After every step each rank is
checked against the oracle (oracle/oracle.py): reduced shard and master / m /
v / bf16 params bit-exact (the clip coefficient is the device's, identical on
every rank; the device norm within 1e-5 of the oracle's), params identical on
all ranks.

Usage: python tests/emu_worker.py --d 4 [--clip 0.02] [--flow step|hooks]
       python tests/emu_worker.py --d 2 --fault timeout|span
"""

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402
from paper_2312_03549_b200 import DistributedOptimizer  # noqa: E402
from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.comm import DPGroup  # noqa: E402
from paper_2312_03549_b200.emulation import EmulatedRow, connections_ok  # noqa: E402
from paper_2312_03549_b200.errors import DeviceError  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def host_grad(g):
    return u16(g) if g.dtype == torch.bfloat16 else g.detach().cpu().numpy()


def build(a, row, dev, gs, span_numel=None):
    opts = []
    for r in range(a.d):
        opts.append(DistributedOptimizer(
            init_params(gs, dev), bucket_size=a.bucket, clip=a.clip if a.clip > 0 else None,
            dp_group=DPGroup(tuple(range(a.d)), r), backend="p2p", keep_reduced=bool(a.keep_reduced),
            barrier_timeout_s=a.timeout, span_numel=(span_numel[r] if span_numel else a.span),
            first_span_numel=(span_numel[r] if span_numel else a.first_span),
            symmetric=row.factory(r), pre_barrier=(a.flow == "hooks"), adamw=a.adamw))
    return opts


def run_step(a, opts, streams, grads, ranks=None):
    ranks = range(a.d) if ranks is None else ranks
    reps = [None] * a.d
    if a.flow == "step":
        for r in ranks:
            with torch.cuda.stream(streams[r]):
                reps[r] = opts[r].step(grads[r])
        return reps
    # hook-driven: interleave the ranks' deliveries in backward order, then
    # finish without waiting and let each rank's "next forward" wait bucket
    # by bucket (first layers = last bucket first)
    for r in ranks:
        with torch.cuda.stream(streams[r]):
            opts[r].begin_step()
    n = len(grads[0])
    for pi in reversed(range(n)):
        for r in ranks:
            with torch.cuda.stream(streams[r]):
                opts[r].grad_ready(pi, grads[r][pi])
    for r in ranks:
        with torch.cuda.stream(streams[r]):
            reps[r] = opts[r].finish_step(wait=False)
            for b in reversed(range(len(opts[r].layout.buckets))):
                opts[r].wait_params(b)
    return reps


def check(a, opts, gs, step, grads, state, reps):
    d = a.d
    L = opts[0].layout
    offs = L.shard_offsets()
    hg = [[host_grad(g) for g in grads[q]] for q in range(d)]
    reduced = []
    for b in L.buckets:
        packs = [oracle.pack([hg[q][s.index] for s in b.slots], [s.offset for s in b.slots], b.numel, 1.0 / d)
                 for q in range(d)]
        reduced.append([oracle.reduce_scatter(packs, r, d) for r in range(d)])
    coef = None
    if a.clip > 0:
        coefs = [np.float32(rp.clip_coef.item()) for rp in reps]
        assert all(c.view(np.uint32) == coefs[0].view(np.uint32) for c in coefs), f"coef differs: {coefs}"
        ss = sum(oracle.sumsq_bf16(x) for bucket in reduced for x in bucket)
        want = float(np.sqrt(ss))
        got = float(reps[0].grad_norm.item())
        assert abs(got - want) <= 1e-5 * want, f"step {step}: norm {got} vs oracle {want}"
        coef = float(coefs[0])
    params = [u16(o.param_buffer) for o in opts]
    for q in range(1, d):
        assert np.array_equal(params[q], params[0]), f"step {step}: rank {q} params differ from rank 0"
    for r in range(d):
        gbuf = u16(opts[r].grad_buffer) if a.keep_reduced else None
        dev_state = [x.cpu().numpy() for x in (opts[r].master, opts[r].exp_avg, opts[r].exp_avg_sq)]
        for bi, b in enumerate(L.buckets):
            n = b.numel // d
            lo = b.start + r * n
            if gbuf is not None:
                assert np.array_equal(gbuf[lo:lo + n], reduced[bi][r]), f"step {step} rank {r} bucket {bi}: RS"
            master, m, v = (x[offs[bi]:offs[bi] + n] for x in state[r])
            want = oracle.adamw(master, m, v, reduced[bi][r], step, coef=coef)
            if getattr(a, "adamw", "exact") == "fast":
                # north-star tolerance (SURVEY §8d norm-relative rule); params
                # are the RNE of the device's own master
                rtol = 1e-6 if step == 1 else 1e-5
                for name, dv, ov in zip(("master", "m", "v"), dev_state, (master, m, v)):
                    got = dv[offs[bi]:offs[bi] + n].astype(np.float64)
                    err = np.abs(got - ov).max() / max(np.abs(ov).max(), 1e-30)
                    assert err <= rtol, f"step {step} rank {r} bucket {bi}: {name} rel err {err}"
                own = torch.from_numpy(dev_state[0][offs[bi]:offs[bi] + n]).to(torch.bfloat16)
                assert np.array_equal(params[0][lo:lo + n], u16(own)), f"step {step} rank {r} bucket {bi}: params"
                continue
            assert np.array_equal(params[0][lo:lo + n], want), f"step {step} rank {r} bucket {bi}: params"
            for name, dv, ov in zip(("master", "m", "v"), dev_state, (master, m, v)):
                assert np.array_equal(dv[offs[bi]:offs[bi] + n].view(np.uint32), ov.view(np.uint32)), \
                    f"step {step} rank {r} bucket {bi}: {name}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=2)
    ap.add_argument("--config", default="odd")
    ap.add_argument("--grad-dtype", default="bf16")
    ap.add_argument("--bucket", type=int, default=100_000)
    ap.add_argument("--span", type=int, default=250_000)
    ap.add_argument("--first-span", type=int, default=50_000)
    ap.add_argument("--clip", type=float, default=0.0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--flow", default="step", choices=["step", "hooks"])
    ap.add_argument("--keep-reduced", type=int, default=1)
    ap.add_argument("--timeout", type=float, default=10.0)
    ap.add_argument("--adamw", default="exact", choices=["exact", "fast"])
    ap.add_argument("--fault", default=None, choices=[None, "timeout", "span", "checkpoint"])
    a = ap.parse_args()
    if not connections_ok():
        raise SystemExit("start with emulation.child_env(): CUDA_DEVICE_MAX_CONNECTIONS=32, CUDA_MODULE_LOADING=EAGER")
    dev = torch.device("cuda", 0)
    gs = config_gradset(a.config)
    gdt = torch.float32 if a.grad_dtype == "f32" else torch.bfloat16
    out = {"d": a.d, "flow": a.flow, "clip": a.clip, "fault": a.fault}
    with EmulatedRow(a.d, dev) as row:
        streams = row.streams()
        if a.fault == "timeout":
            # rank 1 exists (its buffers are the peer's) but never steps: rank 0's
            # first span times out, the update is skipped, and the host raises
            opts = build(a, row, dev, gs)
            grads = [make_grads(gs, 1, r, dev, dtype=gdt) for r in range(a.d)]
            reps = run_step(a, opts, streams, grads, ranks=[0])
            try:
                reps[0].resolve()
            except DeviceError as e:
                out["raised"] = str(e)
            assert "raised" in out and str(nat.HOD_ETIMEOUT) in out["raised"], out
            # the read-back landed: the next step refuses to start
            torch.cuda.synchronize()
            try:
                opts[0].begin_step()
            except DeviceError as e:
                out["next_step_raised"] = str(e)
            assert "next_step_raised" in out, out
        elif a.fault == "span":
            # the two ranks close spans over different buckets (per bucket vs
            # everything at once): the arrival tags differ -> HOD_ESPAN
            opts = build(a, row, dev, gs, span_numel=[1, 1 << 40])
            grads = [make_grads(gs, 1, r, dev, dtype=gdt) for r in range(a.d)]
            reps = run_step(a, opts, streams, grads)
            codes = []
            for r in range(a.d):
                try:
                    reps[r].resolve()
                except DeviceError as e:
                    codes.append(str(e))
            out["raised"] = codes
            assert len(codes) == a.d and all(str(nat.HOD_ESPAN) in c for c in codes), out
        elif a.fault == "checkpoint":
            # save after 2 steps, restore into a fresh row of optimizers with
            # gather, then one more step on both: bit-identical everywhere
            import tempfile

            from paper_2312_03549_b200 import checkpoint

            opts = build(a, row, dev, gs)
            for step in (1, 2):
                grads = [make_grads(gs, step, r, dev, dtype=gdt) for r in range(a.d)]
                for rp in run_step(a, opts, streams, grads):
                    rp.resolve()
            with tempfile.TemporaryDirectory() as tmp:
                for o in opts:
                    checkpoint.save(o, tmp)
                fresh = build(a, row, dev, gs)
                for o in fresh:
                    checkpoint.load(o, tmp, gather=False)   # gather below, all ranks issued first
                for r, o in enumerate(fresh):
                    with torch.cuda.stream(streams[r]):
                        o.gather_params()
                torch.cuda.synchronize()
                for o in fresh:
                    o.check_health()
                for r in range(a.d):
                    assert torch.equal(fresh[r].param_buffer.view(torch.int16), opts[r].param_buffer.view(torch.int16)), \
                        f"rank {r}: gathered params differ after load"
                grads = [make_grads(gs, 3, r, dev, dtype=gdt) for r in range(a.d)]
                for rp in run_step(a, opts, streams, grads) + run_step(a, fresh, streams, grads):
                    rp.resolve()
                torch.cuda.synchronize()
                for r in range(a.d):
                    for name in ("param_buffer", "master", "exp_avg", "exp_avg_sq"):
                        x, y = getattr(opts[r], name), getattr(fresh[r], name)
                        assert torch.equal(x.view(torch.int16) if x.dtype == torch.bfloat16 else x.view(torch.int32),
                                           y.view(torch.int16) if y.dtype == torch.bfloat16 else y.view(torch.int32)), \
                            f"rank {r}: {name} differs after restore + step"
                for o in fresh:
                    o.close()
            out["ok"] = True
        else:
            opts = build(a, row, dev, gs)
            torch.cuda.synchronize()
            state = [[x.cpu().numpy().copy() for x in (o.master, o.exp_avg, o.exp_avg_sq)] for o in opts]
            launches0 = nat.launch_count()
            for step in range(1, a.steps + 1):
                grads = [make_grads(gs, step, r, dev, dtype=gdt) for r in range(a.d)]
                torch.cuda.synchronize()
                reps = run_step(a, opts, streams, grads)
                for rp in reps:
                    rp.resolve()
                torch.cuda.synchronize()
                check(a, opts, gs, step, grads, state, reps)
            out["buckets"] = len(opts[0].layout.buckets)
            out["launches"] = nat.launch_count() - launches0
            out["ok"] = True
        for o in opts:
            o.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
