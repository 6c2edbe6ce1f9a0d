"""BASELINE config 4 in miniature (PP = 2 x DP = 2 or 4) with every rank on ONE GPU.

Launched by tests/test_emulated_pipeline_gpu.py in a fresh process
(emulation.child_env).  The reference-compatible plan places the ranks
(stage, DP row, PP row: planner.optimizer_placement over groups.py Eq. 2/3);
each DP row, each PP row and the world-wide clip-norm group become an
``emulation.EmulatedRow``, so the ranks run the real protocol concurrently on
one device: the per-stage DP optimizers (arrival / params-ready barriers,
the world norm exchange), and in ``--mode pipeline`` the 1F1B stage
hand-offs of ``pipeline.PipelineRunner`` (copy-engine sends into the
neighbour's slot, device-side waits) in the order of
``simulator._one_f_one_b`` (simulator.py:348-356).

Checks after every step / iteration: each stage's reduced shards, master, m,
v and gathered params against the oracle (reduce-scatter semantics of
simulator.py:81-89 over the DP rows of groups.py:137-148; the clip norm over
the whole world, identical coefficient on every rank); in pipeline mode every
hand-off carries exactly what the neighbour sent (compute stand-in: +1 per
stage per direction).
"""

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2312_03549_b200 as hp  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_2312_03549_b200 import DistributedOptimizer  # noqa: E402
from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.comm import DPGroup  # noqa: E402
from paper_2312_03549_b200.emulation import EmulatedRow, connections_ok, grid_cap  # noqa: E402
from paper_2312_03549_b200.pipeline import PipelineRunner  # noqa: E402
from paper_2312_03549_b200.planner import optimizer_placement  # noqa: E402
from paper_2312_03549_b200.scenario_run import ScenarioRank, stage_gradset  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def check(opts, grads, state, coefs, norms, step, clip):
    """Every stage's DP row against the oracle (independent trajectory)."""
    rows = sorted({o.group.ranks for o in opts})
    reduced = {}
    for row in rows:
        o0 = opts[row[0]]
        d = len(row)
        for bi, b in enumerate(o0.layout.buckets):
            packs = [oracle.pack([u16(grads[q][s.index]) for s in b.slots], [s.offset for s in b.slots],
                                 b.numel, 1.0 / d) for q in row]
            for i, q in enumerate(row):
                reduced[(q, bi)] = oracle.reduce_scatter(packs, i, d)
    coef = None
    if clip:
        assert all(np.float32(c).view(np.uint32) == np.float32(coefs[0]).view(np.uint32) for c in coefs), coefs
        ss = sum(oracle.sumsq_bf16(x) for x in reduced.values())
        want = float(np.sqrt(ss))
        assert abs(norms[0] - want) <= 1e-5 * want, f"step {step}: norm {norms[0]} vs oracle {want}"
        coef = float(coefs[0])
    for row in rows:
        params = [u16(opts[q].param_buffer) for q in row]
        for p in params[1:]:
            assert np.array_equal(p, params[0]), f"step {step}: DP row {row} params differ"
        for i, q in enumerate(row):
            o = opts[q]
            offs = o.layout.shard_offsets()
            dev_state = [x.cpu().numpy() for x in (o.master, o.exp_avg, o.exp_avg_sq)]
            gbuf = u16(o.grad_buffer)
            for bi, b in enumerate(o.layout.buckets):
                n = b.numel // len(row)
                lo = b.start + i * n
                red = reduced[(q, bi)]
                assert np.array_equal(gbuf[lo:lo + n], red), f"step {step} rank {q} bucket {bi}: RS"
                master, m, v = (x[offs[bi]:offs[bi] + n] for x in state[q])
                want = oracle.adamw(master, m, v, red, step, coef=coef)
                assert np.array_equal(params[0][lo:lo + n], want), f"step {step} rank {q} bucket {bi}: params"
                for name, dv, ov in zip(("master", "m", "v"), dev_state, (master, m, v)):
                    assert np.array_equal(dv[offs[bi]:offs[bi] + n].view(np.uint32), ov.view(np.uint32)), \
                        f"step {step} rank {q} bucket {bi}: {name}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", required=True)
    ap.add_argument("--mode", default="pipeline", choices=["pipeline", "scenario"])
    ap.add_argument("--clip", type=float, default=0.05)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--micro", type=int, default=4)
    ap.add_argument("--bucket", type=int, default=300_000)
    a = ap.parse_args()
    if not connections_ok():
        raise SystemExit("run with emulation.child_env() (CUDA_DEVICE_MAX_CONNECTIONS=32, EAGER loading)")
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    nat.load()
    s = hp.load_scenario(a.scenario)
    planned = hp.plan_scenario(s)
    part = hp.partition_scenario(s, topo=planned.topology)
    world = planned.config.world_size
    pls = [optimizer_placement(s, g, planned, part) for g in range(world)]
    dp_rows = {row: EmulatedRow(len(row), dev) for row in sorted({pl.dp_ranks for pl in pls})}
    pp_rows = {row: EmulatedRow(len(row), dev) for row in sorted({pl.pp_ranks for pl in pls})}
    norm_row = EmulatedRow(world, dev)
    out = {"mode": a.mode, "world": world, "stages": [pl.stage for pl in pls],
           "dp_rows": [list(r) for r in dp_rows], "pp_rows": [list(r) for r in pp_rows],
           "stage_layers": list(part.stage_layers)}
    nat.set_grid_base(grid_cap(world))
    opts, srs = [], []
    for g, pl in enumerate(pls):
        gs = stage_gradset(s, pl, part)
        srs.append(ScenarioRank(placement=pl, gradset=gs, dp_group=DPGroup(pl.dp_ranks, g), process_group=None,
                                norm_ranks=tuple(range(world)), norm_group=None))
        opts.append(DistributedOptimizer(
            init_params(gs, dev), bucket_size=a.bucket, clip=a.clip if a.clip > 0 else None,
            dp_group=srs[g].dp_group, norm_ranks=srs[g].norm_ranks, backend="p2p", keep_reduced=True,
            barrier_timeout_s=30.0, symmetric=dp_rows[pl.dp_ranks].factory(pl.dp_ranks.index(g)),
            norm_symmetric=norm_row.factory(g)))
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    runners = None
    if a.mode == "pipeline":
        runners = [PipelineRunner(s, srs[g], opts[g], micro_batches=a.micro, compute=False,
                                  symmetric=pp_rows[pl.pp_ranks].factory(pl.pp_ranks.index(g)), stream=streams[g])
                   for g, pl in enumerate(pls)]
        for r in runners:
            r.x.fill_(1.0)
    torch.cuda.synchronize()
    state = [[x.cpu().numpy().copy() for x in (o.master, o.exp_avg, o.exp_avg_sq)] for o in opts]
    for step in range(1, a.steps + 1):
        gstep = 1 if runners else step
        grads = [make_grads(srs[g].gradset, gstep, g, dev) for g in range(world)]
        torch.cuda.synchronize()
        reps = []
        for g in range(world):
            with torch.cuda.stream(streams[g]):
                if runners:
                    runners[g].run_iteration(grads[g])
                else:
                    reps.append(opts[g].step(grads[g]))
        torch.cuda.synchronize()
        for o in opts:
            o.check_health()
        if runners:
            for r in runners:
                r.check()
        coefs = [float(o._coef.item()) for o in opts] if a.clip > 0 else []
        norms = [float(o._norm.item()) for o in opts] if a.clip > 0 else []
        check(opts, grads, state, coefs, norms, step, a.clip > 0)
    if runners:
        traces = []
        for g, r in enumerate(runners):
            tr = [[op, k, float(t.float().mean()), float(t.float().std())] for op, k, t in r.trace]
            traces.append({"rank": g, "stage": r.stage, "trace": tr})
        out["traces"] = traces
    out["ok"] = True
    for o in opts:
        o.close()
    nat.set_grid_base(0)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
