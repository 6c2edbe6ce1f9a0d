"""Measured 1F1B pipeline iteration vs the reference simulator.

    torchrun --nproc-per-node 4 tools/pipeline_vs_sim.py --scenario scenarios/gpt13b_pp2_dp2_hybrid.json
    torchrun --nproc-per-node 2 tools/pipeline_vs_sim.py --scenario scenarios/gpt1p3b_pp2_dp1_node.json

Runs ``pipeline.PipelineRunner`` (the 1F1B order of simulator._one_f_one_b,
stage hand-offs over NVLink peer memory, cuBLAS GEMM stand-ins on the
stage's real parameters, the DP optimizer overlapping the last micro-batch's
backward) and measures, per stage, the forward and backward time of one
micro-batch in isolation at sustained clocks (CUDA events, no hand-off
waits, after ~1 s of back-to-back warm-up).  Those per-op
times calibrate the reference's cost model — ``CostModel(cluster_speeds_tflops=…,
backward_forward_ratio=…)`` so that ``stage_compute_time`` reproduces them —
and ``simulate_iteration`` (the event-driven 1F1B of simulator.py:359-470)
then predicts the iteration, which is compared with the measured one:

* without the optimizer: the simulator's schedule model (warm-up, steady
  1F1B, flush; PP hops priced on the scenario's channels) against the real
  execution;
* with the optimizer: the reference's post-flush DP charge (simulator.py:
  445-452, RS + AG priced on the scenario's NICs) and the overlap hook fed
  with the MEASURED exposed time (``exposed_dp_sync``, §8f.1).
Prints one JSON line (rank 0).
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_03549_b200 as hp  # noqa: E402
from paper_2312_03549_b200 import simulator  # noqa: E402
from paper_2312_03549_b200.pipeline import PipelineRunner  # noqa: E402
from paper_2312_03549_b200.scenario_run import make_optimizer, setup_rank  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402


def _time(fn, reps, stream, warm_s: float = 1.0):
    """Mean time of ``fn`` at SUSTAINED clocks: ~``warm_s`` of back-to-back
    warm-up first (a B200 running GEMMs at full power settles well below its
    burst clock — MEASURED_PEAKS.json: sustained bf16 0.85 of burst), then
    ``reps`` timed calls."""
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    for _ in range(max(1, int(warm_s * 1e3 / max(e0.elapsed_time(e1), 1e-3)))):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def calibrated_model(s, micro: int, tf: dict, tb: dict):
    """The reference's cost model calibrated to measured per-op times:
    ``tf`` / ``tb`` map stage -> forward / backward ms of one micro-batch.
    Returns (planned, partition, model, CostModel) such that
    ``stage_compute_time`` reproduces ``tf`` on every stage (each stage's
    cluster speed solved for) with ``backward_forward_ratio`` = sum(tb) /
    sum(tf); the model's global batch is rescaled so the simulator schedules
    ``micro`` micro-batches."""
    from dataclasses import replace

    planned = hp.plan_scenario(s)
    part = hp.partition_scenario(s, topo=planned.topology)
    cfg, topo, model = planned.config, planned.topology, s.model
    if simulator.micro_batch_count(model, cfg) != micro:
        model = replace(model, global_batch=micro * model.micro_batch * cfg.data)
    ratio = sum(tb.values()) / sum(tf.values())
    speeds = [None] * len(topo.clusters)
    for st in range(1, cfg.pipeline + 1):
        f_at_1tf, _ = simulator.stage_compute_time(part.stage_layers[st - 1], model, cfg, 1.0, 1.0, ratio)
        speeds[simulator._stage_cluster(st, cfg, topo) - 1] = f_at_1tf / (tf[st] / 1e3)
    speeds = [x if x is not None else max(v for v in speeds if v) for x in speeds]
    cost = simulator.CostModel(backward_forward_ratio=ratio, cluster_speeds_tflops=tuple(speeds))
    return planned, part, model, cost


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", required=True)
    ap.add_argument("--micro", type=int, default=8, help="micro-batches per iteration")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--timeline", default=None, help="write measured + simulated StageEvent timelines here")
    a = ap.parse_args()
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    s = hp.load_scenario(a.scenario)
    sr = setup_rank(s, rank)
    opt = make_optimizer(sr, init_params(sr.gradset, dev), clip=1.0, barrier_timeout_s=60.0)
    pr = PipelineRunner(s, sr, opt, micro_batches=a.micro, compute=True)
    grads = make_grads(sr.gradset, 1, rank, dev)

    # per-op compute of this stage in isolation
    dy = torch.randn(pr.tokens, pr.h, device=dev, dtype=torch.bfloat16) * 1e-3
    t_f = _time(lambda: pr._forward(pr.x), 20, pr.stream)
    t_b = _time(lambda: pr._backward(dy, last=False, grads=grads), 20, pr.stream)

    iters = {}
    for with_opt in (False, True):
        for _ in range(2):
            pr.run_iteration(grads, with_optimizer=with_opt)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pr.stream)
        for _ in range(a.iters):
            pr.run_iteration(grads, with_optimizer=with_opt)
        e1.record(pr.stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / a.iters], device=dev, dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        iters[with_opt] = float(ms.item())
    # one instrumented iteration: every stage op's span on its stream, against
    # a common start (barrier + synchronize), in the reference's StageEvent
    # form — the measured counterpart of SimReport.timeline (simulator.py:98-116)
    pr.timed = True
    pr.op_events = []
    torch.cuda.synchronize()
    dist.barrier()
    base = torch.cuda.Event(enable_timing=True)
    base.record(pr.stream)
    pr.run_iteration(grads, with_optimizer=True)
    torch.cuda.synchronize()
    pr.timed = False
    timeline = [{"stage": pr.stage, "rank": rank, "op": op, "micro": k,
                 "start_s": base.elapsed_time(e0) / 1e3, "end_s": base.elapsed_time(e1) / 1e3}
                for op, k, e0, e1 in pr.op_events]
    pr.check()
    opt.check_health()
    per = [None] * dist.get_world_size()
    dist.all_gather_object(per, {"rank": rank, "stage": pr.stage, "t_f_ms": t_f, "t_b_ms": t_b,
                                 "timeline": timeline})
    if rank == 0:
        stage_tf = {}
        stage_tb = {}
        for d in per:
            stage_tf.setdefault(d["stage"], []).append(d["t_f_ms"])
            stage_tb.setdefault(d["stage"], []).append(d["t_b_ms"])
        tf = {st: sum(v) / len(v) for st, v in stage_tf.items()}
        tb = {st: sum(v) / len(v) for st, v in stage_tb.items()}
        planned, part, model, cost = calibrated_model(s, a.micro, tf, tb)
        cfg, topo = planned.config, planned.topology
        speeds, ratio = list(cost.cluster_speeds_tflops), cost.backward_forward_ratio
        sim = lambda **kw: simulator.simulate_iteration(topo, cfg, planned.plan, planned.channels, part,  # noqa: E731
                                                        model, cost, **kw).iter_time_s * 1e3
        sim_no_dp = sim(exposed_dp_sync=0.0)
        exposed = max(0.0, iters[True] - iters[False]) / 1e3
        doc = {"scenario": os.path.basename(a.scenario), "world": dist.get_world_size(),
               "pipeline": cfg.pipeline, "data": cfg.data, "micro_batches": a.micro,
               "stage_layers": list(part.stage_layers),
               "measured_op_ms": {str(st): {"fwd": tf[st], "bwd": tb[st]} for st in sorted(tf)},
               "calibrated_cluster_tflops": speeds, "backward_forward_ratio": ratio,
               "measured_iter_ms_no_opt": iters[False], "simulated_iter_ms_no_dp": sim_no_dp,
               "sim_over_measured": sim_no_dp / iters[False],
               "measured_iter_ms_with_opt": iters[True],
               "simulated_iter_ms_reference_dp_charge": sim(),
               "simulated_iter_ms_measured_exposed_dp": sim(exposed_dp_sync=exposed),
               "measured_exposed_dp_ms": exposed * 1e3,
               "ideal_1f1b_ms": (a.micro + cfg.pipeline - 1) * max(tf[st] + tb[st] for st in tf),
               "note": "per-op times measured in isolation at sustained clocks calibrate the reference cost "
                       "model; the simulator's PP hops are priced on the scenario's channels"}
        print(json.dumps(doc), flush=True)
        if a.timeline:
            # measured (DP-row rank 0 of each stage) and simulated timelines side by side
            first = {}
            for d in per:
                first.setdefault(d["stage"], d)
            sim_rep = simulator.simulate_iteration(topo, cfg, planned.plan, planned.channels, part, model, cost,
                                                   exposed_dp_sync=exposed)
            with open(a.timeline, "w") as f:
                json.dump({"measured": [e for st in sorted(first) for e in first[st]["timeline"]],
                           "simulated": [e.to_json_dict() for e in sim_rep.timeline]}, f)
    opt.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
