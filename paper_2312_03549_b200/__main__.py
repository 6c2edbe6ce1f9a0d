"""Command line: ``python -m paper_2312_03549_b200 <command>``.

JSON conventions follow the reference CLI (cli.py:37: ``indent=2``,
``ensure_ascii=False``, insertion-ordered keys, newline-terminated) and its exit
codes (cli.py:22-24: 0 ok, 1 domain infeasibility, 2 malformed input).  The
reference's planning commands (validate / plan / partition / simulate) are
mirrored because the optimizer consumes their output; the optimizer-specific
commands are new:

  layout          bucket layout (JSON) of a BASELINE gradient set or scenario stage
  placement       stage / DP row / PP row / channel of every rank of a scenario
  optimizer-bench run bench.py (one process per GPU; use torchrun for N > 1)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

from . import planner
from .buckets import build_bucket_layout
from .config import load_scenario
from .errors import ConfigError, PlannerError

EXIT_OK, EXIT_INFEASIBLE, EXIT_MALFORMED = 0, 1, 2


def _emit(doc) -> None:
    sys.stdout.write(json.dumps(doc, indent=2, ensure_ascii=False) + "\n")


def cmd_validate(a) -> int:
    diags = planner.scenario_diagnostics(load_scenario(a.config))
    for dgn in diags:
        print(str(dgn))
    if diags:
        return EXIT_INFEASIBLE
    print("ok")
    return EXIT_OK


def _feasible(s) -> bool:
    diags = planner.scenario_diagnostics(s)
    for dgn in diags:
        print(str(dgn), file=sys.stderr)
    return not diags


def cmd_plan(a) -> int:
    s = load_scenario(a.config)
    if not _feasible(s):
        return EXIT_INFEASIBLE
    _emit(planner.plan_scenario(s, naive=a.naive).to_json_dict())
    return EXIT_OK


def cmd_partition(a) -> int:
    s = load_scenario(a.config)
    if not _feasible(s):
        return EXIT_INFEASIBLE
    plan = planner.partition_scenario(s)
    for note in plan.warnings:
        print(note, file=sys.stderr)
    _emit(plan.to_json_dict())
    return EXIT_OK


def cmd_simulate(a) -> int:
    s = load_scenario(a.config)
    exposed = None if a.exposed_dp_sync is None else float(a.exposed_dp_sync)
    report, planned, part = planner.run_scenario(s, naive=a.naive, exposed_dp_sync=exposed)
    _emit({
        "scenario": s.name,
        "config_fingerprint": s.fingerprint,
        "nic_env": planner.nic_env_label(planned.topology),
        "channel_policy": "naive" if a.naive else "holmes",
        "defaults_applied": list(s.defaults_applied),
        "eta": s.cost.eta,
        "partition": part.to_json_dict(),
        "report": report.to_json_dict(),
        "reduce_scatter": [e.to_json_dict() for e in planner.scenario_reduce_scatter(s, planned, part)],
    })
    return EXIT_OK


def cmd_layout(a) -> int:
    if a.config.endswith(".json"):
        from .scenario_run import stage_gradset

        s = load_scenario(a.config)
        placement = planner.optimizer_placement(s, a.rank)
        gs = stage_gradset(s, placement, planner.partition_scenario(s))
        dp = len(placement.dp_ranks)
    else:
        from .gradsets import config_gradset

        gs = config_gradset(a.config, a.stage)
        dp = a.dp
    _emit(build_bucket_layout(gs.numels, a.bucket_size, dp).to_json_dict())
    return EXIT_OK


def cmd_placement(a) -> int:
    s = load_scenario(a.config)
    if not _feasible(s):
        return EXIT_INFEASIBLE
    planned = planner.plan_scenario(s)
    part = planner.partition_scenario(s, topo=planned.topology)
    _emit([planner.optimizer_placement(s, r, planned, part).to_json_dict()
           for r in range(planned.config.world_size)])
    return EXIT_OK


def cmd_optimizer_bench(a, extra) -> int:
    bench = Path(__file__).resolve().parent.parent / "bench.py"
    return subprocess.call([sys.executable, str(bench), *extra], env=dict(os.environ))


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2312_03549_b200", description=__doc__.splitlines()[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("validate", "plan", "partition", "simulate", "placement"):
        p = sub.add_parser(name)
        p.add_argument("--config", required=True, help="scenario JSON (reference schema)")
        if name in ("plan", "simulate"):
            p.add_argument("--naive", action="store_true")
        if name == "simulate":
            p.add_argument("--exposed-dp-sync", default=None,
                           help="seconds of exposed DP sync per stage (overlap hook, §8f.1)")
    p = sub.add_parser("layout")
    p.add_argument("--config", required=True, help="toy|gpt1.3b|llama7b|gpt13b|odd or a scenario JSON")
    p.add_argument("--stage", type=int, default=1)
    p.add_argument("--rank", type=int, default=0)
    p.add_argument("--dp", type=int, default=1)
    p.add_argument("--bucket-size", type=int, default=25_000_000)
    sub.add_parser("optimizer-bench", help="forwards all further arguments to bench.py")
    return ap


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if argv and argv[0] == "optimizer-bench":
        return cmd_optimizer_bench(None, argv[1:])
    a = build_parser().parse_args(argv)
    handlers = {"validate": cmd_validate, "plan": cmd_plan, "partition": cmd_partition,
                "simulate": cmd_simulate, "layout": cmd_layout, "placement": cmd_placement}
    try:
        return handlers[a.cmd](a)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_MALFORMED
    except PlannerError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INFEASIBLE


if __name__ == "__main__":
    sys.exit(main())
