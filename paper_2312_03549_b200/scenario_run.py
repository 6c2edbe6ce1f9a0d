"""Run the optimizer for a planned scenario on one box (BASELINE config 4).

Every torch rank looks itself up in the reference-compatible plan
(``planner.optimizer_placement``): its pipeline stage and that stage's layer
count (self-adapting partition, Eq. 5), its DP row (Eq. 3, 0-based) and the
clip-norm group (the whole world, so both stages clip with one global norm).
The stage's gradient set is the reference's own parameter-count model
(``_stage_grad_bytes``, simulator.py:268-280) laid out as tensors.  DP rows
become symmetric-memory groups via ``dist.new_subgroups_by_enumeration`` —
collective over the world, as required when several disjoint rows exist.
Heterogeneous NIC clusters are emulated as disjoint GPU subsets of the box.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .comm import DPGroup
from .gradsets import GradSet, gpt_stage_tensors
from .planner import OptimizerPlacement, optimizer_placement, partition_scenario, plan_scenario


@dataclass
class ScenarioRank:
    placement: OptimizerPlacement
    gradset: GradSet
    dp_group: DPGroup
    process_group: object
    norm_ranks: tuple[int, ...]
    norm_group: object


def stage_gradset(scenario, placement: OptimizerPlacement, part) -> GradSet:
    m = scenario.model
    p = scenario.parallel.pipeline
    first = sum(part.stage_layers[:placement.stage - 1])
    return gpt_stage_tensors(placement.stage_layers, m.hidden, m.vocab, stage=placement.stage,
                             pipeline=p, first_layer=first,
                             name=f"{scenario.name}-stage{placement.stage}")


def setup_rank(scenario, global_rank: int) -> ScenarioRank:
    """Collective over the world: every rank must call it."""
    planned = plan_scenario(scenario)
    part = partition_scenario(scenario, topo=planned.topology)
    world = planned.config.world_size
    if dist.get_world_size() != world:
        raise SystemExit(f"scenario needs {world} ranks, torch world is {dist.get_world_size()}")
    placement = optimizer_placement(scenario, global_rank, planned, part)
    rows = [[r - 1 for r in row] for row in planned.plan.dp.rows]
    if len(rows) == 1:
        pg = dist.group.WORLD
    else:
        pg, _ = dist.new_subgroups_by_enumeration(rows)
    return ScenarioRank(placement=placement, gradset=stage_gradset(scenario, placement, part),
                        dp_group=DPGroup(placement.dp_ranks, global_rank), process_group=pg,
                        norm_ranks=tuple(range(world)), norm_group=dist.group.WORLD)


def make_optimizer(sr: ScenarioRank, init_params, **kw):
    from .optimizer import DistributedOptimizer

    return DistributedOptimizer(init_params, dp_group=sr.dp_group, process_group=sr.process_group,
                                norm_ranks=sr.norm_ranks, norm_group=sr.norm_group, **kw)


def device_of(local_rank: int) -> torch.device:
    return torch.device("cuda", local_rank)
