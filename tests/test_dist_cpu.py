"""CPU, world_size 2 over gloo: the host-side logic of the N > 1 path.

* DP rows from the reference GroupPlan -> 0-based communicator members;
* the NCCL unique-id bootstrap through the torch.distributed store;
* every rank's fp32 master shards, gathered, reassemble the whole layout
  (shard bookkeeping of the sharded optimizer).
"""

import os
from pathlib import Path

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2312_03549_b200 as hp
from paper_2312_03549_b200.buckets import build_bucket_layout
from paper_2312_03549_b200.comm import DPGroup, comm_key, exchange_unique_id
from paper_2312_03549_b200.gradsets import odd_tensors
from paper_2312_03549_b200.optimizer import fill_master_shards
from conftest import free_port  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    key = comm_key("dp", 0, tuple(range(world)))
    uid = exchange_unique_id(store, key, rank == 0, lambda: bytes(range(128)))
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    assert all(x == bytes(range(128)) for x in ids)

    gs = odd_tensors()
    gen = torch.Generator().manual_seed(7)
    params = [torch.randn(t.shape, generator=gen) for t in gs.tensors]
    L = build_bucket_layout(gs.numels, 150_000, dp=world)
    group = DPGroup(tuple(range(world)), rank)
    mine = fill_master_shards(L, params, group.index, torch.empty(L.total_numel // world))
    shards = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(shards, mine)
    if rank == 0:
        offs = L.shard_offsets()
        full = torch.zeros(L.total_numel)
        for bi, b in enumerate(L.buckets):
            n = b.numel // world
            for r in range(world):
                full[b.start + r * n:b.start + (r + 1) * n] = shards[r][offs[bi]:offs[bi] + n]
        for b in L.buckets:
            for s in b.slots:
                got = full[b.start + s.offset:b.start + s.offset + s.numel]
                assert torch.equal(got, params[s.index].reshape(-1))
        torch.save({"ok": True}, os.path.join(result_dir, "ok.pt"))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_shards(tmp_path):
    port = free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok.pt").exists()


def test_dp_groups_from_config4_plan():
    s = hp.load_scenario(ROOT / "scenarios" / "gpt13b_pp2_dp4_hybrid.json")
    plan = hp.plan_scenario(s).plan
    groups = [DPGroup.from_plan(plan, r) for r in range(8)]
    assert [g.ranks for g in groups] == [(0, 1, 2, 3)] * 4 + [(4, 5, 6, 7)] * 4
    assert [g.index for g in groups] == [0, 1, 2, 3, 0, 1, 2, 3]
    with pytest.raises(hp.InvalidPlanError):
        DPGroup((0, 1), 5)


def _scenario_worker(rank, world, port, scen, result_dir):
    """Config 4 host logic over gloo: every rank places itself in the
    reference plan, builds its stage's gradient set and joins its DP row's
    subgroup (collective over the world)."""
    import json

    from paper_2312_03549_b200.scenario_run import setup_rank

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sr = setup_rank(hp.load_scenario(scen), rank)
    # the DP row's subgroup really contains exactly the row's ranks
    x = torch.tensor([float(rank + 1)])
    dist.all_reduce(x, group=sr.process_group)
    # the clip-norm group is the world (one global norm for both stages)
    y = torch.tensor([1.0])
    dist.all_reduce(y, group=sr.norm_group)
    doc = {"stage": sr.placement.stage, "dp_ranks": list(sr.dp_group.ranks), "index": sr.dp_group.index,
           "params": sr.gradset.total, "row_sum": float(x), "world_sum": float(y),
           "norm_ranks": list(sr.norm_ranks)}
    with open(os.path.join(result_dir, f"r{rank}.json"), "w") as f:
        json.dump(doc, f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scen,world", [("gpt13b_pp2_dp2_hybrid.json", 4), ("gpt13b_pp2_dp4_hybrid.json", 8)])
def test_scenario_ranks_over_gloo(tmp_path, scen, world):
    import json

    port = free_port()
    mp.spawn(_scenario_worker, args=(world, port, str(ROOT / "scenarios" / scen), str(tmp_path)),
             nprocs=world, join=True)
    docs = [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(world)]
    d = world // 2
    stage_params = {1: 7_497_318_400, 2: 5_609_881_600}      # SURVEY §8a A1 known answers
    for r, doc in enumerate(docs):
        row = list(range(0, d)) if r < d else list(range(d, world))
        assert doc["stage"] == (1 if r < d else 2)            # the IB cluster holds stage 1 ([23, 17])
        assert doc["dp_ranks"] == row and doc["index"] == row.index(r)
        assert doc["params"] == stage_params[doc["stage"]]
        assert doc["row_sum"] == sum(q + 1 for q in row)
        assert doc["world_sum"] == world and doc["norm_ranks"] == list(range(world))
