"""Generate tests/golden/planner_golden.json by RUNNING the reference package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Only this container has /root/reference; the JSON it writes is committed so
the CPU suite (and the GPU box) can check the host-side mirror against the
reference's own outputs without the reference present.  Covered rows
(SURVEY.md §8a): A1 stage grad bytes, A2 collective prices, A3-A4 dp_sync and
the post-flush simulate report, A5 reduce_scatter_report, A6-A8 group
matrices + diagnostics, A9-A10 ordering + channels, A11-A12 partition,
A13 numbering — over every reference scenario, the config-4 preset, the
SURVEY §0.4 quirk variants, and seeded random topologies.
"""

from __future__ import annotations

import copy
import json
import random
import sys
import warnings
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
import holmes_planner as hp  # noqa: E402

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent


def scenario_docs():
    docs = {}
    for p in sorted((REF / "scenarios").glob("*.json")):
        docs[p.stem] = json.loads(p.read_text())
    c4 = json.loads((ROOT / "scenarios" / "gpt13b_pp2_dp4_hybrid.json").read_text())
    docs["gpt13b_pp2_dp4_hybrid"] = c4
    # speeds indexed post-normalisation -> RoCE-first gives [18,22]
    v = copy.deepcopy(c4)
    v["topology"]["clusters"] = list(reversed(v["topology"]["clusters"]))
    v["cost"]["cluster_speeds_tflops"] = [160, 197]
    docs["c4_roce_first_speeds_160_197"] = v
    v = copy.deepcopy(c4)
    v["topology"]["clusters"] = list(reversed(v["topology"]["clusters"]))
    docs["c4_roce_first_speeds_197_160"] = v
    sa = json.loads((REF / "scenarios" / "gpt_3p6b_hybrid_self_adapting.json").read_text())
    v = copy.deepcopy(sa)
    v["partition"]["cluster_alphas"] = [1.2]
    docs["sa_cluster_alphas_1p2"] = v
    v = copy.deepcopy(c4)
    v["partition"]["cluster_mem_budget_gb"] = [80]
    docs["c4_mem_budget_m_minus_1"] = v  # loader accepts, planner raises
    v = copy.deepcopy(c4)
    v["partition"] = {"strategy": "uniform"}
    docs["c4_uniform"] = v
    v = copy.deepcopy(c4)
    del v["cost"]
    docs["c4_eta_only"] = v
    v = copy.deepcopy(sa)
    v["partition"]["alpha"] = 3.0
    docs["sa_alpha_clamp"] = v
    return docs


def run_doc(doc):
    raw = json.dumps(doc).encode()
    out = {}
    try:
        s = hp.parse_scenario(doc, raw)
    except hp.PlannerError as e:
        return {"error": type(e).__name__, "message": str(e)}
    out["diagnostics"] = [[d.code, d.message] for d in hp.scenario_diagnostics(s)]
    try:
        pr = hp.plan_scenario(s)
        out["plan"] = pr.to_json_dict()
        naive = hp.plan_scenario(s, naive=True)
        out["plan_naive"] = naive.to_json_dict()
    except hp.PlannerError as e:
        out["plan_error"] = [type(e).__name__, str(e)]
        return out
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            part = hp.partition_scenario(s, topo=pr.topology)
        out["partition"] = part.to_json_dict()
        out["partition_warnings"] = list(part.warnings)
    except hp.PlannerError as e:
        out["partition_error"] = [type(e).__name__, str(e)]
        return out
    try:
        rep, _, _ = hp.run_scenario(s)
        d = rep.to_json_dict()
        d["timeline_len"] = len(d["timeline"])
        d["timeline"] = d["timeline"][:40] + d["timeline"][-40:]
        out["simulate"] = d
        out["reduce_scatter"] = [e.to_json_dict() for e in hp.scenario_reduce_scatter(s, pr, part)]
        out["stage_grad_bytes"] = [
            hp.simulator._stage_grad_bytes(st, part.stage_layers[st - 1], s.parallel.pipeline, s.model)
            for st in range(1, s.parallel.pipeline + 1)]
    except hp.PlannerError as e:
        out["simulate_error"] = [type(e).__name__, str(e)]
    return out


def random_topologies(n=60, seed=2024):
    rng = random.Random(seed)
    kinds = ["infiniband", "roce", "ethernet"]
    cases = []
    while len(cases) < n:
        m = rng.randint(1, 4)
        g = rng.choice([1, 2, 4, 8])
        clusters = [{"kind": rng.choice(kinds), "bw": rng.choice([25.0, 100.0, 200.0, 400.0]),
                     "nodes": rng.randint(1, 3)} for _ in range(m)]
        N = g * sum(c["nodes"] for c in clusters)
        facts = [(t, p, N // (t * p)) for t in range(1, N + 1) if N % t == 0
                 for p in range(1, N // t + 1) if (N // t) % p == 0]
        t, p, d = rng.choice(facts)
        cases.append({"clusters": clusters, "g": g, "inter": rng.random() < 0.3,
                      "eth": rng.choice([10.0, 25.0]), "cfg": [t, p, d]})
    return cases


def topo_of(case):
    cl = tuple(hp.Cluster(i, c["nodes"], hp.NicSpec(hp.NicKind(c["kind"]), c["bw"]))
               for i, c in enumerate(case["clusters"], 1))
    return hp.ClusterTopology(cl, case["g"], hp.NicSpec(hp.NicKind.ETHERNET, case["eth"]), 2400.0,
                              inter_cluster_rdma=case["inter"])


def run_topo(case):
    topo = topo_of(case)
    cfg = hp.ParallelConfig(*case["cfg"])
    out = {"validate": [[d.code, d.message] for d in hp.validate(cfg, topo)]}
    norm, order = hp.normalize_topology(topo)
    out["order"] = [list(order.order), order.ib_cluster_count]
    out["coords"] = [[c.cluster, c.node, c.gpu] for c in
                     (hp.coord_of(norm, r) for r in range(1, norm.total_devices + 1))]
    try:
        plan = hp.build_plan(cfg, norm)
    except hp.PlannerError as e:
        out["build_error"] = [type(e).__name__, str(e)]
        return out
    out["plan"] = plan.to_json_dict()
    out["channels"] = [a.to_json_dict() for a in hp.assign_channels(plan, norm)]
    out["naive"] = [a.to_json_dict() for a in hp.naive_channels(plan, norm)]
    return out


def partition_grid(seed=99):
    rng = random.Random(seed)
    two, multi = [], []
    for L in (2, 5, 8, 13, 30, 36, 40, 61, 96):
        for s_ib in (50.0, 122.0, 160.0, 197.0, 312.0):
            for s_roce in (10.0, 122.0, 160.0, 197.0):
                for a in (0.01, 0.5, 0.95, 1.0, 1.05, 1.2, 2.0, 3.0):
                    with warnings.catch_warnings(record=True) as w:
                        warnings.simplefilter("always")
                        res = hp.two_nic_split(L, s_ib, s_roce, a)
                    two.append([L, s_ib, s_roce, a, list(res), len(w)])
    for _ in range(300):
        L = rng.randint(1, 96)
        m = rng.randint(1, 4)
        speeds = [round(rng.uniform(50, 400), 3) for _ in range(m)]
        alphas = [round(rng.uniform(0.3, 1.6), 3) for _ in range(m)] if rng.random() < 0.7 else None
        per = round(rng.uniform(0.01, 3.0), 4)
        dmem = [round(rng.uniform(5, 200), 2) for _ in range(m)]
        try:
            with warnings.catch_warnings(record=True) as w:
                warnings.simplefilter("always")
                res = hp.multi_cluster_alloc(L, speeds, alphas, per, dmem)
            multi.append([L, speeds, alphas, per, dmem, res, len(w)])
        except hp.PlannerError as e:
            multi.append([L, speeds, alphas, per, dmem, [type(e).__name__, str(e)], -1])
    return two, multi


def main():
    docs = scenario_docs()
    cases = random_topologies()
    two, multi = partition_grid()
    cm = hp.CostModel()
    chan = hp.ChannelAssignment(hp.GroupKind.DP, 1, hp.Channel.INFINIBAND, 7200.0, 1e-6)
    prices = []
    for nbytes in (0, 1, 2 * 16252928, 2 * 1312817152, 2 * 6738415616):
        for n in (1, 2, 4, 8):
            prices.append([nbytes, n, cm.reduce_scatter(nbytes, n, chan), cm.all_gather(nbytes, n, chan),
                           cm.all_reduce(nbytes, n, chan)])
    golden = {
        "generator": "tests/golden/make_golden.py (runs /root/reference/pkg/src/holmes_planner)",
        "scenarios": {k: {"doc": v, "result": run_doc(v)} for k, v in docs.items()},
        "topologies": [{"case": c, "result": run_topo(c)} for c in cases],
        "two_nic_split": two,
        "multi_cluster_alloc": multi,
        "collective_prices_7200gbps": prices,
    }
    (HERE / "planner_golden.json").write_text(json.dumps(golden, indent=1, sort_keys=True) + "\n")
    print("wrote", HERE / "planner_golden.json")


if __name__ == "__main__":
    main()
