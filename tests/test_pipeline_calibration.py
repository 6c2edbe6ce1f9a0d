"""CPU checks of tools/pipeline_vs_sim.calibrated_model: the
reference's cost model, calibrated to measured per-op times, reproduces them
and its event-driven 1F1B (simulator.py:359-470) then predicts the closed
form for uniform stages."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "tools"))

pytest.importorskip("torch")


def test_calibration_reproduces_the_measured_op_times():
    import paper_2312_03549_b200 as hp
    from paper_2312_03549_b200 import simulator
    from pipeline_vs_sim import calibrated_model

    s = hp.load_scenario(str(ROOT / "scenarios" / "gpt13b_pp2_dp2_hybrid.json"))
    tf, tb = {1: 88.4, 2: 65.3}, {1: 175.4, 2: 128.9}
    planned, part, model, cost = calibrated_model(s, 8, tf, tb)
    assert simulator.micro_batch_count(model, planned.config) == 8
    assert cost.backward_forward_ratio == pytest.approx((175.4 + 128.9) / (88.4 + 65.3))
    for st in (1, 2):
        c = simulator._stage_cluster(st, planned.config, planned.topology)
        f, b = simulator.stage_compute_time(part.stage_layers[st - 1], model, planned.config,
                                            cost.cluster_speeds_tflops[c - 1], 1.0, cost.backward_forward_ratio)
        assert f * 1e3 == pytest.approx(tf[st], rel=1e-12)
        assert b == pytest.approx(cost.backward_forward_ratio * f, rel=1e-12)


def test_uniform_stages_match_the_closed_form():
    import paper_2312_03549_b200 as hp
    from paper_2312_03549_b200 import simulator
    from pipeline_vs_sim import calibrated_model

    s = hp.load_scenario(str(ROOT / "scenarios" / "gpt1p3b_pp2_dp1_node.json"))
    tf, tb = {1: 2.0, 2: 2.0}, {1: 4.0, 2: 4.0}
    planned, part, model, cost = calibrated_model(s, 16, tf, tb)
    rep = simulator.simulate_iteration(planned.topology, planned.config, planned.plan, planned.channels, part,
                                       model, cost, exposed_dp_sync=0.0)
    hop = rep.breakdown["pipeline_p2p"] / 2.0                  # 2 (p - 1) hops charged, p = 2
    assert rep.iter_time_s * 1e3 == pytest.approx((16 + 2 - 1) * (2.0 + 4.0) + 2 * hop * 1e3, rel=1e-9)


@pytest.mark.parametrize("p", [2, 3, 4])
@pytest.mark.parametrize("m", [1, 4, 8])
def test_event_simulation_equals_the_closed_form(tmp_path, p, m):
    """SPEC.md:488's acceptance criterion the reference never tested: with
    uniform stages the event-driven 1F1B equals analytic_makespan."""
    import json

    import paper_2312_03549_b200 as hp
    from paper_2312_03549_b200 import simulator

    doc = json.loads((ROOT / "scenarios" / "gpt1p3b_pp2_dp1_node.json").read_text())
    doc["topology"]["gpus_per_node"] = p
    doc["parallel"]["p"] = p
    doc["model"]["global_batch"] = m
    path = tmp_path / "s.json"
    path.write_text(json.dumps(doc))
    s = hp.load_scenario(str(path))
    planned = hp.plan_scenario(s)
    part = hp.partition_scenario(s, topo=planned.topology)
    assert len(set(part.stage_layers)) == 1                    # uniform stages
    cost = simulator.CostModel()
    rep = simulator.simulate_iteration(planned.topology, planned.config, planned.plan, planned.channels, part,
                                       s.model, cost, exposed_dp_sync=0.0)
    c = simulator._costs(planned.config, planned.topology, simulator.channel_map(planned.channels), part,
                         s.model, cost)
    hop = rep.breakdown["pipeline_p2p"] / (2 * (p - 1))
    want = simulator.analytic_makespan([(x.t_fwd, x.t_bwd) for x in c], m, [hop] * (p - 1))
    assert rep.iter_time_s == pytest.approx(want, rel=1e-12)
