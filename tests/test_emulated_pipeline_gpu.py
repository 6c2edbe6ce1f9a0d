"""BASELINE config 4 in miniature (PP = 2 x DP = 2) on ONE GPU (driver-visible).

tests/pipe_emu_worker.py runs the four ranks of the reference-compatible
plan concurrently on one device (paper_2312_03549_b200/emulation.py): the
per-stage DP optimizers with the world-wide clip norm (§8e), and the 1F1B
stage hand-offs of pipeline.PipelineRunner (§8f.3) in the order of
simulator._one_f_one_b — the same checks as the 4-GPU cases in
tests/test_multigpu_gpu.py, without needing four GPUs.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def run(tmp_path, *args, timeout=900, data=2):
    from paper_2312_03549_b200.emulation import child_env
    from test_multigpu_gpu import MINI_PP_SCENARIO

    doc = json.loads(json.dumps(MINI_PP_SCENARIO))
    if data != 2:
        # config 4's shape: PP = 2 x DP = d, one node of d GPUs per NIC cluster
        doc["topology"]["gpus_per_node"] = data
        doc["parallel"]["d"] = data
        doc["model"]["global_batch"] = 4 * data
    scen = tmp_path / "mini_pp.json"
    scen.write_text(json.dumps(doc))
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "pipe_emu_worker.py"), "--scenario", str(scen),
                        *map(str, args)], capture_output=True, text=True, timeout=timeout, env=child_env(), cwd=ROOT)
    assert p.returncode == 0, f"worker failed ({p.returncode}):\n{p.stdout[-3000:]}\n{p.stderr[-3000:]}"
    return json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("clip", [0.05, 0.0])
def test_pp_dp_scenario_emulated_matches_oracle(tmp_path, clip):
    """Stage placement, DP rows and the partition from the plan; every stage's
    DP row bit-exact against the oracle, one clip coefficient for the world."""
    out = run(tmp_path, "--mode", "scenario", "--clip", clip, "--steps", 3)
    assert out["ok"]
    assert out["stages"] == [1, 1, 2, 2]
    assert out["dp_rows"] == [[0, 1], [2, 3]] and out["pp_rows"] == [[0, 2], [1, 3]]
    assert sum(out["stage_layers"]) == 6


def test_pipeline_1f1b_handoffs_emulated(tmp_path):
    """1F1B over the PP rows: every activation / activation gradient lands
    intact in the neighbour's slot (stand-in compute +1 per stage and
    direction), and the DP optimizers overlapping the last backward stay
    bit-exact with the world clip norm."""
    out = run(tmp_path, "--mode", "pipeline", "--clip", 0.05, "--steps", 2, "--micro", 4)
    assert out["ok"]
    for doc in out["traces"]:
        tr = doc["trace"]
        assert len(tr) == 2 * 4                  # 4 micro-batches x 2 iterations, one direction
        for op, k, mean, std in tr:
            # stage 1 sends x + 1 = 2; stage 2 returns (2 + 1) + 1 = 4
            assert (op, mean, std) == (("fwd", 2.0, 0.0) if doc["stage"] == 2 else ("bwd", 4.0, 0.0))


def test_pp2_dp4_scenario_emulated_matches_oracle(tmp_path):
    """BASELINE config 4's exact shape (PP = 2 x DP = 4, eight ranks: DP rows
    {0..3} / {4..7}, PP rows (q, q + 4), world clip norm over eight ranks) —
    the layout the driver's 8-GPU run uses — with all eight ranks on one GPU."""
    out = run(tmp_path, "--mode", "pipeline", "--clip", 0.05, "--steps", 2, "--micro", 4, data=4)
    assert out["ok"]
    assert out["stages"] == [1, 1, 1, 1, 2, 2, 2, 2]
    assert out["dp_rows"] == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert out["pp_rows"] == [[0, 4], [1, 5], [2, 6], [3, 7]]
    for doc in out["traces"]:
        for op, k, mean, std in doc["trace"]:
            assert (op, mean, std) == (("fwd", 2.0, 0.0) if doc["stage"] == 2 else ("bwd", 4.0, 0.0))
