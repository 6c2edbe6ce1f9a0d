"""bench.py's reference arm (runs on host cores, no GPU): the JSON contract."""

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                           "--warmup", "0", "--ref-seconds", "1", "--config", "toy"],
                          capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_reference_arm_prints_one_contract_line():
    r = _run({})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"] == "optimizer-step params/s" and d["unit"] == "params/s"
    assert d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "params/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_non_zero_rank_is_silent():
    r = _run({"WORLD_SIZE": "2", "RANK": "1"})
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_sweep_row_fractions():
    sys.path.insert(0, str(ROOT))
    import bench

    row = bench._sweep_row({"bucket_MB": 1024.0, "results": {
        "fused_p2p": {"ms": 2.5, "busBW_GBps": 616.0}, "adamw_local": {"ms": 0.1, "busBW_GBps": None},
        "error": 0}})
    assert row["bucket_MB"] == 1024.0
    # headline denominator: 900 GB/s per direction (north star); measured copy beside it
    assert row["fused_p2p"] == {"ms": 2.5, "busBW_GBps": 616.0, "frac_nvlink": 0.684,
                                "frac_nvlink_measured_copy": 0.8}
    assert row["adamw_local"]["frac_nvlink"] is None and "error" not in row


def test_reference_arm_config_equals_gpu_arm_config():
    """Both arms build ``config`` with bench._config_doc from the same args, so
    the driver's same-config check holds; the CPU sample is labelled."""
    sys.path.insert(0, str(ROOT))
    import argparse

    import bench
    from paper_2312_03549_b200.buckets import build_bucket_layout
    from paper_2312_03549_b200.gradsets import config_gradset

    r = _run({})
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    gs = config_gradset("toy")
    args = argparse.Namespace(config="toy", bucket_size=25_000_000)
    nb = len(build_bucket_layout(gs.numels, 25_000_000, dp=1).buckets)
    assert d["config"] == json.loads(json.dumps(bench._config_doc(args, None, gs.total, nb, 1)))
    assert "full step" in d["cpu_baseline"]["sample"] or "bounded sample" in d["cpu_baseline"]["sample"]
