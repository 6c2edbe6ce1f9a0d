"""Real-module integration at d > 1: a LLaMA-style block stack
(attention + SwiGLU MLP + RMSNorms, tests/llama_blocks.py) bound with
``DistributedOptimizer.attach`` — backward hooks launch buckets, forward
pre-hooks wait for each submodule's gathered params — checked against the
oracle every step (tests/module_worker.py).  The emulated cases run d ranks
concurrently on one GPU (driver-visible); the dist case needs 2 GPUs.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def _run(args, env, timeout=900, launcher=None):
    cmd = (launcher or [sys.executable]) + [str(ROOT / "tests" / "module_worker.py"), *map(str, args)]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, f"worker failed ({p.returncode}):\n{p.stdout[-3000:]}\n{p.stderr[-4000:]}"
    return json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("d,clip", [(2, 0.0), (2, 1.0), (4, 0.5)])
def test_llama_blocks_emulated_ranks_match_oracle(d, clip):
    from paper_2312_03549_b200.emulation import child_env

    out = _run(["--mode", "emulated", "--d", d, "--clip", clip, "--steps", 3], child_env())
    assert out["ok"] and out["buckets"] >= 4


def test_llama_blocks_two_gpus_match_oracle():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    from conftest import free_port

    env = dict(os.environ)
    launcher = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(free_port())]
    out = _run(["--mode", "dist", "--clip", 1.0, "--steps", 3], env, launcher=launcher)
    assert out["ok"] and out["d"] == 2
