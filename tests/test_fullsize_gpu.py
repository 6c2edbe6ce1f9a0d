"""Full-size parity (BASELINE configs 2 and 3 at their real sizes): one step of
the whole GPT-3 1.3B / LLaMA-7B gradient set at d = 1, 2, 4 (8 when the box
has it), checked through size-independent properties and oracle-checked
sampled buckets (tests/mp_worker_fullsize.py)."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

from conftest import free_port  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent


def _ngpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("n", [1, 2, 4, 8])
@pytest.mark.parametrize("config,clip", [("gpt1.3b", 0.0), ("llama7b", 1.0)])
def test_fullsize_step_properties(tmp_path, n, config, clip):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={free_port()}",
            str(ROOT / "tests" / "mp_worker_fullsize.py"), "--out", str(tmp_path),
            "--config", config, "--clip", str(clip)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [json.loads((tmp_path / f"result_r{q}.json").read_text()) for q in range(n)]
    assert all(x["ok"] for x in res)
    assert len({tuple(x["param_checksum"]) for x in res}) == 1
    if clip:
        assert len({x["grad_norm"] for x in res}) == 1
