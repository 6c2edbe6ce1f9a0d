"""The full multi-rank protocol on ONE GPU (driver-visible d > 1 parity).

Each case starts tests/emu_worker.py in a fresh process with
CUDA_DEVICE_MAX_CONNECTIONS=32 and eager module loading: d DistributedOptimizer ranks of one DP row
share the device (paper_2312_03549_b200/emulation.py) and run concurrently —
arrival barriers with span tags, params-ready barriers, the 1-CTA pre-span
barrier, the peer-memory norm exchange and the clip, every flag raised by a
live peer kernel.  Three steps per case, each rank checked bit-exactly
against the oracle after every step (reduce-scatter semantics of
simulator.py:81-89 over the DP row of groups.py:137-148).  The fault cases
prove that a barrier timeout and a span mismatch raise DeviceError instead of
leaving stale parameters.
"""

import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent


def run_worker(*args, timeout=600, extra_env=None):
    from paper_2312_03549_b200.emulation import child_env

    env = child_env()
    env.update(extra_env or {})
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "emu_worker.py"), *map(str, args)],
                       capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert p.returncode == 0, f"worker failed ({p.returncode}):\n{p.stdout[-3000:]}\n{p.stderr[-3000:]}"
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("d", [2, 3, 4, 8])
@pytest.mark.parametrize("clip", [0.0, 0.02])
@pytest.mark.parametrize("flow", ["step", "hooks"])
def test_emulated_ranks_match_oracle(d, clip, flow):
    out = run_worker("--d", d, "--clip", clip, "--flow", flow, "--steps", 3)
    assert out["ok"] and out["buckets"] > 3


@pytest.mark.parametrize("flow", ["step", "hooks"])
def test_emulated_ranks_maximum_span(flow):
    """Spans at their maximum of HOD_P2P_MAX_SPAN (32) buckets: a deep model
    of many small tensors, one bucket each, with an unbounded span threshold
    splits into full 32-bucket spans and a remainder (one launch's SpanArgs
    tables filled to capacity)."""
    out = run_worker("--d", 2, "--config", "deep", "--bucket", 20_000, "--span", 10**9, "--first-span", 10**9,
                     "--clip", 0.02, "--flow", flow, "--steps", 2)
    assert out["ok"] and out["buckets"] > 32


@pytest.mark.parametrize("d", [5, 6, 7])
def test_emulated_ranks_non_power_of_two(d):
    """DP rows that are not a power of two (the generic-d kernel paths, shard
    padding to lcm(128, 16 d)) through the concurrent protocol with clipping
    and the hook-driven flow."""
    out = run_worker("--d", d, "--clip", 0.02, "--flow", "hooks", "--steps", 2)
    assert out["ok"]


@pytest.mark.parametrize("d,clip,flow", [(2, 0.0, "step"), (4, 0.02, "step"), (8, 0.0, "step"),
                                         (4, 0.02, "hooks")])
def test_emulated_ranks_tma_span_kernel(d, clip, flow):
    """The TMA-fed span kernel (HOD_SPAN_TMA=2: also under the emulation's
    grid cap) through the concurrent protocol, checked like the default."""
    out = run_worker("--d", d, "--clip", clip, "--flow", flow, "--steps", 3, extra_env={"HOD_SPAN_TMA": "2"})
    assert out["ok"] and out["buckets"] > 3


@pytest.mark.parametrize("flow", ["step", "hooks"])
def test_emulated_baseline_config1_toy_gpt_fp32_dp2(flow):
    """BASELINE config 1 exactly (toy GPT L4 h256, fp32 grads, DP = 2, one
    overlapped step) — the reference's CPU scenario — on one GPU."""
    out = run_worker("--d", 2, "--config", "toy", "--grad-dtype", "f32", "--bucket", 4_000_000,
                     "--span", 8_000_000, "--first-span", 4_000_000, "--flow", flow, "--steps", 2)
    assert out["ok"]


@pytest.mark.parametrize("d,clip", [(2, 0.0), (4, 1.0)])
def test_emulated_fullsize_gpt13b(d, clip):
    """BASELINE config 2 at its real size (GPT-3 1.3B gradient set, 37
    buckets of 25 M elements, bf16 grads) with d ranks running the real
    protocol on one GPU: every bucket of every rank bit-exact against the
    oracle (reduced shard, master, m, v, gathered params)."""
    out = run_worker("--d", d, "--config", "gpt1.3b", "--bucket", 25_000_000, "--span", 268_435_456,
                     "--first-span", 33_554_432, "--clip", clip, "--steps", 1, "--timeout", 60, timeout=1200)
    assert out["ok"] and out["buckets"] == 37


def test_emulated_fp32_grads_without_keep_reduced():
    out = run_worker("--d", 4, "--grad-dtype", "f32", "--keep-reduced", 0, "--clip", 1.0, "--flow", "hooks")
    assert out["ok"]


@pytest.mark.parametrize("d,clip", [(2, 0.0), (4, 0.02)])
def test_emulated_ranks_fast_adamw_within_tolerance(d, clip):
    """adamw='fast' through the fused span kernels: reduce-scatter still
    bit-exact, master / m / v within the north star's tolerance."""
    out = run_worker("--d", d, "--clip", clip, "--adamw", "fast", "--steps", 3)
    assert out["ok"]


@pytest.mark.parametrize("adamw", ["exact", "fast"])
def test_emulated_ranks_100_steps(adamw):
    """The north star's long-run tolerance at d > 1: 100 steps of the real
    protocol (d = 2, clip), every step against the oracle's INDEPENDENT
    trajectory — exact: bit-exact at every step; fast: master / m / v within
    1e-6 after step 1 and 1e-5 after that (norm-relative)."""
    out = run_worker("--d", 2, "--clip", 0.02, "--steps", 100, "--adamw", adamw, timeout=1200)
    assert out["ok"]


def test_barrier_timeout_raises_device_error():
    out = run_worker("--d", 2, "--fault", "timeout", "--timeout", 0.5)
    assert "10003" in out["raised"] and "next_step_raised" in out


def test_span_mismatch_raises_device_error():
    out = run_worker("--d", 2, "--fault", "span", "--timeout", 5)
    assert all("10005" in c for c in out["raised"])


@pytest.mark.parametrize("d", [2, 4])
def test_checkpoint_restore_with_gather_is_bit_exact(d):
    """checkpoint.load(gather=True) at d > 1: every rank's param
    buffer equals the saved model, and a further step matches the optimizer
    that never stopped, bit for bit."""
    out = run_worker("--d", d, "--fault", "checkpoint", "--clip", 0.02)
    assert out["ok"]
