"""CPU: pin the oracle (and the layout rule) before trusting it.

* AdamW / clip restatement vs torch.optim.AdamW + clip_grad_norm_ golden
  vectors (tests/golden/adamw_torch.npz): 1e-6 after 1 step, 1e-5 after 100
  (SURVEY.md §8d tolerance rule |a-b| <= rtol*max|b|).
* pack / reduce-scatter restatements vs independent numpy formulations
  (bit-exact).
* bucket layout: the product's builder == the oracle's loop, SURVEY §8a N1
  known answers (37 / 162 buckets), DP invariance for d | 8, alignment.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_2312_03549_b200 as hp
from paper_2312_03549_b200.buckets import build_bucket_layout
from paper_2312_03549_b200.gradsets import config_gradset, gpt_stage_tensors, odd_tensors

GOLD = Path(__file__).parent / "golden" / "adamw_torch.npz"
N = 4099


def _grad(step):
    import torch

    g = np.random.default_rng(1000 + step).standard_normal(N).astype(np.float32) * np.float32(1e-3)
    return torch.from_numpy(g).to(torch.bfloat16).float().numpy()


def _init():
    return np.random.default_rng(42).standard_normal(N).astype(np.float32) * np.float32(0.02)


def _max_ulp(a, b):
    """Max distance in fp32 units-in-the-last-place (ordered int32 mapping)."""
    def key(x):
        i = np.asarray(x, np.float32).view(np.int32).astype(np.int64)
        return np.where(i < 0, -(i & 0x7FFFFFFF), i)
    return int(np.abs(key(a) - key(b)).max())


@pytest.mark.parametrize("steps,clip,rtol", [(1, None, 1e-6), (100, None, 1e-5),
                                             (1, 0.01, 1e-6), (100, 0.01, 1e-5)])
def test_oracle_adamw_pinned_to_torch(oracle, steps, clip, rtol, record_property):
    gold = np.load(GOLD)
    tag = f"s{steps}_{'clip' if clip else 'noclip'}"
    master, m, v = _init(), np.zeros(N, np.float32), np.zeros(N, np.float32)
    for s in range(1, steps + 1):
        g16 = oracle.f32_to_bf16(_grad(s))
        coef = None
        if clip is not None:
            # the norm itself: our fp64 sum vs torch's fp32 vector_norm (~4e-7 apart)
            ss = oracle.sumsq_bf16(g16)
            tnorm = gold[f"{tag}_norms"][s - 1]
            assert abs(np.sqrt(ss) - tnorm) <= 1e-6 * np.sqrt(ss)
            assert abs(oracle.clip_coef(np.float32(ss), clip) * (tnorm + 1e-6) / clip - 1) <= 1e-6
            # AdamW given the SAME coefficient torch used (clip_grad_norm_ in fp32)
            coef = float(min(np.float32(1.0), np.float32(clip) / (np.float32(tnorm) + np.float32(1e-6))))
        oracle.adamw(master, m, v, g16, s, 1e-4, (0.9, 0.95), 1e-8, 0.1, coef=coef)
    for name, got in (("master", master), ("m", m), ("v", v)):
        want = gold[f"{tag}_{name}"]
        err = np.abs(got.astype(np.float64) - want).max()
        assert err <= rtol * np.abs(want).max(), (name, err, np.abs(want).max())
        # record the max-ULP distance alongside (large only for
        # elements near zero, which is why the pass rule is norm-relative)
        record_property(f"max_ulp_{name}", _max_ulp(got, want))


def _np_bf16(x32):
    u = x32.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(x32)
    r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def test_oracle_bf16_rounding_matches_numpy(oracle):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100_000).astype(np.float32) * 10 ** rng.uniform(-30, 30, 100_000).astype(np.float32),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8,
                                  3.3895314e38], np.float32)])
    np.testing.assert_array_equal(oracle.f32_to_bf16(x), _np_bf16(x))


def test_oracle_pack_and_rs_match_numpy(oracle):
    rng = np.random.default_rng(1)
    sizes = [1000, 37, 4096, 5]
    offs = [0, 1024, 1088, 5184]
    numel = 5248
    for scale in (1.0, 0.25, 1 / 3):
        g32 = [rng.standard_normal(n).astype(np.float32) for n in sizes]
        want = np.zeros(numel, np.uint16)
        for g, o in zip(g32, offs):
            want[o:o + g.size] = _np_bf16(g * np.float32(scale))
        np.testing.assert_array_equal(oracle.pack(g32, offs, numel, scale), want)
        g16 = [_np_bf16(g) for g in g32]
        want16 = np.zeros(numel, np.uint16)
        for g, o in zip(g16, offs):
            want16[o:o + g.size] = _np_bf16(oracle.bf16_to_f32(g) * np.float32(scale))
        np.testing.assert_array_equal(oracle.pack(g16, offs, numel, scale), want16)
    buckets = [_np_bf16(rng.standard_normal(4096).astype(np.float32)) for _ in range(4)]
    acc = np.zeros(1024, np.float32)
    for b in buckets:
        acc = acc + oracle.bf16_to_f32(b[2048:3072])
    np.testing.assert_array_equal(oracle.reduce_scatter(buckets, 2, 4), _np_bf16(acc))


@pytest.mark.parametrize("config,nb,lo,hi", [("gpt1.3b", 37, 33_554_432, 104_857_600),
                                             ("llama7b", 162, 33_554_432, 131_072_000),
                                             ("toy", 1, 16_252_928, 16_252_928)])
def test_layout_known_answers(oracle, config, nb, lo, hi):
    gs = config_gradset(config)
    for d in (1, 2, 4, 8):
        L = build_bucket_layout(gs.numels, 25_000_000, dp=d)
        assert len(L.buckets) == nb
        assert min(b.numel for b in L.buckets) == lo and max(b.numel for b in L.buckets) == hi
        assert L.padding == 0
        O = oracle.bucket_layout(gs.numels, 25_000_000, d)
        assert [(b.start, b.numel, [(s.index, s.offset, s.numel) for s in b.slots]) for b in L.buckets] == \
               [(o["start"], o["numel"], o["params"]) for o in O]


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("bucket", [1, 1000, 150_000, 10**9])
def test_layout_properties_odd_sizes(oracle, d, bucket):
    gs = odd_tensors()
    L = build_bucket_layout(gs.numels, bucket, dp=d)
    O = oracle.bucket_layout(gs.numels, bucket, d)
    assert [(b.start, b.numel, [(s.index, s.offset, s.numel) for s in b.slots]) for b in L.buckets] == \
           [(o["start"], o["numel"], o["params"]) for o in O]
    seen = sorted(s.index for b in L.buckets for s in b.slots)
    assert seen == list(range(len(gs.numels)))            # every param exactly once
    order = [s.index for b in L.buckets for s in b.slots]
    assert order == sorted(order, reverse=True)           # backward order
    pos = 0
    for b in L.buckets:
        assert b.start == pos and b.numel % d == 0
        assert (b.numel // d) % 16 == 0                    # 32-byte bf16 shards
        assert all(s.offset % 64 == 0 for s in b.slots)
        assert b.used <= b.numel
        pos += b.numel
    if d in (1, 2, 4, 8):                                  # DP-invariant layout
        ref = build_bucket_layout(gs.numels, bucket, dp=1)
        assert [(b.start, b.numel) for b in L.buckets] == [(b.start, b.numel) for b in ref.buckets]


def test_gradsets_match_reference_stage_grad_bytes():
    # tensor lists reproduce _stage_grad_bytes exactly
    for L_, h, p in ((4, 256, 1), (24, 2048, 1)):
        gs = gpt_stage_tensors(L_, h)
        model = hp.ModelSpec(layers=L_, hidden=h, heads=16, global_batch=8, micro_batch=1)
        assert gs.total * 2 == hp.stage_grad_bytes(1, L_, p, model)
    model = hp.ModelSpec(layers=40, hidden=5120, heads=40, global_batch=512, micro_batch=4)
    for stage, layers in ((1, 23), (2, 17)):
        gs = config_gradset("gpt13b", stage)
        assert gs.total * 2 == hp.stage_grad_bytes(stage, layers, 2, model)
    assert config_gradset("llama7b").total == 6_738_415_616
    assert config_gradset("toy").total == 16_252_928
    assert config_gradset("gpt1.3b").total == 1_312_817_152


def test_layout_json_roundtrip():
    import json

    L = build_bucket_layout(config_gradset("gpt1.3b").numels, 25_000_000, dp=8)
    doc = json.loads(L.to_json())
    assert doc["total_numel"] == 1_312_817_152 and len(doc["buckets"]) == 37
    assert doc["buckets"][0]["params"][0] == len(config_gradset("gpt1.3b").numels) - 1


def test_sum_slices_equals_reduce_scatter(oracle):
    """The streaming form the full-size check uses (each rank holds only its
    own shard of every rank's bucket) is the reduce-scatter, bit for bit."""
    rng = np.random.default_rng(3)
    d, n = 4, 4096
    packs = [oracle.f32_to_bf16(rng.standard_normal(n).astype(np.float32)) for _ in range(d)]
    sh = n // d
    for r in range(d):
        cut = [p[r * sh:(r + 1) * sh] for p in packs]
        np.testing.assert_array_equal(oracle.sum_slices(cut), oracle.reduce_scatter(packs, r, d))
        np.testing.assert_array_equal(oracle.sum_slices_f64(cut), oracle.reduce_scatter_f64(packs, r, d))
