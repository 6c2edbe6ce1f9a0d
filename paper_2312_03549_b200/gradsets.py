"""Synthetic gradient sets for the BASELINE.json configurations.

Tensor lists follow the reference's parameter-count model:
``_stage_grad_bytes`` (simulator.py:268-280) counts 12*h^2 parameters per
transformer layer (qkv 3h*h, proj h*h, fc1 4h*h, fc2 h*4h) plus the V*h
embedding on each terminal pipeline stage (once when p == 1).
``gpt_stage_tensors`` reproduces exactly that count, tensor by tensor, so
``sum(numels) * bytes_per_param == _stage_grad_bytes(...)`` (tests check it).

LLaMA-7B uses the real HuggingFace parameter list (untied lm_head, RMSNorm
weights, SwiGLU MLP): 6,738,415,616 parameters.

Synthetic data convention: per-rank gradients
g ~ N(0, 1e-3^2) from torch.Generator(seed = 1234 + 1000*step + global_rank),
generated per tensor in registration order; initial parameters
theta0 ~ N(0, 0.02^2) from seed 42.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TensorSpec:
    name: str
    shape: tuple[int, ...]

    @property
    def numel(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n


@dataclass(frozen=True)
class GradSet:
    name: str
    tensors: tuple[TensorSpec, ...]

    @property
    def numels(self) -> tuple[int, ...]:
        return tuple(t.numel for t in self.tensors)

    @property
    def total(self) -> int:
        return sum(self.numels)


def _gpt_layer(i: int, h: int) -> list[TensorSpec]:
    return [
        TensorSpec(f"layers.{i}.attn.qkv.weight", (3 * h, h)),
        TensorSpec(f"layers.{i}.attn.proj.weight", (h, h)),
        TensorSpec(f"layers.{i}.mlp.fc1.weight", (4 * h, h)),
        TensorSpec(f"layers.{i}.mlp.fc2.weight", (h, 4 * h)),
    ]


def gpt_stage_tensors(layers: int, hidden: int, vocab: int = 51200, stage: int = 1,
                      pipeline: int = 1, first_layer: int = 0, name: str = "gpt") -> GradSet:
    """One pipeline stage of a GPT-style model, counted like simulator.py:268-280."""
    ts: list[TensorSpec] = []
    if pipeline == 1 or stage == 1:
        ts.append(TensorSpec("embed.weight", (vocab, hidden)))
    for i in range(first_layer, first_layer + layers):
        ts.extend(_gpt_layer(i, hidden))
    if pipeline > 1 and stage == pipeline:
        ts.append(TensorSpec("lm_head.weight", (vocab, hidden)))
    return GradSet(name, tuple(ts))


def llama7b_tensors() -> GradSet:
    h, f, v, L = 4096, 11008, 32000, 32
    ts = [TensorSpec("model.embed_tokens.weight", (v, h))]
    for i in range(L):
        p = f"model.layers.{i}."
        ts += [
            TensorSpec(p + "self_attn.q_proj.weight", (h, h)),
            TensorSpec(p + "self_attn.k_proj.weight", (h, h)),
            TensorSpec(p + "self_attn.v_proj.weight", (h, h)),
            TensorSpec(p + "self_attn.o_proj.weight", (h, h)),
            TensorSpec(p + "mlp.gate_proj.weight", (f, h)),
            TensorSpec(p + "mlp.up_proj.weight", (f, h)),
            TensorSpec(p + "mlp.down_proj.weight", (h, f)),
            TensorSpec(p + "input_layernorm.weight", (h,)),
            TensorSpec(p + "post_attention_layernorm.weight", (h,)),
        ]
    ts += [TensorSpec("model.norm.weight", (h,)), TensorSpec("lm_head.weight", (v, h))]
    return GradSet("llama-7b", tuple(ts))


def odd_tensors(layers: int = 3, hidden: int = 200, vocab: int = 1001) -> GradSet:
    """Adversarial sizes (odd, non-multiples of 8/64/128) for the padding paths."""
    ts = [TensorSpec("embed.weight", (vocab, hidden))]
    for i in range(layers):
        ts += [
            TensorSpec(f"l{i}.qkv.weight", (3 * hidden + 13, hidden)),
            TensorSpec(f"l{i}.qkv.bias", (3 * hidden + 13,)),
            TensorSpec(f"l{i}.ln.weight", (hidden + 1,)),
            TensorSpec(f"l{i}.fc.weight", (hidden, 4 * hidden + 7)),
            TensorSpec(f"l{i}.scalar", (1,)),
        ]
    return GradSet("odd", tuple(ts))


def config_gradset(config: str, stage: int = 1) -> GradSet:
    """Gradient set of one BASELINE.json configuration (1-based stage for 13B)."""
    if config == "toy":
        return gpt_stage_tensors(4, 256, 51200, name="toy-gpt-l4-h256")
    if config == "gpt1.3b":
        return gpt_stage_tensors(24, 2048, 51200, name="gpt3-1.3b")
    if config == "llama7b":
        return llama7b_tensors()
    if config == "gpt13b":
        # stage layers [23, 17] come from the self-adapting partition of the
        # config-4 scenario (scenarios/gpt13b_pp2_dp4_hybrid.json)
        layers = (23, 17)
        first = 0 if stage == 1 else layers[0]
        return gpt_stage_tensors(layers[stage - 1], 5120, 51200, stage=stage, pipeline=2,
                                 first_layer=first, name=f"gpt3-13b-stage{stage}")
    if config == "odd":
        return odd_tensors()
    if config == "deep":
        # many small tensors: > HOD_P2P_MAX_SPAN buckets at small bucket sizes (test shape)
        return gpt_stage_tensors(40, 128, 1000, name="deep-gpt-l40-h128")
    raise ValueError(f"unknown gradient-set config {config!r}")
