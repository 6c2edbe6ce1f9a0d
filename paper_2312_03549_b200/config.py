"""Scenario documents — mirror of holmes_planner.config
(reference config.py:1-318).

The schema is the reference's, unchanged (Draft 2020-12, ``additionalProperties:
false`` everywhere), so every reference scenario file — and the new config-4
preset ``scenarios/gpt13b_pp2_dp4_hybrid.json`` — loads unchanged.  Optimizer
knobs (bucket size, lr, betas, eps, weight decay, clip) deliberately live in a
SEPARATE document (``OptimizerSettings``) so scenario files still validate.
Fingerprint = sha256 of the raw bytes.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path

import jsonschema

from .errors import ConfigError
from .groups import ParallelConfig
from .partition import ModelSpec, PartitionStrategy
from .simulator import CostModel
from .topology import DEFAULT_INTRA_NODE_LATENCY_S, Cluster, ClusterTopology, NicKind, NicSpec


def _num(exclusive_min=None, minimum=None, maximum=None):
    s = {"type": "number"}
    if exclusive_min is not None:
        s["exclusiveMinimum"] = exclusive_min
    if minimum is not None:
        s["minimum"] = minimum
    if maximum is not None:
        s["maximum"] = maximum
    return s


def _int_min1():
    return {"type": "integer", "minimum": 1}


def _obj(props, required=()):
    d = {"type": "object", "properties": props, "additionalProperties": False}
    if required:
        d["required"] = list(required)
    return d


def _pos_array():
    return {"type": "array", "items": _num(exclusive_min=0)}


_NIC = _obj({"kind": {"type": "string", "enum": ["infiniband", "roce", "ethernet"]},
             "bandwidth_gbps": _num(exclusive_min=0), "latency_s": _num(minimum=0)},
            ("kind", "bandwidth_gbps"))
_ETH = _obj({"bandwidth_gbps": _num(exclusive_min=0), "latency_s": _num(minimum=0)},
            ("bandwidth_gbps",))

SCENARIO_SCHEMA = {
    "$schema": "https://json-schema.org/draft/2020-12/schema",
    **_obj({
        "topology": _obj({
            "clusters": {"type": "array", "minItems": 1,
                         "items": _obj({"nodes": _int_min1(), "nic": _NIC,
                                        "device_tflops_peak": _num(exclusive_min=0),
                                        "device_mem_gb": _num(exclusive_min=0)}, ("nodes",))},
            "gpus_per_node": _int_min1(),
            "ethernet": _ETH,
            "intra_node_bandwidth_gbps": _num(exclusive_min=0),
            "intra_node_latency_s": _num(minimum=0),
            "inter_cluster_rdma": {"type": "boolean"},
        }, ("clusters", "gpus_per_node", "ethernet", "intra_node_bandwidth_gbps")),
        "model": _obj({k: _int_min1() for k in ("layers", "hidden", "heads", "seq_len", "vocab",
                                                 "global_batch", "micro_batch", "bytes_per_param")}
                      | {"per_layer_mem_gb": _num(exclusive_min=0)},
                      ("layers", "hidden", "heads", "global_batch", "micro_batch")),
        "parallel": _obj({"t": _int_min1(), "p": _int_min1(), "d": _int_min1()}, ("t", "p", "d")),
        "partition": _obj({"strategy": {"type": "string", "enum": ["uniform", "self_adapting"]},
                           "alpha": _num(exclusive_min=0), "cluster_alphas": _pos_array(),
                           "cluster_mem_budget_gb": _pos_array()}),
        "cost": _obj({"eta": _num(exclusive_min=0, maximum=1),
                      "backward_forward_ratio": _num(exclusive_min=0),
                      "cluster_speeds_tflops": _pos_array()}),
        "notes": {"type": "string"},
    }, ("topology", "model", "parallel")),
}

_FLAGGED_MODEL_DEFAULTS = ("seq_len", "vocab")


@dataclass(frozen=True)
class PartitionSettings:
    strategy: PartitionStrategy = PartitionStrategy.UNIFORM
    alpha: float = 1.0
    cluster_alphas: tuple[float, ...] | None = None
    cluster_mem_budget_gb: tuple[float, ...] | None = None


@dataclass(frozen=True)
class ScenarioConfig:
    topology: ClusterTopology
    model: ModelSpec
    parallel: ParallelConfig
    partition: PartitionSettings
    cost: CostModel
    fingerprint: str
    name: str = "scenario"
    defaults_applied: tuple[str, ...] = ()
    notes: str | None = None


def _nic(doc: dict, kind: NicKind | None = None) -> NicSpec:
    return NicSpec(kind or NicKind(doc["kind"]), doc["bandwidth_gbps"], doc.get("latency_s"))


def _opt_tuple(doc: dict, key: str):
    return tuple(doc[key]) if key in doc else None


def parse_scenario(doc: dict, raw: bytes, name: str = "scenario") -> ScenarioConfig:
    try:
        jsonschema.validate(doc, SCENARIO_SCHEMA)
    except jsonschema.ValidationError as exc:
        where = ".".join(str(x) for x in exc.absolute_path) or "<root>"
        raise ConfigError(f"invalid scenario at {where}: {exc.message}") from exc
    td = doc["topology"]
    eth = _nic(td["ethernet"], NicKind.ETHERNET)
    clusters = tuple(
        Cluster(index=i, node_count=c["nodes"], rdma_nic=_nic(c["nic"]) if "nic" in c else eth,
                device_tflops_peak=c.get("device_tflops_peak", 312.0),
                device_mem_gb=c.get("device_mem_gb", 80.0))
        for i, c in enumerate(td["clusters"], 1))
    topo = ClusterTopology(clusters, td["gpus_per_node"], eth, td["intra_node_bandwidth_gbps"],
                           td.get("intra_node_latency_s", DEFAULT_INTRA_NODE_LATENCY_S),
                           td.get("inter_cluster_rdma", False))
    md = doc["model"]
    model = ModelSpec(layers=md["layers"], hidden=md["hidden"], heads=md["heads"],
                      global_batch=md["global_batch"], micro_batch=md["micro_batch"],
                      seq_len=md.get("seq_len", 2048), vocab=md.get("vocab", 51200),
                      bytes_per_param=md.get("bytes_per_param", 2),
                      per_layer_mem_gb=md.get("per_layer_mem_gb"))
    pd = doc["parallel"]
    parallel = ParallelConfig(tensor=pd["t"], pipeline=pd["p"], data=pd["d"])
    qd = doc.get("partition", {})
    part = PartitionSettings(PartitionStrategy(qd.get("strategy", "uniform")), qd.get("alpha", 1.0),
                             _opt_tuple(qd, "cluster_alphas"), _opt_tuple(qd, "cluster_mem_budget_gb"))
    cd = doc.get("cost", {})
    cost = CostModel(eta=cd.get("eta", CostModel.eta),
                     backward_forward_ratio=cd.get("backward_forward_ratio",
                                                   CostModel.backward_forward_ratio),
                     cluster_speeds_tflops=_opt_tuple(cd, "cluster_speeds_tflops"))
    m = len(clusters)
    if cost.cluster_speeds_tflops is not None and len(cost.cluster_speeds_tflops) != m:
        raise ConfigError(f"cost.cluster_speeds_tflops has {len(cost.cluster_speeds_tflops)} "
                          f"entries for {m} clusters")
    for key in ("cluster_alphas", "cluster_mem_budget_gb"):
        val = getattr(part, key)
        if val is not None and len(val) not in (m, m - 1):
            raise ConfigError(f"partition.{key} has {len(val)} entries for {m} clusters")
    return ScenarioConfig(
        topology=topo, model=model, parallel=parallel, partition=part, cost=cost,
        fingerprint=hashlib.sha256(raw).hexdigest(), name=name,
        defaults_applied=tuple(f"model.{k}" for k in _FLAGGED_MODEL_DEFAULTS if k not in md),
        notes=doc.get("notes"))


def load_scenario(path) -> ScenarioConfig:
    path = Path(path)
    try:
        raw = path.read_bytes()
    except OSError as exc:
        raise ConfigError(f"cannot read {path}: {exc}") from exc
    try:
        doc = json.loads(raw.decode("utf-8"))
    except UnicodeDecodeError as exc:
        raise ConfigError(f"{path} is not UTF-8: {exc}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigError(f"{path}: {exc.msg} at line {exc.lineno} column {exc.colno}",
                          line=exc.lineno, column=exc.colno) from exc
    if not isinstance(doc, dict):
        raise ConfigError(f"{path}: top level must be a JSON object")
    return parse_scenario(doc, raw, name=path.stem)


# ---------------------------------------------------------------------------
# Optimizer settings: a separate document so scenario files stay schema-valid
# ---------------------------------------------------------------------------
OPTIMIZER_SCHEMA = {
    "$schema": "https://json-schema.org/draft/2020-12/schema",
    **_obj({
        "bucket_size": _int_min1(),
        "lr": _num(exclusive_min=0),
        "betas": {"type": "array", "items": _num(minimum=0, maximum=1), "minItems": 2, "maxItems": 2},
        "eps": _num(exclusive_min=0),
        "weight_decay": _num(minimum=0),
        "clip": {"type": ["number", "null"], "exclusiveMinimum": 0},
        "backend": {"type": "string", "enum": ["auto", "nccl", "p2p", "none"]},
        "grad_dtype": {"type": "string", "enum": ["bf16", "f32"]},
    }),
}


@dataclass(frozen=True)
class OptimizerSettings:
    bucket_size: int = 25_000_000
    lr: float = 1e-4
    betas: tuple[float, float] = (0.9, 0.95)
    eps: float = 1e-8
    weight_decay: float = 0.1
    clip: float | None = None
    backend: str = "auto"
    grad_dtype: str = "bf16"

    def to_json_dict(self) -> dict:
        return {"bucket_size": self.bucket_size, "lr": self.lr, "betas": list(self.betas),
                "eps": self.eps, "weight_decay": self.weight_decay, "clip": self.clip,
                "backend": self.backend, "grad_dtype": self.grad_dtype}


def parse_optimizer_settings(doc: dict) -> OptimizerSettings:
    try:
        jsonschema.validate(doc, OPTIMIZER_SCHEMA)
    except jsonschema.ValidationError as exc:
        where = ".".join(str(x) for x in exc.absolute_path) or "<root>"
        raise ConfigError(f"invalid optimizer settings at {where}: {exc.message}") from exc
    base = OptimizerSettings()
    kw = {k: doc.get(k, getattr(base, k)) for k in base.to_json_dict()}
    kw["betas"] = tuple(kw["betas"])
    return OptimizerSettings(**kw)
