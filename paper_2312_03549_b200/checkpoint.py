"""Sharded optimizer checkpoint.

Each rank writes its own shard files — fp32 master, exp_avg, exp_avg_sq (the
``total/d`` elements of its DP shards, back to back) — plus one JSON
manifest with the ``BucketLayout``, the step count, the hyper-parameters and
a sha256 per array, in the same determinism conventions as the reference's
scenario fingerprint (config.py:292: sha256 of raw bytes).  Loading checks
that the layout and the DP position match, restores the local bf16 param
shards from the master and, with ``gather=True`` (the default), all-gathers
them so every rank's param buffer holds the restored model before the next
forward (``DistributedOptimizer.gather_params``; every rank of the row must
call ``load``).
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import torch

from .errors import ConfigError

_ARRAYS = ("master", "exp_avg", "exp_avg_sq")


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(a.tobytes()).hexdigest()


def save(opt, directory) -> Path:
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    r = opt.group.global_rank
    torch.cuda.synchronize(opt.device)
    manifest = {
        "format": "hod-sharded-optimizer/1",
        "step": opt.step_count,
        "dp": opt.dp,
        "shard_index": opt.shard_index,
        "dp_ranks": list(opt.group.ranks),
        "hparams": {"lr": opt.lr, "betas": list(opt.betas), "eps": opt.eps,
                    "weight_decay": opt.weight_decay, "clip": opt.clip},
        "layout": opt.layout.to_json_dict(),
        "arrays": {},
    }
    for name in _ARRAYS:
        arr = getattr(opt, name).detach().cpu().numpy()
        path = d / f"rank{r:05d}.{name}.npy"
        np.save(path, arr)
        manifest["arrays"][name] = {"file": path.name, "sha256": _sha(arr), "numel": int(arr.size)}
    out = d / f"rank{r:05d}.manifest.json"
    out.write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    return out


def load(opt, directory, gather: bool = True) -> dict:
    d = Path(directory)
    r = opt.group.global_rank
    man = json.loads((d / f"rank{r:05d}.manifest.json").read_text())
    if man["layout"] != opt.layout.to_json_dict():
        raise ConfigError("checkpoint bucket layout differs from the optimizer's")
    if man["dp"] != opt.dp or man["shard_index"] != opt.shard_index:
        raise ConfigError("checkpoint DP position differs from the optimizer's")
    for name in _ARRAYS:
        meta = man["arrays"][name]
        arr = np.load(d / meta["file"])
        if _sha(arr) != meta["sha256"]:
            raise ConfigError(f"checkpoint array {name} is corrupt (sha256 mismatch)")
        getattr(opt, name).copy_(torch.from_numpy(arr).to(opt.device))
    opt.step_count = int(man["step"])
    # the local param shard follows from the master (RNE, as the update
    # kernels round it); the peers' shards come from their owners
    for b, off in zip(opt.layout.buckets, opt.layout.shard_offsets()):
        lo, hi = b.shard_range(opt.shard_index, opt.dp)
        opt.param_buffer[lo:hi].copy_(opt.master[off:off + (hi - lo)].to(torch.bfloat16))
    torch.cuda.synchronize(opt.device)
    if gather and opt.dp > 1:
        opt.gather_params()
    return man
