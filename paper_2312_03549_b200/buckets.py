"""Gradient-bucket layout — pure integer arithmetic.

The reference prices one flat "gradient set" per pipeline stage
(``_stage_grad_bytes``, simulator.py:268-280) and never splits it.  The
overlapped optimizer (Megatron-LLaMA) splits that set into
buckets so bucket k's collective can run while bucket k+1 is still being
produced.  The rule, fixed here and restated independently in
oracle/oracle.py::bucket_layout:

* walk parameters in REVERSE registration order (the order backward
  produces their gradients);
* align every parameter start to ``param_align`` (64) elements, so each
  tensor starts on a 128-byte (bf16) / 256-byte (fp32) boundary;
* close the bucket as soon as it holds >= ``bucket_size`` elements; a
  parameter is never split across buckets;
* pad every bucket to a multiple of lcm(128, 16*d) elements, so every
  rank's shard is a whole number of 32-byte bf16 vectors; for d | 8 the
  multiple is 128 and the layout does not depend on d (DP-invariant);
* shard r of a bucket of n elements is [start + r*n/d, start + (r+1)*n/d).

HBM layout built on top of it: one flat bf16
param buffer and one flat bf16 gradient-bucket buffer of ``total_numel``
elements, and fp32 master / exp_avg / exp_avg_sq buffers of
``total_numel / d`` elements holding this rank's shards back to back.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass


@dataclass(frozen=True)
class ParamSlot:
    """Where one parameter lives inside the flat buffers."""

    index: int          # registration index of the parameter
    bucket: int         # bucket id (0 = first bucket produced by backward)
    offset: int         # element offset inside its bucket
    numel: int

    def to_json_dict(self) -> dict:
        return {"index": self.index, "bucket": self.bucket, "offset": self.offset,
                "numel": self.numel}


@dataclass(frozen=True)
class Bucket:
    index: int
    start: int                       # element offset in the flat buffer
    numel: int                       # padded size
    slots: tuple[ParamSlot, ...]     # in bucket order (reverse registration)

    @property
    def used(self) -> int:
        last = self.slots[-1]
        return last.offset + last.numel

    def shard_numel(self, dp: int) -> int:
        return self.numel // dp

    def shard_range(self, rank: int, dp: int) -> tuple[int, int]:
        """[begin, end) of rank's shard in flat-buffer coordinates."""
        n = self.numel // dp
        return self.start + rank * n, self.start + (rank + 1) * n

    def to_json_dict(self) -> dict:
        return {"index": self.index, "start": self.start, "numel": self.numel,
                "params": [s.index for s in self.slots],
                "offsets": [s.offset for s in self.slots]}


@dataclass(frozen=True)
class BucketLayout:
    buckets: tuple[Bucket, ...]
    numels: tuple[int, ...]          # per parameter, registration order
    bucket_size: int
    dp: int
    param_align: int
    pad_multiple: int

    @property
    def total_numel(self) -> int:
        return sum(b.numel for b in self.buckets)

    @property
    def param_numel(self) -> int:
        return sum(self.numels)

    @property
    def padding(self) -> int:
        return self.total_numel - self.param_numel

    def slot(self, param_index: int) -> ParamSlot:
        return self._slot_map()[param_index]

    def _slot_map(self) -> dict[int, ParamSlot]:
        return {s.index: s for b in self.buckets for s in b.slots}

    def shard_offsets(self) -> list[int]:
        """Offset of each bucket's shard inside this rank's fp32 state buffers."""
        out, acc = [], 0
        for b in self.buckets:
            out.append(acc)
            acc += b.numel // self.dp
        return out

    def to_json_dict(self) -> dict:
        return {
            "bucket_size": self.bucket_size,
            "dp": self.dp,
            "param_align": self.param_align,
            "pad_multiple": self.pad_multiple,
            "total_numel": self.total_numel,
            "param_numel": self.param_numel,
            "buckets": [b.to_json_dict() for b in self.buckets],
        }

    def to_json(self) -> str:
        return json.dumps(self.to_json_dict(), indent=2, ensure_ascii=False) + "\n"


def pad_multiple_for(dp: int, pad_base: int = 128) -> int:
    return math.lcm(pad_base, 16 * dp)


def _ceil_to(x: int, m: int) -> int:
    return -(-x // m) * m


def build_bucket_layout(numels, bucket_size: int, dp: int = 1, param_align: int = 64,
                        pad_base: int = 128) -> BucketLayout:
    """Lay out parameters of the given element counts into buckets (rule above)."""
    numels = tuple(int(n) for n in numels)
    if dp < 1:
        raise ValueError(f"dp must be >= 1, got {dp}")
    if bucket_size < 1:
        raise ValueError(f"bucket_size must be >= 1, got {bucket_size}")
    if any(n < 0 for n in numels):
        raise ValueError("parameter sizes must be >= 0")
    pad = pad_multiple_for(dp, pad_base)
    buckets: list[Bucket] = []
    pending: list[ParamSlot] = []
    fill = 0
    start = 0
    for idx in range(len(numels) - 1, -1, -1):
        off = _ceil_to(fill, param_align)
        pending.append(ParamSlot(idx, len(buckets), off, numels[idx]))
        fill = off + numels[idx]
        if fill >= bucket_size:
            size = _ceil_to(fill, pad)
            buckets.append(Bucket(len(buckets), start, size, tuple(pending)))
            start += size
            pending, fill = [], 0
    if pending:
        size = max(_ceil_to(fill, pad), pad)
        buckets.append(Bucket(len(buckets), start, size, tuple(pending)))
    return BucketLayout(tuple(buckets), numels, bucket_size, dp, param_align, pad)
