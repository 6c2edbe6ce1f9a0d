"""NCCL communicators for DP rows, built through the C ABI (include/hod.h).

A ``DPGroup`` is one row of the reference's DP matrix (``build_dp``,
groups.py:137-148) converted to 0-based torch/NCCL ranks (reference rank
minus 1, topology.py:159-176).  Communicator bootstrap exchanges the
128-byte NCCL unique id through the torch.distributed key-value store, so
the only torch.distributed requirement is an initialised default group
(env:// rendezvous, one process per GPU).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _native as nat
from .errors import InvalidPlanError


@dataclass(frozen=True)
class DPGroup:
    """Members (0-based global ranks, in GroupPlan order) and this rank's slot."""

    ranks: tuple[int, ...]
    global_rank: int

    def __post_init__(self):
        if self.global_rank not in self.ranks:
            raise InvalidPlanError(f"rank {self.global_rank} is not in DP row {self.ranks}")

    @property
    def size(self) -> int:
        return len(self.ranks)

    @property
    def index(self) -> int:
        """Position of this rank inside the row == the shard it owns."""
        return self.ranks.index(self.global_rank)

    @classmethod
    def single(cls, global_rank: int = 0) -> "DPGroup":
        return cls((global_rank,), global_rank)

    @classmethod
    def from_plan(cls, plan, global_rank: int) -> "DPGroup":
        """The DP row of a GroupPlan that contains ``global_rank`` (0-based)."""
        for row in plan.dp.rows:
            zero_based = tuple(r - 1 for r in row)
            if global_rank in zero_based:
                return cls(zero_based, global_rank)
        raise InvalidPlanError(f"rank {global_rank} is in no DP row of the plan")


def comm_key(tag: str, serial: int, ranks) -> str:
    """Store key of one communicator's bootstrap (unique per member set)."""
    return f"hod/nccl/{tag}/{serial}/{'-'.join(map(str, ranks))}"


def exchange_unique_id(store, key: str, is_root: bool, make_id) -> bytes:
    """Root creates the 128-byte id and publishes it; the others wait for it."""
    if is_root:
        raw = make_id()
        if len(raw) != 128:
            raise InvalidPlanError("NCCL unique id must be 128 bytes")
        store.set(key, raw)
        return raw
    raw = store.get(key)
    if len(raw) != 128:
        raise InvalidPlanError(f"bad unique id under {key}")
    return bytes(raw)


def _store():
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        raise InvalidPlanError("torch.distributed must be initialised for a multi-rank group")
    return dist.distributed_c10d._get_default_store()


class NcclComm:
    """One NCCL communicator over ``ranks`` (this process must be a member)."""

    _serial: dict[str, int] = {}

    def __init__(self, ranks, global_rank: int, tag: str):
        self.ranks = tuple(ranks)
        self.rank = self.ranks.index(global_rank)
        self.size = len(self.ranks)
        n = NcclComm._serial.get(tag, 0)
        NcclComm._serial[tag] = n + 1
        key = comm_key(tag, n, self.ranks)

        def make_id() -> bytes:
            buf = (ctypes.c_uint8 * 128)()
            nat.call("hod_nccl_unique_id", ctypes.cast(buf, ctypes.c_void_p))
            return bytes(buf)

        raw = exchange_unique_id(_store(), key, self.rank == 0, make_id)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(raw)
        handle = ctypes.c_void_p()
        nat.call("hod_nccl_comm_init", ctypes.cast(uid, ctypes.c_void_p), self.size, self.rank,
                 ctypes.byref(handle))
        self.handle = handle.value

    def reduce_scatter_bf16(self, send_ptr: int, recv_ptr: int, recvcount: int, stream) -> None:
        nat.call("hod_reduce_scatter_bf16", send_ptr, recv_ptr, recvcount, self.handle,
                 nat.stream_ptr(stream))

    def all_gather_bf16(self, send_ptr: int, recv_ptr: int, sendcount: int, stream) -> None:
        nat.call("hod_all_gather_bf16", send_ptr, recv_ptr, sendcount, self.handle,
                 nat.stream_ptr(stream))

    def all_reduce_f32(self, ptr: int, n: int, stream) -> None:
        nat.call("hod_all_reduce_f32", ptr, n, self.handle, nat.stream_ptr(stream))

    def check(self) -> None:
        """Raise DeviceError if NCCL recorded an asynchronous error on this
        communicator (ncclCommGetAsyncError; no synchronisation)."""
        if self.handle:
            nat.call("hod_comm_async_error", self.handle)

    def close(self) -> None:
        if self.handle:
            nat.call("hod_comm_destroy", self.handle)
            self.handle = None
