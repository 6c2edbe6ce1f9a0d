"""Symmetric (peer-mapped + NVLS multicast) buffers for the fused collectives.

Allocation and the handle exchange are plumbing borrowed from
``torch.distributed._symmetric_memory`` (cuMem VMM under the hood); all data
movement on these buffers is done by our own kernels (csrc/hod_p2p.cu).  Each
rank of the DP row maps every peer's copy (``ptrs[q]``) and, when the box
supports NVLS, one multicast address (``mc``) whose loads reduce across all
copies (multimem.ld_reduce) and whose stores land in all of them.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .errors import DeviceError


# torch's symmetric memory is a private API: the calls used here exist with
# these semantics from torch 2.6 on (empty / rendezvous / buffer_ptrs /
# multicast_ptr); checked once, with a clear error instead of an AttributeError
# deep inside a step
_MIN_TORCH = (2, 6)


def _symm():
    ver = tuple(int(x) for x in torch.__version__.split("+")[0].split(".")[:2])
    if ver < _MIN_TORCH:
        raise DeviceError(f"torch {torch.__version__}: symmetric memory needs torch >= 2.6 "
                          "(use backend='nccl')")
    try:
        import torch.distributed._symmetric_memory as symm_mem
    except ImportError as e:
        raise DeviceError(f"torch.distributed._symmetric_memory unavailable ({e}); use backend='nccl'") from e
    for name in ("empty", "rendezvous"):
        if not hasattr(symm_mem, name):
            raise DeviceError(f"torch {torch.__version__}: _symmetric_memory.{name} missing; "
                              "use backend='nccl'")
    return symm_mem


class SymmetricTensor:
    """One symmetric allocation over ``group``: the local tensor + peer/mc pointers."""

    def __init__(self, numel: int, dtype: torch.dtype, device, group, zero: bool = False):
        symm_mem = _symm()
        self.tensor = symm_mem.empty(numel, dtype=dtype, device=device)
        if zero:
            self.tensor.zero_()
        name = group.group_name if group is not None else dist.group.WORLD.group_name
        self.handle = symm_mem.rendezvous(self.tensor, name)
        if not hasattr(self.handle, "buffer_ptrs"):
            raise DeviceError(f"torch {torch.__version__}: symmetric memory handle has no buffer_ptrs")
        self.ptrs = [int(p) for p in self.handle.buffer_ptrs]
        self.mc = int(self.handle.multicast_ptr or 0)
        self.rank = int(self.handle.rank)
        self.world = int(self.handle.world_size)
        if self.ptrs[self.rank] != self.tensor.data_ptr():
            raise DeviceError("symmetric rendezvous returned an unexpected local pointer")

    def peer(self, q: int, byte_offset: int = 0) -> int:
        return self.ptrs[q] + byte_offset

    def multicast(self, byte_offset: int = 0) -> int:
        if not self.mc:
            raise DeviceError("NVLS multicast is not available on this group/box")
        return self.mc + byte_offset


def group_for(ranks, world_group_ranks=None):
    """Process group over ``ranks``: the WORLD when it spans everybody.

    Any other member set needs a group that every rank of the world created
    in the same call (``dist.new_group`` is collective over the WORLD and
    must see identical arguments everywhere): build all DP rows at once with
    ``dist.new_subgroups_by_enumeration`` (``scenario_run.setup_rank`` does)
    and pass the row's group as ``process_group`` / ``norm_group``."""
    from .errors import InfeasibleConfigError

    ranks = tuple(ranks)
    if len(ranks) == dist.get_world_size() and sorted(ranks) == list(range(len(ranks))):
        return dist.group.WORLD
    raise InfeasibleConfigError(
        f"ranks {ranks} are not the whole world: pass the row's process group (create every row on every "
        "rank with dist.new_subgroups_by_enumeration, e.g. scenario_run.setup_rank)")
