"""d data-parallel ranks of one DP row on ONE GPU, running the real protocol.

The driver's GPU tests run on a single B200, so the cross-GPU half of the
step — arrival barriers, span tags, params-ready barriers, the peer-memory
norm exchange — would otherwise never execute concurrently on its hardware.
An ``EmulatedRow`` gives every emulated rank ordinary allocations on the one
device in place of symmetric memory: ``peer(q)`` of rank r is simply rank q's
allocation, so the fused kernels (csrc/hod_p2p.cu) load, store and signal
exactly as they do over NVLink, only through local HBM.  Every rank owns its
own ``DistributedOptimizer`` with its own streams; the host thread issues the
ranks' steps one after another without synchronising, and the GPU runs them
concurrently, so every flag is raised by a real peer kernel (nothing is
pre-arrived).

Three things keep d ranks' spinning kernels from starving each other on one
GPU: a standing CTA cap (``grid_cap``) so that every rank's pack, span and
barrier kernels fit on the 148 SMs at once; eager module loading
(``CUDA_MODULE_LOADING=EAGER``) — with lazy loading, the first launch of a
kernel that is not loaded yet waits behind a kernel already spinning on the
device (measured, tools/emu_probe.py: a 3 s barrier timeout that disappears
with EAGER); and enough hardware work queues (``CUDA_DEVICE_MAX_CONNECTIONS``
= 32).  Both variables must be set before CUDA initialises, i.e. in the
environment of a fresh process (``child_env()``).  NVLS multicast has no one-GPU stand-in
(a multicast object binds one physical allocation per device), so only the
p2p backend is emulated.  This is a test and profiling harness; production
ranks get ``symm.SymmetricTensor``.
"""

from __future__ import annotations

import os

import torch

from . import _native as nat
from .errors import DeviceError

_SMS = 148


def grid_cap(d: int) -> int:
    """CTAs per launch so that d ranks x (pack + span + barrier kernels) are
    co-resident: the span kernel holds 2 CTAs per SM, so the 296 slots are
    shared three ways per rank."""
    return max(4, (2 * _SMS) // (3 * d))


def child_env(env=None) -> dict:
    """Environment for a process that runs emulated ranks."""
    env = dict(os.environ if env is None else env)
    env.update(CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER")
    return env


def connections_ok() -> bool:
    """True when this process was started with ``child_env()``."""
    return (int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) >= 32
            and os.environ.get("CUDA_MODULE_LOADING", "") == "EAGER")


class EmulatedSymmetric:
    """Stand-in for symm.SymmetricTensor: rank ``rank``'s buffer of one
    symmetric allocation of the row; peers resolve to the other ranks'."""

    mc = 0

    def __init__(self, row: "EmulatedRow", key, rank: int, tensor: torch.Tensor):
        self.row, self.key, self.rank, self.tensor = row, key, rank, tensor
        self.world = row.d

    def peer(self, q: int, byte_offset: int = 0) -> int:
        t = self.row.buffers[self.key][q]
        if t is None:
            raise DeviceError(f"emulated rank {q} has not allocated symmetric buffer {self.key} yet")
        return t.data_ptr() + byte_offset

    def multicast(self, byte_offset: int = 0) -> int:
        raise DeviceError("NVLS multicast has no one-GPU emulation; use backend='p2p'")


class EmulatedRow:
    """The symmetric allocations of a d-rank row, all on ``device``.

    ``factory(rank)`` is the ``symmetric=`` argument of rank ``rank``'s
    DistributedOptimizer; the k-th allocation of every rank forms one
    symmetric buffer (the same order every rank's constructor follows)."""

    def __init__(self, d: int, device=None):
        if d < 1 or d > nat.HOD_P2P_MAX_RANKS:
            raise DeviceError(f"emulated row of {d} ranks (1..{nat.HOD_P2P_MAX_RANKS})")
        self.d = d
        self.device = torch.device(device) if device is not None else torch.device("cuda", 0)
        self.buffers: dict = {}
        self._count = [0] * d

    def factory(self, rank: int):
        def make(numel, dtype, device, zero=False):
            k = self._count[rank]
            self._count[rank] += 1
            t = (torch.zeros if zero else torch.empty)(numel, dtype=dtype, device=self.device)
            slots = self.buffers.setdefault(k, [None] * self.d)
            for other in slots:
                if other is not None and (other.numel() != numel or other.dtype != dtype):
                    raise DeviceError(f"emulated symmetric buffer {k}: ranks disagree on its shape")
            slots[rank] = t
            return EmulatedSymmetric(self, k, rank, t)
        return make

    def streams(self):
        """One 'current' stream per rank: each rank's step is issued inside
        ``torch.cuda.stream(streams[r])`` so no rank waits on another's
        default-stream work."""
        return [torch.cuda.Stream(device=self.device) for _ in range(self.d)]

    def __enter__(self):
        """Standing CTA cap for the ranks' launches (restored on exit)."""
        self._prev = nat.grid_base()
        nat.set_grid_base(grid_cap(self.d))
        return self

    def __exit__(self, *exc):
        nat.set_grid_base(self._prev)
        return False
