"""ctypes binding of the in-tree sm_100a library ``libhod.so`` (include/hod.h).

This is the only door from Python to the device data path.  There is no
fallback: if the library is missing or cannot be loaded the import of any
compute entry point raises, loudly, instead of silently running something
else on the CPU.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import DeviceError

# HOD_LIB: an alternative build of the same library (A/B tuning runs only)
LIB_PATH = Path(os.environ.get("HOD_LIB", Path(__file__).resolve().parent / "libhod.so"))

HOD_PACK_MAX_ENTRIES = 64
HOD_SUMSQ_PARTIALS = 296
HOD_DTYPE_BF16 = 0
HOD_DTYPE_F32 = 1

# every symbol include/hod.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "hod_abi_version", "hod_last_error", "hod_launch_count", "hod_set_grid_limit",
    "hod_pack_bf16", "hod_pack_adamw", "hod_pack_sumsq", "hod_sumsq_bf16", "hod_sum_partials", "hod_clip_coef",
    "hod_adamw_bf16", "hod_adamw_f32", "hod_adamw", "hod_sumsq",
    "hod_nccl_unique_id", "hod_nccl_comm_init", "hod_comm_destroy", "hod_comm_async_error",
    "hod_reduce_scatter_bf16", "hod_all_gather_bf16", "hod_all_reduce_f32",
    "hod_p2p_step", "hod_set_span_tma", "hod_p2p_barrier", "hod_p2p_norm", "hod_p2p_signal", "hod_p2p_wait", "hod_ce_copy",
)


class PackEntry(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("numel", ctypes.c_int64), ("dst_offset", ctypes.c_int64)]


HOD_P2P_MAX_RANKS = 8
HOD_P2P_FUSED, HOD_P2P_RS, HOD_P2P_ADAMW_AG = 0, 1, 2
HOD_P2P_MAX_SPAN = 32
HOD_NORM_TAG = 0x4E4F524D
HOD_ETIMEOUT, HOD_ESPAN = 10003, 10005
ERROR_NAMES = {HOD_ETIMEOUT: "cross-GPU barrier timeout (a peer never arrived)",
               HOD_ESPAN: "span mismatch (peers closed a span over different buckets)"}


def span_tag(first: int, last: int) -> int:
    """HOD_SPAN_TAG(first, last) of include/hod.h."""
    return (first & 0xFFFF) | ((last & 0xFFFF) << 16)


class P2PSpan(ctypes.Structure):
    """Mirror of hod_p2p_span (include/hod.h)."""

    _fields_ = [
        ("grad", ctypes.c_void_p * HOD_P2P_MAX_RANKS),
        ("param", ctypes.c_void_p * HOD_P2P_MAX_RANKS),
        ("flags", ctypes.c_void_p * HOD_P2P_MAX_RANKS),
        ("local_grad", ctypes.c_void_p),
        ("master", ctypes.c_void_p), ("exp_avg", ctypes.c_void_p), ("exp_avg_sq", ctypes.c_void_p),
        ("partials", ctypes.c_void_p), ("clip_coef", ctypes.c_void_p), ("err", ctypes.c_void_p),
        ("bucket_start", ctypes.c_int64 * HOD_P2P_MAX_SPAN),
        ("shard_numel", ctypes.c_int64 * HOD_P2P_MAX_SPAN),
        ("n_buckets", ctypes.c_int), ("d", ctypes.c_int), ("rank", ctypes.c_int), ("nvls", ctypes.c_int),
        ("keep_reduced", ctypes.c_int), ("slot", ctypes.c_int),
        ("epoch", ctypes.c_uint32), ("tag", ctypes.c_uint32), ("timeout_ns", ctypes.c_ulonglong),
    ]


HOD_ADAMW_EXACT, HOD_ADAMW_FAST = 0, 1


class AdamWParams(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double), ("step", ctypes.c_int64),
                ("mode", ctypes.c_int32), ("reserved", ctypes.c_int32)]


ABI_VERSION = 3          # HOD_ABI_VERSION of include/hod.h

_lib = None
_grid_base = 0


def load(build_if_missing: bool = True):
    """Load libhod.so (building it in-tree first if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    import torch  # noqa: F401  (loads the pip libnccl.so.2 our library links to)

    if not LIB_PATH.exists() and build_if_missing:
        from .build_native import build

        build()
    if not LIB_PATH.exists():
        raise DeviceError(f"CUDA library {LIB_PATH} is missing; run "
                          "`python -m paper_2312_03549_b200.build_native`")
    L = ctypes.CDLL(str(LIB_PATH))
    L.hod_abi_version.restype = ctypes.c_int
    if L.hod_abi_version() != ABI_VERSION:
        raise DeviceError(f"{LIB_PATH} has ABI {L.hod_abi_version()}, this package needs {ABI_VERSION}: "
                          "rebuild with `python -m paper_2312_03549_b200.build_native --force`")
    P, I64, I, F = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float
    sig = {
        "hod_abi_version": ([], I),
        "hod_last_error": ([], ctypes.c_char_p),
        "hod_launch_count": ([], ctypes.c_longlong),
        "hod_set_grid_limit": ([I], I),
        "hod_pack_bf16": ([ctypes.POINTER(PackEntry), I, P, I64, F, I, P], I),
        "hod_sumsq_bf16": ([P, I64, P, P], I),
        "hod_pack_adamw": ([ctypes.POINTER(PackEntry), I, I64, F, I, P, P, P, P,
                            ctypes.POINTER(AdamWParams), P, P], I),
        "hod_sum_partials": ([P, I64, P, P], I),
        "hod_pack_sumsq": ([ctypes.POINTER(PackEntry), I, I64, F, I, P, P], I),
        "hod_clip_coef": ([P, F, P, P, P], I),
        "hod_adamw_bf16": ([P, P, P, P, P, I64, ctypes.POINTER(AdamWParams), P, P], I),
        "hod_adamw": ([P, P, P, P, P, I64, F, F, F, F, F, I64, P, P], I),
        "hod_sumsq": ([P, I64, P, P], I),
        "hod_adamw_f32": ([P, P, P, P, P, I64, ctypes.POINTER(AdamWParams), P, P], I),
        "hod_nccl_unique_id": ([P], I),
        "hod_nccl_comm_init": ([P, I, I, ctypes.POINTER(ctypes.c_void_p)], I),
        "hod_comm_destroy": ([P], I),
        "hod_comm_async_error": ([P], I),
        "hod_reduce_scatter_bf16": ([P, P, ctypes.c_size_t, P, P], I),
        "hod_all_gather_bf16": ([P, P, ctypes.c_size_t, P, P], I),
        "hod_all_reduce_f32": ([P, ctypes.c_size_t, P, P], I),
        "hod_p2p_step": ([ctypes.POINTER(P2PSpan), I, ctypes.POINTER(AdamWParams), P], I),
        "hod_set_span_tma": ([I], I),
        "hod_p2p_barrier": ([P, I, I, I, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_ulonglong, P, P], I),
        "hod_p2p_norm": ([P, I64, P, P, I, I, I, ctypes.c_uint32, ctypes.c_ulonglong, P, F, P, P, P, P], I),
        "hod_ce_copy": ([P, P, ctypes.c_size_t, P], I),
        "hod_p2p_signal": ([P, ctypes.c_uint32, P], I),
        "hod_p2p_wait": ([P, ctypes.c_uint32, ctypes.c_ulonglong, P, P], I),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().hod_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed (code {rc}): {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def set_grid_base(max_ctas: int) -> None:
    """Standing CTA cap of every launch of this process (0 = none).  The
    optimizer's temporary ``sm_budget`` caps are taken relative to it and
    restore it afterwards (emulation.EmulatedRow keeps d ranks' kernels
    co-resident on one GPU with it)."""
    global _grid_base
    call("hod_set_grid_limit", int(max_ctas))
    _grid_base = int(max_ctas)


def grid_base() -> int:
    return _grid_base


def launch_count() -> int:
    """Kernels launched by libhod.so so far in this process."""
    return int(load().hod_launch_count())


def stream_ptr(stream) -> int:
    """cudaStream_t handle of a torch.cuda.Stream (0 = legacy default)."""
    return int(stream.cuda_stream) if stream is not None else 0
