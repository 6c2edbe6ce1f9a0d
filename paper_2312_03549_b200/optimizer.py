"""The Overlapped Distributed Optimizer: host side of the B200 data path.

Per bucket b:

    K1 pack/cast(b)  ->  C1 reduce-scatter(b)  ->  [K3 sumsq(b)]
                     ->  K2 AdamW(shard b)     ->  C2 all-gather(b)

K1 runs on a pack stream as soon as bucket b's gradients are ready (either
``grad_ready`` calls from backward hooks, or ``step(grads)``), the
collectives run on a communication stream and the update on an optimizer
stream; CUDA events carry every dependency, the host never synchronises.
With gradient clipping the update of every bucket waits for the global norm
(K3 partials -> C3 all-reduce -> clip coefficient in device memory).

This replaces the reference's *priced* DP synchronisation — reduce-scatter
plus all-gather of the stage's gradient bytes charged after the pipeline
flush (simulator.py:327-333, 445-452) — with the real,
overlapped operation.  The ``backend`` selects how C1/C2 move bytes:

* ``"p2p"`` (``"auto"`` at d = 2, and at any d with clipping) — our fused
  kernels over NVLink peer memory: one kernel per span of consecutive packed
  buckets does the cross-GPU arrival barrier, the reduce-scatter (P2P loads,
  fp32 rank-order sum: deterministic and bit-exact with the oracle), the
  AdamW update and the all-gather (P2P stores); with clipping the RS and the
  AdamW+AG halves run as two kernels around the peer-memory norm exchange.
* ``"nvls"`` (``"auto"`` from d = 4 without clipping) — the same fused kernel
  with NVSwitch in-switch reduction (multimem.ld_reduce) and multicast
  stores (multimem.st).
* ``"nccl"`` — NCCL ReduceScatter / AllGather (bf16, sum) around our K2; the
  library baseline the fused path is measured against.
* ``"none"`` — d == 1: no collective, AdamW reads the packed bucket.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os
from dataclasses import dataclass, field

import torch

from . import _native as nat
from .buckets import BucketLayout, build_bucket_layout
from .comm import DPGroup, NcclComm
from .errors import DeviceError, InfeasibleConfigError

# fused pack+AdamW launches are chained with programmatic dependent launch
# unless HOD_PDL=0 (read by the library too, csrc/hod_kernels.cu)
_PDL = os.environ.get("HOD_PDL", "1") != "0"

_BF16 = torch.bfloat16
BACKENDS = ("none", "nccl", "p2p", "nvls")
_CORESIDENT_CTAS = 148       # one CTA per SM (include/hod.h hod_set_grid_limit)
_SPAN_MAX_BUCKETS = 0xFFFF   # bucket indices fit the 16-bit halves of a span tag


@dataclass
class StepReport:
    """What one ``step`` did.  Device-side values stay on the device until
    ``resolve()`` is called (after the caller synchronises)."""

    step: int
    buckets: int
    params_updated: int           # elements of this rank's shards updated
    grad_norm: torch.Tensor | None = None
    clip_coef: torch.Tensor | None = None
    start: torch.cuda.Event | None = None
    end: torch.cuda.Event | None = None
    err: torch.Tensor | None = None   # device error word of the fused collectives
    resolved: dict = field(default_factory=dict)

    def resolve(self) -> dict:
        """Wait for the step and return its figures; raises DeviceError if a
        cross-GPU barrier of the step timed out or met a mismatched span."""
        if self.end is not None:
            self.end.synchronize()
        if self.err is not None:
            raise_device_error(int(self.err.item()))
        if not self.resolved:
            doc = {"step": self.step, "buckets": self.buckets,
                   "params_updated": self.params_updated}
            if self.start is not None and self.end is not None:
                doc["step_ms"] = self.start.elapsed_time(self.end)
            if self.grad_norm is not None:
                doc["grad_norm"] = float(self.grad_norm.item())
                doc["clip_coef"] = float(self.clip_coef.item())
            self.resolved = doc
        return self.resolved


def raise_device_error(code: int) -> None:
    """DeviceError for a nonzero device error word (include/hod.h HOD_E*)."""
    if code:
        raise DeviceError(f"fused collective failed on the device: code {code} "
                          f"({nat.ERROR_NAMES.get(code, 'unknown')}); the step's update was skipped")


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def shard_pieces(layout: BucketLayout, shard_index: int):
    """Yield (param_index, src_begin, dst_begin, length): which slice of which
    parameter lands where in rank ``shard_index``'s concatenated fp32 shards.
    Padding inside a shard is left untouched (zero)."""
    offs = layout.shard_offsets()
    for b, off in zip(layout.buckets, offs):
        lo, hi = b.shard_range(shard_index, layout.dp)
        for s in b.slots:
            a = b.start + s.offset
            x0, x1 = max(a, lo), min(a + s.numel, hi)
            if x0 < x1:
                yield s.index, x0 - a, off + (x0 - lo), x1 - x0


def fill_master_shards(layout: BucketLayout, init_params, shard_index: int,
                       master: torch.Tensor) -> torch.Tensor:
    """Write the fp32 initial values of this rank's shards into ``master``
    (exact for fp32 inputs).  Works on any device (CPU in the gloo tests)."""
    master.zero_()
    for pi, src0, dst0, n in shard_pieces(layout, shard_index):
        flat = init_params[pi].detach().reshape(-1)
        master[dst0:dst0 + n].copy_(flat[src0:src0 + n].to(master.device).float())
    return master


class DistributedOptimizer:
    """Sharded, bucketed, overlapped AdamW over one DP row.

    Parameters
    ----------
    init_params : list of tensors (registration order) giving the initial
        values; their dtype may be fp32 (exact master init) or bf16.
    dp_group : DPGroup of this rank (``DPGroup.from_plan(plan, rank)`` maps a
        reference GroupPlan DP row); ``None`` means a single rank.
    norm_ranks : ranks over which the clip norm is summed (default: the DP
        row; the whole world for PP x DP so every stage sees one norm).
    grad_scale : multiplier fused into the pack (default 1/d: gradient mean).
    adamw : ``"exact"`` (default: IEEE operations in the oracle's order,
        bit-exact against it) or ``"fast"`` (FMAs + MUFU sqrt/reciprocal,
        ~25 instead of ~90 instructions per element; within the north star's
        1e-6 / 1e-5 tolerance — include/hod.h HOD_ADAMW_FAST).
    symmetric, norm_symmetric : factories ``(numel, dtype, device, zero) ->``
        symmetric buffer (``.tensor``, ``.peer(q)``, ``.multicast()``, ``.mc``,
        ``.rank``, ``.world``) for the DP row / the clip-norm ranks; default:
        torch symmetric memory over the process group (symm.SymmetricTensor).
        ``emulation.EmulatedRow`` supplies one-GPU stand-ins that run the same
        protocol with d ranks on one device.
    """

    def __init__(self, init_params, *, lr: float = 1e-4, betas=(0.9, 0.95), eps: float = 1e-8,
                 weight_decay: float = 0.1, clip: float | None = None,
                 bucket_size: int = 25_000_000, dp_group: DPGroup | None = None,
                 norm_ranks=None, grad_scale: float | None = None, backend: str = "auto",
                 device=None, param_align: int = 64, process_group=None, norm_group=None,
                 keep_reduced: bool = False, barrier_timeout_s: float = 20.0,
                 sm_budget: int | None = None, span_numel: int = 256 * 2**20,
                 param_barriers: bool = True, pre_barrier: bool | None = None,
                 first_span_numel: int | None = None, symmetric=None, norm_symmetric=None,
                 adamw: str = "exact", corun_span_numel: int | None = None):
        if clip is not None and not clip > 0:
            raise InfeasibleConfigError(f"clip must be positive, got {clip}")
        init_params = list(init_params)
        if not init_params:
            raise InfeasibleConfigError("optimizer got an empty parameter list")
        self.device = (torch.device("cuda", torch.cuda.current_device()) if device is None
                       else torch.device(device))
        self.lr, self.betas, self.eps, self.weight_decay = lr, tuple(betas), eps, weight_decay
        self.clip = clip
        if adamw not in ("exact", "fast"):
            raise InfeasibleConfigError(f"adamw must be 'exact' or 'fast', got {adamw!r}")
        self.adamw_mode = adamw
        self.group = dp_group or DPGroup.single(0)
        self.dp = self.group.size
        self.shard_index = self.group.index
        self.grad_scale = (1.0 / self.dp) if grad_scale is None else float(grad_scale)
        auto = backend == "auto"
        if auto:
            # measured choice (tools/p2p_microbench.py, bench.py): P2P
            # loads/stores at d = 2 (NVLS loops the own shard through the switch);
            # NVLS from d = 4 (measured 6.61 vs 6.80 ms/step at d = 4), and at
            # d = 8 it moves 18n instead of 28n bytes per direction per GPU
            # (falls back to p2p when multicast is unavailable)
            # With clipping the RS and the update+AG run as separate phases around
            # the global norm; alone, each NVLS phase is lopsided (RS: 2P out,
            # AG: 2P in per GPU) while p2p moves 2P(d-1)/d each way, so clip -> p2p.
            backend = ("none" if self.dp == 1 else
                       ("nvls" if self.dp >= 4 and clip is None else "p2p"))
        if backend not in BACKENDS:
            raise InfeasibleConfigError(f"unknown backend {backend!r} (choose from {BACKENDS})")
        if (backend == "none") != (self.dp == 1):
            raise InfeasibleConfigError(f"backend {backend!r} does not fit a DP row of {self.dp}")
        if backend in ("p2p", "nvls") and self.dp > nat.HOD_P2P_MAX_RANKS:
            raise InfeasibleConfigError(f"{backend} supports at most {nat.HOD_P2P_MAX_RANKS} ranks")
        self.backend = backend
        self.keep_reduced = keep_reduced
        # CTAs per launch while backward still runs; the last bucket, step()
        # and the post-backward phase always get the whole GPU.  None (auto):
        # 148 = one CTA per SM, the CO-RESIDENT mode of hod_set_grid_limit —
        # each optimizer CTA fits beside a resident cuBLAS GEMM CTA and shares
        # its SM (HBM/NVLink vs tensor cores) instead of time-slicing it
        # (tools/corun_probe.py: 0.55-0.72 of a co-resident update hidden,
        # ~0 with full-GPU grids).  0 = whole GPU; env HOD_SM_BUDGET overrides.
        env = os.environ.get("HOD_SM_BUDGET")
        if env is not None:
            sm_budget = int(env)
        self.sm_budget = _CORESIDENT_CTAS if sm_budget is None else int(sm_budget)
        # p2p/nvls: consecutive packed buckets are coalesced into one fused
        # launch until the span holds >= span_numel elements (1 = per bucket)
        self.span_numel = int(span_numel)
        # the step's first span waits for its packs before any NVLink traffic
        # starts: a smaller first span shortens that lead-in
        env = os.environ.get("HOD_FIRST_SPAN")
        if env is not None:
            first_span_numel = int(env)
        self.first_span_numel = (min(self.span_numel, 32 * 2**20) if first_span_numel is None
                                 else int(first_span_numel))
        # co-resident spans (buckets delivered during backward) close early:
        # a bucket that waits for its span to fill would otherwise run only
        # after backward, at the end of the step, as exposed time
        env = os.environ.get("HOD_CORUN_SPAN")
        self.corun_span_numel = (int(env) if env is not None else
                                 min(self.span_numel, 32 * 2**20) if corun_span_numel is None
                                 else int(corun_span_numel))
        self._spans_launched = 0
        self._whole_step = False
        # p2p/nvls: a params-ready barrier after every span (enables per-bucket
        # wait_params for a forward-overlapped all-gather) instead of a single
        # end-of-step barrier
        self.param_barriers = bool(param_barriers)
        # arrival barrier as a 1-CTA kernel ahead of each RS/fused span launch:
        # the wide kernel then never occupies SMs while a late peer catches up.
        # Measured trade-off (profiles/r01_overlap_prebarrier.jsonl): exposed
        # share of a training iteration drops at d = 2 14.1 -> 12.8 % (1.3B),
        # 11.3 -> 9.7 % (LLaMA-7B clip), at d = 4 10.5 -> 9.4 % and 7.4 ->
        # 6.2 %, but the standalone step pays ~20 us per span (LLaMA-7B
        # d = 4: 34.7 -> 35.4 ms).  Default (None): on for buckets delivered
        # by grad_ready during backward (hooks: backward kernels share the
        # SMs), off inside step() (resident gradients); env HOD_PRE_BARRIER=0/1
        # forces.
        env = os.environ.get("HOD_PRE_BARRIER")
        if env is not None:
            pre_barrier = env == "1"
        self.pre_barrier = pre_barrier
        self._pending_span: list[int] = []
        self.timeout_ns = int(barrier_timeout_s * 1e9)
        nat.load()

        shapes = [tuple(p.shape) for p in init_params]
        numels = [math.prod(s) for s in shapes]
        self.layout: BucketLayout = build_bucket_layout(numels, bucket_size, self.dp, param_align)
        L = self.layout
        total = L.total_numel
        dev = self.device
        nb = len(L.buckets)
        self._sym = None
        if nb > _SPAN_MAX_BUCKETS:
            raise InfeasibleConfigError(f"{nb} buckets: at most {_SPAN_MAX_BUCKETS} (raise bucket_size)")
        self._emulated = symmetric is not None
        if backend in ("p2p", "nvls"):
            if symmetric is None:
                from .symm import SymmetricTensor, group_for

                pg = process_group if process_group is not None else group_for(self.group.ranks)
                self._pg = pg

                def symmetric(numel, dtype, device, zero=False, _pg=pg):
                    return SymmetricTensor(numel, dtype, device, _pg, zero=zero)
            self._symmetric = symmetric
            self._sym_grad = symmetric(total, _BF16, dev, False)
            self._sym_param = symmetric(total, _BF16, dev, True)
            # 64-bit barrier flags (epoch << 32 | tag), slots: [0, nb) span
            # arrival, nb end of step, nb+1+b span b's params ready
            self._sym_flags = symmetric((2 * nb + 1) * nat.HOD_P2P_MAX_RANKS, torch.int64, dev, True)
            if self._sym_grad.rank != self.shard_index:
                raise InfeasibleConfigError("process group order differs from the DP row order")
            if backend == "nvls" and not (self._sym_grad.mc and self._sym_param.mc):
                if not auto:
                    raise InfeasibleConfigError("NVLS multicast unavailable; use backend='p2p'")
                self.backend = backend = "p2p"
            self.param_buffer = self._sym_param.tensor
            self.grad_buffer = self._sym_grad.tensor
            self._norm_group = norm_group
        else:
            self.param_buffer = torch.zeros(total, dtype=_BF16, device=dev)
            self.grad_buffer = torch.empty(total, dtype=_BF16, device=dev)
        # device error word of the fused collectives (HOD_ETIMEOUT / HOD_ESPAN),
        # read back asynchronously after every step into pinned memory and
        # checked at the next begin_step without a host synchronisation
        self._err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._err_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._ev_err = torch.cuda.Event()
        self._err_pending = False
        shard_total = total // self.dp
        self.master = torch.empty(shard_total, dtype=torch.float32, device=dev)
        self.exp_avg = torch.zeros(shard_total, dtype=torch.float32, device=dev)
        self.exp_avg_sq = torch.zeros(shard_total, dtype=torch.float32, device=dev)
        self._shard_off = L.shard_offsets()

        # model-visible bf16 params are views into the flat buffer
        self.params: list[torch.Tensor] = [None] * len(shapes)  # type: ignore[list-item]
        for b in L.buckets:
            for s in b.slots:
                lo = b.start + s.offset
                view = self.param_buffer[lo:lo + s.numel].view(shapes[s.index])
                view.copy_(init_params[s.index].detach().to(dev).to(_BF16))
                self.params[s.index] = view
        fill_master_shards(L, init_params, self.shard_index, self.master)

        # streams / events (one set per bucket, reused every step)
        # high-priority streams: when an SM frees up between backward GEMM
        # tiles, the optimizer's CTAs are dispatched first
        hi = torch.cuda.Stream.priority_range()[1] if hasattr(torch.cuda.Stream, "priority_range") else -1
        self.s_pack = torch.cuda.Stream(device=dev, priority=hi)
        # HOD_COMM_PRIORITY_DROP (tuning): the collective stream this many
        # levels below the pack stream
        comm_prio = hi + int(os.environ.get("HOD_COMM_PRIORITY_DROP", "0"))
        self.s_comm = torch.cuda.Stream(device=dev, priority=comm_prio) if self.dp > 1 else self.s_pack
        self.s_opt = torch.cuda.Stream(device=dev, priority=hi) if self.dp > 1 else self.s_pack
        nb = len(L.buckets)
        self._ev_packed = [torch.cuda.Event() for _ in range(nb)]
        self._ev_reduced = [torch.cuda.Event() for _ in range(nb)]
        self._ev_updated = [torch.cuda.Event() for _ in range(nb)]
        self._ev_params = [torch.cuda.Event() for _ in range(nb)]
        self._ev_norm = torch.cuda.Event()
        self._ev_start = torch.cuda.Event(enable_timing=True)
        self._ev_end = torch.cuda.Event(enable_timing=True)

        if self.clip is not None:
            self._partials = torch.zeros(nb * nat.HOD_SUMSQ_PARTIALS, dtype=torch.float32, device=dev)
            self._sumsq = torch.zeros(1, dtype=torch.float32, device=dev)
            self._coef = torch.ones(1, dtype=torch.float32, device=dev)
            self._norm = torch.zeros(1, dtype=torch.float32, device=dev)

        # communicators
        self.comm = None
        self.norm_comm = None
        if self.backend == "nccl":
            self.comm = NcclComm(self.group.ranks, self.group.global_rank, "dp")
        norm_ranks = tuple(norm_ranks) if norm_ranks is not None else self.group.ranks
        self.norm_ranks = norm_ranks
        if self.clip is not None and len(norm_ranks) > 1:
            if self.backend in ("p2p", "nvls"):
                if norm_ranks == self.group.ranks:
                    nsym = self._symmetric
                elif norm_symmetric is not None:
                    nsym = norm_symmetric
                else:
                    from .symm import SymmetricTensor, group_for

                    ng = self._norm_group if self._norm_group is not None else group_for(norm_ranks)

                    def nsym(numel, dtype, device, zero=False, _ng=ng):
                        return SymmetricTensor(numel, dtype, device, _ng, zero=zero)
                self._norm_xchg = nsym(nat.HOD_P2P_MAX_RANKS, torch.float64, dev, True)
                self._norm_flags = nsym(nat.HOD_P2P_MAX_RANKS, torch.int64, dev, True)
                self._norm_rank = self._norm_xchg.rank
                self._norm_d = self._norm_xchg.world
            else:
                self.norm_comm = (self.comm if norm_ranks == self.group.ranks and self.comm is not None
                                  else NcclComm(norm_ranks, self.group.global_rank, "norm"))
        if self.backend in ("p2p", "nvls"):
            torch.cuda.synchronize(dev)
            if not self._emulated:
                import torch.distributed as dist

                dist.barrier()  # every rank's zeroed flags exist before anyone signals

        self._ktiming = None
        self._krun = None                # open run of PDL-chained launches (timing)
        self._grads_resident = False
        self._staging = None
        self._ev_staging_free = None
        self.step_count = 0              # AdamW bias-correction step (restored by checkpoint.load)
        self._epoch = 0                  # barrier epoch: monotonic, never restored
        self._pending_grads: list[dict[int, torch.Tensor]] = []
        self._launched: list[bool] = []
        self._deferred_ag: list[int] = []
        self._in_step = False
        self._finish_wait = True
        self._corun_active = False
        self._ev_span_end = torch.cuda.Event()
        self._sync_enabled = True

    # ------------------------------------------------------------------ API
    def bucket_layout(self) -> BucketLayout:
        return self.layout

    def begin_step(self) -> None:
        if self._in_step:
            raise InfeasibleConfigError("begin_step called twice without finish_step")
        self.poll_error()
        self._in_step = True
        self.step_count += 1
        self._epoch += 1
        nb = len(self.layout.buckets)
        self._pending_grads = [dict() for _ in range(nb)]
        self._launched = [False] * nb
        self._deferred_ag = []
        self._pending_span = []
        self._spans_launched = 0
        self._deferred_pa = []
        self._ev_start.record(torch.cuda.current_stream(self.device))
        if self.dp > 1 and self._epoch > 1:
            # this step's packs overwrite the grad buckets the previous step's
            # reduce-scatter read (peers included): order them after its
            # params-ready points even if the caller skipped wait_params
            for ev in self._ev_params:
                self.s_pack.wait_event(ev)
        if self.clip is not None and self.backend in ("p2p", "nvls"):
            # span starts (hence the partial slots written) may differ between steps
            with torch.cuda.stream(self.s_comm):
                self._partials.zero_()

    def grad_ready(self, param_index: int, grad: torch.Tensor) -> None:
        """Backward produced ``grad`` for parameter ``param_index`` (call from a
        post-accumulate-grad hook).  Launches the bucket once it is complete.

        Each parameter is delivered once per step, between ``begin_step`` and
        ``finish_step``: a second delivery (gradient accumulation without
        ``no_sync``, a backward outside the step) would relaunch its bucket
        against barrier slots its peers already passed, so it raises."""
        if not self._in_step:
            raise InfeasibleConfigError(
                f"grad_ready({param_index}) outside begin_step/finish_step (wrap accumulation "
                "micro-batches in no_sync())")
        slot = self.layout.slot(param_index)
        if self._launched[slot.bucket]:
            raise InfeasibleConfigError(
                f"gradient of param {param_index} delivered again after bucket {slot.bucket} was launched")
        pend = self._pending_grads[slot.bucket]
        if param_index in pend:
            raise InfeasibleConfigError(f"gradient of param {param_index} delivered twice in one step")
        pend[param_index] = grad
        b = self.layout.buckets[slot.bucket]
        if len(pend) == len(b.slots):
            self._launch_bucket(slot.bucket)

    def finish_step(self, wait: bool = True) -> StepReport:
        """Launch whatever is left, run the clip barrier if needed, and return.

        ``wait=False`` leaves the current stream free: the next forward then
        calls ``wait_params(b)`` before it touches bucket b (p2p/nvls buckets
        become ready span by span — in reverse bucket order after a clip norm,
        i.e. first-layer parameters first), overlapping the all-gather with
        the next forward."""
        L = self.layout
        for b in range(len(L.buckets)):
            if not self._launched[b]:
                missing = [s.index for s in L.buckets[b].slots if s.index not in self._pending_grads[b]]
                raise InfeasibleConfigError(f"bucket {b} is missing gradients for params {missing[:8]}")
        self._finish_wait = wait
        if self.backend in ("p2p", "nvls"):
            self._p2p_finish()
        elif self._deferred_pa:
            self._norm_then_pack_adamw()
        elif self.clip is not None:
            self._clip_and_update()
        else:
            self._flush_deferred_ag()
        self._close_run()
        cur = torch.cuda.current_stream(self.device)
        if wait:
            for ev in self._ev_params:
                cur.wait_event(ev)
            self._ev_end.record(cur)
        else:
            self._ev_end.record(self.s_comm if self.backend in ("p2p", "nvls") else self.s_opt)
        self._in_step = False
        if self.backend in ("p2p", "nvls"):
            # asynchronous read-back of the error word (checked at the next
            # begin_step once it has landed; StepReport.resolve checks it too)
            s = self.s_comm
            with torch.cuda.stream(s):
                self._err_host.copy_(self._err, non_blocking=True)
            self._ev_err.record(s)
            self._err_pending = True
        rep = StepReport(self.step_count, len(L.buckets), L.total_numel // self.dp,
                         start=self._ev_start, end=self._ev_end,
                         err=self._err if self.backend in ("p2p", "nvls") else None)
        if self.clip is not None:
            rep.grad_norm, rep.clip_coef = self._norm, self._coef
        return rep

    def step(self, grads) -> StepReport:
        """One optimizer step over ``grads`` (registration order), issued in
        backward order as if every gradient had just become ready."""
        host = grads[0].device.type == "cpu"
        if host:
            self._ensure_staging(grads)
            # the staging buffers are reused: this step's uploads must not
            # overwrite them before the previous step's packs have read them
            if self._ev_staging_free is not None:
                self.s_h2d.wait_event(self._ev_staging_free)
        self.begin_step()
        if not host:
            # every gradient is already complete on the current stream: one
            # wait here instead of one per bucket keeps the pack stream a pure
            # chain of kernels (programmatic dependent launch can then overlap
            # bucket k+1's ramp with bucket k's tail)
            self.s_pack.wait_stream(torch.cuda.current_stream(self.device))
            self._grads_resident = True
        # step() returns with every bucket's params gathered (finish_step waits
        # for all of them), so per-span params-ready barriers buy nothing
        # here: one end-of-step barrier instead (measured d = 4: -0.06 ms)
        self._whole_step = True
        try:
            self._step_buckets(grads, host)
            rep = self.finish_step()
        finally:
            self._grads_resident = False
            self._whole_step = False
        if host:
            # every read of the staging buffers (packs, fused pack+AdamW, the
            # post-norm pass at d = 1) runs on s_pack and is enqueued by now
            if self._ev_staging_free is None:
                self._ev_staging_free = torch.cuda.Event()
            self._ev_staging_free.record(self.s_pack)
        return rep

    def _step_buckets(self, grads, host: bool) -> None:
        for b in self.layout.buckets:
            if host:
                # host->device copy of this bucket's gradients on the copy
                # engine; the pack of bucket b waits only for its own copy
                with torch.cuda.stream(self.s_h2d):
                    for s in b.slots:
                        self._staging[s.index].copy_(grads[s.index], non_blocking=True)
                self._ev_h2d[b.index].record(self.s_h2d)
                self.s_pack.wait_event(self._ev_h2d[b.index])
            for s in b.slots:
                self.grad_ready(s.index, self._staging[s.index] if host else grads[s.index])

    def _ensure_staging(self, grads) -> None:
        if (self._staging is not None and self._staging[0].dtype == grads[0].dtype):
            return
        self._staging = [torch.empty(g.shape, dtype=g.dtype, device=self.device) for g in grads]
        self.s_h2d = torch.cuda.Stream(device=self.device)
        self._ev_h2d = [torch.cuda.Event() for _ in self.layout.buckets]

    def gather_params(self) -> None:
        """All-gather every bucket's bf16 param shard from its owner into
        every rank's param buffer (after ``checkpoint.load`` restored only the
        local shards).  p2p/nvls: copy-engine stores of the own shard into each
        peer's buffer, then an end-of-step barrier; nccl: AllGather per
        bucket.  Stream-ordered, no host synchronisation; every rank calls it."""
        if self._in_step:
            raise InfeasibleConfigError("gather_params inside a step")
        cur = torch.cuda.current_stream(self.device)
        s = self.s_comm
        s.wait_stream(cur)
        L = self.layout
        if self.backend == "nccl":
            for b in L.buckets:
                lo, hi = b.shard_range(self.shard_index, self.dp)
                self.comm.all_gather_bf16(_ptr(self.param_buffer) + 2 * lo, _ptr(self.param_buffer) + 2 * b.start,
                                          hi - lo, s)
        elif self.backend in ("p2p", "nvls"):
            for b in L.buckets:
                lo, hi = b.shard_range(self.shard_index, self.dp)
                for q in range(self.dp):
                    if q != self.shard_index:
                        nat.call("hod_ce_copy", self._sym_param.peer(q, 2 * lo), _ptr(self.param_buffer) + 2 * lo,
                                 2 * (hi - lo), nat.stream_ptr(s))
            self._epoch += 1
            nb = len(L.buckets)
            nat.call("hod_p2p_barrier", self._flag_ptrs(self._sym_flags), self.dp, self.shard_index, nb,
                     self._epoch, nb, self.timeout_ns, _ptr(self._err), nat.stream_ptr(s))
        for ev in self._ev_params:
            ev.record(s)
        cur.wait_stream(s)

    def wait_params(self, bucket: int, stream=None) -> None:
        """Make ``stream`` (default: current) wait until bucket's params are gathered."""
        (stream or torch.cuda.current_stream(self.device)).wait_event(self._ev_params[bucket])

    def register_hooks(self, module_params) -> list:
        """Attach post-accumulate-grad hooks: parameter i's gradient feeds
        ``grad_ready(i)``.  ``module_params[i]`` must be the model parameter
        for registration index i.  Backward passes of accumulation
        micro-batches run under ``no_sync()`` (the hooks stay silent and the
        gradients accumulate in ``p.grad``); the last micro-batch's backward,
        inside ``begin_step``/``finish_step``, delivers the sums."""
        handles = []
        for i, p in enumerate(module_params):
            def hook(param, i=i):
                if self._sync_enabled:
                    self.grad_ready(i, param.grad)
            handles.append(p.register_post_accumulate_grad_hook(hook))
        return handles

    def attach(self, model) -> list:
        """Bind ``model`` (an nn.Module whose ``parameters()`` are, in order,
        the optimizer's registration order) to the flat buffers:

        * every parameter's storage becomes its view of the bf16 param buffer
          (the forward reads what the all-gather wrote);
        * post-accumulate-grad hooks deliver gradients (``register_hooks``):
          buckets launch during backward, in backward order;
        * a forward pre-hook on every submodule that owns parameters waits
          for their buckets (``wait_params``): after ``finish_step(wait=False)``
          the all-gather of the last spans overlaps the next forward.

        This is the integration point of the imported overlapped optimizer
        (Megatron-LLaMA) that the reference prices as
        non-overlapped.  Returns the hook handles."""
        params = list(model.parameters())
        if len(params) != len(self.params):
            raise InfeasibleConfigError(f"model has {len(params)} parameters, optimizer {len(self.params)}")
        index = {}
        for i, (p, view) in enumerate(zip(params, self.params)):
            if tuple(p.shape) != tuple(view.shape):
                raise InfeasibleConfigError(f"parameter {i}: shape {tuple(p.shape)} vs {tuple(view.shape)}")
            p.data = view
            index[id(p)] = i
        handles = self.register_hooks(params)
        for mod in model.modules():
            own = [index[id(p)] for p in mod.parameters(recurse=False) if id(p) in index]
            if not own:
                continue
            buckets = sorted({self.layout.slot(i).bucket for i in own})

            def pre(_mod, _inp, buckets=buckets):
                for b in buckets:
                    self.wait_params(b)
            handles.append(mod.register_forward_pre_hook(pre))
        return handles

    def no_sync(self):
        """Context manager: hooks registered by ``register_hooks`` do not
        deliver gradients inside it (gradient-accumulation micro-batches)."""

        @contextlib.contextmanager
        def ctx():
            prev, self._sync_enabled = self._sync_enabled, False
            try:
                yield
            finally:
                self._sync_enabled = prev
        return ctx()

    def poll_error(self) -> None:
        """Raise DeviceError if an earlier step's read-back error word is
        nonzero, or if a NCCL communicator holds an asynchronous error.
        Never blocks: a read-back still in flight is checked later."""
        for c in (self.comm, self.norm_comm):
            if c is not None:
                c.check()
        if self._err_pending and self._ev_err.query():
            self._err_pending = False
            raise_device_error(int(self._err_host[0]))

    def close(self) -> None:
        for c in {id(x): x for x in (self.comm, self.norm_comm) if x is not None}.values():
            c.close()
        self.comm = self.norm_comm = None

    # ------------------------------------------------------------ internals
    def _hp(self) -> nat.AdamWParams:
        return nat.AdamWParams(self.lr, self.betas[0], self.betas[1], self.eps, self.weight_decay,
                               self.step_count,
                               nat.HOD_ADAMW_FAST if self.adamw_mode == "fast" else nat.HOD_ADAMW_EXACT)

    def _grad_shard(self, b) -> tuple[int, int]:
        """(ptr, numel) of this rank's reduced-gradient shard of bucket b."""
        lo, hi = b.shard_range(self.shard_index, self.dp)
        return _ptr(self.grad_buffer) + 2 * lo, hi - lo

    def _coresident(self, on: bool):
        """Context: launches inside it use the co-resident grid (sm_budget)
        when ``on`` — they share the SMs with the caller's GEMMs."""

        @contextlib.contextmanager
        def ctx():
            if not on or not self.sm_budget:
                yield
                return
            base = nat.grid_base()
            nat.call("hod_set_grid_limit", min(int(self.sm_budget), base) if base else int(self.sm_budget))
            self._corun_active = True
            try:
                yield
            finally:
                self._corun_active = False
                nat.call("hod_set_grid_limit", base)
        return ctx()

    def _launch_bucket(self, bi: int) -> None:
        last = sum(self._launched) == len(self._launched) - 1
        # step(): no backward to share the SMs with; the last bucket finds
        # backward (nearly) done
        with self._coresident(not last and not self._whole_step):
            self._launch_bucket_body(bi)

    def _launch_bucket_body(self, bi: int) -> None:
        b = self.layout.buckets[bi]
        grads = self._pending_grads[bi]
        cur = torch.cuda.current_stream(self.device)
        if not self._grads_resident:
            self.s_pack.wait_stream(cur)
        # keep gradient memory alive until the pack has consumed it
        for s in b.slots:
            g = grads[s.index]
            if g.numel() != s.numel:
                raise InfeasibleConfigError(
                    f"gradient for param {s.index} has {g.numel()} elements, expected {s.numel}")
            g.record_stream(self.s_pack)
        first = grads[b.slots[0].index]
        if first.dtype == torch.float32:
            dtype = nat.HOD_DTYPE_F32
        elif first.dtype == _BF16:
            dtype = nat.HOD_DTYPE_BF16
        else:
            raise InfeasibleConfigError(f"gradient dtype {first.dtype} not supported (bf16/fp32)")
        entries = (nat.PackEntry * len(b.slots))()
        for k, s in enumerate(b.slots):
            g = grads[s.index]
            if not g.is_contiguous() or g.dtype != first.dtype:
                raise InfeasibleConfigError(f"gradient {s.index} must be contiguous {first.dtype}")
            entries[k].src = _ptr(g)
            entries[k].numel = s.numel
            entries[k].dst_offset = s.offset
        bucket_ptr = _ptr(self.grad_buffer) + 2 * b.start
        src_bytes = 4 if dtype == nat.HOD_DTYPE_F32 else 2
        if self.backend == "none" and not self.keep_reduced:
            # d == 1: nothing to exchange, so K1 and K2 fuse (no bucket round
            # trip).  With clipping the norm needs every bucket first: a
            # 2 B/element norm pass now, the fused update after the norm.
            self._launched[bi] = True
            if self.clip is None:
                self._pack_adamw(bi, entries, dtype, None)
                return
            part = _ptr(self._partials) + 4 * nat.HOD_SUMSQ_PARTIALS * bi
            t0 = self._timed_event(self.s_pack, run="pack_sumsq" if self._grads_resident else None)
            nat.call("hod_pack_sumsq", entries, len(b.slots), b.numel, ctypes.c_float(self.grad_scale),
                     dtype, part, nat.stream_ptr(self.s_pack))
            self._timed_close("pack_sumsq", t0, self.s_pack, src_bytes * b.numel)
            self._deferred_pa.append((bi, entries, dtype))
            return
        chained = self._grads_resident   # back-to-back launches: timed as one PDL run
        t0 = self._timed_event(self.s_pack, run="pack" if chained else None)
        nat.call("hod_pack_bf16", entries, len(b.slots), bucket_ptr, b.numel,
                 ctypes.c_float(self.grad_scale), dtype, nat.stream_ptr(self.s_pack))
        self._timed_close("pack", t0, self.s_pack, (src_bytes + 2) * b.numel)
        self._ev_packed[bi].record(self.s_pack)
        self._launched[bi] = True

        if self.backend in ("p2p", "nvls"):
            self._queue_p2p(bi)
            return

        reduced = self._ev_packed[bi]
        if self.backend == "nccl":
            self.s_comm.wait_event(self._ev_packed[bi])
            shard_ptr, shard_n = self._grad_shard(b)
            self.comm.reduce_scatter_bf16(bucket_ptr, shard_ptr, shard_n, self.s_comm)
            self._ev_reduced[bi].record(self.s_comm)
            reduced = self._ev_reduced[bi]

        if self.clip is not None:
            shard_ptr, shard_n = self._grad_shard(b)
            part = _ptr(self._partials) + 4 * nat.HOD_SUMSQ_PARTIALS * bi
            nat.call("hod_sumsq_bf16", shard_ptr, shard_n, part, nat.stream_ptr(self.s_comm))
        else:
            self._update_bucket(bi, reduced, clip_coef_ptr=None)
            # all-gather of the previous bucket goes behind this RS (pipelining)
            self._flush_deferred_ag(keep_last=True)

    def _pack_adamw(self, bi: int, entries, dtype, coef_ptr, chained: bool | None = None) -> None:
        """Fused pack+AdamW of bucket bi (d == 1).  ``chained``: launched back to
        back with other bucket kernels (a PDL chain, timed as one run)."""
        b = self.layout.buckets[bi]
        off = self._shard_off[bi]
        hp = self._hp()
        src_bytes = 4 if dtype == nat.HOD_DTYPE_F32 else 2
        chained = self._grads_resident if chained is None else chained
        t0 = self._timed_event(self.s_pack, run="pack_adamw" if chained else None)
        nat.call("hod_pack_adamw", entries, len(entries), b.numel, ctypes.c_float(self.grad_scale),
                 dtype, _ptr(self.master) + 4 * off, _ptr(self.exp_avg) + 4 * off,
                 _ptr(self.exp_avg_sq) + 4 * off, _ptr(self.param_buffer) + 2 * b.start,
                 ctypes.byref(hp), coef_ptr, nat.stream_ptr(self.s_pack))
        self._timed_close("pack_adamw", t0, self.s_pack, (src_bytes + 26) * b.numel)
        self._ev_params[bi].record(self.s_pack)

    def _update_bucket(self, bi: int, ready: torch.cuda.Event, clip_coef_ptr) -> None:
        b = self.layout.buckets[bi]
        self.s_opt.wait_event(ready)
        shard_ptr, shard_n = self._grad_shard(b)
        lo, _ = b.shard_range(self.shard_index, self.dp)
        off = self._shard_off[bi]
        hp = self._hp()
        t0 = self._timed_event(self.s_opt)
        nat.call("hod_adamw_bf16", _ptr(self.master) + 4 * off, _ptr(self.exp_avg) + 4 * off,
                 _ptr(self.exp_avg_sq) + 4 * off, shard_ptr, _ptr(self.param_buffer) + 2 * lo,
                 shard_n, ctypes.byref(hp), clip_coef_ptr, nat.stream_ptr(self.s_opt))
        self._timed_close("adamw", t0, self.s_opt, 28 * shard_n)
        self._ev_updated[bi].record(self.s_opt)
        if self.backend == "nccl":
            self._deferred_ag.append(bi)
        else:
            self._ev_params[bi].record(self.s_opt)

    def _issue_ag(self, bi: int) -> None:
        b = self.layout.buckets[bi]
        self.s_comm.wait_event(self._ev_updated[bi])
        lo, hi = b.shard_range(self.shard_index, self.dp)
        self.comm.all_gather_bf16(_ptr(self.param_buffer) + 2 * lo, _ptr(self.param_buffer) + 2 * b.start,
                                  hi - lo, self.s_comm)
        self._ev_params[bi].record(self.s_comm)

    def _flush_deferred_ag(self, keep_last: bool = False) -> None:
        while len(self._deferred_ag) > (1 if keep_last else 0):
            self._issue_ag(self._deferred_ag.pop(0))

    # ------------------------------------------------- fused peer-memory path
    def _flag_ptrs(self, sym) -> ctypes.Array:
        arr = (ctypes.c_void_p * sym.world)()
        for q in range(sym.world):
            arr[q] = sym.peer(q)
        return arr

    def _p2p(self, bis, mode: int, partials=None, coef_ptr=None) -> None:
        """One fused launch over the consecutive buckets ``bis`` (a span)."""
        L = self.layout
        d = self.dp
        sp = nat.P2PSpan()
        if self.backend == "nvls":
            sp.grad[0] = self._sym_grad.multicast()
            sp.param[0] = self._sym_param.multicast()
        else:
            for q in range(d):
                sp.grad[q] = self._sym_grad.peer(q)
                sp.param[q] = self._sym_param.peer(q)
        for q in range(d):
            sp.flags[q] = self._sym_flags.peer(q)
        off = self._shard_off[bis[0]]
        sp.local_grad = _ptr(self.grad_buffer)
        sp.master = _ptr(self.master) + 4 * off
        sp.exp_avg = _ptr(self.exp_avg) + 4 * off
        sp.exp_avg_sq = _ptr(self.exp_avg_sq) + 4 * off
        sp.partials = partials
        sp.clip_coef = coef_ptr
        sp.err = _ptr(self._err)
        n_total = 0
        for k, bi in enumerate(bis):
            b = L.buckets[bi]
            sp.bucket_start[k] = b.start
            sp.shard_numel[k] = b.numel // d
            n_total += b.numel // d
        sp.n_buckets = len(bis)
        sp.d, sp.rank, sp.nvls = d, self.shard_index, int(self.backend == "nvls")
        sp.keep_reduced = int(self.keep_reduced)
        sp.slot, sp.epoch, sp.timeout_ns = bis[0], self._epoch, self.timeout_ns
        sp.tag = nat.span_tag(bis[0], bis[-1])
        hp = self._hp()
        name = {nat.HOD_P2P_FUSED: "fused", nat.HOD_P2P_RS: "rs", nat.HOD_P2P_ADAMW_AG: "adamw_ag"}[mode]
        # algorithmic bytes per launch: local HBM (state 24 B + own param 2 B +
        # own grad 2 B per owned element) — NVLink bytes are reported separately
        nbytes = {"fused": 28 * n_total, "rs": 2 * d * n_total + 2 * n_total, "adamw_ag": 28 * n_total}[name]
        pre = (not self._whole_step) if self.pre_barrier is None else self.pre_barrier
        if pre and mode != nat.HOD_P2P_ADAMW_AG:
            nat.call("hod_p2p_barrier", self._flag_ptrs(self._sym_flags), d, self.shard_index, sp.slot,
                     sp.epoch, sp.tag, self.timeout_ns, _ptr(self._err), nat.stream_ptr(self.s_comm))
        t0 = self._timed_event(self.s_comm)
        nat.call("hod_p2p_step", ctypes.byref(sp), mode, ctypes.byref(hp), nat.stream_ptr(self.s_comm))
        self._timed_close(name, t0, self.s_comm, nbytes)

    def _spans(self, bis):
        """Split consecutive bucket ids into spans of >= span_numel elements
        (at most HOD_P2P_MAX_SPAN buckets each)."""
        out, cur, acc = [], [], 0
        for bi in bis:
            cur.append(bi)
            acc += self.layout.buckets[bi].numel
            if acc >= self.span_numel or len(cur) == nat.HOD_P2P_MAX_SPAN:
                out.append(cur)
                cur, acc = [], 0
        if cur:
            out.append(cur)
        return out

    def _queue_p2p(self, bi: int, final: bool = False) -> None:
        """Bucket bi is packed: extend the pending span, launch it when full."""
        if bi is not None:
            if self._pending_span and bi != self._pending_span[-1] + 1:
                # spans must be consecutive buckets (their state is contiguous)
                self._queue_p2p(None, final=True)
            self._pending_span.append(bi)
        pend = self._pending_span
        target = (self.first_span_numel if self._spans_launched == 0 else
                  self.corun_span_numel if self._corun_active else self.span_numel)
        full = (sum(self.layout.buckets[x].numel for x in pend) >= target
                or len(pend) == nat.HOD_P2P_MAX_SPAN)
        if pend and (full or final):
            self._pending_span = []
            self._spans_launched += 1
            # the pack stream is in order: the span's last pack implies the others
            self.s_comm.wait_event(self._ev_packed[pend[-1]])
            if self.clip is None:
                self._p2p(pend, nat.HOD_P2P_FUSED)
                self._span_done(pend)
            else:
                part = _ptr(self._partials) + 4 * nat.HOD_SUMSQ_PARTIALS * pend[0]
                self._p2p(pend, nat.HOD_P2P_RS, partials=part)
            if self._corun_active:
                # co-resident: the next pack starts after this span, so at most
                # one optimizer CTA sits on an SM — a pack CTA beside a span CTA
                # would leave too few registers for a GEMM CTA (22.5 K free)
                self._ev_span_end.record(self.s_comm)
                self.s_pack.wait_event(self._ev_span_end)

    def _p2p_finish(self) -> None:
        nb = len(self.layout.buckets)
        s = self.s_comm
        if self.clip is not None:
            self._queue_p2p(None, final=True)
            if len(self.norm_ranks) == 1:
                nat.call("hod_sum_partials", _ptr(self._partials), nb * nat.HOD_SUMSQ_PARTIALS,
                         _ptr(self._sumsq), nat.stream_ptr(s))
                nat.call("hod_clip_coef", _ptr(self._sumsq), ctypes.c_float(self.clip),
                         _ptr(self._coef), _ptr(self._norm), nat.stream_ptr(s))
            else:
                xchg = self._flag_ptrs(self._norm_xchg)
                flags = self._flag_ptrs(self._norm_flags)
                nat.call("hod_p2p_norm", _ptr(self._partials), nb * nat.HOD_SUMSQ_PARTIALS, xchg, flags,
                         self._norm_d, self._norm_rank, 0, self._epoch, self.timeout_ns,
                         _ptr(self._err), ctypes.c_float(self.clip), _ptr(self._coef), _ptr(self._norm),
                         _ptr(self._sumsq), nat.stream_ptr(s))
            # reverse bucket order: the last bucket holds the first layers, which
            # the next forward needs first.  With finish_step(wait=False) the
            # forward runs concurrently: the first span gets the whole GPU (the
            # forward waits for it), the others run co-resident beside the
            # forward GEMMs
            for k, span in enumerate(reversed(self._spans(range(nb)))):
                with self._coresident(k > 0 and not self._finish_wait and not self._whole_step):
                    self._p2p(span, nat.HOD_P2P_ADAMW_AG, coef_ptr=_ptr(self._coef))
                self._span_done(span)
        else:
            self._queue_p2p(None, final=True)
        if not self.param_barriers or self._whole_step:
            # end-of-step barrier: every rank's param stores (and reads of our
            # buckets) are complete before anyone uses the params or repacks
            nat.call("hod_p2p_barrier", self._flag_ptrs(self._sym_flags), self.dp, self.shard_index, nb,
                     self._epoch, nb, self.timeout_ns, _ptr(self._err), nat.stream_ptr(s))
            for ev in self._ev_params:
                ev.record(s)

    def _span_done(self, span) -> None:
        """Per-span params-ready barrier: once every rank passed it, all peers'
        stores into this span's param buckets (and all reads of our grad
        buckets) are complete, so the span's params may be used / repacked."""
        if not self.param_barriers or self._whole_step:
            return
        nb = len(self.layout.buckets)
        nat.call("hod_p2p_barrier", self._flag_ptrs(self._sym_flags), self.dp, self.shard_index,
                 nb + 1 + span[0], self._epoch, nat.span_tag(span[0], span[-1]), self.timeout_ns,
                 _ptr(self._err), nat.stream_ptr(self.s_comm))
        for b in span:
            self._ev_params[b].record(self.s_comm)

    def check_health(self) -> None:
        """Raise DeviceError if a cross-GPU barrier timed out or met a
        mismatched span, or NCCL reported an asynchronous error (synchronises)."""
        for c in (self.comm, self.norm_comm):
            if c is not None:
                c.check()
        raise_device_error(int(self._err.item()))

    def _norm_then_pack_adamw(self) -> None:
        """d == 1 with clipping: every bucket's norm partials exist; finish the
        norm on the pack stream and run the fused pack+AdamW per bucket."""
        nb = len(self.layout.buckets)
        s = self.s_pack
        nat.call("hod_sum_partials", _ptr(self._partials), nb * nat.HOD_SUMSQ_PARTIALS,
                 _ptr(self._sumsq), nat.stream_ptr(s))
        nat.call("hod_clip_coef", _ptr(self._sumsq), ctypes.c_float(self.clip), _ptr(self._coef),
                 _ptr(self._norm), nat.stream_ptr(s))
        # one launch per bucket, chained by programmatic dependent launch, in
        # DESCENDING bucket order so the first layers' parameters (last bucket)
        # are ready first for the next forward.  (Merging consecutive buckets
        # into one launch measured slower: 6.37 vs 6.55 TB/s on LLaMA-7B — a
        # grid striding over a ~37 GB range loses DRAM locality.)
        coef = _ptr(self._coef)
        # with finish_step(wait=False) the next forward runs concurrently: the
        # first update gets the whole GPU (the forward waits for it), the rest
        # run co-resident beside the forward GEMMs (as the p2p post-norm spans)
        for k, (bi, entries, dtype) in enumerate(sorted(self._deferred_pa, key=lambda t: t[0], reverse=True)):
            with self._coresident(k > 0 and not self._finish_wait and not self._whole_step):
                self._pack_adamw(bi, entries, dtype, coef, chained=True)
        self._deferred_pa = []

    def _clip_and_update(self) -> None:
        nb = len(self.layout.buckets)
        s = self.s_comm
        nat.call("hod_sum_partials", _ptr(self._partials), nb * nat.HOD_SUMSQ_PARTIALS,
                 _ptr(self._sumsq), nat.stream_ptr(s))
        if self.norm_comm is not None:
            self.norm_comm.all_reduce_f32(_ptr(self._sumsq), 1, s)
        nat.call("hod_clip_coef", _ptr(self._sumsq), ctypes.c_float(self.clip), _ptr(self._coef),
                 _ptr(self._norm), nat.stream_ptr(s))
        self._ev_norm.record(s)
        for bi in range(nb):
            self._update_bucket(bi, self._ev_norm, clip_coef_ptr=_ptr(self._coef))
            if self.backend == "nccl" and len(self._deferred_ag) > 1:
                self._issue_ag(self._deferred_ag.pop(0))
        self._flush_deferred_ag()

    # ------------------------------------------------------------ timing
    def enable_kernel_timing(self, on: bool = True) -> None:
        """Record CUDA events around every K1/K2 launch, on the launching
        stream, for live per-kernel bandwidth (bench.py roofline)."""
        self._ktiming = [] if on else None

    def kernel_timing(self) -> dict:
        """{kernel: (launches, total_ms, algorithmic_bytes)} — synchronises.

        Launches chained by programmatic dependent launch (fused pack+AdamW at
        d = 1) overlap each other's ramp and tail, so they are timed as one run
        (events before the first and after the last launch of the run): the
        run's time divided by its launches is their effective duration."""
        self._close_run()
        out: dict = {}
        for name, e0, e1, nbytes, nl in self._ktiming or []:
            e1.synchronize()
            n, ms, by = out.get(name, (0, 0.0, 0))
            out[name] = (n + nl, ms + e0.elapsed_time(e1), by + nbytes)
        return out

    def reset_kernel_timing(self) -> None:
        if self._ktiming is not None:
            self._ktiming = []

    _RUN = object()   # token: launch belongs to the open PDL run

    def _timed_event(self, stream, run: str | None = None):
        """Start timing a launch.  ``run``: kernel name whose consecutive
        launches on ``stream`` form one PDL chain — a timing event between them
        would serialise the chain, so the run gets one start / one end event."""
        if getattr(self, "_ktiming", None) is None:
            return None
        if run is not None and _PDL:
            if self._krun is not None and (self._krun[0] != run or self._krun[2] is not stream):
                self._close_run()
            if self._krun is None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                self._krun = [run, ev, stream, 0, 0]
            return self._RUN
        self._close_run()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        return ev

    def _timed_close(self, name, e0, stream, nbytes) -> None:
        if e0 is None:
            return
        if e0 is self._RUN:
            self._krun[3] += 1
            self._krun[4] += nbytes
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream)
        self._ktiming.append((name, e0, e1, nbytes, 1))

    def _close_run(self) -> None:
        if self._krun is None:
            return
        name, e0, stream, nl, nbytes = self._krun
        self._krun = None
        if nl:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            self._ktiming.append((name, e0, e1, nbytes, nl))

    # ------------------------------------------------------------ helpers
    def full_master(self) -> torch.Tensor:
        """This rank's fp32 master shards, concatenated (debug / checkpoint)."""
        return self.master
