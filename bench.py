#!/usr/bin/env python
"""Optimizer-step benchmark: BASELINE.json metric on B200.

``python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt1.3b]``
(one process per GPU; for N > 1 launch under torch.distributed.run).

A step is one Overlapped Distributed Optimizer step over one synthetic
gradient set: per bucket pack/cast -> reduce-scatter ->
sharded AdamW -> all-gather.  ``value`` = parameters updated per second for
the whole job (every parameter of the set is updated once per step, the
shards of all N ranks together) with inputs resident in HBM; ``e2e`` is the
same metric through ``DistributedOptimizer.step`` fed from pinned HOST
gradients (H2D inside the timed region) with a device->host read of the
step result.  ``--impl reference`` times the CPU restatement of the same
step (the reference has no optimizer of its own) on the host
cores instead.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "optimizer-step params/s"
UNIT = "params/s"
CONFIGS = {
    "toy": dict(grad_dtype="f32", clip=None, desc="toy GPT L4 h256 V51200, fp32 grads"),
    "gpt1.3b": dict(grad_dtype="bf16", clip=None, desc="GPT-3 1.3B-shape gradient set (L24 h2048 V51200), bf16 grads, fp32 master AdamW"),
    "llama7b": dict(grad_dtype="bf16", clip=1.0, desc="LLaMA-7B real tensor list, bf16 grads, grad-norm clip 1.0"),
}
FALLBACK_HBM_GBS = 6650.0
NVLINK_MEASURED = 770.0   # GB/s per direction per GPU, peer copy (B200_PROFILING.md)
NVLINK_NOMINAL = 900.0    # NVLink 5, 18 links: the north star's and SURVEY §8d's denominator
NVLINK_PEAK = NVLINK_NOMINAL   # headline roofline denominator; the measured copy is reported beside it

KERNEL_NAMES = {
    "adamw": "hod adamw_vec_kernel (K2)",
    "pack": "hod pack_kernel (K1)",
    "pack_adamw": "hod pack_adamw_kernel (K1+K2 fused, d=1)",
    "fused": "hod {span} FUSED (barrier+RS+AdamW+AG)",
    "rs": "hod {span} RS (+sumsq)",
    "adamw_ag": "hod {span} ADAMW_AG",
}


def _kernel_name(dom: str, backend: str) -> str:
    """Full-GPU p2p span launches run the TMA-fed kernel, NVLS the register one."""
    span = "span_tma_kernel" if backend == "p2p" else "p2p_step_kernel"
    return KERNEL_NAMES.get(dom, dom).format(span=span)


def _desc(cfg, clip) -> str:
    """Workload text with the clip actually used (``--clip`` may override it)."""
    base = cfg["desc"].replace(", grad-norm clip 1.0", "")
    return base + (f", grad-norm clip {clip}" if clip else ", no clip")


def _config_doc(args, clip, params, buckets, dp, scen=None) -> dict:
    """The ``config`` object of the JSON line — identical for both arms (the
    driver compares them); implementation details live outside it."""
    cfg = CONFIGS[args.config]
    hbm_gb = {"gpt1.3b": 37, "llama7b": 190, "toy": 0.5}.get(args.config, 0)
    return {"workload": (f"scenario {scen['scenario']}: GPT stages {scen['stage_layers']} "
                         "(reference self-adapting partition), PP x DP, world clip norm"
                         if scen else _desc(cfg, clip)),
            "config": "scenario" if scen else args.config, "params": params,
            "scenario": scen, "buckets": buckets, "bucket_size": args.bucket_size, "dp": dp, "clip": clip,
            "l2": f"inputs (~{hbm_gb} GB per step) >> 126 MB L2, no flush needed"}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling DURING the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_setup(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _barrier(world):
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def _max_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x: float, world: int) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


def _traffic_from_profile(kernel: str):
    """dram bytes per launch of ``kernel`` from the committed ncu summary."""
    for p in sorted((ROOT / "profiles").glob("*ncu_summary.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
        except Exception:
            continue
        k = d.get("kernels", {}).get(kernel)
        if k and k.get("dram_bytes_per_launch"):
            return k["dram_bytes_per_launch"], k.get("algorithmic_bytes_per_launch"), p.name
    return None, None, None


# best per-direction NVLink rate SM- or TMA-issued peer traffic reached on
# this box for the span kernels' access mix (profiles/r02_peer_bw_tma_n2.jsonl,
# r01_peer_bw_n4.jsonl, r01_nvls_bw_n4.jsonl); None where not measured
_PRACTICAL_NVLINK = {
    ("p2p", 2): (692.4, "d=2 TMA peer read + peer write (tma_both), r02_peer_bw_tma_n2.jsonl"),
    ("p2p", 4): (659.9, "d=4 SM peer reads from 3 peers, r01_nvls_bw_n4.jsonl"),
    ("nvls", 4): (580.0, "d=4 multimem.ld_reduce + multimem.st both ways, r01_nvls_bw_n4.jsonl"),
}


def _practical_nvlink(d: int, dom: str, backend: str):
    v = _PRACTICAL_NVLINK.get((backend, d))
    if v is None:
        return None
    return {"ceiling_gbps": v[0], "source": v[1]}


def _emulated_traffic_ratio(dom: str, d: int, backend: str):
    """DRAM traffic / algorithmic bytes of the span kernel from the one-GPU
    emulated ncu capture (profiles/*_ncu_each.json, tools/ncu_each.py): a
    multi-rank kernel cannot be replayed under ncu, its peers' copies are
    local there.  p2p only (multicast has no single-GPU stand-in)."""
    if backend != "p2p":
        return None
    # full-GPU p2p launches run the TMA-fed span kernel (round-2 captures name
    # it span_tma_*); round-1 captures hold the register kernel as span_*
    for p in sorted((ROOT / "profiles").glob("*ncu_each.json"), reverse=True):
        try:
            kernels = json.loads(p.read_text())["kernels"]
        except Exception:
            continue
        for name in (f"span_tma_{dom}_d{d}", f"span_{dom}_d{d}"):
            k = kernels.get(name)
            if k and k.get("traffic_over_algorithmic"):
                return {"traffic_over_algorithmic": k["traffic_over_algorithmic"], "source": f"{p.name}:{name}",
                        "note": "one-GPU emulation of the d-way kernel (peer copies local), cold cache"}
    return None


def parity_probe(opt, gs, rank: int, dev, gdtype, world: int) -> dict:
    """Self-check AFTER the timed region (the line then carries its own
    correctness): one more step of the benchmarked optimizer over
    the same gradients, then the first, middle and last bucket of this rank
    against the oracle (oracle/oracle.py — the checker, never the measured
    path): every DP peer's gradients are regenerated from their seeds,
    packed and reduce-scattered by the oracle (rank-order fp32 sum of
    simulator.py:81-89 semantics over the DP row of groups.py:137-148;
    NVLS / NCCL within d/2 bf16 ulp of sum|x|), then the oracle AdamW from
    the pre-step state with the device's reduced shard and clip coefficient
    must give master / m / v / the gathered bf16 params bit-exactly; the
    clip coefficient must be bit-identical on every rank.  ``ok`` is the AND
    over all ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from oracle import oracle
    from paper_2312_03549_b200.errors import DeviceError
    from paper_2312_03549_b200.synthetic import make_grads

    def u16(t):
        return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)

    t0 = time.perf_counter()
    oracle.set_threads(max(1, len(os.sched_getaffinity(0)) // max(1, torch.cuda.device_count())))
    L = opt.layout
    nb = len(L.buckets)
    sample = sorted({0, nb // 2, nb - 1})
    offs = L.shard_offsets()
    d, me = opt.dp, opt.shard_index
    out = {"buckets_checked": sample, "dp": d, "backend": opt.backend, "ok": False}
    errors = []
    pre = {}
    for bi in sample:
        n = L.buckets[bi].numel // d
        pre[bi] = tuple(x[offs[bi]:offs[bi] + n].cpu().numpy().copy() for x in (opt.master, opt.exp_avg, opt.exp_avg_sq))
    keep = opt.keep_reduced
    opt.keep_reduced = d > 1                 # leave the reduced shard in place for the check
    grads = None
    try:
        grads = make_grads(gs, 1, opt.group.global_rank, dev, dtype=gdtype)
        rep = opt.step(grads)
        rep.resolve()
    except DeviceError as e:
        errors.append(f"device: {e}")
        rep = None
    finally:
        opt.keep_reduced = keep
    del grads
    torch.cuda.empty_cache()
    coef = None
    if rep is not None and rep.clip_coef is not None:
        c = rep.clip_coef.reshape(1).clone()
        if world > 1:
            cs = [torch.zeros_like(c) for _ in range(world)]
            dist.all_gather(cs, c)
            if any(not torch.equal(x.view(torch.int32), c.view(torch.int32)) for x in cs):
                errors.append("clip coefficient differs between ranks")
        coef = float(c.item())
    if rep is not None:
        slices = {bi: [] for bi in sample}
        for q in opt.group.ranks:
            gq = make_grads(gs, 1, q, dev, dtype=gdtype)
            for bi in sample:
                b = L.buckets[bi]
                srcs = [(u16(gq[s.index]) if gdtype == torch.bfloat16 else gq[s.index].cpu().numpy()).reshape(-1)
                        for s in b.slots]
                full = oracle.pack(srcs, [s.offset for s in b.slots], b.numel, opt.grad_scale)
                sh = b.numel // d
                slices[bi].append(full[me * sh:(me + 1) * sh].copy())
                del full, srcs
            del gq
            torch.cuda.empty_cache()
        exact = opt.backend in ("p2p", "none")
        out["reduce_scatter_rule"] = ("bit-exact rank-order fp32 sum" if exact
                                      else "within d/2 bf16 ulp of sum|x| (switch / ring order)")
        out["adamw_rule"] = ("bit-exact" if opt.adamw_mode == "exact"
                             else "fast mode: within 1e-6 norm-relative, params = RNE(master)")
        step = opt.step_count
        checked = 0
        for bi in sample:
            b = L.buckets[bi]
            lo, hi = b.shard_range(me, d)
            if d > 1:
                dev_red = u16(opt.grad_buffer[lo:hi])
                if exact:
                    if not np.array_equal(dev_red, oracle.sum_slices(slices[bi])):
                        errors.append(f"bucket {bi}: reduced shard")
                else:
                    f64 = oracle.sum_slices_f64(slices[bi])
                    absum = sum(np.abs(oracle.bf16_to_f32(x).astype(np.float64)) for x in slices[bi])
                    err = np.abs(oracle.bf16_to_f32(dev_red).astype(np.float64) - f64)
                    ulp = np.exp2(np.floor(np.log2(np.maximum(absum, np.finfo(np.float32).tiny))) - 7)
                    if not np.all(err <= d * 0.5 * ulp + 1e-30):
                        errors.append(f"bucket {bi}: reduced shard outside the bf16 bound")
            else:
                dev_red = slices[bi][0]
            master, m, v = (x.copy() for x in pre[bi])
            want_p = oracle.adamw(master, m, v, dev_red, step, opt.lr, opt.betas, opt.eps, opt.weight_decay,
                                  coef=coef)
            o, n = offs[bi], hi - lo
            fast = opt.adamw_mode == "fast"
            for name, want, got in (("master", master, opt.master), ("m", m, opt.exp_avg), ("v", v, opt.exp_avg_sq)):
                g = got[o:o + n].cpu().numpy()
                if fast:    # one step from the same state: north-star 1e-6, norm-relative
                    err = float(np.abs(g.astype(np.float64) - want).max() / max(np.abs(want).max(), 1e-30))
                    out.setdefault("max_norm_rel_err", {})[name] = max(err, out.get("max_norm_rel_err", {}).get(name, 0))
                    if err > 1e-6:
                        errors.append(f"bucket {bi}: {name} rel err {err:.2e}")
                elif not np.array_equal(g.view(np.uint32), want.view(np.uint32)):
                    errors.append(f"bucket {bi}: {name}")
            want_p = u16(opt.master[o:o + n].to(torch.bfloat16)) if fast else want_p
            if not np.array_equal(u16(opt.param_buffer[lo:hi]), want_p):
                errors.append(f"bucket {bi}: gathered params")
            checked += n
        out["elements_checked_per_rank"] = checked
    ok = torch.tensor([0 if errors else 1], dtype=torch.int32, device=dev)
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    out["ok"] = bool(ok.item())
    out["errors_rank"] = errors[:8]
    out["seconds"] = round(time.perf_counter() - t0, 1)
    return out


def cpu_baseline(config: str, gs, seconds: float = 10.0) -> dict:
    """Oracle (CPU port) timed on a bounded sample: pack + AdamW over whole
    buckets of the workload, repeated until ``seconds`` elapse."""
    import numpy as np

    from oracle import oracle
    from paper_2312_03549_b200.buckets import build_bucket_layout

    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    L = build_bucket_layout(gs.numels, 25_000_000, dp=1)
    b = max(L.buckets, key=lambda x: -x.numel)  # smallest whole bucket
    rng = np.random.default_rng(0)
    grads = [oracle.f32_to_bf16(rng.standard_normal(s.numel, dtype=np.float32) * 1e-3) for s in b.slots]
    master = (rng.standard_normal(b.numel, dtype=np.float32) * 0.02)
    m = np.zeros(b.numel, np.float32)
    v = np.zeros(b.numel, np.float32)
    offs = [s.offset for s in b.slots]
    done, t0, step = 0, time.perf_counter(), 0
    while True:
        step += 1
        bucket = oracle.pack(grads, offs, b.numel, 1.0)
        oracle.adamw(master, m, v, bucket, step)
        done += b.numel
        if time.perf_counter() - t0 >= seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": oracle.threads(), "kind": "port",
            "sample": f"{step} x (pack + AdamW) over one {b.numel}-element bucket of {config} "
                      f"(d=1 step restated by oracle/hod_oracle.c, OpenMP {oracle.threads()} threads, {dt:.1f} s)"}


_CPU_REF: dict = {}


def cpu_reference_step(gs, d: int, clip, bucket_size: int, budget_s: float) -> dict:
    """One optimizer step of the whole job restated on the host cores by the
    oracle (oracle/hod_oracle.c, OpenMP): for every bucket, the pack of each of
    the d ranks' gradients (dp-scale + bf16 cast), the rank-order reduce-scatter
    sum, the clip norm and the AdamW update of every shard — the reference's
    own CPU path for this step, since the reference has no optimizer.
    Buckets stream through reused host buffers (the work and DRAM traffic per
    bucket are those of the real step).  If the full step would exceed
    ``budget_s`` the step is cut after the buckets that fit (a bounded sample,
    labelled as such); params/s = parameters updated / seconds."""
    import numpy as np

    from oracle import oracle
    from paper_2312_03549_b200.buckets import build_bucket_layout

    key = (gs.name, d, bucket_size)
    if key not in _CPU_REF:
        L = build_bucket_layout(gs.numels, bucket_size, dp=d)
        rng = np.random.default_rng(0)
        block = oracle.f32_to_bf16(rng.standard_normal(1 << 20, dtype=np.float32) * 1e-3)
        big = max(b.numel for b in L.buckets)
        grads = {t_i: (np.tile(block, -(-n // block.size))[:n] if n else np.zeros(0, np.uint16))
                 for t_i, n in enumerate(gs.numels)}
        _CPU_REF.clear()
        _CPU_REF[key] = (L, grads, rng.standard_normal(big, dtype=np.float32) * 0.02,
                         np.zeros(big, np.float32), np.zeros(big, np.float32))
    L, grads, master, m, v = _CPU_REF[key]
    t0 = time.perf_counter()
    done = 0
    nb = 0
    for b in L.buckets:
        srcs = [grads[s.index] for s in b.slots]
        offs = [s.offset for s in b.slots]
        packs = [oracle.pack(srcs, offs, b.numel, 1.0 / d) for _ in range(d)]
        shards = [oracle.reduce_scatter(packs, r, d) if d > 1 else packs[0] for r in range(d)]
        coef = None
        if clip:
            ss = sum(oracle.sumsq_bf16(x) for x in shards)
            coef = oracle.clip_coef(np.float32(ss), clip)
        n = b.numel // d
        for r in range(d):
            oracle.adamw(master[:n], m[:n], v[:n], shards[r], 1, coef=coef)
        done += b.numel
        nb += 1
        if time.perf_counter() - t0 > budget_s and nb < len(L.buckets):
            break
    dt = time.perf_counter() - t0
    full = nb == len(L.buckets)
    return {"params": done, "seconds": dt, "buckets": nb, "of": len(L.buckets), "full": full}


def run_reference(args) -> None:
    """--impl reference: the job's optimizer step on the host cores (rank 0
    only; the other ranks exit 0 without work), same config / metric / unit."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    from paper_2312_03549_b200.buckets import build_bucket_layout
    from paper_2312_03549_b200.gradsets import config_gradset

    cfg = CONFIGS[args.config]
    clip = cfg["clip"] if args.clip is None else (None if args.clip <= 0 else args.clip)
    gs = config_gradset(args.config)
    d = args.gpus
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    vals, last = [], None
    for i in range(args.warmup + args.steps):
        r = cpu_reference_step(gs, d, clip, args.bucket_size, budget_s=args.ref_seconds)
        if i >= args.warmup:
            vals.append(r["params"] / r["seconds"])
            last = r
    value = statistics.median(vals)
    nbk = len(build_bucket_layout(gs.numels, args.bucket_size, dp=d).buckets)
    sample = (f"{'full step' if last['full'] else 'bounded sample'}: {last['buckets']} of {last['of']} buckets "
              f"x (pack of {d} ranks + reduce-scatter + {'clip + ' if clip else ''}AdamW) per timed step, "
              f"oracle/hod_oracle.c OpenMP {oracle.threads()} threads"
              + ("" if last["full"] else "; params/s extrapolates the sample to the step"))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * gs.total / value, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16-grads/f32-adamw", "data": "synthetic",
        "impl": "reference",
        "config": _config_doc(args, clip, gs.total, nbk, d),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference has no optimizer implementation (SPEC.md:14): its CPU path for this step is "
                "the oracle restatement (SURVEY §8c)",
    }
    print(json.dumps(line), flush=True)


def north_star_probe(args, world: int, rank: int, dev) -> dict:
    """BASELINE.json's target workload measured inside the default run at
    N >= 4: the LLaMA-7B real tensor list, bf16 grads, clip 1.0, DP = N —
    standalone step time (CUDA events, max over ranks) and the exposure of
    the optimizer inside a training iteration (synthetic cuBLAS fwd/bwd of
    ``--overlap-tokens`` tokens per GPU, tools/overlap_bench.py)."""
    import torch

    from paper_2312_03549_b200 import DistributedOptimizer
    from paper_2312_03549_b200.comm import DPGroup
    from paper_2312_03549_b200.gradsets import config_gradset
    from paper_2312_03549_b200.synthetic import init_params, make_grads

    gs = config_gradset("llama7b")
    p0 = init_params(gs, dev)
    opt = DistributedOptimizer(p0, bucket_size=args.bucket_size, clip=1.0, adamw=args.adamw,
                               dp_group=DPGroup(tuple(range(world)), rank), span_numel=args.span_numel)
    del p0
    torch.cuda.empty_cache()
    grads = make_grads(gs, 1, rank, dev)
    for _ in range(3):
        opt.step(grads)
    _barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 5
    e0.record()
    for _ in range(steps):
        opt.step(grads)
    e1.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(e0.elapsed_time(e1) / steps, world)
    del grads
    torch.cuda.empty_cache()
    sys.path.insert(0, str(ROOT / "tools"))
    from overlap_bench import measure

    o = measure(opt, gs, args.overlap_tokens, 3, world, dev)
    parity = None if args.no_parity else parity_probe(opt, gs, rank, dev, torch.bfloat16, world)
    P, d = gs.total, world
    peak, _ = _peaks()
    hbm = 4 * P + 30 * P / d                  # pack + AdamW 28 B + norm read 2 B per owned element
    nvl = 4 * P * (d - 1) / d
    t_roof = max(hbm / (peak * 1e9), nvl / (NVLINK_PEAK * 1e9)) * 1e3
    out = {"workload": f"LLaMA-7B real tensor list, bf16 grads, grad-norm clip 1.0, DP={world} "
                       f"(BASELINE.json target; backend {opt.backend})",
           "params": gs.total, "ms_per_step": ms, "params_per_s": gs.total / (ms / 1e3), "steps": steps,
           "parity": parity,
           "step_roofline": {"t_roof_ms": t_roof, "frac": t_roof / ms,
                             "nvlink_peak_gbps": NVLINK_PEAK,
                             "bound": "hbm" if hbm / (peak * 1e9) >= nvl / (NVLINK_PEAK * 1e9) else "nvlink"},
           "overlap": {"tokens_per_gpu": args.overlap_tokens,
                       "exposed_frac_iteration": o["iteration"]["exposed_frac"],
                       "t_fwd_bwd_ms": o["iteration"]["t_fwd_bwd_ms"],
                       "t_fwd_bwd_opt_ms": o["iteration"]["t_fwd_bwd_opt_ms"],
                       "exposed_comm_frac_survey": o["exposed_comm_frac_survey"],
                       "t_optimizer_alone_ms": o["t_optimizer_alone_ms"],
                       "hidden_frac_of_optimizer": o["hidden_frac_of_optimizer"]}}
    opt.close()
    torch.cuda.empty_cache()
    return out


def scenario_probe(args, path: Path, world: int, rank: int, dev) -> dict:
    """BASELINE config 4 inside the default run: the reference planner's
    self-adapting partition and DP rows for ``path`` (PP x DP over the world),
    every stage's DP row running its own optimizer, world clip norm; step time
    = max over ranks (CUDA events)."""
    import torch
    import torch.distributed as dist

    import paper_2312_03549_b200 as hp
    from paper_2312_03549_b200.scenario_run import make_optimizer, setup_rank
    from paper_2312_03549_b200.synthetic import init_params, make_grads

    scenario = hp.load_scenario(str(path))
    sr = setup_rank(scenario, rank)
    gs = sr.gradset
    p0 = init_params(gs, dev)
    opt = make_optimizer(sr, p0, bucket_size=args.bucket_size, clip=1.0, span_numel=args.span_numel,
                         adamw=args.adamw)
    del p0
    torch.cuda.empty_cache()
    grads = make_grads(gs, 1, rank, dev)
    for _ in range(3):
        opt.step(grads)
    _barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 5
    e0.record()
    for _ in range(steps):
        opt.step(grads)
    e1.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(e0.elapsed_time(e1) / steps, world)
    parity = None if args.no_parity else parity_probe(opt, gs, rank, dev, torch.bfloat16, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, {sr.placement.stage: gs.total})
    totals = {}
    for dct in gathered:
        totals.update(dct)
    out = {"scenario": path.name, "stage_layers": list(hp.partition_scenario(scenario).stage_layers),
           "stage_params": totals, "dp_ranks_rank0": list(sr.placement.dp_ranks), "backend": opt.backend,
           "ms_per_step": ms, "params_per_s": sum(totals.values()) / (ms / 1e3), "steps": steps,
           "parity": parity}
    opt.close()
    del grads, opt
    torch.cuda.empty_cache()
    return out


def sweep_probe(world: int, rank: int, dev) -> list:
    """BASELINE config 5 inside the default run: one bucket of 1 MB .. 1 GB,
    fused RS+AdamW+AG (p2p, nvls) vs NCCL ReduceScatter+AllGather, busBW
    (tools/p2p_microbench.py)."""
    import torch

    from paper_2312_03549_b200.comm import NcclComm

    sys.path.insert(0, str(ROOT / "tools"))
    from p2p_microbench import measure_bucket

    comm = NcclComm(tuple(range(world)), rank, "sweep")
    rows = []
    for numel in (1 << 19, 1 << 23, 1 << 26, 1 << 29):     # 1 MB, 16 MB, 128 MB, 1 GB of bf16
        iters = max(5, min(50, int(2e9 // (numel * 2))))
        doc = measure_bucket(numel, iters, world, rank, dev, comm,
                             cases=("fused_p2p", "fused_nvls", "nccl_rs+ag"))
        rows.append(_sweep_row(doc))
    comm.close()
    torch.cuda.empty_cache()
    return rows


def _sweep_row(doc: dict) -> dict:
    """One bucket size of the sweep: time and busBW per case, with busBW as a
    fraction of the measured (770) and nominal (900 GB/s) NVLink roofline."""
    row = {"bucket_MB": doc["bucket_MB"]}
    for k, v in doc["results"].items():
        if not isinstance(v, dict):
            continue
        bus = v.get("busBW_GBps")
        row[k] = {"ms": v["ms"], "busBW_GBps": bus,
                  "frac_nvlink": round(bus / NVLINK_PEAK, 3) if bus else None,
                  "frac_nvlink_measured_copy": round(bus / NVLINK_MEASURED, 3) if bus else None}
    return row


def _guarded(name, fn, world):
    """Run one add-on probe; a failure is recorded in the line, not fatal."""
    try:
        out = fn()
    except Exception as e:  # noqa: BLE001  (the main measurement must still print)
        out = {"error": f"{type(e).__name__}: {e}"[:300]}
    _barrier(world)
    return out


def run_ours(args) -> None:
    import torch

    from paper_2312_03549_b200 import DistributedOptimizer, _native
    from paper_2312_03549_b200.comm import DPGroup
    from paper_2312_03549_b200.gradsets import config_gradset
    from paper_2312_03549_b200.synthetic import init_params, make_grads

    world, rank, local = _dist_setup(args)
    cfg = CONFIGS[args.config]
    clip = cfg["clip"] if args.clip is None else (None if args.clip <= 0 else args.clip)
    dev = torch.device("cuda", local)
    gdtype = torch.float32 if cfg["grad_dtype"] == "f32" else torch.bfloat16
    scen = None
    if args.scenario:
        # BASELINE config 4: PP x DP from the reference-compatible planner; every
        # stage updates its own gradient set, the clip norm spans the world
        import paper_2312_03549_b200 as hp
        from paper_2312_03549_b200.scenario_run import make_optimizer, setup_rank

        scenario = hp.load_scenario(args.scenario)
        sr = setup_rank(scenario, rank)
        gs = sr.gradset
        clip = 1.0 if args.clip is None else (None if args.clip <= 0 else args.clip)
        p0 = init_params(gs, dev)
        opt = make_optimizer(sr, p0, bucket_size=args.bucket_size, clip=clip, backend=args.backend, adamw=args.adamw,
                             span_numel=args.span_numel)
        stage_params = {sr.placement.stage: gs.total}
        gathered = [None] * world
        import torch.distributed as dist

        dist.all_gather_object(gathered, stage_params)
        totals = {}
        for dct in gathered:
            totals.update(dct)
        scen = {"scenario": Path(args.scenario).name, "stage_layers": None, "stage_params": totals,
                "placement": sr.placement.to_json_dict()}
        scen["stage_layers"] = list(hp.partition_scenario(scenario).stage_layers)
    else:
        gs = config_gradset(args.config)
        p0 = init_params(gs, dev)
        group = DPGroup(tuple(range(world)), rank)
        opt = DistributedOptimizer(p0, bucket_size=args.bucket_size, clip=clip, dp_group=group, adamw=args.adamw,
                                   backend=args.backend, span_numel=args.span_numel,
                                   first_span_numel=args.first_span_numel,
                                   param_barriers=bool(args.param_barriers))
    del p0
    torch.cuda.empty_cache()
    grads = make_grads(gs, 1, rank, dev, dtype=gdtype)

    # ---- device-resident timed region -------------------------------------
    for _ in range(args.warmup):
        opt.step(grads)
    _barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    opt.enable_kernel_timing(True)
    launches0 = _native.launch_count()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _barrier(world)
    start.record()
    for _ in range(args.steps):
        opt.step(grads)
    end.record()
    torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    _barrier(world)
    clk = clocks.stop()
    ms = start.elapsed_time(end) / args.steps
    ms = _max_over_ranks(ms, world)
    kt = opt.kernel_timing()
    opt.enable_kernel_timing(False)
    # every parameter of the set (of every stage, for a PP x DP scenario) is
    # updated once per step
    params_per_step = sum(scen["stage_params"].values()) if scen else gs.total
    value = params_per_step / (ms / 1e3)

    # ---- roofline of the dominant kernel ----------------------------------
    # (largest share of timed kernel time; HBM-bound at d = 1, the fused
    # RS+AdamW+AG kernel is NVLink-bound at d > 1 and reports both views)
    peak, peak_src = _peaks()
    dom = max(kt, key=lambda k: kt[k][1]) if kt else "adamw"
    n_launch, ktime, kbytes = kt.get(dom, (0, 0.0, 0))
    achieved = (kbytes / (ktime / 1e3)) / 1e9 if ktime > 0 else None
    traffic, alg_per_launch, prof = _traffic_from_profile(dom)
    roof = {"kernel": _kernel_name(dom, opt.backend), "bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
            "traffic": traffic, "traffic_source": prof, "peak_source": peak_src,
            "traffic_launch_algorithmic_bytes": alg_per_launch,
            "algorithmic_bytes_per_launch": kbytes / max(1, n_launch),
            "avg_launch_ms": ktime / max(1, n_launch), "launches_timed": n_launch,
            "bytes_per_element": 28}
    if achieved and achieved > peak:
        roof["peak_note"] = ("the measured peak is a torch copy_ (1:1 read/write, MEASURED_PEAKS.json); this "
                             "kernel's mixed read/write stream runs slightly above it — at the HBM roofline")
    if dom in ("fused", "adamw_ag", "rs") and opt.dp > 1:
        # a collective span kernel: the binding resource is whichever of local
        # HBM (28 B per owned element for the update; RS: own shard read +
        # reduced shard write) and NVLink per direction (SURVEY §8d algorithmic
        # bytes: RS in + AG out = 2(d-1) B each per owned element) needs longer
        d_ = opt.dp
        elems = kbytes / 28 if dom != "rs" else kbytes / (2 * d_ + 2)
        per_elem = {"fused": 4, "adamw_ag": 2, "rs": 2}[dom] * (d_ - 1)
        hbm_elem = {"fused": 28, "adamw_ag": 28, "rs": 4}[dom]
        nvl = elems * per_elem / (ktime / 1e3) / 1e9 if ktime > 0 else None
        hbm = elems * hbm_elem / (ktime / 1e3) / 1e9 if ktime > 0 else None
        hbm_view = {"achieved": hbm, "peak": peak, "frac": hbm / peak if hbm else None,
                    "bytes_per_owned_element": hbm_elem}
        nvl_view = {"achieved": nvl, "peak": NVLINK_PEAK, "frac": nvl / NVLINK_PEAK if nvl else None,
                    "frac_measured_copy": nvl / NVLINK_MEASURED if nvl else None,
                    "bytes_per_owned_element": per_elem}
        if opt.backend == "nvls":
            # what the switch actually moves per GPU and direction (the larger of
            # egress / ingress): fused 2(d+1), RS egress 2d, AG ingress 2d
            phys = {"fused": 2 * (d_ + 1), "adamw_ag": 2 * d_, "rs": 2 * d_}[dom]
            nvl_view["physical_bytes_per_owned_element"] = phys
            nvl_view["physical_achieved"] = elems * phys / (ktime / 1e3) / 1e9 if ktime > 0 else None
        # what SM/TMA-issued peer traffic reaches on this box (tools/peer_bw.py):
        # the practical ceiling the span kernels are measured against
        ceil = _practical_nvlink(d_, dom, opt.backend)
        if ceil and nvl:
            # NVLS ceilings are physical switch traffic: compare like with like
            rate = nvl_view.get("physical_achieved") or nvl
            nvl_view["practical"] = dict(ceil, achieved=rate, frac=rate / ceil["ceiling_gbps"])
        roof["traffic_emulated"] = _emulated_traffic_ratio(dom, d_, opt.backend)
        if hbm_elem / peak >= per_elem / NVLINK_PEAK:
            roof.update({"bound": "hbm", "achieved": hbm, "frac": hbm_view["frac"],
                         "bytes_per_element": hbm_elem, "nvlink_view": nvl_view})
        else:
            roof.update({"bound": "nvlink", "achieved": nvl, "peak": NVLINK_PEAK, "frac": nvl_view["frac"],
                         "peak_source": "NVLink 5 nominal 900 GB/s per direction (north star, SURVEY §8d); "
                         "frac_measured_copy against the 770 GB/s peer copy of B200_PROFILING.md",
                         "frac_measured_copy": nvl_view["frac_measured_copy"], "hbm_view": hbm_view,
                         "practical": nvl_view.get("practical"),
                         "nvlink_bytes_per_owned_element": per_elem, "bytes_per_element": per_elem})
            if "physical_achieved" in nvl_view:
                roof["nvlink_physical"] = {k: nvl_view[k] for k in
                                           ("physical_bytes_per_owned_element", "physical_achieved")}
    kernels = {k: {"launches": n, "ms_total": t, "GBps": (b / (t / 1e3)) / 1e9 if t else None}
               for k, (n, t, b) in kt.items()}
    # step-level roofline: max(HBM bytes / peak, NVLink bytes / link bandwidth)
    d = opt.dp
    P = gs.total  # this rank's stage
    src_b = 4 if gdtype == torch.float32 else 2
    if d == 1 and not clip:   # K1+K2 fuse: grad read + 24 B state + 2 B param, no bucket
        hbm_bytes = (src_b + 26) * P
    elif d == 1:              # norm pass over the tensors, then the fused update
        hbm_bytes = src_b * P + (src_b + 26) * P
    else:
        hbm_bytes = (src_b + 2) * P + 28 * P / d + (2 * P / d if clip else 0)
    nvl_bytes = 4 * P * (d - 1) / d
    # NVLink denominator: 900 GB/s per direction (north star, SURVEY §8d,
    # BASELINE.md's table); the measured 770 GB/s peer copy is reported beside it
    t_roof = _max_over_ranks(max(hbm_bytes / (peak * 1e9), nvl_bytes / (NVLINK_PEAK * 1e9)), world)
    t_roof_meas = _max_over_ranks(max(hbm_bytes / (peak * 1e9), nvl_bytes / (NVLINK_MEASURED * 1e9)), world)
    # physically each GPU's HBM also serves its peers' NVLink traffic: their
    # reads of its packed bucket and their stores into its param buffer
    # (2P(d-1)/d each) — the floor the step actually runs against at d = 2
    hbm_phys = hbm_bytes + (4 * P * (d - 1) / d if opt.backend in ("p2p", "nvls") else 0)
    t_roof_phys = _max_over_ranks(max(hbm_phys / (peak * 1e9), nvl_bytes / (NVLINK_PEAK * 1e9)), world)
    step_roof = {"t_roof_ms": t_roof * 1e3, "frac": (t_roof * 1e3) / ms,
                 "t_roof_measured_copy_ms": t_roof_meas * 1e3, "frac_measured_copy": (t_roof_meas * 1e3) / ms,
                 "physical": {"hbm_bytes_per_gpu": hbm_phys, "t_roof_ms": t_roof_phys * 1e3,
                              "frac": (t_roof_phys * 1e3) / ms,
                              "note": "HBM bytes incl. the peers' NVLink reads/stores served by this GPU"},
                 "hbm_bytes_per_gpu": hbm_bytes, "nvlink_bytes_per_gpu_per_dir": nvl_bytes,
                 "nvlink_peak_gbps": NVLINK_PEAK,
                 "bound": "hbm" if hbm_bytes / (peak * 1e9) >= nvl_bytes / (NVLINK_PEAK * 1e9) else "nvlink"}

    # ---- e2e through the public API with host buffers ---------------------
    e2e = None
    if not args.no_e2e:
        host = [g.cpu().pin_memory() for g in grads]
        res_host = torch.empty(1, dtype=torch.float32).pin_memory()
        del grads
        torch.cuda.empty_cache()
        for _ in range(max(1, min(args.warmup, 2))):
            opt.step(host)
        _barrier(world)
        e_steps = max(1, min(args.steps, 5))
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(e_steps):
            rep = opt.step(host)
            # device->host read of the step result: grad norm (clip) or first updated param
            src = rep.grad_norm if rep.grad_norm is not None else opt.params[0].reshape(-1)[:2].view(torch.float32)
            res_host.copy_(src, non_blocking=True)
        t1.record()
        torch.cuda.synchronize()
        ems = _max_over_ranks(t0.elapsed_time(t1) / e_steps, world)
        h2d = _sum_over_ranks(float(sum(h.numel() * h.element_size() for h in host)), world)
        e2e = {"value": params_per_step / (ems / 1e3), "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4 * world,
               "steps": e_steps, "path": "DistributedOptimizer.step(pinned host grads)"}

    # ---- exposure inside a training iteration (N > 1) --------------------
    # synthetic cuBLAS forward/backward of 8192 tokens per GPU around the
    # optimizer driven as under autograd hooks (grad_ready per tensor, per-span
    # params-ready, wait_params before each bucket's first forward use):
    # exposed = iteration with the optimizer - iteration without (north star
    # <= 10 %), plus SURVEY §8d's tail definition (tools/overlap_bench.py)
    overlap = None
    if world > 1 and not scen and not args.no_overlap:
        if not args.no_e2e:
            del host
        torch.cuda.empty_cache()
        sys.path.insert(0, str(ROOT / "tools"))
        from overlap_bench import measure

        o = measure(opt, gs, args.overlap_tokens, 5, world, dev)
        overlap = {"tokens_per_gpu": args.overlap_tokens, "exposed_frac_iteration": o["iteration"]["exposed_frac"],
                   "t_fwd_bwd_ms": o["iteration"]["t_fwd_bwd_ms"],
                   "t_fwd_bwd_opt_ms": o["iteration"]["t_fwd_bwd_opt_ms"],
                   "exposed_comm_frac_survey": o["exposed_comm_frac_survey"],
                   "t_backward_ms": o["t_backward_ms"], "t_backward_with_opt_ms": o["t_overlapped_ms"],
                   "t_optimizer_alone_ms": o["t_optimizer_alone_ms"],
                   "hidden_frac_of_optimizer": o["hidden_frac_of_optimizer"],
                   "note": "synthetic GEMM fwd/bwd (real cuBLAS bf16 GEMMs on the config's weight shapes); "
                           "exposed_frac_iteration = (iter with optimizer - iter without) / iter with, "
                           "steady state: (T(3 iterations) - T(1)) / 2 per block, blocks alternated with / "
                           "without, medians (tools/overlap_bench.py)"}

    opt_info = {"buckets": len(opt.layout.buckets), "dp": opt.dp, "backend": opt.backend}
    # ---- self-check after every timed measurement (one more step vs the oracle)
    parity = None
    if not args.no_parity:
        parity = _guarded("parity", lambda: parity_probe(opt, gs, rank, dev, gdtype, world), world)
    extras = None
    if args.extras == 1 or (args.extras == -1 and world >= 4 and not scen and args.config == "gpt1.3b"):
        # the driver's multi-GPU runs use the default config: measure the other
        # BASELINE configs at this N too (config 3 target, config 4, config 5)
        opt.close()
        opt = None
        torch.cuda.empty_cache()
        scen_file = ROOT / "scenarios" / ("gpt13b_pp2_dp4_hybrid.json" if world == 8 else
                                          "gpt13b_pp2_dp2_hybrid.json")
        extras = {"north_star_llama7b": _guarded("llama", lambda: north_star_probe(args, world, rank, dev), world)}
        if world in (4, 8):
            extras["config4_scenario"] = _guarded("scenario", lambda: scenario_probe(args, scen_file, world, rank,
                                                                                      dev), world)
        extras["config5_sweep"] = _guarded("sweep", lambda: sweep_probe(world, rank, dev), world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, gs, seconds=args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16-grads/f32-adamw", "data": "synthetic",
            "config": _config_doc(args, clip, params_per_step, opt_info["buckets"], opt_info["dp"], scen),
            "backend": opt_info["backend"], "adamw": args.adamw, "parity": parity,
            "roofline": roof, "step_roofline": step_roof, "kernels": kernels,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
            "overlap": overlap, "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if opt is not None:
        opt.close()
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="gpt1.3b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scenario", default=None,
                    help="scenario JSON (reference schema) for a PP x DP run, e.g. "
                         "scenarios/gpt13b_pp2_dp4_hybrid.json (BASELINE config 4, 8 GPUs)")
    ap.add_argument("--bucket-size", type=int, default=25_000_000)
    ap.add_argument("--span-numel", type=int, default=256 * 2**20,
                    help="p2p/nvls: coalesce packed buckets into fused launches of >= this many elements")
    ap.add_argument("--first-span-numel", type=int, default=None,
                    help="p2p/nvls: threshold of the step's first span (default: min(--span-numel, 32M))")
    ap.add_argument("--param-barriers", type=int, default=1, choices=[0, 1],
                    help="p2p/nvls, hook-driven flows (the overlap measurement): params-ready barrier per "
                         "span (1) or one end-of-step barrier (0); step() always ends with one barrier")
    ap.add_argument("--backend", default="auto")
    ap.add_argument("--adamw", default="exact", choices=["exact", "fast"],
                    help="AdamW arithmetic: exact (bit-exact vs the oracle) or fast (FMA + MUFU, within 1e-6/1e-5)")
    ap.add_argument("--clip", type=float, default=None, help="override clip (<=0 disables)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true", help="skip the N > 1 iteration-exposure measurement")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-measurement self-check of sampled buckets against the oracle")
    ap.add_argument("--overlap-tokens", type=int, default=8192)
    ap.add_argument("--extras", type=int, default=-1, choices=[-1, 0, 1],
                    help="also measure BASELINE configs 3 (LLaMA-7B clip DP=N: step + iteration exposure), "
                         "4 (13B PP=2 x DP=N/2 scenario) and 5 (bucket sweep) at this N; "
                         "-1 = on for the default config at N >= 4")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="--impl reference: time budget of one timed CPU step (a longer step is cut to a "
                         "bounded, labelled sample of its buckets)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
