"""Pipeline-parallel iteration around the optimizer.

Executes the flush-synchronised 1F1B schedule the reference SIMULATES
(``_schedule_ops`` simulator.py:348-356, mirrored as
``simulator._one_f_one_b``) on real GPUs, with the stage-boundary transfers
(activations forward, activation gradients backward; ``b*s*h`` bf16 elements,
``_activation_bytes`` simulator.py:283-284) moved over NVLink peer memory:

* each PP row (``build_pp`` Eq. 2, groups.py:126-134) is a symmetric-memory
  group; every rank owns receive slots ``fwd_in[k]`` / ``bwd_in[k]`` for the
  m micro-batches of an iteration and a flag per slot;
* a send is a copy-engine transfer (``hod_ce_copy``) into the neighbour's
  slot followed by ``hod_p2p_signal`` (system fence + release store of the iteration epoch);
  a receive is ``hod_p2p_wait`` on the local flag before the consumer runs —
  sends never block (one slot per micro-batch), so the 1F1B order cannot
  deadlock the way paired blocking send/recv can;
* stage compute is a stand-in made of cuBLAS GEMMs on the stage's real bf16
  parameters (the optimizer's flat buffer): 24*b*s*h^2 forward FLOPs per layer
  (qkv, proj, fc1, fc2) and twice that backward (dgrad + wgrad);
* during the LAST micro-batch's backward, each layer's weight gradients go to
  ``DistributedOptimizer.grad_ready`` as they are produced, so the DP
  reduce-scatter of a stage's buckets overlaps the rest of that backward;
  ``finish_step`` closes the iteration (the post-flush point of
  simulator.py:445-452, now mostly hidden).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _native as nat
from .simulator import _one_f_one_b
from .symm import SymmetricTensor


class PipelineRunner:
    def __init__(self, scenario, sr, opt, micro_batches: int | None = None, compute: bool = True,
                 timeout_s: float = 30.0, symmetric=None, stream=None):
        """``sr``: scenario_run.ScenarioRank of this rank; ``opt``: its optimizer.

        ``symmetric``: factory ``(numel, dtype, device, zero) ->`` symmetric
        buffer over this rank's PP row (default: torch symmetric memory over a
        PP-row process group, created collectively);
        ``emulation.EmulatedRow(p).factory(stage - 1)`` runs the stages of a
        row in one process on one GPU (the one-GPU test of the 1F1B
        hand-offs).  ``stream``: the stream this rank's iteration runs on."""
        self.s, self.sr, self.opt = scenario, sr, opt
        self.device = opt.device
        m = scenario.model
        self.p = scenario.parallel.pipeline
        self.stage = sr.placement.stage
        self.pp_ranks = sr.placement.pp_ranks
        self.pos = self.pp_ranks.index(sr.placement.global_rank)     # == stage - 1
        d = scenario.parallel.data
        full_m = m.global_batch // (m.micro_batch * d)
        self.m = micro_batches or full_m
        self.tokens = m.micro_batch * m.seq_len
        self.h = m.hidden
        self.compute = compute
        self.timeout_ns = int(timeout_s * 1e9)
        self.epoch = 0
        emulated = symmetric is not None
        if symmetric is None:
            rows = [[r - 1 for r in row] for row in self._pp_rows()]
            pg, _ = dist.new_subgroups_by_enumeration(rows)

            def symmetric(numel, dtype, device, zero=False, _pg=pg):
                return SymmetricTensor(numel, dtype, device, _pg, zero=zero)
        act = self.m * self.tokens * self.h
        self.fwd_in = symmetric(act, torch.bfloat16, self.device, True)
        self.bwd_in = symmetric(act, torch.bfloat16, self.device, True)
        self.flags = symmetric(2 * self.m, torch.int32, self.device, True)
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.trace: list = []     # compute=False: (op, micro, received tensor) for data-flow tests
        self.op_events: list = []  # timed=True: (op, micro, start, end) CUDA events per stage op
        self.timed = False
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.s_send = torch.cuda.Stream(device=self.device)
        # stand-in layer weights: views of the optimizer's bf16 params, per layer
        self.layers = self._layer_weights()
        self.x = torch.randn(self.tokens, self.h, device=self.device, dtype=torch.bfloat16)
        widths = (self.h, 3 * self.h, 4 * self.h)
        self.act = {w: torch.randn(self.tokens, w, device=self.device, dtype=torch.bfloat16) for w in widths}
        self.gout = {w: torch.randn(self.tokens, w, device=self.device, dtype=torch.bfloat16) * 1e-3
                     for w in widths}
        torch.cuda.synchronize(self.device)
        if not emulated:
            dist.barrier()

    # ------------------------------------------------------------ plumbing
    def _pp_rows(self):
        from .planner import plan_scenario

        return plan_scenario(self.s).plan.pp.rows

    def _layer_weights(self):
        gs = self.sr.gradset
        by_layer: dict[str, list[int]] = {}
        for i, t in enumerate(gs.tensors):
            if t.name.startswith("layers."):
                by_layer.setdefault(t.name.split(".")[1], []).append(i)
        return [by_layer[k] for k in sorted(by_layer, key=int)]

    def _own_slot(self, sym, k: int) -> torch.Tensor:
        """Micro-batch k's slot of this rank's receive buffer."""
        n = self.tokens * self.h
        return sym.tensor[k * n:(k + 1) * n].view(self.tokens, self.h)

    def _peer_slot_ptr(self, sym, q: int, k: int) -> int:
        """Device address of micro-batch k's slot in rank q's receive buffer
        (peer-mapped; a copy destination)."""
        return sym.peer(q, 2 * k * self.tokens * self.h)

    def _flag_ptr(self, q: int, kind: int, k: int) -> int:
        return self.flags.peer(q, 4 * (kind * self.m + k))

    def _send(self, kind: int, k: int, t: torch.Tensor) -> None:
        """kind 0: activation to the next stage; 1: gradient to the previous one."""
        q = self.pos + 1 if kind == 0 else self.pos - 1
        dst = self._peer_slot_ptr(self.fwd_in if kind == 0 else self.bwd_in, q, k)
        # copy engine over NVLink (one peer: ~0.75 TB/s, tools/ce_probe.py) on a
        # side stream: no SM leaves the stage's GEMMs for the hand-off, and the
        # stage's next op does not queue behind the copy
        t = t.contiguous()
        self.s_send.wait_stream(self.stream)
        t.record_stream(self.s_send)
        nat.call("hod_ce_copy", dst, t.data_ptr(), t.numel() * t.element_size(),
                 nat.stream_ptr(self.s_send))
        nat.call("hod_p2p_signal", self._flag_ptr(q, kind, k), self.epoch, nat.stream_ptr(self.s_send))

    def _recv(self, kind: int, k: int) -> torch.Tensor:
        nat.call("hod_p2p_wait", self._flag_ptr(self.pos, kind, k), self.epoch, self.timeout_ns,
                 self.err.data_ptr(), nat.stream_ptr(self.stream))
        return self._own_slot(self.fwd_in if kind == 0 else self.bwd_in, k)

    # ------------------------------------------------------------ compute
    def _forward(self, x: torch.Tensor) -> torch.Tensor:
        if not self.compute:
            return x + 1
        params = self.opt.params
        for qkv, proj, fc1, fc2 in self.layers:
            a = x @ params[qkv].t()                      # h -> 3h
            a = a[:, : self.h] @ params[proj].t()        # h -> h
            f = a @ params[fc1].t()                      # h -> 4h
            x = f @ params[fc2].t()                      # 4h -> h
        return x

    def _backward(self, dy: torch.Tensor, last: bool, grads) -> torch.Tensor:
        """dgrad + wgrad GEMMs per weight (twice the forward FLOPs); the chain of
        width-h activation gradients carries the received tensor through."""
        if not self.compute:
            if last:
                for layer in reversed(self.layers):
                    for i in reversed(layer):
                        self.opt.grad_ready(i, grads[i])
            return dy + 1
        params = self.opt.params
        for layer in reversed(self.layers):
            for i in reversed(layer):                                  # fc2, fc1, proj, qkv
                w = params[i]
                out_f, in_f = w.shape
                g = dy if out_f == self.h else self.gout[out_f]
                torch.matmul(g.t(), self.act[in_f], out=grads[i])      # wgrad (out x in)
                dx = g @ w                                             # dgrad (T x in)
                if in_f == self.h:
                    dy = dx
                if last:
                    self.opt.grad_ready(i, grads[i])
        return dy

    # ------------------------------------------------------------ iteration
    def run_iteration(self, grads, with_optimizer: bool = True) -> None:
        """One 1F1B iteration (+ the DP optimizer step of this stage)."""
        self.epoch += 1
        ops = _one_f_one_b(self.p, self.stage, self.m)
        outs = {}
        if with_optimizer:
            self.opt.begin_step()
            # embedding / head gradients are produced outside the GEMM chain
            for i, t in enumerate(self.sr.gradset.tensors):
                if not t.name.startswith("layers."):
                    self.opt.grad_ready(i, grads[i])
        for op, k in ops:
            idx = k - 1
            if self.timed:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            if op == "fwd":
                x = self.x if self.stage == 1 else self._recv(0, idx)
                if self.timed:
                    ev[0].record(self.stream)     # compute starts once the input is here
                if not self.compute and self.stage > 1:
                    self.trace.append(("fwd", k, x.clone()))
                y = self._forward(x)
                outs[idx] = y
                if self.stage < self.p:
                    self._send(0, idx, y)
            else:
                dy = outs.pop(idx) if self.stage == self.p else self._recv(1, idx)
                if self.timed:
                    ev[0].record(self.stream)
                if not self.compute and self.stage < self.p:
                    self.trace.append(("bwd", k, dy.clone()))
                dx = self._backward(dy, last=(with_optimizer and k == self.m), grads=grads)
                if self.stage > 1:
                    self._send(1, idx, dx)
            if self.timed:
                # the op's compute on this stage's stream (from its input's
                # arrival to its output's hand-off)
                ev[1].record(self.stream)
                self.op_events.append((op, k, ev[0], ev[1]))
        # the next iteration reuses the neighbours' receive slots: its sends
        # (and this iteration's end) are ordered after this iteration's sends
        self.stream.wait_stream(self.s_send)
        if with_optimizer:
            self.opt.finish_step()

    def check(self) -> None:
        if int(self.err.item()):
            from .errors import DeviceError

            raise DeviceError("pipeline hand-off timed out")
