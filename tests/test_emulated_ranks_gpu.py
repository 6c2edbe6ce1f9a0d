"""All DP degrees of the fused p2p kernels on ONE GPU, ranks emulated in turn.

The box used for development has at most 4 GPUs, but the driver's scaling run
uses 8.  Here every rank's buffers live on the same device: for rank r the
barrier flags of all d "peers" are pre-set (everybody has already arrived),
so each launch runs straight through — no kernel ever waits on another
(the launches are sequential in one stream) — while the kernel executes the
exact d-way code path (the D = 2/4/8 template instantiations and the generic
d path for 3, 5, 6, 7): reduce-scatter from d bucket copies, AdamW, and the
all-gather stores into d param copies.  Checked bit-exactly against the oracle.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.buckets import build_bucket_layout  # noqa: E402
from paper_2312_03549_b200.gradsets import odd_tensors  # noqa: E402

DEV = "cuda"


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.fixture(params=["tma", "register"])
def span_kernel(request, native):
    """Both span kernels: the TMA-fed one (default for full-GPU launches) and
    the register-streaming one (co-resident launches, NVLS)."""
    nat.call("hod_set_span_tma", 1 if request.param == "tma" else 0)
    yield request.param
    nat.call("hod_set_span_tma", 1)


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("clip", [None, 0.02])
def test_emulated_d_way_fused_step(oracle, native, span_kernel, d, clip):
    gs = odd_tensors()
    L = build_bucket_layout(gs.numels, 200_000, dp=d)
    total, nb = L.total_numel, len(L.buckets)
    gen = torch.Generator(device=DEV).manual_seed(100 + d)
    packs = [torch.randn(total, generator=gen, device=DEV).mul_(1e-3).to(torch.bfloat16) for _ in range(d)]
    grads = [p.clone() for p in packs]      # per-rank grad buffers (RS writes in place)
    params = [torch.zeros(total, dtype=torch.bfloat16, device=DEV) for _ in range(d)]
    flags = [torch.zeros((2 * nb + 1) * 8, dtype=torch.int64, device=DEV) for _ in range(d)]
    shard_total = total // d
    state = [[torch.randn(shard_total, generator=gen, device=DEV).mul_(0.02),
              torch.rand(shard_total, generator=gen, device=DEV).mul_(1e-3),
              torch.rand(shard_total, generator=gen, device=DEV).mul_(1e-6)] for _ in range(d)]
    cpu_state = [[x.cpu().numpy().copy() for x in st] for st in state]
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    partials = torch.zeros(d, nb * nat.HOD_SUMSQ_PARTIALS, device=DEV)
    coef = torch.tensor([1.0], device=DEV)
    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)
    offs = L.shard_offsets()
    spans = [[b.index] for b in L.buckets]
    if nb >= 3:
        spans = [[0, 1], list(range(2, nb))]    # exercise multi-bucket spans too

    def span_struct(r, span):
        sp = nat.P2PSpan()
        for q in range(d):
            sp.grad[q], sp.param[q], sp.flags[q] = grads[q].data_ptr(), params[q].data_ptr(), flags[q].data_ptr()
        sp.local_grad = grads[r].data_ptr()
        o = offs[span[0]]
        sp.master, sp.exp_avg, sp.exp_avg_sq = (x.data_ptr() + 4 * o for x in state[r])
        sp.err = err.data_ptr()
        for k, bi in enumerate(span):
            sp.bucket_start[k], sp.shard_numel[k] = L.buckets[bi].start, L.buckets[bi].numel // d
        sp.n_buckets, sp.d, sp.rank, sp.nvls, sp.keep_reduced = len(span), d, r, 0, 1
        sp.slot, sp.epoch, sp.timeout_ns = span[0], 1, 5_000_000_000
        sp.tag = nat.span_tag(span[0], span[-1])
        return sp

    def arrive_all(slot):
        for q in range(d):
            tag = nat.span_tag(slot, next(sp_[-1] for sp_ in spans if sp_[0] == slot))
            flags[q].view(-1, 8)[slot, :d] = (1 << 32) | tag   # every peer has signalled epoch 1

    if clip is None:
        for span in spans:
            arrive_all(span[0])
            for r in range(d):
                nat.call("hod_p2p_step", ctypes.byref(span_struct(r, span)), nat.HOD_P2P_FUSED,
                         ctypes.byref(hp), 0)
    else:
        for span in spans:
            arrive_all(span[0])
            for r in range(d):
                sp = span_struct(r, span)
                sp.partials = partials[r].data_ptr() + 4 * nat.HOD_SUMSQ_PARTIALS * span[0]
                nat.call("hod_p2p_step", ctypes.byref(sp), nat.HOD_P2P_RS, ctypes.byref(hp), 0)
        torch.cuda.synchronize()
        ss = float(partials.double().sum())
        coef.fill_(min(1.0, clip / (np.sqrt(np.float32(ss)) + 1e-6)))
        for span in spans:
            for r in range(d):
                sp = span_struct(r, span)
                sp.clip_coef = coef.data_ptr()
                nat.call("hod_p2p_step", ctypes.byref(sp), nat.HOD_P2P_ADAMW_AG, ctypes.byref(hp), 0)
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    for q in range(1, d):
        assert torch.equal(params[q].view(torch.int16), params[0].view(torch.int16))
    host_packs = [u16(p) for p in packs]
    full = u16(params[0])
    cf = float(coef.item()) if clip is not None else None
    for bi, b in enumerate(L.buckets):
        bucket_packs = [hp_[b.start:b.start + b.numel] for hp_ in host_packs]
        n = b.numel // d
        for r in range(d):
            red = oracle.reduce_scatter(bucket_packs, r, d)
            np.testing.assert_array_equal(u16(grads[r])[b.start + r * n:b.start + (r + 1) * n], red)
            master, m, v = (x[offs[bi]:offs[bi] + n] for x in cpu_state[r])
            want = oracle.adamw(master, m, v, red, 1, coef=cf)
            np.testing.assert_array_equal(full[b.start + r * n:b.start + (r + 1) * n], want)
            dev_master = state[r][0][offs[bi]:offs[bi] + n].cpu().numpy()
            np.testing.assert_array_equal(dev_master.view(np.uint32), master.view(np.uint32))
