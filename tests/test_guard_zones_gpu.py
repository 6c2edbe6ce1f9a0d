"""Out-of-bounds checks of every kernel without compute-sanitizer.

compute-sanitizer is refused on this GPU pool (profiles/r02_sanitizer_closed.txt),
so each C entry point runs on buffers embedded in guard zones:

* every OUTPUT buffer sits between two 64 KiB guard zones filled with a
  canary pattern: after the launch both zones must be byte-identical (no
  stray write, including by the bulk-copy engine of the TMA kernel);
* every INPUT buffer sits between guard zones of NaNs: a read past its end
  would pull NaNs into the result, which then no longer equals the oracle.

Sizes are odd (scalar tails, partial tiles and chunks, misaligned starts) —
exactly where an index bug would step outside.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_03549_b200 import _native as nat  # noqa: E402

DEV = "cuda"
GUARD_BYTES = 64 * 1024


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


class Guarded:
    """``n`` elements of ``dtype`` between two guard zones."""

    def __init__(self, n, dtype, role, fill=None, gen=None, scale=1.0, offset=0):
        esz = torch.empty(0, dtype=dtype).element_size()
        self.g = GUARD_BYTES // esz
        self.n = n
        self.full = torch.empty(self.g + offset + n + self.g, dtype=dtype, device=DEV)
        if role == "out":
            self.full.view(torch.uint8).fill_(0xA5)            # canary
        else:
            self.full.fill_(float("nan"))                       # reading these poisons the result
        lo = self.g + offset
        self.t = self.full[lo:lo + n]
        if fill is not None:
            self.t.copy_(fill)
        elif gen is not None:
            self.t.copy_((torch.randn(n, generator=gen, device=DEV) * scale).to(dtype))
        self.lo = lo
        self.before = self.full[:lo].clone()
        self.after = self.full[lo + n:].clone()

    def check(self, what):
        assert torch.equal(self.full[:self.lo].view(torch.uint8), self.before.view(torch.uint8)), \
            f"{what}: write before the buffer"
        assert torch.equal(self.full[self.lo + self.n:].view(torch.uint8), self.after.view(torch.uint8)), \
            f"{what}: write past the buffer"


@pytest.mark.parametrize("n,offset", [(1, 0), (255, 0), (257, 0), (4099, 1), (100_003, 3)])
def test_adamw_stays_inside_its_buffers(oracle, native, n, offset):
    gen = torch.Generator(device=DEV).manual_seed(n)
    master = Guarded(n, torch.float32, "io", gen=gen, scale=0.02, offset=offset)
    m = Guarded(n, torch.float32, "io", fill=torch.zeros(n), offset=offset)
    v = Guarded(n, torch.float32, "io", fill=torch.zeros(n), offset=offset)
    g = Guarded(n, torch.bfloat16, "in", gen=gen, scale=1e-3, offset=offset)
    p = Guarded(n, torch.bfloat16, "out", offset=offset)
    cm, cv, cp = (master.t.cpu().numpy().copy(), np.zeros(n, np.float32), np.zeros(n, np.float32))
    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)
    for buf in (master, m, v):     # in-place state: its zones are outputs too
        buf.full[:buf.lo].view(torch.uint8).fill_(0xA5)
        buf.full[buf.lo + n:].view(torch.uint8).fill_(0xA5)
        buf.before, buf.after = buf.full[:buf.lo].clone(), buf.full[buf.lo + n:].clone()
    nat.call("hod_adamw_bf16", master.t.data_ptr(), m.t.data_ptr(), v.t.data_ptr(), g.t.data_ptr(),
             p.t.data_ptr(), n, ctypes.byref(hp), None, 0)
    torch.cuda.synchronize()
    want = oracle.adamw(cm, cv, cp, u16(g.t), 1)
    np.testing.assert_array_equal(u16(p.t), want)
    for name, buf in (("master", master), ("m", m), ("v", v), ("param", p)):
        buf.check(f"adamw n={n} {name}")


@pytest.mark.parametrize("sizes", [[1], [7, 9], [4099, 65, 3], [100_003, 257]])
def test_pack_stays_inside_its_buffers(oracle, native, sizes):
    gen = torch.Generator(device=DEV).manual_seed(len(sizes))
    srcs = [Guarded(k, torch.bfloat16, "in", gen=gen, scale=1e-2) for k in sizes]
    offs, o = [], 0
    for k in sizes:
        offs.append(o)
        o += -(-k // 64) * 64                    # 64-element aligned starts, as the layout
    total = -(-o // 128) * 128
    bucket = Guarded(total, torch.bfloat16, "out")
    e = (nat.PackEntry * len(sizes))()
    for i, (s, off) in enumerate(zip(srcs, offs)):
        e[i].src, e[i].numel, e[i].dst_offset = s.t.data_ptr(), s.n, off
    nat.call("hod_pack_bf16", e, len(sizes), bucket.t.data_ptr(), total, ctypes.c_float(0.5), 0, 0)
    torch.cuda.synchronize()
    want = oracle.pack([u16(s.t) for s in srcs], offs, total, 0.5)
    np.testing.assert_array_equal(u16(bucket.t), want)
    bucket.check(f"pack {sizes}")


def test_norm_kernels_stay_inside_their_buffers(native):
    gen = torch.Generator(device=DEV).manual_seed(3)
    x = Guarded(100_003, torch.bfloat16, "in", gen=gen, scale=1e-2)
    parts = Guarded(nat.HOD_SUMSQ_PARTIALS, torch.float32, "out")
    nat.call("hod_sumsq_bf16", x.t.data_ptr(), x.n, parts.t.data_ptr(), 0)
    out = Guarded(1, torch.float32, "out")
    nat.call("hod_sum_partials", parts.t.data_ptr(), nat.HOD_SUMSQ_PARTIALS, out.t.data_ptr(), 0)
    coef, norm = Guarded(1, torch.float32, "out"), Guarded(1, torch.float32, "out")
    nat.call("hod_clip_coef", out.t.data_ptr(), ctypes.c_float(0.5), coef.t.data_ptr(), norm.t.data_ptr(), 0)
    torch.cuda.synchronize()
    want = float((x.t.float().double() ** 2).sum())
    assert abs(float(out.t.item()) - want) <= 1e-5 * want
    for name, buf in (("partials", parts), ("sum", out), ("coef", coef), ("norm", norm)):
        buf.check(name)


@pytest.mark.parametrize("kernel", ["tma", "register"])
@pytest.mark.parametrize("d", [2, 4])
@pytest.mark.parametrize("mode", ["fused", "rs", "adamw_ag"])
def test_span_kernels_stay_inside_their_buffers(oracle, native, kernel, d, mode):
    """One emulated span launch (all d ranks' buffers on this GPU, flags
    pre-set) over two buckets with odd shard sizes: every peer's grad and
    param buffer and the state between guard zones; results vs the oracle."""
    nat.call("hod_set_span_tma", 1 if kernel == "tma" else 0)
    try:
        shards = [2048 * 3 + 8, 520]                   # partial tiles / chunks
        numels = [s * d for s in shards]
        starts = [0, -(-numels[0] // 64) * 64]
        total = starts[1] + numels[1]
        n_owned = sum(shards)
        gen = torch.Generator(device=DEV).manual_seed(d)
        # grads: read by every rank (inputs) and, for RS / keep_reduced, the
        # own shard written in place: canary zones around the whole buffer
        grads = [Guarded(total, torch.bfloat16, "out") for _ in range(d)]
        for g in grads:
            g.t.copy_((torch.randn(total, generator=gen, device=DEV) * 1e-3).to(torch.bfloat16))
        params = [Guarded(total, torch.bfloat16, "out") for _ in range(d)]
        master = Guarded(n_owned, torch.float32, "out")
        master.t.copy_(torch.randn(n_owned, generator=gen, device=DEV) * 0.02)
        m = Guarded(n_owned, torch.float32, "out")
        m.t.zero_()
        v = Guarded(n_owned, torch.float32, "out")
        v.t.zero_()
        parts = Guarded(nat.HOD_SUMSQ_PARTIALS, torch.float32, "out")
        coef = torch.tensor([0.75], device=DEV)
        flags = [torch.full((64,), 1 << 32, dtype=torch.int64, device=DEV) for _ in range(d)]
        err = torch.zeros(1, dtype=torch.int32, device=DEV)
        for buf in grads + params + [master, m, v, parts]:
            buf.before, buf.after = buf.full[:buf.lo].clone(), buf.full[buf.lo + buf.n:].clone()
        host_packs = [u16(g.t) for g in grads]
        cm, cv, cp = master.t.cpu().numpy().copy(), np.zeros(n_owned, np.float32), np.zeros(n_owned, np.float32)
        sp = nat.P2PSpan()
        for q in range(d):
            sp.grad[q], sp.param[q], sp.flags[q] = grads[q].t.data_ptr(), params[q].t.data_ptr(), flags[q].data_ptr()
        sp.local_grad = grads[0].t.data_ptr()
        sp.master, sp.exp_avg, sp.exp_avg_sq = master.t.data_ptr(), m.t.data_ptr(), v.t.data_ptr()
        sp.err = err.data_ptr()
        for k in range(2):
            sp.bucket_start[k], sp.shard_numel[k] = starts[k], shards[k]
        sp.n_buckets, sp.d, sp.rank, sp.nvls, sp.keep_reduced = 2, d, 0, 0, 1
        sp.slot, sp.epoch, sp.timeout_ns = 0, 1, 5_000_000_000
        hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)
        if mode == "rs":
            sp.partials = parts.t.data_ptr()
        reduced = [oracle.reduce_scatter([hpk[starts[k]:starts[k] + numels[k]] for hpk in host_packs], 0, d)
                   for k in range(2)]
        if mode == "adamw_ag":
            # the update half reads the reduced shard kept in place
            for k in range(2):
                grads[0].t[starts[k]:starts[k] + shards[k]].copy_(
                    torch.from_numpy(reduced[k].view(np.int16)).to(DEV).view(torch.bfloat16))
            sp.clip_coef = coef.data_ptr()
        mnum = {"fused": nat.HOD_P2P_FUSED, "rs": nat.HOD_P2P_RS, "adamw_ag": nat.HOD_P2P_ADAMW_AG}[mode]
        nat.call("hod_p2p_step", ctypes.byref(sp), mnum, ctypes.byref(hp), 0)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        own = u16(grads[0].t)
        s0 = 0
        for k in range(2):
            if mode != "adamw_ag":
                np.testing.assert_array_equal(own[starts[k]:starts[k] + shards[k]], reduced[k])
            if mode != "rs":
                sl = slice(s0, s0 + shards[k])
                want = oracle.adamw(cm[sl], cv[sl], cp[sl], reduced[k], 1,
                                    coef=0.75 if mode == "adamw_ag" else None)
                for q in range(d):
                    np.testing.assert_array_equal(u16(params[q].t)[starts[k]:starts[k] + shards[k]], want)
            s0 += shards[k]
        for i, buf in enumerate(grads):
            buf.check(f"grad[{i}]")
        for i, buf in enumerate(params):
            buf.check(f"param[{i}]")
        for name, buf in (("master", master), ("m", m), ("v", v), ("partials", parts)):
            buf.check(name)
    finally:
        nat.call("hod_set_span_tma", 1)


def test_guard_zone_harness_detects_a_stray_write():
    """The harness itself: one element written past the end is caught."""
    buf = Guarded(1000, torch.float32, "out")
    buf.full[buf.lo + buf.n].fill_(1.0)
    with pytest.raises(AssertionError, match="past the buffer"):
        buf.check("self-test")
