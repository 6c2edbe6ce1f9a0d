"""K1/K2/K3 sm_100a kernels vs the CPU oracle, through the C ABI (bit-exact).

Every comparison is on identical inputs: tensors are generated once and the
same bytes are handed to the device kernel and to oracle/hod_oracle.c.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.buckets import build_bucket_layout  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset, odd_tensors  # noqa: E402

DEV = "cuda"


def u16(t):
    """bf16 tensor -> numpy uint16 bit pattern."""
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def pack_gpu(grads, slots, bucket_numel, scale):
    bucket = torch.full((bucket_numel,), 7.0, dtype=torch.bfloat16, device=DEV)  # garbage
    entries = (nat.PackEntry * len(slots))()
    for k, (g, off) in enumerate(zip(grads, slots)):
        entries[k].src, entries[k].numel, entries[k].dst_offset = g.data_ptr(), g.numel(), off
    dtype = nat.HOD_DTYPE_F32 if grads[0].dtype == torch.float32 else nat.HOD_DTYPE_BF16
    nat.call("hod_pack_bf16", entries, len(slots), bucket.data_ptr(), bucket_numel,
             ctypes.c_float(scale), dtype, 0)
    torch.cuda.synchronize()
    return bucket


@pytest.mark.parametrize("src_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("scale", [1.0, 0.5, 1.0 / 3.0])
def test_pack_bit_exact_odd_sizes(oracle, native, src_dtype, scale):
    gs = odd_tensors()
    layout = build_bucket_layout(gs.numels, 150_000, dp=3)
    gen = torch.Generator(device=DEV).manual_seed(5)
    grads = [torch.randn(t.shape, generator=gen, device=DEV).mul_(1e-2).to(src_dtype)
             for t in gs.tensors]
    for b in layout.buckets:
        gl = [grads[s.index].reshape(-1) for s in b.slots]
        offs = [s.offset for s in b.slots]
        got = u16(pack_gpu(gl, offs, b.numel, scale))
        cpu = [g.cpu().numpy() if src_dtype == torch.float32 else u16(g) for g in gl]
        want = oracle.pack(cpu, offs, b.numel, scale)
        np.testing.assert_array_equal(got, want)


def test_pack_many_entries_splits_windows(oracle, native):
    # 150 tiny tensors -> more than HOD_PACK_MAX_ENTRIES per bucket
    numels = [64 * (1 + (i % 5)) for i in range(150)]
    layout = build_bucket_layout(numels, 10**9, dp=1)
    (b,) = layout.buckets
    gen = torch.Generator(device=DEV).manual_seed(9)
    grads = [torch.randn(n, generator=gen, device=DEV).to(torch.bfloat16) for n in numels]
    gl = [grads[s.index] for s in b.slots]
    offs = [s.offset for s in b.slots]
    got = u16(pack_gpu(gl, offs, b.numel, 0.25))
    want = oracle.pack([u16(g) for g in gl], offs, b.numel, 0.25)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("src_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("clip", [None, 0.3])
def test_pack_adamw_fused_equals_pack_then_adamw(oracle, native, src_dtype, clip):
    """K1+K2 fused (d == 1) is bit-identical to pack -> AdamW on the bucket."""
    gs = odd_tensors()
    layout = build_bucket_layout(gs.numels, 150_000, dp=1)
    gen = torch.Generator(device=DEV).manual_seed(21)
    grads = [torch.randn(t.shape, generator=gen, device=DEV).mul_(1e-2).to(src_dtype) for t in gs.tensors]
    coef = None if clip is None else torch.tensor([clip], device=DEV)
    for b in layout.buckets:
        gl = [grads[s.index].reshape(-1) for s in b.slots]
        offs = [s.offset for s in b.slots]
        master = torch.randn(b.numel, generator=gen, device=DEV).mul_(0.02)
        m = torch.rand(b.numel, generator=gen, device=DEV).mul_(1e-3)
        v = torch.rand(b.numel, generator=gen, device=DEV).mul_(1e-6)
        cm, cv, cp = master.cpu().numpy().copy(), m.cpu().numpy().copy(), v.cpu().numpy().copy()
        out = torch.empty(b.numel, dtype=torch.bfloat16, device=DEV)
        entries = (nat.PackEntry * len(gl))()
        for k, (g, off) in enumerate(zip(gl, offs)):
            entries[k].src, entries[k].numel, entries[k].dst_offset = g.data_ptr(), g.numel(), off
        hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 7)
        dt = nat.HOD_DTYPE_F32 if src_dtype == torch.float32 else nat.HOD_DTYPE_BF16
        nat.call("hod_pack_adamw", entries, len(gl), b.numel, ctypes.c_float(0.5), dt, master.data_ptr(),
                 m.data_ptr(), v.data_ptr(), out.data_ptr(), ctypes.byref(hp),
                 None if coef is None else coef.data_ptr(), 0)
        torch.cuda.synchronize()
        cpu = [g.cpu().numpy() if src_dtype == torch.float32 else u16(g) for g in gl]
        packed = oracle.pack(cpu, offs, b.numel, 0.5)
        want = oracle.adamw(cm, cv, cp, packed, 7, coef=None if clip is None else np.float32(clip))
        np.testing.assert_array_equal(u16(out), want)
        np.testing.assert_array_equal(master.cpu().numpy().view(np.uint32), cm.view(np.uint32))
        np.testing.assert_array_equal(v.cpu().numpy().view(np.uint32), cp.view(np.uint32))


def _adamw_gpu(master, m, v, grad, n, step, coef=None, out_offset=0, mode=0):
    out = torch.empty(n + out_offset, dtype=torch.bfloat16, device=DEV)
    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, step, mode)
    fn = "hod_adamw_f32" if grad.dtype == torch.float32 else "hod_adamw_bf16"
    coef_ptr = None if coef is None else coef.data_ptr()
    nat.call(fn, master.data_ptr(), m.data_ptr(), v.data_ptr(), grad.data_ptr(),
             out[out_offset:].data_ptr(), n, ctypes.byref(hp), coef_ptr, 0)
    return out[out_offset:]


@pytest.mark.parametrize("n,offset", [(1, 0), (7, 0), (8, 0), (4099, 0), (1_000_003, 0),
                                      (65_536, 1), (33_333, 3)])
@pytest.mark.parametrize("grad_dtype", [torch.bfloat16, torch.float32])
def test_adamw_bit_exact_100_steps(oracle, native, n, offset, grad_dtype):
    gen = torch.Generator(device=DEV).manual_seed(n)
    base = torch.randn(n + offset, generator=gen, device=DEV).mul_(0.02)
    master = base[offset:].clone() if offset == 0 else base[offset:]   # offset => misaligned path
    m = torch.zeros(n + offset, device=DEV)[offset:]
    v = torch.zeros(n + offset, device=DEV)[offset:]
    cm, cv, cp = (master.cpu().numpy().copy(), np.zeros(n, np.float32), np.zeros(n, np.float32))
    for step in range(1, 101):
        g = torch.randn(n + offset, generator=gen, device=DEV).mul_(1e-3).to(grad_dtype)[offset:]
        p = _adamw_gpu(master, m, v, g, n, step)
        gc = g.cpu().numpy() if grad_dtype == torch.float32 else u16(g)
        want_p = oracle.adamw(cm, cv, cp, gc, step)
        if step in (1, 2, 50, 100):
            torch.cuda.synchronize()
            np.testing.assert_array_equal(master.cpu().numpy().view(np.uint32), cm.view(np.uint32))
            np.testing.assert_array_equal(m.cpu().numpy().view(np.uint32), cv.view(np.uint32))
            np.testing.assert_array_equal(v.cpu().numpy().view(np.uint32), cp.view(np.uint32))
            np.testing.assert_array_equal(u16(p), want_p)


def _norm_rel(gpu, cpu):
    """SURVEY §8d pass rule: ||gpu - cpu||_inf / ||cpu||_inf."""
    gpu, cpu = np.asarray(gpu, np.float64), np.asarray(cpu, np.float64)
    return float(np.abs(gpu - cpu).max() / max(np.abs(cpu).max(), 1e-30))


@pytest.mark.parametrize("n,offset", [(1_000_003, 0), (65_536, 1)])
@pytest.mark.parametrize("clip", [None, 0.37])
def test_adamw_fast_mode_within_north_star_tolerance(oracle, native, n, offset, clip):
    """HOD_ADAMW_FAST (FMAs, MUFU sqrt / reciprocal) against the exact oracle:
    master / m / v within 1e-6 norm-relative after 1 step and 1e-5 after
    100 (the north star's tolerance, SURVEY §8d rule); the bf16 params are
    the RNE of the device's own master."""
    gen = torch.Generator(device=DEV).manual_seed(n + 5)
    base = torch.randn(n + offset, generator=gen, device=DEV).mul_(0.02)
    master = base[offset:].clone() if offset == 0 else base[offset:]
    m = torch.zeros(n + offset, device=DEV)[offset:]
    v = torch.zeros(n + offset, device=DEV)[offset:]
    coef = None if clip is None else torch.tensor([clip], device=DEV)
    cm, cv, cp = (master.cpu().numpy().copy(), np.zeros(n, np.float32), np.zeros(n, np.float32))
    worst = {}
    for step in range(1, 101):
        g = torch.randn(n + offset, generator=gen, device=DEV).mul_(1e-3).to(torch.bfloat16)[offset:]
        p = _adamw_gpu(master, m, v, g, n, step, coef=coef, mode=nat.HOD_ADAMW_FAST)
        oracle.adamw(cm, cv, cp, u16(g), step, coef=None if clip is None else np.float32(clip))
        if step in (1, 100):
            torch.cuda.synchronize()
            rtol = 1e-6 if step == 1 else 1e-5
            for name, dev_t, ref in (("master", master, cm), ("m", m, cv), ("v", v, cp)):
                err = _norm_rel(dev_t.cpu().numpy(), ref)
                worst[f"{name}@{step}"] = err
                assert err <= rtol, (name, step, err)
            assert torch.equal(p.view(torch.int16), master.to(torch.bfloat16).view(torch.int16))
    print("fast-mode norm-relative errors", worst)


def test_adamw_with_clip_coef(oracle, native):
    n = 100_000
    gen = torch.Generator(device=DEV).manual_seed(3)
    master = torch.randn(n, generator=gen, device=DEV).mul_(0.02)
    m, v = torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)
    g = torch.randn(n, generator=gen, device=DEV).to(torch.bfloat16)
    coef = torch.tensor([0.37], device=DEV)
    cm, cv, cp = master.cpu().numpy().copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    p = _adamw_gpu(master, m, v, g, n, 1, coef=coef)
    want = oracle.adamw(cm, cv, cp, u16(g), 1, coef=np.float32(0.37))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u16(p), want)
    np.testing.assert_array_equal(master.cpu().numpy(), cm)


def test_sumsq_deterministic_and_close(oracle, native):
    n = 3_000_017
    gen = torch.Generator(device=DEV).manual_seed(11)
    x = torch.randn(n, generator=gen, device=DEV).to(torch.bfloat16)
    parts = torch.empty(nat.HOD_SUMSQ_PARTIALS, device=DEV)
    out = torch.empty(2, device=DEV)
    for k in range(2):
        nat.call("hod_sumsq_bf16", x.data_ptr(), n, parts.data_ptr(), 0)
        nat.call("hod_sum_partials", parts.data_ptr(), nat.HOD_SUMSQ_PARTIALS, out[k:].data_ptr(), 0)
    torch.cuda.synchronize()
    a, b = out.cpu().numpy()
    assert a == b  # bit-reproducible
    want = oracle.sumsq_bf16(u16(x))
    assert abs(a - want) <= 1e-5 * want
    # clip coefficient from the same sumsq is bit-exact
    coef = torch.empty(1, device=DEV)
    nrm = torch.empty(1, device=DEV)
    nat.call("hod_clip_coef", out.data_ptr(), ctypes.c_float(1.0), coef.data_ptr(), nrm.data_ptr(), 0)
    torch.cuda.synchronize()
    assert coef.item() == oracle.clip_coef(np.float32(a), 1.0)


@pytest.mark.parametrize("src_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("scale", [1.0, 1.0 / 3.0])
def test_pack_sumsq_matches_packed_norm(oracle, native, src_dtype, scale):
    """hod_pack_sumsq (d = 1 clip norm read straight from the tensors) equals the
    sum of squares of the oracle's packed bucket, gaps and padding included."""
    gs = odd_tensors()
    layout = build_bucket_layout(gs.numels, 150_000, dp=1)
    gen = torch.Generator(device=DEV).manual_seed(9)
    grads = [torch.randn(t.shape, generator=gen, device=DEV).mul_(1e-2).to(src_dtype)
             for t in gs.tensors]
    parts = torch.empty(nat.HOD_SUMSQ_PARTIALS, device=DEV)
    out = torch.empty(2, device=DEV)
    for b in layout.buckets:
        gl = [grads[s.index].reshape(-1) for s in b.slots]
        offs = [s.offset for s in b.slots]
        entries = (nat.PackEntry * len(gl))()
        for k, (g, off) in enumerate(zip(gl, offs)):
            entries[k].src, entries[k].numel, entries[k].dst_offset = g.data_ptr(), g.numel(), off
        dtype = nat.HOD_DTYPE_F32 if src_dtype == torch.float32 else nat.HOD_DTYPE_BF16
        for k in range(2):
            nat.call("hod_pack_sumsq", entries, len(gl), b.numel, ctypes.c_float(scale), dtype,
                     parts.data_ptr(), 0)
            nat.call("hod_sum_partials", parts.data_ptr(), nat.HOD_SUMSQ_PARTIALS, out[k:].data_ptr(), 0)
        torch.cuda.synchronize()
        a, a2 = out.cpu().numpy()
        assert a == a2  # bit-reproducible
        cpu = [g.cpu().numpy() if src_dtype == torch.float32 else u16(g) for g in gl]
        want = oracle.sumsq_bf16(oracle.pack(cpu, offs, b.numel, scale))
        assert abs(a - want) <= 1e-5 * want


def test_survey_spellings_match(oracle, native):
    """hod_adamw (scalar args) and hod_sumsq (accumulating) — the SURVEY §8b
    spellings — give the same bits as hod_adamw_bf16 / hod_sumsq_bf16."""
    n = 1_000_003
    gen = torch.Generator(device=DEV).manual_seed(21)
    g = (torch.randn(n, generator=gen, device=DEV) * 1e-3).to(torch.bfloat16)
    st = [torch.randn(n, generator=gen, device=DEV) * 0.02, torch.zeros(n, device=DEV), torch.zeros(n, device=DEV)]
    st2 = [t.clone() for t in st]
    p1 = torch.empty(n, dtype=torch.bfloat16, device=DEV)
    p2 = torch.empty_like(p1)
    f = [float(np.float32(x)) for x in (1e-4, 0.9, 0.95, 1e-8, 0.1)]
    hp = nat.AdamWParams(*f, 1)
    nat.call("hod_adamw_bf16", *[t.data_ptr() for t in st], g.data_ptr(), p1.data_ptr(), n, ctypes.byref(hp), None, 0)
    nat.call("hod_adamw", *[t.data_ptr() for t in st2], g.data_ptr(), p2.data_ptr(), n, *f, 1, None, 0)
    torch.cuda.synchronize()
    for a, b in zip(st + [p1], st2 + [p2]):
        assert torch.equal(a.view(torch.int32) if a.dtype == torch.float32 else a.view(torch.int16),
                           b.view(torch.int32) if b.dtype == torch.float32 else b.view(torch.int16))
    parts = torch.empty(nat.HOD_SUMSQ_PARTIALS, device=DEV)
    ref = torch.empty(1, device=DEV)
    nat.call("hod_sumsq_bf16", g.data_ptr(), n, parts.data_ptr(), 0)
    nat.call("hod_sum_partials", parts.data_ptr(), nat.HOD_SUMSQ_PARTIALS, ref.data_ptr(), 0)
    acc = torch.zeros(1, device=DEV)
    nat.call("hod_sumsq", g.data_ptr(), n, acc.data_ptr(), 0)
    torch.cuda.synchronize()
    assert acc.item() == ref.item()
    nat.call("hod_sumsq", g.data_ptr(), n, acc.data_ptr(), 0)
    torch.cuda.synchronize()
    assert acc.item() == 2 * ref.item()


def test_bad_arguments_raise_device_error(native):
    from paper_2312_03549_b200.errors import DeviceError

    hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 0)  # step 0 is invalid
    x = torch.zeros(16, device=DEV)
    with pytest.raises(DeviceError, match="step"):
        nat.call("hod_adamw_f32", x.data_ptr(), x.data_ptr(), x.data_ptr(), x.data_ptr(),
                 x.data_ptr(), 16, ctypes.byref(hp), None, 0)


def test_layout_of_gpt13b_stage_is_padding_free():
    for stage in (1, 2):
        gs = config_gradset("gpt13b", stage)
        L = build_bucket_layout(gs.numels, 25_000_000, dp=4)
        assert L.padding == 0
