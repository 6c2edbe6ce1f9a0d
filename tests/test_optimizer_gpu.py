"""DistributedOptimizer (d = 1 on one GPU) vs the oracle's whole-step restatement.

Multi-rank parity (d = 2/4/8) lives in tests/test_multigpu_gpu.py.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_03549_b200 import DistributedOptimizer  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402

DEV = "cuda"


def u16(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def _oracle_state(oracle, layout, params_cpu):
    """Per-bucket [(master, m, v)] for a single rank from fp32 initial params."""
    state = []
    for b in layout.buckets:
        flat = np.zeros(b.numel, np.float32)
        for s in b.slots:
            flat[s.offset:s.offset + s.numel] = params_cpu[s.index].reshape(-1)
        state.append([(flat, np.zeros(b.numel, np.float32), np.zeros(b.numel, np.float32))])
    return state


@pytest.mark.parametrize("keep_reduced", [False, True])   # False: K1+K2 fused at d = 1
@pytest.mark.parametrize("config,grad_dtype,clip,bucket",
                         [("toy", torch.float32, None, 25_000_000),
                          ("toy", torch.bfloat16, 1.0, 2_000_000),
                          ("odd", torch.bfloat16, 0.01, 100_000),
                          ("odd", torch.float32, None, 10**9),
                          ("odd", torch.bfloat16, None, 70_000)])
def test_single_rank_steps_match_oracle(oracle, native, config, grad_dtype, clip, bucket, keep_reduced):
    gs = config_gradset(config)
    p0 = init_params(gs, DEV)
    opt = DistributedOptimizer(p0, bucket_size=bucket, clip=clip, keep_reduced=keep_reduced)
    L = opt.layout
    state = _oracle_state(oracle, L, [p.cpu().numpy() for p in p0])
    for step in (1, 2, 3):
        grads = make_grads(gs, step, 0, DEV, dtype=grad_dtype)
        rep = opt.step(grads)
        torch.cuda.synchronize()
        gcpu = [[g.cpu().numpy() if grad_dtype == torch.float32 else u16(g) for g in grads]]
        params, norm = oracle.step_all_ranks(gcpu, [
            {"params": [(s.index, s.offset, s.numel) for s in b.slots], "numel": b.numel}
            for b in L.buckets], state, step, opt.lr, opt.betas, opt.eps, opt.weight_decay,
            clip=clip)
        if clip is not None:
            got = rep.resolve()
            assert abs(got["grad_norm"] - norm) <= 1e-5 * norm
            # the coefficient the device used is fed back: AdamW parity is exact
        pb = u16(opt.param_buffer)
        for bi, b in enumerate(L.buckets):
            master, m, v = state[bi][0]
            off = L.shard_offsets()[bi]
            dev_master = opt.master[off:off + b.numel].cpu().numpy()
            if clip is None:
                np.testing.assert_array_equal(pb[b.start:b.start + b.numel], params[bi])
                np.testing.assert_array_equal(dev_master, master)
            else:
                # clip coefficient differs by <= 1 ulp (norm order) => 1e-6 relative
                np.testing.assert_allclose(dev_master, master, rtol=1e-6, atol=1e-6 * np.abs(master).max())
                np.testing.assert_allclose(opt.exp_avg[off:off + b.numel].cpu().numpy(), m,
                                           rtol=1e-6, atol=1e-6 * np.abs(m).max())
        # model views alias the flat buffer
        for i, p in enumerate(opt.params):
            s = L.slot(i)
            b = L.buckets[s.bucket]
            assert p.data_ptr() == opt.param_buffer.data_ptr() + 2 * (b.start + s.offset)
    opt.close()


def test_padding_stays_zero_and_params_alias(native):
    gs = config_gradset("odd")
    opt = DistributedOptimizer(init_params(gs, DEV), bucket_size=50_000, keep_reduced=True)
    opt.step(make_grads(gs, 1, 0, DEV))
    torch.cuda.synchronize()
    pad_mask = torch.ones(opt.layout.total_numel, dtype=torch.bool, device=DEV)
    for b in opt.layout.buckets:
        for s in b.slots:
            pad_mask[b.start + s.offset:b.start + s.offset + s.numel] = False
    assert torch.count_nonzero(opt.grad_buffer[pad_mask]).item() == 0
    assert torch.count_nonzero(opt.param_buffer[pad_mask]).item() == 0


@pytest.mark.parametrize("clip", [None, 1.0])
def test_host_gradient_steps_match_resident(native, clip):
    """step() fed from pinned HOST gradients (the e2e path: H2D into reused
    staging buffers) equals the resident-gradient step over several steps
    with a different gradient set each step — the uploads of step k+1 must
    not overwrite staging that step k's packs still read."""
    gs = config_gradset("toy")
    p0 = init_params(gs, DEV)
    a = DistributedOptimizer(p0, bucket_size=2_000_000, clip=clip)
    b = DistributedOptimizer(p0, bucket_size=2_000_000, clip=clip)
    for step in (1, 2, 3, 4):
        grads = make_grads(gs, step, 0, DEV)
        host = [g.cpu().pin_memory() for g in grads]
        a.step(grads)
        b.step(host)
    torch.cuda.synchronize()
    assert torch.equal(a.param_buffer, b.param_buffer)
    assert torch.equal(a.master, b.master)
    a.close()
    b.close()


@pytest.mark.parametrize("clip", [None, 0.5])
@pytest.mark.parametrize("keep_reduced", [False, True])
def test_ragged_and_empty_tensors_match_oracle(oracle, native, clip, keep_reduced):
    """Zero-element, single-element and odd-sized tensors (empty slots, padding
    tails, buckets that hold only padding) through the whole d = 1 step."""
    shapes = [(0,), (1,), (3, 5), (0, 7), (129,), (64,), (2, 63), (1000,), (0,)]
    g = torch.Generator(device="cpu").manual_seed(7)
    p0 = [(torch.randn(s, generator=g) * 0.02).to(DEV) for s in shapes]
    opt = DistributedOptimizer(p0, bucket_size=100, clip=clip, keep_reduced=keep_reduced)
    L = opt.layout
    state = _oracle_state(oracle, L, [p.cpu().numpy() for p in p0])
    for step in (1, 2):
        grads = [(torch.randn(s, generator=g) * 1e-3).to(torch.bfloat16).to(DEV) for s in shapes]
        opt.step(grads)
        torch.cuda.synchronize()
        params, _ = oracle.step_all_ranks([[u16(x) for x in grads]], [
            {"params": [(s.index, s.offset, s.numel) for s in b.slots], "numel": b.numel}
            for b in L.buckets], state, step, opt.lr, opt.betas, opt.eps, opt.weight_decay, clip=clip)
        pb = u16(opt.param_buffer)
        for bi, b in enumerate(L.buckets):
            if clip is None:
                np.testing.assert_array_equal(pb[b.start:b.start + b.numel], params[bi])
            else:
                master = state[bi][0][0]
                off = L.shard_offsets()[bi]
                np.testing.assert_allclose(opt.master[off:off + b.numel].cpu().numpy(), master,
                                           rtol=1e-6, atol=1e-6 * max(1e-30, np.abs(master).max()))
    for i, p in enumerate(opt.params):
        assert tuple(p.shape) == shapes[i]
    opt.close()


def test_empty_parameter_list_is_rejected(native):
    from paper_2312_03549_b200.errors import InfeasibleConfigError

    with pytest.raises(InfeasibleConfigError):
        DistributedOptimizer([])


@pytest.mark.parametrize("clip", [0.01, None])
def test_long_pack_table_bucket_beside_short_one(oracle, native, clip):
    """d = 1: one bucket holding 71 tensors (> HOD_PACK_MAX_ENTRIES, windowed
    norm pass and update) next to a 1-tensor bucket.  Round 1 sent the long
    bucket down a route that never updated it when clipping deferred the
    short one; every bucket must match the oracle."""
    shapes = [(50_000,), (100_000,)] + [(257,)] * 70
    g = torch.Generator(device="cpu").manual_seed(11)
    p0 = [(torch.randn(s, generator=g) * 0.02).to(DEV) for s in shapes]
    opt = DistributedOptimizer(p0, bucket_size=30_000, clip=clip)
    L = opt.layout
    assert [len(b.slots) for b in L.buckets] == [71, 1]
    state = _oracle_state(oracle, L, [p.cpu().numpy() for p in p0])
    for step in (1, 2, 3):
        grads = [(torch.randn(s, generator=g) * 1e-3).to(torch.bfloat16).to(DEV) for s in shapes]
        rep = opt.step(grads)
        torch.cuda.synchronize()
        params, norm = oracle.step_all_ranks([[u16(x) for x in grads]], [
            {"params": [(s.index, s.offset, s.numel) for s in b.slots], "numel": b.numel}
            for b in L.buckets], state, step, opt.lr, opt.betas, opt.eps, opt.weight_decay, clip=clip)
        if clip is not None:
            assert abs(rep.resolve()["grad_norm"] - norm) <= 1e-5 * norm
        pb = u16(opt.param_buffer)
        for bi, b in enumerate(L.buckets):
            master = state[bi][0][0]
            off = L.shard_offsets()[bi]
            dev_master = opt.master[off:off + b.numel].cpu().numpy()
            if clip is None:
                np.testing.assert_array_equal(pb[b.start:b.start + b.numel], params[bi])
                np.testing.assert_array_equal(dev_master, master)
            else:
                np.testing.assert_allclose(dev_master, master, rtol=1e-6, atol=1e-6 * np.abs(master).max())
                assert not np.array_equal(dev_master, p0_master(p0, b)), f"bucket {bi} never updated"
    opt.close()


def p0_master(p0, b):
    flat = np.zeros(b.numel, np.float32)
    for s in b.slots:
        flat[s.offset:s.offset + s.numel] = p0[s.index].cpu().numpy().reshape(-1)
    return flat


def test_grad_delivery_errors_and_no_sync(native):
    """grad_ready outside a step, twice for one param, or after its bucket
    launched raises; no_sync() silences the hooks for accumulation
    micro-batches and the last backward delivers the accumulated sum."""
    from paper_2312_03549_b200.errors import InfeasibleConfigError

    gs = config_gradset("odd")
    p0 = init_params(gs, DEV)
    opt = DistributedOptimizer(p0, bucket_size=100_000)
    g = make_grads(gs, 1, 0, DEV)
    with pytest.raises(InfeasibleConfigError):
        opt.grad_ready(0, g[0])
    opt.begin_step()
    last = len(g) - 1
    opt.grad_ready(last, g[last])
    b = opt.layout.slot(last).bucket
    if len(opt.layout.buckets[b].slots) > 1:
        with pytest.raises(InfeasibleConfigError):
            opt.grad_ready(last, g[last])
    for s in opt.layout.buckets[b].slots:
        if s.index != last:
            opt.grad_ready(s.index, g[s.index])
    with pytest.raises(InfeasibleConfigError):   # bucket b already launched
        opt.grad_ready(last, g[last])
    for i in range(len(g)):
        if opt.layout.slot(i).bucket != b:
            opt.grad_ready(i, g[i])
    opt.finish_step()
    opt.close()

    # accumulation: two micro-batches under no_sync + one delivering == one
    # step on the sum of the three
    params = [torch.nn.Parameter(p.clone()) for p in p0]
    ref = DistributedOptimizer(p0, bucket_size=100_000)
    acc = DistributedOptimizer(p0, bucket_size=100_000)
    acc.register_hooks(params)
    micro = [make_grads(gs, k, 0, DEV, dtype=torch.float32) for k in (1, 2, 3)]
    for k, mg in enumerate(micro):
        loss = sum((p * x).sum() for p, x in zip(params, mg))
        if k < 2:
            with acc.no_sync():
                loss.backward()
        else:
            acc.begin_step()
            loss.backward()
            acc.finish_step()
    ref.step([p.grad.clone() for p in params])
    torch.cuda.synchronize()
    assert torch.equal(acc.param_buffer, ref.param_buffer)
    ref.close()
    acc.close()


@pytest.mark.parametrize("clip", [None, 1.0])
def test_fast_adamw_single_rank_within_tolerance(oracle, native, clip):
    """adamw='fast' on the d = 1 fused pack+AdamW path: master within 1e-6
    norm-relative of the exact oracle after step 1, 1e-5 after step 3."""
    gs = config_gradset("odd")
    p0 = init_params(gs, DEV)
    opt = DistributedOptimizer(p0, bucket_size=100_000, clip=clip, adamw="fast")
    L = opt.layout
    state = _oracle_state(oracle, L, [p.cpu().numpy() for p in p0])
    for step in (1, 2, 3):
        grads = make_grads(gs, step, 0, DEV)
        opt.step(grads)
        torch.cuda.synchronize()
        oracle.step_all_ranks([[u16(g) for g in grads]], [
            {"params": [(s.index, s.offset, s.numel) for s in b.slots], "numel": b.numel}
            for b in L.buckets], state, step, opt.lr, opt.betas, opt.eps, opt.weight_decay, clip=clip)
        rtol = 1e-6 if step == 1 else 1e-5
        for bi, b in enumerate(L.buckets):
            off = L.shard_offsets()[bi]
            got = opt.master[off:off + b.numel].cpu().numpy().astype(np.float64)
            want = state[bi][0][0]
            assert np.abs(got - want).max() / np.abs(want).max() <= rtol
            assert torch.equal(opt.param_buffer[b.start:b.start + b.numel].view(torch.int16),
                               opt.master[off:off + b.numel].to(torch.bfloat16).view(torch.int16))
    opt.close()
