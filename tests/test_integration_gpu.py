"""Real-module integration and sharded checkpoint (§8f.4), d = 1.

* hooks: a torch nn.Module whose parameters alias the optimizer's flat bf16
  buffer; post-accumulate-grad hooks launch each bucket during backward; the
  result must be bit-identical to feeding the same gradients to ``step``.
* checkpoint: save -> fresh optimizer -> load reproduces master/m/v/params and
  the next step bit-for-bit.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2312_03549_b200 import DistributedOptimizer, checkpoint  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset  # noqa: E402
from paper_2312_03549_b200.synthetic import init_params, make_grads  # noqa: E402

DEV = "cuda"


def _model():
    torch.manual_seed(0)
    layers = []
    for _ in range(4):
        layers += [torch.nn.Linear(256, 512, bias=True), torch.nn.GELU(), torch.nn.Linear(512, 256, bias=False)]
    return torch.nn.Sequential(*layers).to(DEV, torch.bfloat16)


def test_backward_hooks_launch_buckets_and_match_step():
    model = _model()
    params = list(model.parameters())
    init = [p.detach().float().clone() for p in params]
    opt = DistributedOptimizer(init, bucket_size=200_000)
    twin = DistributedOptimizer(init, bucket_size=200_000)
    for p, view in zip(params, opt.params):
        p.data = view                      # the model now reads the optimizer's buffer
    seen = []
    handles = opt.register_hooks(params)
    orig = opt._launch_bucket

    def spy(bi):
        seen.append(bi)
        orig(bi)

    opt._launch_bucket = spy
    x = torch.randn(64, 256, device=DEV, dtype=torch.bfloat16)
    for _ in range(2):
        opt.begin_step()
        loss = model(x).float().pow(2).mean()
        loss.backward()
        grads = [p.grad.detach().clone() for p in params]
        opt.finish_step()
        twin.step(grads)
        for p in params:
            p.grad = None
    torch.cuda.synchronize()
    assert seen[:len(opt.layout.buckets)] == list(range(len(opt.layout.buckets)))  # backward order
    assert torch.equal(opt.param_buffer.view(torch.int16), twin.param_buffer.view(torch.int16))
    assert torch.equal(opt.master, twin.master)
    for h in handles:
        h.remove()


def test_checkpoint_round_trip(tmp_path):
    gs = config_gradset("odd")
    p0 = init_params(gs, DEV)
    a = DistributedOptimizer(p0, bucket_size=100_000)
    a.step(make_grads(gs, 1, 0, DEV))
    checkpoint.save(a, tmp_path)
    b = DistributedOptimizer([torch.zeros_like(p) for p in p0], bucket_size=100_000)
    man = checkpoint.load(b, tmp_path)
    assert man["step"] == 1
    for name in ("master", "exp_avg", "exp_avg_sq"):
        assert torch.equal(getattr(a, name), getattr(b, name))
    assert torch.equal(a.param_buffer.view(torch.int16), b.param_buffer.view(torch.int16))
    g2 = make_grads(gs, 2, 0, DEV)
    a.step(g2)
    b.step(g2)
    torch.cuda.synchronize()
    assert torch.equal(a.master, b.master)
    assert np.array_equal(a.param_buffer.view(torch.int16).cpu().numpy(),
                          b.param_buffer.view(torch.int16).cpu().numpy())
    # corruption is detected
    f = next(tmp_path.glob("*.master.npy"))
    arr = np.load(f)
    arr[0] += 1
    np.save(f, arr)
    from paper_2312_03549_b200.errors import ConfigError

    with pytest.raises(ConfigError, match="corrupt"):
        checkpoint.load(b, tmp_path)
