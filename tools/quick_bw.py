"""Quick device-time check of K1/K2/K3 bandwidth (CUDA events, warm, large n)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2312_03549_b200 import _native as nat  # noqa: E402

nat.load()
dev = "cuda"
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000_000
p = torch.randn(n, device=dev)
m = torch.zeros(n, device=dev)
v = torch.zeros(n, device=dev)
g = torch.randn(n, device=dev).to(torch.bfloat16)
out = torch.empty(n, dtype=torch.bfloat16, device=dev)
hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)


def timeit(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


t = timeit(lambda: nat.call("hod_adamw_bf16", p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                            out.data_ptr(), n, ctypes.byref(hp), None, 0))
print(f"adamw n={n}: {t:.3f} ms  {28 * n / t / 1e6:.0f} GB/s  {n / t / 1e6:.1f} Gelem/s")
src = torch.randn(n, device=dev).to(torch.bfloat16)
e = (nat.PackEntry * 1)()
e[0].src, e[0].numel, e[0].dst_offset = src.data_ptr(), n, 0
t = timeit(lambda: nat.call("hod_pack_bf16", e, 1, out.data_ptr(), n, ctypes.c_float(0.125), 0, 0))
print(f"pack bf16 n={n}: {t:.3f} ms  {4 * n / t / 1e6:.0f} GB/s")
src32 = torch.randn(n, device=dev)
e[0].src = src32.data_ptr()
t = timeit(lambda: nat.call("hod_pack_bf16", e, 1, out.data_ptr(), n, ctypes.c_float(0.125), 1, 0))
print(f"pack f32 n={n}: {t:.3f} ms  {6 * n / t / 1e6:.0f} GB/s")
parts = torch.empty(nat.HOD_SUMSQ_PARTIALS, device=dev)
t = timeit(lambda: nat.call("hod_sumsq_bf16", g.data_ptr(), n, parts.data_ptr(), 0))
print(f"sumsq n={n}: {t:.3f} ms  {2 * n / t / 1e6:.0f} GB/s")
c = torch.empty_like(p)
t = timeit(lambda: c.copy_(p))
print(f"torch copy fp32 n={n}: {t:.3f} ms  {8 * n / t / 1e6:.0f} GB/s")
for lim in (148, 74, 48, 32, 16):
    nat.call("hod_set_grid_limit", lim * 4)
    t = timeit(lambda: nat.call("hod_adamw_bf16", p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                                out.data_ptr(), n, ctypes.byref(hp), None, 0))
    nat.call("hod_set_grid_limit", 0)
    print(f"adamw_vec ctas={lim * 4} (~{lim} SMs): {t:.3f} ms  {28 * n / t / 1e6:.0f} GB/s")

# bucket-sized launches (LLaMA-7B: ~33.5M-element buckets of 1-3 tensors)
nb = 33_554_432
srcs = [torch.randn(nb // 2, device=dev).to(torch.bfloat16) for _ in range(2)]
eb = (nat.PackEntry * 2)()
for k, t_ in enumerate(srcs):
    eb[k].src, eb[k].numel, eb[k].dst_offset = t_.data_ptr(), t_.numel(), k * (nb // 2)
t = timeit(lambda: nat.call("hod_pack_sumsq", eb, 2, nb, ctypes.c_float(1.0), 0, parts.data_ptr(), 0), 50)
print(f"pack_sumsq bucket n={nb}: {t * 1e3:.1f} us  {2 * nb / t / 1e6:.0f} GB/s")
t = timeit(lambda: nat.call("hod_sumsq_bf16", g.data_ptr(), nb, parts.data_ptr(), 0), 50)
print(f"sumsq bucket n={nb}: {t * 1e3:.1f} us  {2 * nb / t / 1e6:.0f} GB/s")
t = timeit(lambda: nat.call("hod_pack_adamw", eb, 2, nb, ctypes.c_float(1.0), 0, p.data_ptr(), m.data_ptr(),
                            v.data_ptr(), out.data_ptr(), ctypes.byref(hp), None, 0), 50)
print(f"pack_adamw bucket n={nb}: {t * 1e3:.1f} us  {28 * nb / t / 1e6:.0f} GB/s")
e1 = (nat.PackEntry * 1)()
e1[0].src, e1[0].numel, e1[0].dst_offset = g.data_ptr(), n, 0
t = timeit(lambda: nat.call("hod_pack_adamw", e1, 1, n, ctypes.c_float(1.0), 0, p.data_ptr(), m.data_ptr(),
                            v.data_ptr(), out.data_ptr(), ctypes.byref(hp), None, 0))
print(f"pack_adamw 1 entry n={n}: {t:.3f} ms  {28 * n / t / 1e6:.0f} GB/s")
for nn in (nb, 4 * nb):
    t = timeit(lambda: nat.call("hod_adamw_bf16", p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(),
                                out.data_ptr(), nn, ctypes.byref(hp), None, 0), 50)
    print(f"adamw n={nn}: {t * 1e3:.1f} us  {28 * nn / t / 1e6:.0f} GB/s")
    e1[0].numel = nn
    t = timeit(lambda: nat.call("hod_pack_adamw", e1, 1, nn, ctypes.c_float(1.0), 0, p.data_ptr(), m.data_ptr(),
                                v.data_ptr(), out.data_ptr(), ctypes.byref(hp), None, 0), 50)
    print(f"pack_adamw 1 entry n={nn}: {t * 1e3:.1f} us  {28 * nn / t / 1e6:.0f} GB/s")
