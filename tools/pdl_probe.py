"""Back-to-back fused pack+AdamW launches over the GPT-3 1.3B bucket layout
(d = 1, no events between launches): device time of the whole sequence.
Run with HOD_PDL=0 / 1 to see what programmatic dependent launch buys."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03549_b200 import _native as nat  # noqa: E402
from paper_2312_03549_b200.buckets import build_bucket_layout  # noqa: E402
from paper_2312_03549_b200.gradsets import config_gradset  # noqa: E402

nat.load()
gs = config_gradset(sys.argv[1] if len(sys.argv) > 1 else "gpt1.3b")
L = build_bucket_layout(gs.numels, 25_000_000, 1)
N = L.total_numel
dev = "cuda"
g = torch.randn(N, device=dev).mul_(1e-3).to(torch.bfloat16)
p = torch.randn(N, device=dev).mul_(0.02)
m = torch.zeros(N, device=dev)
v = torch.zeros(N, device=dev)
out = torch.empty(N, dtype=torch.bfloat16, device=dev)
hp = nat.AdamWParams(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)
tables = []
for b in L.buckets:
    e = (nat.PackEntry * len(b.slots))()
    for k, s in enumerate(b.slots):
        e[k].src, e[k].numel, e[k].dst_offset = g.data_ptr() + 2 * (b.start + s.offset), s.numel, s.offset
    tables.append((b, e))


EVENTS = os.environ.get("PROBE_EVENTS", "0") == "1"   # an event record after every launch
TIMING = os.environ.get("PROBE_TIMING", "0") == "1"   # timing events around every launch (bench style)
evs = [torch.cuda.Event(enable_timing=TIMING) for _ in tables]
evs0 = [torch.cuda.Event(enable_timing=True) for _ in tables]


def step():
    for (b, e), ev, ev0 in zip(tables, evs, evs0):
        if TIMING:
            ev0.record()
        nat.call("hod_pack_adamw", e, len(b.slots), b.numel, ctypes.c_float(1.0), nat.HOD_DTYPE_BF16,
                 p.data_ptr() + 4 * b.start, m.data_ptr() + 4 * b.start, v.data_ptr() + 4 * b.start,
                 out.data_ptr() + 2 * b.start, ctypes.byref(hp), None, 0)
        if EVENTS or TIMING:
            ev.record()


for _ in range(3):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"HOD_PDL={os.environ.get('HOD_PDL', '1')} events={int(EVENTS)} timing={int(TIMING)} buckets={len(L.buckets)} step {ms:.3f} ms "
      f"{28 * N / ms / 1e6:.0f} GB/s (28 B/elem)")
