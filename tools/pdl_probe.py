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
CLIP = os.environ.get("PROBE_CLIP", "0") == "1"      # pass a clip coefficient (kClip variant)
MERGE = os.environ.get("PROBE_MERGE", "0") == "1"    # runs of consecutive buckets (<= 64 tensors) per launch
coef = torch.ones(1, device=dev)


class Run:
    def __init__(self, start, numel, slots):
        self.start, self.numel, self.slots = start, numel, slots


runs = []
for b in L.buckets:
    sl = [(b.start + s.offset, s.numel) for s in b.slots]
    if MERGE and runs and len(runs[-1].slots) + len(sl) <= nat.HOD_PACK_MAX_ENTRIES:
        r = runs[-1]
        r.slots += sl
        r.numel = b.start + b.numel - r.start
    else:
        runs.append(Run(b.start, b.numel, sl))
tables = []
for r in runs:
    e = (nat.PackEntry * len(r.slots))()
    for k, (off, n) in enumerate(r.slots):
        e[k].src, e[k].numel, e[k].dst_offset = g.data_ptr() + 2 * off, n, off - r.start
    tables.append((r, e))


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
                 out.data_ptr() + 2 * b.start, ctypes.byref(hp), coef.data_ptr() if CLIP else None, 0)
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
print(f"HOD_PDL={os.environ.get('HOD_PDL', '1')} events={int(EVENTS)} timing={int(TIMING)} clip={int(CLIP)} merge={int(MERGE)} launches={len(runs)} step {ms:.3f} ms "
      f"{28 * N / ms / 1e6:.0f} GB/s (28 B/elem)")
