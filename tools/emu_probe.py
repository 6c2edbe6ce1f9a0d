"""Probe: can two emulated ranks' spinning barrier kernels meet on one GPU?

    CUDA_DEVICE_MAX_CONNECTIONS=32 python tools/emu_probe.py

Case 'barrier': rank 0's 1-CTA barrier kernel on stream A, then rank 1's on
stream B (flags in one device allocation per rank).  Case 'busy': the same
with a 100 ms kernel queued on B ahead of rank 1's barrier.  Prints the time
each case takes and the error words (0 = met).
"""

import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_03549_b200 import _native as nat  # noqa: E402


def main():
    nat.load()
    dev = torch.device("cuda", 0)
    d = 2
    flags = [torch.zeros(64 * 8, dtype=torch.int64, device=dev) for _ in range(d)]
    errs = [torch.zeros(1, dtype=torch.int32, device=dev) for _ in range(d)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(d)]
    import ctypes
    arr = (ctypes.c_void_p * d)(*[f.data_ptr() for f in flags])
    print("connections", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"), flush=True)
    extra = torch.cuda.Stream(device=dev)
    from cuda.bindings import runtime as cudart

    raw = []
    for _ in range(d):
        err, h = cudart.cudaStreamCreateWithFlags(cudart.cudaStreamNonBlocking)
        raw.append(torch.cuda.ExternalStream(int(h), device=dev))
    cases = ["barrier", "late", "busy", "busy_other", "busy_first", "prio", "busy_raw"]
    for epoch, case in enumerate(cases, start=1):
        torch.cuda.synchronize()
        t0 = time.time()
        ss = streams
        if case == "prio":
            hi = torch.cuda.Stream.priority_range()[1]
            ss = [torch.cuda.Stream(device=dev, priority=hi) for _ in range(d)]
        if case == "busy_raw":
            ss = raw
        order = [1, 0] if case == "busy_first" else [0, 1]
        for r in order:
            if r == 1 and case in ("busy", "busy_first", "busy_raw"):
                with torch.cuda.stream(ss[1]):
                    torch.cuda._sleep(100_000_000)
            if r == 1 and case == "busy_other":
                with torch.cuda.stream(extra):
                    torch.cuda._sleep(100_000_000)
            if r == 1 and case == "late":
                time.sleep(0.05)
            nat.call("hod_p2p_barrier", arr, d, r, 0, epoch, 7, 3_000_000_000, errs[r].data_ptr(),
                     nat.stream_ptr(ss[r]))
        torch.cuda.synchronize()
        print(case, "s=%.3f" % (time.time() - t0), "err", [int(e.item()) for e in errs], flush=True)
        for e in errs:
            e.zero_()


if __name__ == "__main__":
    main()
