"""Probe: peer pointers + NVLS multicast availability via torch symmetric memory."""
import os

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
try:
    from cuda.bindings import driver as cu

    dev = cu.cuDeviceGet(rank)[1]
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
        attr = getattr(cu.CUdevice_attribute, name)
        print(rank, name, cu.cuDeviceGetAttribute(attr, dev))
except Exception as e:  # noqa: BLE001
    print("cuda-python probe failed", e)
print(rank, "backend", symm_mem.get_backend(torch.device("cuda", rank)) if hasattr(symm_mem, "get_backend") else "?")
t = symm_mem.empty(1 << 20, dtype=torch.bfloat16, device=f"cuda:{rank}")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "ptrs", [hex(p) for p in h.buffer_ptrs], "mc", hex(h.multicast_ptr) if h.multicast_ptr else h.multicast_ptr,
      "signal", [hex(p) for p in h.signal_pad_ptrs][:2], "sig_size", h.signal_pad_size)
print(rank, [a for a in dir(h) if not a.startswith("_")])
# peer write check through torch
t.fill_(rank + 1)
torch.cuda.synchronize()
dist.barrier()
peer = h.get_buffer((rank + 1) % world, (16,), torch.bfloat16)
print(rank, "peer value", peer[:4].tolist())
dist.destroy_process_group()
