#!/bin/bash
# One-off environment probe on the GPU box (nvidia-smi, topology, host cores, symmetric memory).
set -x
nvidia-smi
nvidia-smi topo -m
nproc; lscpu | head -20; free -g
python - <<'PY'
import torch, os
print(torch.__version__, torch.cuda.device_count(), torch.cuda.get_device_name(0))
p = torch.cuda.get_device_properties(0)
print(p)
print("affinity", len(os.sched_getaffinity(0)))
PY
