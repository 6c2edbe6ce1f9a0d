#!/bin/bash
# co-residency probe: carveout off/on x kernels (adamw, fused d=2 span, pack)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for k in adamw fused_d2 pack; do
  for c in 0 1; do
    HOD_CARVEOUT=$c timeout 300 python tools/corun_probe.py --kernel $k --grids 0,74,148,296 >> gpurun_out/r2e_corun.jsonl 2>> gpurun_out/r2e_corun.err
  done
done
