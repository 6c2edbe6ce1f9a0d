#!/bin/bash
# GEMM + optimizer kernel launch footprints (ncu launch__* metrics)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=launch__registers_per_thread,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static,launch__shared_mem_config_size,launch__block_size,launch__grid_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_warps,launch__occupancy_limit_blocks,launch__cluster_dim_x,launch__cluster_dim_y,launch__cluster_max_active,launch__sm_count,gpu__time_duration.sum
timeout 600 ncu --metrics $M --csv -k regex:"nvjet|gemm|cutlass|xmma|Kernel|hod" -c 60 python tools/corun_probe.py --reps 1 --numel 16777216 > gpurun_out/r2d_footprint.csv 2> gpurun_out/r2d_ncu.err
timeout 600 ncu --metrics $M --csv -c 40 -k regex:"hod" python tools/fused_emulated.py > gpurun_out/r2d_footprint_hod.csv 2>> gpurun_out/r2d_ncu.err
