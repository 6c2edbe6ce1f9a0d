#!/bin/bash
# round-2 one-GPU check (the driver's configuration): GPU suite, GEMM/optimizer
# co-residency probe, cuBLAS GEMM launch footprint (ncu), compute-sanitizer
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2c_tests.log
timeout 600 python tools/corun_probe.py > gpurun_out/r2c_corun.jsonl 2> gpurun_out/r2c_corun.err
timeout 600 ncu --metrics launch__registers_per_thread,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static,launch__block_size,launch__grid_size,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem,launch__occupancy_limit_warps,launch__cluster_dim_x,launch__cluster_dim_y,launch__occupancy_per_block_size --csv -c 40 python tools/corun_probe.py --reps 1 --numel 16777216 > gpurun_out/r2c_gemm_footprint.csv 2> gpurun_out/r2c_ncu.err
timeout 2400 bash tools/sanitize.sh > gpurun_out/r2c_sanitize.txt 2>&1
