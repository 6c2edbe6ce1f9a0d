#!/bin/bash
# compute-sanitizer over the kernel tests (K1-K3, fused span kernels in the
# one-GPU d-way emulation, d = 1 optimizer steps).  Summaries -> gpurun_out/san_*.log
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_kernels_gpu.py tests/test_emulated_ranks_gpu.py tests/test_optimizer_gpu.py"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 2400 $CS --tool $tool $extra --target-processes all --print-limit 20 --error-exitcode 99 \
    python -m pytest $T -m gpu -q -x -p no:cacheprovider -k "not 100_steps and not long_pack_table" > gpurun_out/san_$tool.log 2>&1
  echo "tool=$tool rc=$?" >> gpurun_out/san_$tool.log
done
grep -h "ERROR SUMMARY\|tool=\|passed\|failed" gpurun_out/san_*.log
