#!/bin/bash
# one GPU (driver configuration), final code: GPU suite, smoke, default bench; ncu of every hot kernel
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/r3j_tests_1gpu.log 2>&1; echo "rc=$?" >> $O/r3j_tests_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r3j_smoke.log 2>&1; echo "rc=$?" >> $O/r3j_smoke.log
timeout 600 python bench.py > $O/r3j_bench_n1.log 2>&1
bash tools/run_r2n.sh
