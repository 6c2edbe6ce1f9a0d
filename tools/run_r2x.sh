#!/bin/bash
# one GPU (the driver's round-end configuration): build from scratch, GPU suite, smoke, default bench
cd "$(dirname "$0")/.."
O=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $O/r2x_build.log 2>&1; echo "build rc=$?" >> $O/r2x_build.log
timeout 2400 python -m pytest tests -m gpu -q > $O/r2x_tests_1gpu.log 2>&1; echo "rc=$?" >> $O/r2x_tests_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r2x_smoke.log 2>&1; echo "rc=$?" >> $O/r2x_smoke.log
timeout 600 python bench.py > $O/r2x_bench_n1.log 2>&1; echo "rc=$?" >> $O/r2x_bench_n1.log
