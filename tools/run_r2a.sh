#!/bin/bash
# round-2 check on a 2-GPU box: GPU suite, bench N=1 and N=2 (parity key)
cd "$(dirname "$0")/.."
python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r2a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_n1.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_n1.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2a_n2.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_n2.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a_ref1.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_ref1.log
