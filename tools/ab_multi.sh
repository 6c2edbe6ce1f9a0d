#!/bin/bash
# bench.py under several env settings on N GPUs (same box, back to back).
#   bash tools/ab_multi.sh N "bench args" "ENV1=a ENV2=b" "ENV1=c" ...
N=$1; ARGS=$2; shift 2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29750
for rep in 1 2; do
  for setting in "$@"; do
    port=$((port+1))
    env $setting timeout 600 $TR --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $ARGS 2>/dev/null \
      | grep '"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$setting', round(d['ms_per_step'],3), {k:(round(x['ms_total']/d['steps'],2)) for k,x in d['kernels'].items()})"
  done
done
