#!/bin/bash
# A/B of an env knob on the N-GPU bench (same box, back to back, alternating).
#   bash tools/ab_env.sh N VAR "v1 v2" "bench args..."
N=$1; VAR=$2; VALS=$3; ARGS=$4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
port=29700
for rep in 1 2; do
  for v in $VALS; do
    port=$((port+1))
    env $VAR=$v timeout 600 $TR --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $ARGS 2>/dev/null \
      | grep '"metric"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['ms_per_step'],3), {k:(round(x['ms_total']/d['steps'],2)) for k,x in d['kernels'].items()})"
  done
done
