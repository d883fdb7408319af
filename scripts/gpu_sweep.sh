#!/bin/bash
# C5 sweep on the GPU: step ms and measured max/mean for each executable plan
# at N GPUs (run under gpurun --gpus N). Output: gpurun_out/sweep_N<N>.jsonl
N=${1:-2}
OUT=gpurun_out/sweep_N${N}.jsonl
: > $OUT
for spec in "atomic-ownership 1" "alpha-balanced 0" "alpha-balanced 0.25" "alpha-balanced 0.5" "alpha-balanced 1"; do
  set -- $spec
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 3 --warmup 2 --no-e2e \
    --method $1 --alpha $2 2>/dev/null | grep '^{' >> $OUT
done
wc -l $OUT
