#!/bin/bash
# A/B of the stage-sequence overlap (NCCL RS-v/AG-v path and DP x TP path) on
# a 4-GPU box: each line once with OSH_OVERLAP=0 and once with the default.
# Output: gpurun_out/seq_ab/*.json
mkdir -p gpurun_out/seq_ab
run() {  # name, extra bench args
  local name=$1; shift
  for ov in 0 1; do
    OSH_OVERLAP=$ov timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 4 \
      --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
      > gpurun_out/seq_ab/${name}_ov${ov}.json 2> gpurun_out/seq_ab/${name}_ov${ov}.err
    echo "$name ov=$ov rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/seq_ab/${name}_ov${ov}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d.get('phases_ms_rank0'), d['max_mean_rank_load'].get('per_rank_compute_ms'))" 2>&1 | tail -1)"
  done
}
run tp2 --tp 2
run nccl4 --collectives nccl
