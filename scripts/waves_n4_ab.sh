#!/bin/bash
# N=4 NVLS wave-count sweep (OSH_MIN_WAVES 8 vs 16), interleaved
mkdir -p gpurun_out/waves_n4
for rep in 1 2; do
  for w in 8 16; do
    OSH_MIN_WAVES=$w timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 4 \
      --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/waves_n4/w${w}_${rep}.json 2> gpurun_out/waves_n4/w${w}_${rep}.err
    echo "w=$w rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/waves_n4/w${w}_${rep}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['max_mean_rank_load']['per_rank_compute_ms'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
