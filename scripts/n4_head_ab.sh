#!/bin/bash
# N=4 NVLS A/B of the opt-in tapered head (OSH_TAPER_HEAD=1 vs default), interleaved.
mkdir -p gpurun_out/n4_head
for rep in 1 2; do
  for th in 0 1; do
    OSH_TAPER_HEAD=$th timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 4 \
      --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/n4_head/th${th}_${rep}.json 2> gpurun_out/n4_head/th${th}_${rep}.err
    echo "th=$th rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/n4_head/th${th}_${rep}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['max_mean_rank_load']['per_rank_compute_ms'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
