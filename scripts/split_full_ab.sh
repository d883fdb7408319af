#!/bin/bash
# Shampoo refresh: Newton products on symmetric tiles + mirror (default) vs all tiles (OSH_SPLIT_FULL=1)
mkdir -p gpurun_out/split_full
OSH_SPLIT_FULL=1 timeout 300 python -m pytest tests/test_gpu_shampoo.py -q -x > gpurun_out/split_full/tests_full.log 2>&1; echo "rc=$?" >> gpurun_out/split_full/tests_full.log
for rep in 1 2; do
  for sf in 0 1; do
    OSH_SPLIT_FULL=$sf timeout 600 python bench.py --config configs/qwen3-1p7b-like.cfg --optimizer shampoo --steps 6 --warmup 3 \
      --no-e2e --no-cpu-baseline > gpurun_out/split_full/sf${sf}_${rep}.json 2> gpurun_out/split_full/sf${sf}_${rep}.err
    echo "sf=$sf rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/split_full/sf${sf}_${rep}.json').read().strip().splitlines()[-1]); x=d['shampoo']; print(d['ms_per_step'], x['refresh_step_ms'], x['refresh_by_mode_rank0'].get('split'), d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
