#!/bin/bash
# N=1 wave-count sweep (OSH_MIN_WAVES), interleaved
mkdir -p gpurun_out/${OUTD:-waves_ab}
for rep in 1 2; do
  for w in ${WAVES:-8 6 12 16}; do
    OSH_MIN_WAVES=$w timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${OUTD:-waves_ab}/w${w}_${rep}.json 2> gpurun_out/${OUTD:-waves_ab}/w${w}_${rep}.err
    echo "w=$w rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/${OUTD:-waves_ab}/w${w}_${rep}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['gpu_launches'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
