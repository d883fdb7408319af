#!/bin/bash
# Same-box A/B of the tapered head (OSH_TAPER_HEAD=0 vs default), N=1 bench with e2e.
mkdir -p gpurun_out/head_ab
for rep in 1 2; do
  for th in 0 1; do
    OSH_TAPER_HEAD=$th timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 4 --no-cpu-baseline \
      > gpurun_out/head_ab/th${th}_${rep}.json 2> gpurun_out/head_ab/th${th}_${rep}.err
    echo "th=$th rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/head_ab/th${th}_${rep}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'], d['gpu_launches'])" 2>&1 | tail -1)"
  done
done
