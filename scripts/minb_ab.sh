#!/bin/bash
# 2-CTA GEMM momentum CTAs per SM (OSH_MOM_MINB 2 / 4 default / 8), N=1 step, interleaved
mkdir -p gpurun_out/minb_ab
for rep in 1 2; do
  for v in 4 2 8; do
    if [ $v = 4 ]; then unset OSH_LIB; else export OSH_LIB=ab/libosh_mb$v.so; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/minb_ab/s${v}_${rep}.json 2> gpurun_out/minb_ab/s${v}_${rep}.err
    echo "st=$v rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/minb_ab/s${v}_${rep}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
