#!/bin/bash
# FINAL epilogue W staging depth (kFinBufs 2 / 3 default / 4), N=1 step, interleaved
mkdir -p gpurun_out/fin_ab
for rep in 1 2; do
  for v in 3 2 4; do
    if [ $v = 3 ]; then unset OSH_LIB; else export OSH_LIB=ab/libosh_fin$v.so; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fin_ab/f${v}_${rep}.json 2> gpurun_out/fin_ab/f${v}_${rep}.err
    echo "fin=$v rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/fin_ab/f${v}_${rep}.json').read().strip().splitlines()[-1]); r=d['roofline']['by_mode']; print(d['ms_per_step'], r['final']['ms_per_step'], r['update']['ms_per_step'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
