#!/bin/bash
# Same-box A/B of the upper-tile form (default) vs full mirrored symmetric matrices (OSH_UPPER_FORM=0), N=1
mkdir -p gpurun_out/upper_ab
for rep in 1 2 3; do
  for uf in 0 1; do
    OSH_UPPER_FORM=$uf timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/upper_ab/uf${uf}_${rep}.json 2> gpurun_out/upper_ab/uf${uf}_${rep}.err
    echo "uf=$uf rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/upper_ab/uf${uf}_${rep}.json').read().strip().splitlines()[-1]); r=d['roofline']['by_mode']; print(d['ms_per_step'], {k: (v.get('ms_per_step'), v.get('tflops_exec')) for k, v in r.items() if k in ('gram','poly','update','final')}, d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
