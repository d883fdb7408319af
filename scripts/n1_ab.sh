#!/bin/bash
# Same-box A/B of two builds on the default N=1 step (OSH_LIB=ab/libosh_base.so
# vs the in-tree libosh.so), interleaved, plus poly_ab for the GEMM alone.
mkdir -p gpurun_out/n1_ab
for rep in 1 2 3; do
  for lib in base new; do
    if [ $lib = base ]; then export OSH_LIB=ab/libosh_base.so; else unset OSH_LIB; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      > gpurun_out/n1_ab/${lib}_${rep}.json 2> gpurun_out/n1_ab/${lib}_${rep}.err
    echo "$lib $rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/n1_ab/${lib}_${rep}.json').read().strip().splitlines()[-1]); r=d['roofline']['by_mode']; print(d['ms_per_step'], {k: (v.get('ms_per_step'), v.get('tflops_exec')) for k, v in r.items() if k in ('gram','poly','update','final')}, d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
