#!/bin/bash
# Same-box A/B of two builds on the Shampoo / SOAP steps (1 GPU, 1.7B shapes):
#   OSH_LIB=ab/libosh_base.so vs the in-tree libosh.so, interleaved.
mkdir -p gpurun_out/precond_ab
for rep in 1 2; do
  for opt in shampoo soap; do
    for lib in base new; do
      if [ $lib = base ]; then export OSH_LIB=ab/libosh_base.so; else unset OSH_LIB; fi
      timeout 600 python bench.py --config configs/qwen3-1p7b-like.cfg --optimizer $opt --steps 6 --warmup 3 \
        --no-e2e --no-cpu-baseline > gpurun_out/precond_ab/${opt}_${lib}_${rep}.json 2> gpurun_out/precond_ab/${opt}_${lib}_${rep}.err
      echo "$opt $lib $rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/precond_ab/${opt}_${lib}_${rep}.json').read().strip().splitlines()[-1]); r=d['roofline']['by_mode']; x=d.get('shampoo') or d.get('soap'); print(d['ms_per_step'], x['refresh_step_ms'], x['timed_steps_refresh_free'], {k: (v.get('ms'), v.get('tflops_alg')) for k, v in x['refresh_by_mode_rank0'].items() if k in ('stat','split','gram','update')}, d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
    done
  done
done
