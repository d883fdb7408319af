# a*I folded into the POLY epilogue (UPDATE without aux): parity + N=1 bench with / without.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_ns_properties.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for aux in 0 1 0 1; do
  OSH_NS_AUX=$aux timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/fold_$aux.log 2>&1
  grep '^{' gpurun_out/fold_$aux.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('aux=$aux', d['value'], d['clocks']['sm_mhz'], r['by_mode']['update'], r['by_mode']['poly'])"
done
