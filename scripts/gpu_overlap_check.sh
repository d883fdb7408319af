# Overlapped-wave schedule: GPU parity (1 GPU tests + 4-GPU NVLS check) and bench N=1 / N=4
# with and without overlap (OSH_OVERLAP=0).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multi.py > gpurun_out/ov_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/ov_pytest.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514"
timeout 300 $T scripts/multi_gpu_check.py 3 nvls > gpurun_out/ov_check4.log 2>&1; echo rc=$?
grep '^{' gpurun_out/ov_check4.log | tail -1 | head -c 200; echo
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ov_n1.log 2>&1; echo rc=$?
OSH_OVERLAP=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ov_n1_off.log 2>&1; echo rc=$?
timeout 400 $T bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ov_n4.log 2>&1; echo rc=$?
OSH_OVERLAP=0 timeout 400 $T bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ov_n4_off.log 2>&1; echo rc=$?
for f in gpurun_out/ov_n*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', d['value'], d['phases_ms_rank0'], r['gemm_ms_per_step'], d['clocks']['sm_mhz'])
for k,v in r['by_mode'].items(): print('   ', k, v)"; done
