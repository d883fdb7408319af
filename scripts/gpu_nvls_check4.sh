# 4-GPU: NVLS / NCCL parity checks, multi-GPU pytest, bench N=4 both collective paths.
set -x
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512"
timeout 300 $T scripts/multi_gpu_check.py 3 nvls > gpurun_out/nv4_check_nvls.log 2>&1; echo rc=$?
grep '^{' gpurun_out/nv4_check_nvls.log | tail -1 | head -c 300
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/nv4_pytest_multi.log 2>&1; echo rc=$?
tail -3 gpurun_out/nv4_pytest_multi.log
timeout 400 $T bench.py --gpus 4 --steps 5 --warmup 3 --collectives nvls --no-cpu-baseline --no-e2e > gpurun_out/nv4_bench_nvls.log 2>&1; echo rc=$?
timeout 400 $T bench.py --gpus 4 --steps 5 --warmup 3 --collectives nccl --no-cpu-baseline --no-e2e > gpurun_out/nv4_bench_nccl.log 2>&1; echo rc=$?
for f in gpurun_out/nv4_bench_*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$f', d['value'], d['config']['collectives'], d['max_mean_rank_load'], d['phases_ms_rank0'])"; done
