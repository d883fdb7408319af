# Per-launch breakdown (GEMM + elementwise CUDA-event timing) at N=1 and N=4 (NVLS).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bd_n1.log 2>&1; echo rc=$?
if [ "$(nvidia-smi -L | wc -l)" -ge 4 ]; then
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bd_n4.log 2>&1; echo rc=$?
fi
for f in gpurun_out/bd_n*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', d['value'], d['phases_ms_rank0'], r['gemm_ms_per_step'])
for k,v in r['by_mode'].items(): print('   ', k, v)"; done
