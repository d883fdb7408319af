# Shampoo on several GPUs: NVLS parity vs the spec oracle (N=2), bench at N=4 (8B shapes).
set -x
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 scripts/multi_gpu_check.py 3 auto shampoo > gpurun_out/sh_check2.log 2>&1; echo rc=$?
grep '^{' gpurun_out/sh_check2.log | tail -1 | head -c 600; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --optimizer shampoo --no-e2e > gpurun_out/sh_bench_n4.log 2>&1; echo rc=$?
tail -5 gpurun_out/sh_bench_n4.log | cut -c1-3000
