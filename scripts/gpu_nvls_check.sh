# 2-GPU check of the NVLS-fused collectives: oracle parity (nvls, nccl) + bench.
# usage (on a gpurun box): bash scripts/gpu_nvls_check.sh
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
NCCL_DEBUG=WARN timeout 300 $T scripts/multi_gpu_check.py 3 nvls > gpurun_out/nv2_check_nvls.log 2>&1; echo rc=$?
tail -c 1500 gpurun_out/nv2_check_nvls.log
timeout 300 $T scripts/multi_gpu_check.py 3 nccl > gpurun_out/nv2_check_nccl.log 2>&1; echo rc=$?
tail -c 300 gpurun_out/nv2_check_nccl.log
timeout 400 $T bench.py --gpus 2 --steps 5 --warmup 3 --collectives nvls --no-cpu-baseline > gpurun_out/nv2_bench_nvls.log 2>&1; echo rc=$?
tail -c 1200 gpurun_out/nv2_bench_nvls.log
