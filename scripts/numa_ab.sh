#!/bin/bash
# e2e A/B of NUMA-local pinned host buffers (OSH_BENCH_NUMA=1, default) vs not, N=4 and N=1
mkdir -p gpurun_out/numa_ab
nvidia-smi topo -m > gpurun_out/numa_ab/topo.txt 2>&1
lscpu > gpurun_out/numa_ab/lscpu.txt 2>&1
for rep in 1 2; do
  for nu in 0 1; do
    OSH_BENCH_NUMA=$nu timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus 4 \
      --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/numa_ab/n4_nu${nu}_${rep}.json 2> gpurun_out/numa_ab/n4_nu${nu}_${rep}.err
    echo "n4 nu=$nu rep=$rep rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/numa_ab/n4_nu${nu}_${rep}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])" 2>&1 | tail -1)"
  done
done
for nu in 0 1; do
  CUDA_VISIBLE_DEVICES=0 OSH_BENCH_NUMA=$nu timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline \
    > gpurun_out/numa_ab/n1_nu${nu}.json 2> gpurun_out/numa_ab/n1_nu${nu}.err
  echo "n1 nu=$nu rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/numa_ab/n1_nu${nu}.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['value'])" 2>&1 | tail -1)"
done
