# LPT tile schedule: GPU tests (1 GPU) and bench N=1 / N=4 with and without it.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_multi.py > gpurun_out/lpt_pytest.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/lpt_pytest.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551"
for l in 1 0; do
OSH_GEMM_LPT=$l timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/lpt_n1_$l.log 2>&1
OSH_GEMM_LPT=$l timeout 600 $T bench.py --gpus 4 --no-e2e > gpurun_out/lpt_n4_$l.log 2>&1
done
for f in gpurun_out/lpt_n*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$f', d['value'], d['max_mean_rank_load']['per_rank_compute_ms'], r['gemm_ms_per_step'], r['achieved_executed'], d['clocks']['sm_mhz'])"; done
