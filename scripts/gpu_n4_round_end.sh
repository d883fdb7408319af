# 4-GPU round-end evidence: default bench (alpha auto), the
# SOAP step at DP4 (NVLS), and the 4-rank multi-GPU checks.
mkdir -p gpurun_out
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 "$@"; }
run --no-cpu-baseline > gpurun_out/n4_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/n4_bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'], d['max_mean_rank_load'], d.get('e2e'))"
run --no-cpu-baseline --no-e2e --optimizer soap --steps 4 --warmup 3 > gpurun_out/n4_soap.log 2>&1; echo soap rc=$?
grep '^{' gpurun_out/n4_soap.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['max_mean_rank_load'], d['soap']['refresh_step_ms'], d['soap']['amortized_step_ms'])"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -k "dp4 or tp2" > gpurun_out/n4_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/n4_pytest.log
