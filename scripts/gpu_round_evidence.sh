# Round evidence on a 4-GPU box: full GPU test suite, bench N=1 (with CPU baseline + e2e),
# N=2 and N=4 (NVLS), DP2xTP2, and the ncu launch list of the N=1 bench (1 GPU, after it exited 0).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ev_pytest.log 2>&1; echo rc=$?
tail -3 gpurun_out/ev_pytest.log
timeout 900 python bench.py > gpurun_out/ev_n1.log 2>&1; echo rc=$?
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n > gpurun_out/ev_n$n.log 2>&1; echo rc=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29529 bench.py --gpus 4 --tp 2 > gpurun_out/ev_n4_tp2.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/ev_launches_n1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu.log 2>&1; echo rc=$?
for f in gpurun_out/ev_n*.log; do grep '^{' $f | tail -1 | head -c 400; echo; done
