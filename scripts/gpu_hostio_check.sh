# Host-buffer (e2e) path: parity tests, full-size oracle test, bench e2e at N=1 and N=2 (NCCL + NVLS).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_host_io.py tests/test_gpu_fullsize.py -x -q > gpurun_out/hio_pytest.log 2>&1; echo rc=$?
tail -15 gpurun_out/hio_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/hio_n1.log 2>&1; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --collectives nccl > gpurun_out/hio_n2_nccl.log 2>&1; echo rc=$?
for f in gpurun_out/hio_n*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$f', d['value'], d['e2e'], d['phases_ms_rank0'])"; done
