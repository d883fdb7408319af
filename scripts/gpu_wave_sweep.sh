# Sweep the minimum wave count of the overlapped schedule at N=1 and N=4 (NVLS).
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515"
for mw in ${WAVES:-3 6 8 12}; do
  OSH_MIN_WAVES=$mw timeout 400 $T bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ws_n4_$mw.log 2>&1
  OSH_MIN_WAVES=$mw timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ws_n1_$mw.log 2>&1
done
for f in gpurun_out/ws_n*.log; do grep '^{' $f | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; b=r['by_mode']
print('$f', d['value'], d['phases_ms_rank0']['compute_ms'], r['gemm_ms_per_step'], d['clocks']['sm_mhz'], b['momentum_matrix']['launches']//5, b['momentum_matrix']['ms_per_step'], b['apply_update']['ms_per_step'])"; done
