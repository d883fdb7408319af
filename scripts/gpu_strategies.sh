# The paper's DP strategies executed on B200: parity of the SC / NV-layerwise baselines (N=2)
# and the 8B step for sc, nv-layerwise, ASC (atomic ownership) and LB-ASC at N=2 and N=4.
mkdir -p gpurun_out
T2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571"
for s in sc nv-layerwise; do
  timeout 300 $T2 scripts/multi_gpu_check.py 2 auto muon - $s 2>&1 | grep '^{' | head -c 160; echo
done
: > gpurun_out/strategies.jsonl
for n in 2 4; do
  T="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n"
  for spec in "sc alpha-balanced" "nv-layerwise alpha-balanced" "sharded atomic-ownership" "sharded alpha-balanced"; do
    set -- $spec
    timeout 600 $T bench.py --gpus $n --steps 3 --warmup 2 --no-e2e --strategy $1 --method $2 2>/dev/null | grep '^{' >> gpurun_out/strategies.jsonl
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/strategies.jsonl"):
    d = json.loads(l)
    print(d["n_gpus"], d["config"]["strategy"], d["config"]["plan"], d["value"], d["phases_ms_rank0"], d["max_mean_rank_load"]["measured_compute_ms"])
PY
