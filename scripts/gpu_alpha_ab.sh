# Same-box A/B of the plan's alpha at N=4 (NVLS): alpha = 1 (paper default)
# against alpha = 0.25 (the best planned NS-flop balance at R=4), interleaved.
mkdir -p gpurun_out
: > gpurun_out/alpha_ab.jsonl
for al in 1 0.25 1 0.25; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 4 --no-cpu-baseline --no-e2e --steps 10 --warmup 3 --alpha $al 2>/dev/null | grep '^{' >> gpurun_out/alpha_ab.jsonl
done
python -c "
import json
for l in open('gpurun_out/alpha_ab.jsonl'):
    d=json.loads(l); print(d['config']['plan'][:40], d['value'], d['clocks']['sm_mhz'], d['max_mean_rank_load'])
"
