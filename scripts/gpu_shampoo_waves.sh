mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_shampoo.py tests/test_gpu_checkpoint.py -q 2>&1 | tail -1
OSH_SIMRANK_OPT=shampoo OSH_SIMRANK_WS_GB=16 timeout 1500 python scripts/simulated_ranks.py configs/qwen3-32b-real.cfg 8 alpha-balanced 1.0 3 1 > gpurun_out/c4b_simranks.log 2>&1; echo c4 rc=$?
grep '^{' gpurun_out/c4b_simranks.log > gpurun_out/c4b_simranks.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/c4b_simranks.jsonl').read())
print(d['per_rank_compute_ms'], d['per_rank_refresh_ms'], d['per_rank_amortized_ms'], d['measured_max_mean'])
"
