# Wave reorder + alpha auto: parity tests, default bench, simulated 8-rank
# per-rank compute with and without the reorder (1 GPU).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_host_io.py tests/test_gpu_c1.py -x -q > gpurun_out/ro_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/ro_pytest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ro_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/ro_bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d.get('e2e'), d.get('clocks'))"
: > gpurun_out/ro_simranks.jsonl
OSH_SIMRANK_BREAKDOWN=1 timeout 900 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced auto 3 2 2>/dev/null | grep '^{' >> gpurun_out/ro_simranks.jsonl
OSH_SIMRANK_BREAKDOWN=1 timeout 900 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced 1.0 3 2 2>/dev/null | grep '^{' >> gpurun_out/ro_simranks.jsonl
OSH_WAVE_REORDER=0 OSH_SIMRANK_BREAKDOWN=1 timeout 900 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced auto 3 2 2>/dev/null | grep '^{' >> gpurun_out/ro_simranks.jsonl
python -c "
import json
for l in open('gpurun_out/ro_simranks.jsonl'):
    d=json.loads(l); print(d['alpha'], d['measured_max_mean'], d['plan_nsflops_max_mean'], d['per_rank_compute_ms'], d['per_rank_alg_tflops'])
"
