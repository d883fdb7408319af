: > gpurun_out/simranks2.jsonl
for a in 0.25 0.5 0.75; do
  timeout 900 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced $a 2>/dev/null | grep '^{' >> gpurun_out/simranks2.jsonl
done
for a in 0.25 0.5; do
  timeout 900 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 4 alpha-balanced $a 2>/dev/null | grep '^{' >> gpurun_out/simranks2.jsonl
done
timeout 900 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 4 alpha-balanced 1.0 2>/dev/null | grep '^{' >> gpurun_out/simranks2.jsonl
cat gpurun_out/simranks2.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ranks'], d['alpha'], d['max_compute_ms'], d['measured_max_mean'], d['plan_numel_max_mean'])"
