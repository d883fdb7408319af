# 8-rank configs measured one rank at a time on one B200 (C2: 1.7B DP8; M0: 8B DP8).
mkdir -p gpurun_out
: > gpurun_out/simranks.jsonl
for spec in "qwen3-8b-like 8 alpha-balanced 1.0" "qwen3-8b-like 8 atomic-ownership 1.0" \
            "qwen3-1p7b-like 8 alpha-balanced 1.0" "qwen3-1p7b-like 8 atomic-ownership 1.0"; do
  set -- $spec
  timeout 900 python scripts/simulated_ranks.py configs/$1.cfg $2 $3 $4 2>/dev/null | grep '^{' >> gpurun_out/simranks.jsonl
done
cat gpurun_out/simranks.jsonl
