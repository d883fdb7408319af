# Default bench line (N=1) after the wave reorder; config C4: Qwen3-32B
# (f=25600) blocked-Shampoo step at DP=8, ranks measured one at a time.
mkdir -p gpurun_out
#timeout 900 python bench.py --no-cpu-baseline > gpurun_out/c4_bench.log 2>&1; echo bench rc=$?
grep '^{' gpurun_out/c4_bench.log | head -c 400; echo
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
OSH_SIMRANK_OPT=shampoo OSH_SIMRANK_WS_GB=16 timeout 1500 python scripts/simulated_ranks.py configs/qwen3-32b-real.cfg 8 alpha-balanced 1.0 3 1 > gpurun_out/c4_simranks.log 2>&1; echo c4 rc=$?
grep '^{' gpurun_out/c4_simranks.log > gpurun_out/c4_simranks.jsonl; tail -3 gpurun_out/c4_simranks.log | head -c 1500
