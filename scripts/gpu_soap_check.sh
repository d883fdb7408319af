# SOAP: GPU parity vs the fp64 spec, Shampoo / GEMM regressions, and the
# 8B SOAP step at DP=8 measured rank by rank (config C4-style, 8B shapes).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_soap.py tests/test_gpu_shampoo.py tests/test_gpu_gemm.py -q > gpurun_out/soap_pytest.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/soap_pytest.log
OSH_SIMRANK_OPT=soap OSH_SIMRANK_BREAKDOWN=1 timeout 1200 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced 1.0 3 1 > gpurun_out/soap_simranks.log 2>&1; echo simranks rc=$?
grep '^{' gpurun_out/soap_simranks.log > gpurun_out/soap_simranks.jsonl; tail -5 gpurun_out/soap_simranks.log | head -c 3000
