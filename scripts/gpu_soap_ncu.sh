# SOAP: parity, the 8B DP8 per-rank step and refresh, ncu of the step GEMMs
# and of the refresh's Cholesky / basis kernels (CSV exported on the box;
# the .ncu-rep files are not brought back).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_soap.py -q > gpurun_out/sn_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/sn_pytest.log
OSH_SIMRANK_OPT=soap OSH_SIMRANK_BREAKDOWN=1 timeout 1200 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced 1.0 3 1 > gpurun_out/soap_simranks.log 2>&1; echo simranks rc=$?
grep "^{" gpurun_out/soap_simranks.log > gpurun_out/soap_simranks.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/soap_simranks.jsonl').read())
print(d['per_rank_compute_ms'], d['per_rank_refresh_ms'])
print(d['per_rank_modes_ms'][0]['refresh_step'])
"
M=gpu__time_duration.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"ns_gemm_kernel|soap_" --csv python scripts/ncu_soap.py > gpurun_out/sn_step.csv 2> gpurun_out/sn_step.err; echo ncu-step rc=$?
timeout 900 ncu --profile-from-start off --metrics $M --clock-control none -k regex:"soap_chol|soap_basis|soap_split|ns_gemm" -c 12 --csv python scripts/ncu_soap.py --refresh > gpurun_out/sn_refresh.csv 2> gpurun_out/sn_refresh.err; echo ncu-refresh rc=$?
ls -la gpurun_out | head
