mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_soap.py -q > gpurun_out/sn_pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/sn_pytest.log
timeout 300 python scripts/ncu_soap.py > gpurun_out/sn_plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"ns_gemm_kernel|soap_" -o gpurun_out/sn_step python scripts/ncu_soap.py > gpurun_out/sn_ncu_step.log 2>&1; echo ncu-step rc=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"soap_chol|soap_basis" -c 4 -o gpurun_out/sn_refresh python scripts/ncu_soap.py --refresh > gpurun_out/sn_ncu_refresh.log 2>&1; echo ncu-refresh rc=$?
OSH_SIMRANK_OPT=soap OSH_SIMRANK_BREAKDOWN=1 timeout 1200 python scripts/simulated_ranks.py configs/qwen3-8b-like.cfg 8 alpha-balanced 1.0 3 1 > gpurun_out/soap_simranks.log 2>&1; echo simranks rc=$?
grep "^{" gpurun_out/soap_simranks.log > gpurun_out/soap_simranks.jsonl
python -c "
import json
d=json.loads(open('gpurun_out/soap_simranks.jsonl').read())
print(d['per_rank_compute_ms'], d['per_rank_refresh_ms'])
print(d['per_rank_modes_ms'][0]['refresh_step'])
"
