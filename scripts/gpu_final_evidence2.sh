# Round-1 closing evidence (1 GPU), after the wave reorder / alpha auto / SOAP
# changes: smoke, the full GPU suite, the default bench line, the reference
# arm, the ncu launch list of the bench, ncu captures of the SOAP kernels.
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f2_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/f2_smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f2_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/f2_pytest.log
timeout 1200 python bench.py > gpurun_out/f2_bench.log 2>&1; echo bench rc=$?
timeout 1200 python bench.py --impl reference > gpurun_out/f2_ref.log 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/f2_ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ns_gemm_kernel|soap_chol|soap_prep|soap_basis" -c 12 -o gpurun_out/f2_soap python scripts/ncu_soap.py > gpurun_out/f2_ncu_soap.log 2>&1; echo ncu-soap rc=$?
grep '^{' gpurun_out/f2_bench.log | tail -1 | head -c 400; echo
grep '^{' gpurun_out/f2_ref.log | tail -1 | head -c 300; echo
