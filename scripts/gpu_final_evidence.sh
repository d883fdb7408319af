# Final round evidence on 1 GPU: smoke(), the default bench line, the reference arm,
# the ncu launch list of the bench (after it exited 0), and ncu --set full captures
# of the 2-CTA GEMM (UPDATE / GRAM / POLY) and of the elementwise kernels.
set -x
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; echo smoke rc=$?
tail -2 gpurun_out/fin_smoke.log
timeout 1200 python bench.py > gpurun_out/fin_bench.log 2>&1; echo bench rc=$?
timeout 1200 python bench.py --impl reference > gpurun_out/fin_ref.log 2>&1; echo ref rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/fin_ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ns_gemm_kernel -c 3 -o gpurun_out/fin_gemm python scripts/ncu_gemm.py --sym > gpurun_out/fin_ncu_gemm.log 2>&1; echo ncu-gemm rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"momentum_matrix|apply_update" -c 2 -o gpurun_out/fin_elem python scripts/ncu_elementwise.py > gpurun_out/fin_ncu_elem.log 2>&1; echo ncu-elem rc=$?
grep '^{' gpurun_out/fin_bench.log | tail -1 | head -c 600; echo
grep '^{' gpurun_out/fin_ref.log | tail -1 | head -c 600; echo
