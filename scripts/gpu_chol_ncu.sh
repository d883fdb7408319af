mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"soap_chol" -c 1 -o /tmp/chol python scripts/ncu_soap.py --refresh > gpurun_out/chol_ncu.log 2>&1; echo ncu rc=$?
ncu -i /tmp/chol.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/chol_source_mixed.csv 2>&1
ncu -i /tmp/chol.ncu-rep --page details --csv > gpurun_out/chol_details.csv 2>&1
ls -la gpurun_out
