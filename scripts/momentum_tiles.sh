# momentum pass: consecutive tiles per CTA (OSH_MOM_TILES), standalone (OSH_OVERLAP=0), ncu durations
m() { OSH_OVERLAP=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:momentum_matrix -c 4 python scripts/ncu_elementwise.py > gpurun_out/r02_momt_$1.log 2>&1; }
for v in 1 2 4 1 2 4; do
  make -C paper_2602_06079_b200/csrc clean > /dev/null; make -j8 -C paper_2602_06079_b200/csrc NVEXTRA="-DOSH_MOM_TILES=$v" > gpurun_out/r02_momt_build.log 2>&1
  m "t${v}_$RANDOM"
done
make -C paper_2602_06079_b200/csrc clean > /dev/null; make -j8 -C paper_2602_06079_b200/csrc > /dev/null 2>&1
