# momentum pass variants (standalone, OSH_OVERLAP=0): launch bounds / 256-bit streaming accesses
m() { OSH_OVERLAP=0 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:momentum_matrix -c 2 python scripts/ncu_elementwise.py > gpurun_out/r02_mom_$1.log 2>&1; }
m base
for v in "STREAM=1" "MINB=5" "MINB=3 STREAM=1" "STREAM=1" ; do
  flags=""; for kv in $v; do flags="$flags -DOSH_MOM_$kv"; done
  make -C paper_2602_06079_b200/csrc clean > /dev/null; make -j8 -C paper_2602_06079_b200/csrc NVEXTRA="$flags" > gpurun_out/r02_mom_build.log 2>&1
  m "$(echo $v | tr ' =' '__')_$RANDOM"
done
m base_again_after_last
