mkdir -p gpurun_out
for cfg in "libpfcs 1024" "libpfcs_r16 1024" "libpfcs 512"; do
  set -- $cfg
  PFCS_LIB_PATH=paper_2603_26818_b200/$1.so timeout 600 ncu --set full --clock-control none -k regex:k_strided_tma -s 1 -c 1 \
     -o /tmp/y_$1_$2 python tools/prof_kernel.py strided $2 2 > gpurun_out/ncu_y_$1_$2.log 2>&1
  ncu -i /tmp/y_$1_$2.ncu-rep --page raw --csv > gpurun_out/ncu_y_$1_$2.csv 2>&1
done
