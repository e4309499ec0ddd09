#!/bin/bash
# Round-2 ncu evidence (run on the GPU box from the repo root; one GPU):
#  1. launch list of a short bench run (per-launch device times, cold-cache)
#  2. --set full captures of the top kernels at bench sizes
set -u
O=gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-multi"
$CMD > $O/r2n_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/r2n_launches.csv $CMD \
  > $O/r2n_ncu_launches.log 2>&1
echo launches_rc=$?
for spec in "cube_x 1024 k_cube_ls" "update_z 1024 k_pfc_z" "strided 1024 k_strided_tma" "irfft_x 512 k_real_x" "rfft_x 512 k_real_x" "zlines 512 k_lines"; do
  set -- $spec
  python tools/prof_kernel.py $1 $2 3 > $O/r2n_plain_$1_$2.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o $O/r2n_$1_$2 \
      python tools/prof_kernel.py $1 $2 3 > $O/r2n_ncu_$1_$2.log 2>&1
  echo $1 $2 rc=$?
done
