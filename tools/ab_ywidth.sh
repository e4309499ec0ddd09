mkdir -p gpurun_out
{
for tt in 8 4 2; do PFCS_TMA_T=$tt python tools/prof_kernel.py strided 512 30; done
for tt in 4 8; do PFCS_TMA_T=$tt python tools/prof_kernel.py strided 1024 10; done
PFCS_TMA=0 python tools/prof_kernel.py strided 1024 10
PFCS_TMA=0 python tools/prof_kernel.py strided 512 30
} > gpurun_out/ab_ywidth.txt 2>&1
