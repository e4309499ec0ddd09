mkdir -p gpurun_out
{
for lib in libpfcs_notsm libpfcs libpfcs_notsm libpfcs; do
  for k in "strided 1024 10" "strided 512 30"; do
    PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python tools/prof_kernel.py $k | sed "s/^/$lib /"
  done
done
timeout 600 python -m pytest tests/test_gpu_tma.py tests/test_gpu_fft.py tests/test_gpu_pfc.py -x -q 2>&1 | tail -2
for lib in libpfcs_notsm libpfcs libpfcs_notsm libpfcs; do
  PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['value'], d['pfc']['value'], d['pfc']['kernels']['fft_axis1_inv']['avg_ms'], d['pfc']['kernels']['fft_axis1_fwd']['avg_ms'])" || true
done
} > gpurun_out/ab_tsm.txt 2>&1
