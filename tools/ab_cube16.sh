mkdir -p gpurun_out
{
for lib in libpfcs libpfcs_cube16; do
  for k in "cube_x 1024" "cube_x 512" "cube_x 1024"; do
    PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python tools/prof_kernel.py $k 20 | sed "s/^/$lib /"
  done
done
PFCS_LIB_PATH=paper_2603_26818_b200/libpfcs_cube16.so timeout 900 python -m pytest tests/test_gpu_pfc.py tests/test_gpu_tma.py tests/test_gpu_fft.py -x -q 2>&1 | tail -3
for lib in libpfcs_cube16 libpfcs libpfcs_cube16; do
  PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['extra'] if 'extra' in d else {}; print('$lib', d['value'], json.dumps(d)[:100]); [print('  ',k, v.get('value'), v.get('kernels',{}).get('pfc_cube_x')) for k,v in d.items() if isinstance(v,dict) and 'kernels' in v]" || true
done
} > gpurun_out/ab_cube16.txt 2>&1
