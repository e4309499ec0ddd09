set -e
mkdir -p gpurun_out
for lib in libpfcs libpfcs_lines1 libpfcs_y1 libpfcs_ly1; do
  for k in "zlines 512" "zlines 1024" "strided 512" "strided 1024"; do
    for rep in 1 2; do
      PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python tools/prof_kernel.py $k 30 | sed "s/^/$lib /"
    done
  done
done > gpurun_out/ab_twl.txt 2>&1
for lib in libpfcs libpfcs_ly1 libpfcs libpfcs_ly1; do
  PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python bench.py --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', d['value'], d.get('extra', d.get('pfc', ''))) " >> gpurun_out/ab_twl.txt || true
done
