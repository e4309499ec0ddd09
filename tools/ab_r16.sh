mkdir -p gpurun_out
{
for lib in libpfcs libpfcs_r16; do
  for tt in 4 2; do
    for k in "strided 1024" "strided 2048"; do
      PFCS_TMA_T=$tt PFCS_LIB_PATH=paper_2603_26818_b200/$lib.so python tools/prof_kernel.py $k 20 | sed "s/^/$lib T=$tt /"
    done
  done
done
PFCS_LIB_PATH=paper_2603_26818_b200/libpfcs_r16.so python - <<'PY'
import torch, numpy as np
from paper_2603_26818_b200 import _native as nat
n=1024; nh=8
a=torch.randn(nh,n,n,dtype=torch.complex128,device='cuda')
b=torch.empty_like(a)
nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(b), nh, n, n, 1, 1, nat.stream_ptr())
ref=torch.fft.fft(a,dim=1)
print("r16 strided fwd relerr", ((b-ref).abs().max()/ref.abs().max()).item())
nat.call("pfcs_fft_axis_c2c", nat.ptr(a), nat.ptr(b), nh, n, n, 0, 1, nat.stream_ptr())
ref=torch.fft.ifft(a,dim=1)
print("r16 strided inv relerr", ((b-ref).abs().max()/ref.abs().max()).item())
PY
} > gpurun_out/ab_r16.txt 2>&1
