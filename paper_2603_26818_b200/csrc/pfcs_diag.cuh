// pfcs_diag.cuh — NaN-propagating block maxima into striped diagnostic slots.
//
// The per-step diagnostics of pfc.pfc_step (pfc.py:100-105 realness ratio,
// pfc.py:122-124 finiteness + max|psi|) are produced as side outputs of the
// fused passes.  Each CTA reduces its values in registers/shared memory and
// issues ONE atomicMax per value into slot (blockIdx.x % PFCS_DIAG_SLOTS), so
// the L2 atomic units never see more than a few thousand same-address
// operations per launch.  Values are >= 0 (or NaN), whose IEEE bit patterns
// order like unsigned integers, so the max is an integer max and NaN (bit
// pattern above +inf) wins, i.e. divergence is never masked.
#pragma once
#include <cuda_runtime.h>

#define PFCS_DIAG_SLOTS 64
#define PFCS_DIAG_VALS 4

namespace pfcs {

__device__ __forceinline__ double dmax_bits(double a, double b) {
  const unsigned long long ua = (unsigned long long)__double_as_longlong(a);
  const unsigned long long ub = (unsigned long long)__double_as_longlong(b);
  return __longlong_as_double((long long)(ua > ub ? ua : ub));
}
__device__ __forceinline__ double fmax_nan(double a, double b) { return dmax_bits(a, b); }

__device__ __forceinline__ double warp_max_bits(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = dmax_bits(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// All threads of the CTA must call.  diag may be NULL (no diagnostics).
__device__ __forceinline__ void diag_block_max(double* diag, double a, double b, double c) {
  __shared__ double red[3][32];
  if (diag == nullptr) return;
  a = warp_max_bits(a);
  b = warp_max_bits(b);
  c = warp_max_bits(c);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  if (lane == 0) {
    red[0][w] = a;
    red[1][w] = b;
    red[2][w] = c;
  }
  __syncthreads();
  if (w == 0) {
    a = lane < nw ? red[0][lane] : 0.0;
    b = lane < nw ? red[1][lane] : 0.0;
    c = lane < nw ? red[2][lane] : 0.0;
    a = warp_max_bits(a);
    b = warp_max_bits(b);
    c = warp_max_bits(c);
    if (lane == 0) {
      unsigned long long* s =
          (unsigned long long*)(diag + (blockIdx.x % PFCS_DIAG_SLOTS) * PFCS_DIAG_VALS);
      atomicMax(s + 0, (unsigned long long)__double_as_longlong(a));
      atomicMax(s + 1, (unsigned long long)__double_as_longlong(b));
      atomicMax(s + 2, (unsigned long long)__double_as_longlong(c));
    }
  }
}

// Warp-aggregated "non-finite seen" flag into value 3 of the slot.
__device__ __forceinline__ void diag_flag_nonfinite(double* diag, bool bad) {
  if (diag == nullptr) return;
  const unsigned m = __ballot_sync(0xffffffffu, bad);
  if (m && (threadIdx.x & 31) == __ffs(m) - 1) {
    unsigned long long* s =
        (unsigned long long*)(diag + (blockIdx.x % PFCS_DIAG_SLOTS) * PFCS_DIAG_VALS);
    atomicMax(s + 3, (unsigned long long)__double_as_longlong(1.0));
  }
}

}  // namespace pfcs
