// pfcs_pro.cuh — pointwise prologues fused into the first pass of a
// transform (the hydro / multiphysics pointwise products of
// hydro.py:77-107 that immediately feed an fft_nd), so the product never
// makes its own HBM round trip.  Arithmetic is exactly the standalone
// kernels' (pfcs_hydro.cu k_mul_deriv / k_cmul, pfcs_z.cu k_pfc_cube), so
// fused and unfused results are bit-identical.
#pragma once
#include "pfcs_fft.cuh"

namespace pfcs {

enum { PRO_NONE = 0, PRO_CUBE = 1, PRO_CMUL = 2, PRO_DERIV = 3 };

struct Pro {
  int kind;         // PRO_*
  const void* aux;  // PRO_CMUL: double2 array (same shape); PRO_DERIV: double vector
  int axis;         // PRO_DERIV: which coordinate indexes the vector
  int n1, n2;       // PRO_DERIV: grid extents to decode (x, y, z) from a flat index
};

// Prologue on element `idx` (flat C index of the (n0, n1, n2) grid) whose
// coordinate along p.axis is `c` (used by PRO_DERIV only; callers derive it
// from their line/tile indices instead of dividing idx per element).
__device__ __forceinline__ double2 apply_pro(const Pro& p, double2 v, i64 idx, i64 c) {
  if (p.kind == PRO_CUBE) {
    const double a = v.x, b = v.y;
    const double cr = __dsub_rn(__dmul_rn(a, a), __dmul_rn(b, b));
    const double ci = __dadd_rn(__dmul_rn(a, b), __dmul_rn(b, a));
    return make_double2(__dsub_rn(__dmul_rn(a, cr), __dmul_rn(b, ci)), __dadd_rn(__dmul_rn(a, ci), __dmul_rn(b, cr)));
  }
  if (p.kind == PRO_CMUL) {  // aux * v (k_cmul(a = aux, b = v))
    const double2 a = __ldg((const double2*)p.aux + idx);
    return make_double2(__dsub_rn(__dmul_rn(a.x, v.x), __dmul_rn(a.y, v.y)),
                        __dadd_rn(__dmul_rn(a.x, v.y), __dmul_rn(a.y, v.x)));
  }
  if (p.kind == PRO_DERIV) {  // i d_axis[c] v
    const double dk = __ldg((const double*)p.aux + c);
    return make_double2(-__dmul_rn(dk, v.y), __dmul_rn(dk, v.x));
  }
  return v;
}

}  // namespace pfcs
