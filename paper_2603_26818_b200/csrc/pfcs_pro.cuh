// pfcs_pro.cuh — pointwise prologues fused into the first pass of a
// transform (the hydro / multiphysics pointwise products of
// hydro.py:77-107 that immediately feed an fft_nd), so the product never
// makes its own HBM round trip.  Arithmetic is exactly the standalone
// kernels' (pfcs_hydro.cu k_mul_deriv / k_cmul, pfcs_z.cu k_pfc_cube), so
// fused and unfused results are bit-identical.
#pragma once
#include "pfcs_diag.cuh"
#include "pfcs_fft.cuh"
#include "pfcs_hydro_math.cuh"

namespace pfcs {

enum { PRO_NONE = 0, PRO_CUBE = 1, PRO_CMUL = 2, PRO_DERIV = 3, PRO_UPD_PSI = 4, PRO_UPD_VEL = 5, PRO_UPD_CH = 6 };

struct Pro {
  int kind;         // PRO_*
  const void* aux;  // PRO_CMUL: double2 array (same shape); PRO_DERIV: double vector;
                    // PRO_UPD_*: nl_hat / force / f_hat
  int axis;         // PRO_DERIV: which coordinate indexes the vector
  int n1, n2;       // PRO_DERIV / PRO_UPD_*: grid extents to decode (x, y, z) from a flat index
  // PRO_UPD_* (a spectral update fused into the first pass of the following
  // inverse transform): the loaded element is the OLD state; the prologue
  // writes the new state to out2 and transforms it
  const void* aux2;  // adv_hat (psi / c updates; may be null)
  void* out2;        // new state (may alias the loaded array)
  const double *kx, *ky, *kz;
  double c0, c1, c2;  // psi: eps, dt; vel: dt/rho, (dt/rho) gamma, -a0^2/2; c: mobility, kappa, dt
  double* diag;       // non-finite flag (value 3 of a slot), or null
  int pass;           // axis of the transform the prologue feeds (strided passes: 0 or 1)
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

// PRO_UPD_*: the update of element `idx` of the old state v, given its
// |k|^2 (the caller forms kx^2 + ky^2 once per line, then adds kz^2 —
// k2_grid's order, so the sum is the standalone kernels' bit for bit).
__device__ __forceinline__ double2 apply_upd(const Pro& p, double2 v, double2 a, double2 b, i64 idx, double k2) {
  const double2 nw = p.kind == PRO_UPD_PSI ? psi_update(v, a, b, k2, p.c0, p.c1)
                     : p.kind == PRO_UPD_VEL ? vel_update(v, a, k2, p.c0, p.c1, p.c2)
                                             : ch_update(v, a, b, k2, p.c0, p.c1, p.c2);
  ((double2*)p.out2)[idx] = nw;
  if (p.diag && !isfinite(nw.x))
    atomicMax((unsigned long long*)(p.diag + (blockIdx.x % PFCS_DIAG_SLOTS) * PFCS_DIAG_VALS) + 3,
              (unsigned long long)__double_as_longlong(1.0));
  return nw;
}

}  // namespace pfcs
