// pfcs_pfcmath.cuh — per-mode arithmetic shared by the fused PFC passes
// (pfcs_x.cu cube pass, pfcs_z.cu update pass, pfcs_pfc2d.cu whole-loop
// kernel), kept in one place so every path rounds identically.
#pragma once
#include "pfcs_fft.cuh"

#ifndef PFCS_Z_TWL
#define PFCS_Z_TWL 1  // twiddle loads per butterfly in the fused z update (B200 1024^3: 1 -> 6.46 ms, 3 -> 8.05 ms)
#endif

namespace pfcs {

// exp(-2 pi i e / 16): for R = 8 the post/pre-twiddle W_N^k of element
// k = j + P e (N = 2M = 16 P) is W_N^j * W_16^e, one table load per thread.
__device__ __forceinline__ double2 w16(int e) {
  constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  constexpr double h = 0.70710678118654752440;
  switch (e & 7) {
    case 0: return make_double2(1.0, 0.0);
    case 1: return make_double2(c1, -s1);
    case 2: return make_double2(h, -h);
    case 3: return make_double2(s1, -c1);
    case 4: return make_double2(0.0, -1.0);
    case 5: return make_double2(-s1, -c1);
    case 6: return make_double2(-h, -h);
    default: return make_double2(-c1, -s1);
  }
}

// W_N^k for k = j + P e with N = 2M = 2 R P: W_N^j * W_{2R}^e = W_N^j * W_16^{e 8/R}
template <int R>
__device__ __forceinline__ double2 twiddle_k(const double2* __restrict__ twN, double2 wj, int j, int e, int P) {
  if constexpr (R == 8 || R == 4) {
    return cmul(wj, w16(e * (8 / R)));
  } else {
    return __ldg(&twN[j + P * e]);
  }
}

struct PfcSym {
  double eps, dt;
};

__device__ __forceinline__ double k2_of(double kx, double ky, double kz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(kx, kx), __dmul_rn(ky, ky)), __dmul_rn(kz, kz));
}

// returns (lap, fl(1/(1 - dt*linear)))
__device__ __forceinline__ void pfc_symbols(double k2, double eps, double dt, double& lap,
                                            double& rden) {
  lap = -k2;
  const double a = __dsub_rn(1.0, k2);
  const double b = __dsub_rn(4.0 / 3.0, k2);
  const double two_ring = __dmul_rn(__dmul_rn(a, a), __dmul_rn(b, b));
  const double op = __dadd_rn(eps, two_ring);
  const double lin = __dmul_rn(lap, op);
  const double den = __dsub_rn(1.0, __dmul_rn(dt, lin));
  rden = __drcp_rn(den);
}

}  // namespace pfcs
