// pfcs_hydro_math.cuh — per-mode spectral updates of the hydrodynamic /
// multiphysics model (hydro.py:86-88, 103-104 and the composition update),
// in numpy's evaluation order, shared by the standalone update kernels
// (pfcs_hydro.cu) and the update prologues fused into the inverse z pass
// (pfcs_pro.cuh), so both forms round identically.
#pragma once
#include <cuda_runtime.h>

namespace pfcs {

// k^2 = (kx*kx + ky*ky) + kz*kz at flat index idx of an (n0, n1, n2) grid
__device__ __forceinline__ double k2_grid(const double* kx, const double* ky, const double* kz, long long idx,
                                          int n1, int n2) {
  const long long line = idx / n2;
  const int z = (int)(idx - line * n2);
  const long long x = line / n1;
  const int y = (int)(line - x * n1);
  const double a = __ldg(&kx[x]), b = __ldg(&ky[y]), c = __ldg(&kz[z]);
  return __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c));
}

// psi_hat <- (psi_hat + dt*(lap*nl_hat - adv_hat)) / (1 - dt*linear)
__device__ __forceinline__ double2 psi_update(double2 ph, double2 nl, double2 ad, double k2, double eps,
                                              double dt) {
  const double lap = -k2;
  const double a = __dsub_rn(1.0, k2);
  const double b = __dsub_rn(4.0 / 3.0, k2);
  const double op = __dadd_rn(eps, __dmul_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
  const double rden = __drcp_rn(__dsub_rn(1.0, __dmul_rn(dt, __dmul_rn(lap, op))));
  const double tr = __dsub_rn(__dmul_rn(lap, nl.x), ad.x);
  const double ti = __dsub_rn(__dmul_rn(lap, nl.y), ad.y);
  return make_double2(__dmul_rn(__dadd_rn(ph.x, __dmul_rn(dt, tr)), rden),
                      __dmul_rn(__dadd_rn(ph.y, __dmul_rn(dt, ti)), rden));
}

// v_hat <- (v_hat - ((dt/rho)*cg)*force) / (1 - ((dt/rho)*gamma)*lap),
// cg = exp(-a0^2 k^2 / 2); c_cg = dt/rho, c_den = (dt/rho)*gamma, c_exp = -a0^2/2
__device__ __forceinline__ double2 vel_update(double2 v, double2 f, double k2, double c_cg, double c_den,
                                              double c_exp) {
  const double lap = -k2;
  const double cg = exp(__dmul_rn(c_exp, k2));
  const double w = __dmul_rn(c_cg, cg);
  const double rden = __drcp_rn(__dsub_rn(1.0, __dmul_rn(c_den, lap)));
  return make_double2(__dmul_rn(__dsub_rn(v.x, __dmul_rn(w, f.x)), rden),
                      __dmul_rn(__dsub_rn(v.y, __dmul_rn(w, f.y)), rden));
}

// c_hat <- (c_hat + dt*(M lap f_hat - adv_hat)) / (1 + dt*M*kappa*lap^2)
__device__ __forceinline__ double2 ch_update(double2 ch, double2 f, double2 ad, double k2, double mob,
                                             double kappa, double dt) {
  const double lap = -k2;
  const double ml = __dmul_rn(mob, lap);
  const double rden =
      __drcp_rn(__dadd_rn(1.0, __dmul_rn(__dmul_rn(dt, __dmul_rn(mob, kappa)), __dmul_rn(lap, lap))));
  const double tr = __dsub_rn(__dmul_rn(ml, f.x), ad.x);
  const double ti = __dsub_rn(__dmul_rn(ml, f.y), ad.y);
  return make_double2(__dmul_rn(__dadd_rn(ch.x, __dmul_rn(dt, tr)), rden),
                      __dmul_rn(__dadd_rn(ch.y, __dmul_rn(dt, ti)), rden));
}

}  // namespace pfcs
