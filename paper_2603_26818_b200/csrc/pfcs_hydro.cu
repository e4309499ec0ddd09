// pfcs_hydro.cu — pointwise spectral/physical operators of the hydrodynamic
// PFC model (reference hydro.py:77-107), on full-grid complex128 fields.
//
// Every operation reproduces numpy's evaluation order and rounding
// (no FMA contraction; complex/real division as numerator * fl(1/den)), so:
//   * the viscous decay v_hat / (1 - (dt/rho) gamma lap) is bit-exact
//     (test_hydro.py:31-39),
//   * with v = 0 the density update equals the PFC update bit for bit
//     (test_hydro.py:72-107).
// The only non-bit-reproducible factor is the Gaussian cg = exp(-a0^2 k^2/2)
// (CUDA exp vs numpy exp differ in the last ulp on a few % of inputs).
#include "pfcs_diag.cuh"
#include "pfcs_hydro_math.cuh"
#include "pfcs_internal.h"

namespace pfcs {

typedef long long i64;

__device__ __forceinline__ double k2_at(const double* kx, const double* ky, const double* kz, i64 idx,
                                        int n1, int n2) {
  const i64 line = idx / n2;
  const int z = (int)(idx - line * n2);
  const i64 x = line / n1;
  const int y = (int)(line - x * n1);
  const double a = __ldg(&kx[x]), b = __ldg(&ky[y]), c = __ldg(&kz[z]);
  return __dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c));
}

__device__ __forceinline__ double2 cmul_np(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

static inline int grid_for(i64 n) {
  i64 b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (int)(b < 1 ? 1 : b);
}

// Grid-stride loop that keeps warps converged for the ballot at the end.
#define PFCS_FOR_ALL(n)                                                        \
  const i64 _stride = (i64)gridDim.x * blockDim.x;                             \
  const i64 _n = (n);                                                          \
  const i64 _round = ((_n + _stride - 1) / _stride) * _stride;                 \
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < _round; i += _stride) \
    if (i < _n)

// out = (i d_axis) * in, d the Nyquist-zeroed wavenumbers (grid.py:167-176):
// numpy's (±0 + i d)(a + i b) = (-d b, d a).
__global__ void k_mul_deriv(const double2* in, double2* out, i64 n, int n1, int n2,
                            const double* __restrict__ d, int axis) {
  PFCS_FOR_ALL(n) {
    const i64 line = i / n2;
    const int z = (int)(i - line * n2);
    const i64 x = line / n1;
    const int y = (int)(line - x * n1);
    const double dk = __ldg(&d[axis == 0 ? x : (axis == 1 ? y : z)]);
    const double2 a = in[i];
    out[i] = make_double2(-__dmul_rn(dk, a.y), __dmul_rn(dk, a.x));
  }
}

__global__ void k_cmul(const double2* a, const double2* b, double2* out, i64 n) {
  PFCS_FOR_ALL(n) { out[i] = cmul_np(a[i], b[i]); }
}

// adv = v1*x1 + v2*x2 + v3*x3 (hydro.py:83-85, left to right)
__global__ void k_advect(const double2* v1, const double2* x1, const double2* v2, const double2* x2,
                         const double2* v3, const double2* x3, double2* out, i64 n) {
  PFCS_FOR_ALL(n) {
    const double2 a = cmul_np(v1[i], x1[i]);
    const double2 b = cmul_np(v2[i], x2[i]);
    const double2 c = cmul_np(v3[i], x3[i]);
    const double2 s = make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
    out[i] = make_double2(__dadd_rn(s.x, c.x), __dadd_rn(s.y, c.y));
  }
}

// psi_hat <- (psi_hat + dt*(lap*nl_hat - adv_hat)) / (1 - dt*linear)   (hydro.py:86-87)
// psi_in may equal psi_hat (in place); distinct = out of place (no state copy)
__global__ void k_hydro_psi_update(const double2* psi_in, double2* psi_hat, const double2* nl_hat, const double2* adv_hat, i64 n,
                                   int n1, int n2, const double* __restrict__ kx,
                                   const double* __restrict__ ky, const double* __restrict__ kz,
                                   double eps, double dt, double* diag) {
  bool bad = false;
  PFCS_FOR_ALL(n) {
    const double2 ad = adv_hat ? adv_hat[i] : make_double2(0.0, 0.0);
    const double2 nw = psi_update(psi_in[i], nl_hat[i], ad, k2_at(kx, ky, kz, i, n1, n2), eps, dt);
    bad |= !isfinite(nw.x);  // hydro._check_finite looks at the real part (hydro.py:72-74)
    psi_hat[i] = nw;
  }
  diag_flag_nonfinite(diag, bad);
}

// mu_hat = nl_hat + op * f_hat   (hydro.py:101)
__global__ void k_hydro_mu(const double2* nl_hat, const double2* f_hat, double2* out, i64 n, int n1, int n2,
                           const double* __restrict__ kx, const double* __restrict__ ky,
                           const double* __restrict__ kz, double eps) {
  PFCS_FOR_ALL(n) {
    const double k2 = k2_at(kx, ky, kz, i, n1, n2);
    const double a = __dsub_rn(1.0, k2);
    const double b = __dsub_rn(4.0 / 3.0, k2);
    const double op = __dadd_rn(eps, __dmul_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
    const double2 x = nl_hat[i], f = f_hat[i];
    out[i] = make_double2(__dadd_rn(x.x, __dmul_rn(op, f.x)), __dadd_rn(x.y, __dmul_rn(op, f.y)));
  }
}

// v_hat <- (v_hat - ((dt/rho)*cg)*force) / (1 - ((dt/rho)*gamma)*lap)  (hydro.py:103-104)
// c_cg = dt/rho, c_den = (dt/rho)*gamma, c_exp = -0.5*a0**2 (host-evaluated)
__global__ void k_hydro_vel_update(const double2* v_in, double2* v_hat, const double2* force, i64 n, int n1, int n2,
                                   const double* __restrict__ kx, const double* __restrict__ ky,
                                   const double* __restrict__ kz, double c_cg, double c_den,
                                   double c_exp, double* diag) {
  bool bad = false;
  PFCS_FOR_ALL(n) {
    const double2 f = force ? force[i] : make_double2(0.0, 0.0);
    const double2 nw = vel_update(v_in[i], f, k2_at(kx, ky, kz, i, n1, n2), c_cg, c_den, c_exp);
    bad |= !isfinite(nw.x);
    v_hat[i] = nw;
  }
  diag_flag_nonfinite(diag, bad);
}

// ------------------------------------------------- composition field (new) --
// Cahn-Hilliard composition c advected by v (multiphysics mode, no reference
// counterpart; oracle/ref_numpy.py restates it):
//   mu_c = alpha (c^3 - c) - kappa lap c,   dc/dt = M lap mu_c - v . grad c
//   c_hat <- (c_hat + dt (M lap F[alpha (c^3 - c)] - F[v . grad c])) / (1 + dt M kappa lap^2)

// out = alpha * (c*(c*c) - c), complex, numpy order
__global__ void k_ch_nonlin(const double2* c, double2* out, i64 n, double alpha) {
  PFCS_FOR_ALL(n) {
    const double2 a = c[i];
    const double2 c3 = cmul_np(a, cmul_np(a, a));
    out[i] = make_double2(__dmul_rn(alpha, __dsub_rn(c3.x, a.x)), __dmul_rn(alpha, __dsub_rn(c3.y, a.y)));
  }
}

__global__ void k_ch_update(const double2* c_in, double2* c_hat, const double2* f_hat, const double2* adv_hat, i64 n,
                            int n1, int n2,
                            const double* __restrict__ kx, const double* __restrict__ ky,
                            const double* __restrict__ kz, double mob, double kappa, double dt, double* diag) {
  bool bad = false;
  PFCS_FOR_ALL(n) {
    const double2 ad = adv_hat ? adv_hat[i] : make_double2(0.0, 0.0);
    const double2 nw = ch_update(c_in[i], f_hat[i], ad, k2_at(kx, ky, kz, i, n1, n2), mob, kappa, dt);
    bad |= !isfinite(nw.x);
    c_hat[i] = nw;
  }
  diag_flag_nonfinite(diag, bad);
}

// mu_c_hat = f_hat - kappa * lap * c_hat
__global__ void k_ch_mu(const double2* f_hat, const double2* c_hat, double2* out, i64 n, int n1, int n2,
                        const double* __restrict__ kx, const double* __restrict__ ky,
                        const double* __restrict__ kz, double kappa) {
  PFCS_FOR_ALL(n) {
    const double kl = __dmul_rn(kappa, -k2_at(kx, ky, kz, i, n1, n2));
    const double2 f = f_hat[i], ch = c_hat[i];
    out[i] = make_double2(__dsub_rn(f.x, __dmul_rn(kl, ch.x)), __dsub_rn(f.y, __dmul_rn(kl, ch.y)));
  }
}

// out = (a + b) + c  (the advection sum assembled from per-rank products)
__global__ void k_add3(const double2* a, const double2* b, const double2* c, double2* out, i64 n) {
  PFCS_FOR_ALL(n) {
    const double2 x = a[i], y = b[i], z = c[i];
    out[i] = make_double2(__dadd_rn(__dadd_rn(x.x, y.x), z.x), __dadd_rn(__dadd_rn(x.y, y.y), z.y));
  }
}

// out = a + w * b (force accumulation: F[psi d mu_psi] + beta F[c d mu_c])
__global__ void k_axpy(const double2* a, const double2* b, double2* out, i64 n, double w) {
  PFCS_FOR_ALL(n) {
    const double2 x = a[i], y = b[i];
    out[i] = make_double2(__dadd_rn(x.x, __dmul_rn(w, y.x)), __dadd_rn(x.y, __dmul_rn(w, y.y)));
  }
}

}  // namespace pfcs

using namespace pfcs;

// Real-field pointwise operators of the R2C multiphysics path (physical
// fields are real there, so every product / nonlinearity reads and writes
// 8-byte samples; hydro.py:83-86, 100-103 and the composition model).
// Two samples per thread (16-byte loads); numpy's evaluation order, no FMA.
enum { RPW_CUBE = 0, RPW_MUL = 1, RPW_ADV3 = 2, RPW_CHNL = 3, RPW_ADD3 = 4 };

__device__ __forceinline__ double rpw_one(int kind, double a, double b, double c, double d, double e, double f,
                                          double alpha) {
  switch (kind) {
    case RPW_CUBE: return __dmul_rn(__dmul_rn(a, a), a);                          // psi**3
    case RPW_MUL: return __dmul_rn(a, b);                                          // psi * g
    case RPW_ADV3:                                                                  // v1 x1 + v2 x2 + v3 x3
      return __dadd_rn(__dadd_rn(__dmul_rn(a, b), __dmul_rn(c, d)), __dmul_rn(e, f));
    case RPW_CHNL: return __dmul_rn(alpha, __dsub_rn(__dmul_rn(a, __dmul_rn(a, a)), a));  // alpha (c^3 - c)
    default: return __dadd_rn(__dadd_rn(a, b), c);                                 // (a + b) + c
  }
}

__global__ void k_real_pw(int kind, const double* a, const double* b, const double* c, const double* d,
                          const double* e, const double* f, double* out, i64 n, double alpha) {
  const i64 n2 = n >> 1;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const bool two = kind == RPW_MUL || kind == RPW_ADV3 || kind == RPW_ADD3;
  const bool six = kind == RPW_ADV3;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 x = __ldg((const double2*)a + i);
    const double2 y = two ? __ldg((const double2*)b + i) : make_double2(0.0, 0.0);
    const double2 z = two && kind != RPW_MUL ? __ldg((const double2*)c + i) : make_double2(0.0, 0.0);
    const double2 w = six ? __ldg((const double2*)d + i) : make_double2(0.0, 0.0);
    const double2 u = six ? __ldg((const double2*)e + i) : make_double2(0.0, 0.0);
    const double2 v = six ? __ldg((const double2*)f + i) : make_double2(0.0, 0.0);
    ((double2*)out)[i] = make_double2(rpw_one(kind, x.x, y.x, z.x, w.x, u.x, v.x, alpha),
                                      rpw_one(kind, x.y, y.y, z.y, w.y, u.y, v.y, alpha));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const i64 k = n - 1;
    out[k] = rpw_one(kind, a[k], two ? b[k] : 0.0, (two && kind != RPW_MUL) ? c[k] : 0.0, six ? d[k] : 0.0,
                     six ? e[k] : 0.0, six ? f[k] : 0.0, alpha);
  }
}

extern "C" {

int pfcs_mul_deriv(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, const double* d,
                   int axis, void* stream) {
  if (axis < 0 || axis > 2) return fail(PFCS_E_ARG, "axis must be 0, 1 or 2");
  const i64 n = n0 * n1 * n2;
  if (n <= 0) return PFCS_OK;
  k_mul_deriv<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)in, (double2*)out, n, (int)n1,
                                                            (int)n2, d, axis);
  return check_launch("k_mul_deriv");
}

int pfcs_cmul(const void* a, const void* b, void* out, int64_t n, void* stream) {
  if (n <= 0) return PFCS_OK;
  k_cmul<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)a, (const double2*)b, (double2*)out, n);
  return check_launch("k_cmul");
}

int pfcs_hydro_advect(const void* v1, const void* x1, const void* v2, const void* x2, const void* v3,
                      const void* x3, void* out, int64_t n, void* stream) {
  if (n <= 0) return PFCS_OK;
  k_advect<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)v1, (const double2*)x1, (const double2*)v2, (const double2*)x2, (const double2*)v3,
      (const double2*)x3, (double2*)out, n);
  return check_launch("k_advect");
}

int pfcs_hydro_psi_update_to(const void* psi_in, void* psi_out, const void* nl_hat, const void* adv_hat, int64_t n0,
                             int64_t n1, int64_t n2, const double* kx, const double* ky, const double* kz,
                             double eps, double dt, double* diag, void* stream) {
  const i64 n = n0 * n1 * n2;
  if (n <= 0) return PFCS_OK;
  k_hydro_psi_update<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)psi_in, (double2*)psi_out, (const double2*)nl_hat, (const double2*)adv_hat, n, (int)n1,
      (int)n2, kx, ky, kz, eps, dt, diag);
  return check_launch("k_hydro_psi_update");
}

int pfcs_hydro_psi_update(void* psi_hat, const void* nl_hat, const void* adv_hat, int64_t n0, int64_t n1,
                          int64_t n2, const double* kx, const double* ky, const double* kz, double eps,
                          double dt, double* diag, void* stream) {
  return pfcs_hydro_psi_update_to(psi_hat, psi_hat, nl_hat, adv_hat, n0, n1, n2, kx, ky, kz, eps, dt, diag, stream);
}

int pfcs_hydro_mu(const void* nl_hat, const void* f_hat, void* out, int64_t n0, int64_t n1, int64_t n2,
                  const double* kx, const double* ky, const double* kz, double eps, void* stream) {
  const i64 n = n0 * n1 * n2;
  if (n <= 0) return PFCS_OK;
  k_hydro_mu<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)nl_hat, (const double2*)f_hat,
                                                           (double2*)out, n, (int)n1, (int)n2, kx, ky, kz,
                                                           eps);
  return check_launch("k_hydro_mu");
}

int pfcs_hydro_vel_update_to(const void* v_in, void* v_out, const void* force, int64_t n0, int64_t n1, int64_t n2,
                             const double* kx, const double* ky, const double* kz, double c_cg, double c_den,
                             double c_exp, double* diag, void* stream) {
  const i64 n = n0 * n1 * n2;
  if (n <= 0) return PFCS_OK;
  k_hydro_vel_update<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)v_in, (double2*)v_out, (const double2*)force, n, (int)n1, (int)n2, kx, ky, kz, c_cg, c_den,
      c_exp, diag);
  return check_launch("k_hydro_vel_update");
}

int pfcs_hydro_vel_update(void* v_hat, const void* force, int64_t n0, int64_t n1, int64_t n2,
                          const double* kx, const double* ky, const double* kz, double c_cg, double c_den,
                          double c_exp, double* diag, void* stream) {
  return pfcs_hydro_vel_update_to(v_hat, v_hat, force, n0, n1, n2, kx, ky, kz, c_cg, c_den, c_exp, diag, stream);
}

int pfcs_ch_nonlin(const void* c, void* out, int64_t n, double alpha, void* stream) {
  if (n <= 0) return PFCS_OK;
  k_ch_nonlin<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)c, (double2*)out, n, alpha);
  return check_launch("k_ch_nonlin");
}

int pfcs_ch_update_to(const void* c_in, void* c_out, const void* f_hat, const void* adv_hat, int64_t n0, int64_t n1,
                      int64_t n2, const double* kx, const double* ky, const double* kz, double mobility,
                      double kappa, double dt, double* diag, void* stream) {
  const i64 n = n0 * n1 * n2;
  if (n <= 0) return PFCS_OK;
  k_ch_update<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(
      (const double2*)c_in, (double2*)c_out, (const double2*)f_hat, (const double2*)adv_hat, n, (int)n1, (int)n2,
      kx, ky, kz, mobility, kappa, dt, diag);
  return check_launch("k_ch_update");
}

int pfcs_ch_update(void* c_hat, const void* f_hat, const void* adv_hat, int64_t n0, int64_t n1, int64_t n2,
                   const double* kx, const double* ky, const double* kz, double mobility, double kappa,
                   double dt, double* diag, void* stream) {
  return pfcs_ch_update_to(c_hat, c_hat, f_hat, adv_hat, n0, n1, n2, kx, ky, kz, mobility, kappa, dt, diag, stream);
}

int pfcs_ch_mu(const void* f_hat, const void* c_hat, void* out, int64_t n0, int64_t n1, int64_t n2,
               const double* kx, const double* ky, const double* kz, double kappa, void* stream) {
  const i64 n = n0 * n1 * n2;
  if (n <= 0) return PFCS_OK;
  k_ch_mu<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)f_hat, (const double2*)c_hat,
                                                        (double2*)out, n, (int)n1, (int)n2, kx, ky, kz, kappa);
  return check_launch("k_ch_mu");
}

int pfcs_real_pointwise(int kind, const double* a, const double* b, const double* c, const double* d,
                        const double* e, const double* f, double* out, int64_t n, double alpha, void* stream) {
  if (n <= 0) return PFCS_OK;
  if (kind < RPW_CUBE || kind > RPW_ADD3) return fail(PFCS_E_ARG, "pfcs_real_pointwise: unknown kind");
  const bool two = kind == RPW_MUL || kind == RPW_ADV3 || kind == RPW_ADD3;
  if (!a || !out || (two && !b) || ((kind == RPW_ADV3 || kind == RPW_ADD3) && !c) ||
      (kind == RPW_ADV3 && (!d || !e || !f)))
    return fail(PFCS_E_ARG, "pfcs_real_pointwise: missing operand");
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c | (uintptr_t)d | (uintptr_t)e | (uintptr_t)f | (uintptr_t)out) & 15)
    return fail(PFCS_E_ARG, "pfcs_real_pointwise: operands must be 16-byte aligned");
  k_real_pw<<<grid_for((n + 1) / 2), 256, 0, (cudaStream_t)stream>>>(kind, a, b, c, d, e, f, out, n, alpha);
  return check_launch("k_real_pw");
}

int pfcs_add3(const void* a, const void* b, const void* c, void* out, int64_t n, void* stream) {
  if (n <= 0) return PFCS_OK;
  k_add3<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)a, (const double2*)b, (const double2*)c,
                                                       (double2*)out, n);
  return check_launch("k_add3");
}

int pfcs_axpy(const void* a, const void* b, void* out, int64_t n, double w, void* stream) {
  if (n <= 0) return PFCS_OK;
  k_axpy<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>((const double2*)a, (const double2*)b, (double2*)out, n, w);
  return check_launch("k_axpy");
}

}  // extern "C"
