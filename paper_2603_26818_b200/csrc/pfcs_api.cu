// pfcs_api.cu — the extern "C" boundary of libpfcs (see include/pfcs.h) plus
// host utilities: thread-local errors, per-device twiddle tables, shared
// memory opt-in.  No torch types cross this boundary: device pointers, sizes
// and a cudaStream_t passed as void*.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "pfcs_fft.cuh"
#include "pfcs_internal.h"
#include "pfcs_pro.cuh"

namespace pfcs {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PFCS_OK;
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return PFCS_E_CUDA;
}
int check_launch(const char* what) { return check_cuda(cudaGetLastError(), what); }

// exp(-2 pi i m / N) with exact values at the quadrant points and the octant
// symmetry built in; long double keeps every entry within 0.5 ulp + epsilon.
static void twiddle_value(long long m, long long N, double* c, double* s) {
  m %= N;
  const long long q = (4 * m) / N;  // quadrant
  long long r = 4 * m - q * N;      // theta = (pi/2) * (q + r/N)
  long double cp, sp;
  const long double half_pi = 1.5707963267948966192313216916397514L;
  if (r == 0) {
    cp = 1.0L;
    sp = 0.0L;
  } else if (2 * r <= N) {
    const long double phi = half_pi * (long double)r / (long double)N;
    cp = cosl(phi);
    sp = sinl(phi);
  } else {
    const long double phi = half_pi * (long double)(N - r) / (long double)N;
    cp = sinl(phi);
    sp = cosl(phi);
  }
  long double ct, st;
  switch (q) {
    case 0: ct = cp; st = sp; break;
    case 1: ct = -sp; st = cp; break;
    case 2: ct = -cp; st = -sp; break;
    default: ct = sp; st = -cp; break;
  }
  *c = (double)ct;
  *s = -(double)st;  // exp(-i theta)
}

static std::mutex g_tw_mu;
static std::map<std::pair<int, int>, double2*> g_tw;

const double2* twiddles(int N) {
  int dev = 0;
  if (check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return nullptr;
  std::lock_guard<std::mutex> lk(g_tw_mu);
  auto key = std::make_pair(dev, N);
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  std::vector<double2> h((size_t)N);
  for (int m = 0; m < N; ++m) twiddle_value(m, N, &h[m].x, &h[m].y);
  double2* d = nullptr;
  if (check_cuda(cudaMalloc(&d, sizeof(double2) * (size_t)N), "cudaMalloc twiddles")) return nullptr;
  if (check_cuda(cudaMemcpy(d, h.data(), sizeof(double2) * (size_t)N, cudaMemcpyHostToDevice),
                 "cudaMemcpy twiddles")) {
    cudaFree(d);
    return nullptr;
  }
  g_tw[key] = d;
  return d;
}

static std::mutex g_smem_mu;
static std::map<std::pair<int, const void*>, size_t> g_smem;

int ensure_smem(const void* func, size_t bytes) {
  if (bytes == 0) return PFCS_OK;
  int dev = 0;
  if (check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return PFCS_E_CUDA;
  std::lock_guard<std::mutex> lk(g_smem_mu);
  auto key = std::make_pair(dev, func);
  auto it = g_smem.find(key);
  if (it != g_smem.end() && it->second >= bytes) return PFCS_OK;
  if (check_cuda(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                 "cudaFuncSetAttribute(smem)"))
    return PFCS_E_CUDA;
  g_smem[key] = bytes;
  return PFCS_OK;
}

static std::mutex g_occ_mu;
struct OccKey {
  int dev;
  const void* f;
  int threads;
  size_t smem;
  bool operator<(const OccKey& o) const {
    if (dev != o.dev) return dev < o.dev;
    if (f != o.f) return f < o.f;
    if (threads != o.threads) return threads < o.threads;
    return smem < o.smem;
  }
};
static std::map<OccKey, int> g_occ;
static std::map<int, int> g_sms;

int persistent_grid(const void* func, int threads, size_t smem, long long ntiles, int* grid) {
  if (threads > 1024) return fail(PFCS_E_UNSUPPORTED, "tile too large (threads > 1024)");
  if (smem > 227 * 1024) return fail(PFCS_E_UNSUPPORTED, "tile too large (shared memory > 227 KB)");
  if (int rc = ensure_smem(func, smem)) return rc;
  int dev = 0;
  if (int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
  int per_sm = 0, sms = 0;
  {
    std::lock_guard<std::mutex> lk(g_occ_mu);
    OccKey k{dev, func, threads, smem};
    auto it = g_occ.find(k);
    if (it == g_occ.end()) {
      if (int rc = check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem),
                              "occupancy"))
        return rc;
      if (per_sm < 1) return fail(PFCS_E_UNSUPPORTED, "kernel cannot be resident (registers/smem)");
      g_occ[k] = per_sm;
    } else {
      per_sm = it->second;
    }
    auto is = g_sms.find(dev);
    if (is == g_sms.end()) {
      if (int rc = check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "SM count"))
        return rc;
      g_sms[dev] = sms;
    } else {
      sms = is->second;
    }
  }
  long long g = (long long)per_sm * sms;
  if (ntiles < g) g = ntiles;
  if (g < 1) g = 1;
  *grid = (int)g;
  return PFCS_OK;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = getenv("PFCS_PDL");
    return !(v && *v && atoi(v) == 0);
  }();
  return on;
}

int tune_variant(int kind, int n, int dflt) {
  char name[64];
  snprintf(name, sizeof(name), "PFCS_VARIANT_%d_%d", kind, n);
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  const int s = atoi(v);
  return (s < 0 || s > 7) ? dflt : s;
}

// defined in the other translation units
int launch_real_x(const void* in, void* out, long long nx, long long inner, int mode, double* diag,
                  cudaStream_t st);
int launch_cube_c2c(void* data, long long nx, long long inner, double* diag, cudaStream_t st);
int launch_rfft_x_pro(const double* in, void* out, long long nx, long long inner, int kind, const double* aux,
                      double alpha, cudaStream_t st);
int launch_xmul(void* data, const double* aux, long long nx, long long inner, cudaStream_t st);
bool xdot3_supported(long long nx, long long inner);
int launch_upd_zz(const double2* state, const double2* aux, const double2* aux2, double2* state_out, double2* zout,
                  long long nlines, int n1, int n, const double* kx, const double* ky, const double* kz, int kind,
                  double c0, double c1, double c2, int flags, double* diag, cudaStream_t st);
int launch_mu_z(const double2* nl, const double2* f, double2* mu, double2* nl_out, long long nlines, int n1, int n,
                const double* kx, const double* ky, const double* kz, double eps, cudaStream_t st, double2* t0_out,
                double2* tz_out, const double* dz);
int launch_xdot3(const void* const* spec, const double* v0, const double* v1, const double* v2, void* out,
                 long long nx, long long inner, const double* dx, cudaStream_t st);
int launch_pfc_z(const double2* nl, double2* psi_hat, double2* next, long long cx, long long ny,
                 long long nz, int g_in, int g_out, const double* kx, const double* ky,
                 const double* kz, double eps, double dt, double* diag, cudaStream_t st,
                 const PeerTable* dst);
int launch_pfc_cube(void* data, long long n, int real, double* diag, cudaStream_t st);
int launch_pfc_update(const double2* nl, double2* psi_hat, long long cx, long long ny, long long nz,
                      const double* kx, const double* ky, const double* kz, double eps, double dt,
                      double* diag, cudaStream_t st);
int launch_apply_op(const double2* in, double2* out, long long cx, long long ny, long long nz,
                    const double* kx, const double* ky, const double* kz, double eps,
                    cudaStream_t st);
int launch_energy_sum(const double* a, long long sa, const double* b, long long sb, long long n,
                      double* out, double* scratch, cudaStream_t st);
long long energy_scratch_bytes(long long n);
int launch_absmax(const double* a, long long sa, long long n, double* out, cudaStream_t st);

}  // namespace pfcs

using namespace pfcs;

static inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

extern "C" {

int pfcs_version(void) { return 100; }  // 0.1.0

const char* pfcs_last_error(void) { return g_err.c_str(); }

int pfcs_device_count(int* count) { return check_cuda(cudaGetDeviceCount(count), "cudaGetDeviceCount"); }

int pfcs_fft_axis_c2c(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, int axis,
                      int forward, void* stream) {
  if (axis < 0 || axis > 2) return fail(PFCS_E_ARG, "axis must be 0, 1 or 2");
  if (n0 < 0 || n1 < 0 || n2 < 0) return fail(PFCS_E_ARG, "negative extent");
  const int64_t total = n0 * n1 * n2;
  if (total == 0) return PFCS_OK;
  const int64_t n = axis == 0 ? n0 : (axis == 1 ? n1 : n2);
  if (n == 1) {  // fftcore.py:36-37: length-1 axes are copied
    if (in != out)
      return check_cuda(cudaMemcpyAsync(out, in, (size_t)total * 16, cudaMemcpyDeviceToDevice, S(stream)),
                        "copy");
    return PFCS_OK;
  }
  if (n > 16384) return fail(PFCS_E_UNSUPPORTED, "line length > 16384");
  const int64_t outer = axis == 0 ? 1 : (axis == 1 ? n0 : n0 * n1);
  const int64_t inner = axis == 0 ? n1 * n2 : (axis == 1 ? n2 : 1);
  if (inner == 1)
    return launch_lines_c2c((const double2*)in, (double2*)out, outer, (int)n, 1, 1, forward != 0, S(stream));
  return launch_strided_c2c((const double2*)in, (double2*)out, outer, (int)n, inner, forward != 0, S(stream));
}

int pfcs_update_zinv(int kind, const void* state_in, const void* aux, const void* aux2, void* state_out, void* zout,
                     int64_t n0, int64_t n1, int64_t n2, const double* kx, const double* ky, const double* kz,
                     double c0, double c1, double c2, double* diag, void* stream) {
  if (kind < 0 || kind > 2) return fail(PFCS_E_ARG, "update kind must be 0 (psi), 1 (velocity) or 2 (composition)");
  if (!state_in || !aux || !state_out || !zout || !kx || !ky || !kz) return fail(PFCS_E_ARG, "null argument");
  if (zout == state_in || zout == state_out || zout == aux || (aux2 && zout == aux2))
    return fail(PFCS_E_ARG, "zout must not alias the state or the operands");
  if (n0 < 0 || n1 < 0 || n2 < 0) return fail(PFCS_E_ARG, "negative extent");
  if (n0 * n1 * n2 == 0) return PFCS_OK;
  Pro p{};
  p.kind = PRO_UPD_PSI + kind;
  p.aux = aux;
  p.aux2 = kind == 1 ? nullptr : aux2;
  p.out2 = state_out;
  p.axis = 2;
  p.n1 = (int)n1;
  p.n2 = (int)n2;
  p.kx = kx;
  p.ky = ky;
  p.kz = kz;
  p.c0 = c0;
  p.c1 = c1;
  p.c2 = c2;
  p.diag = diag;
  if (n2 > 1) {
    const int rc = launch_lines_pro((const double2*)state_in, (double2*)zout, n0 * n1, (int)n2, p, false, S(stream));
    if (rc != 1) return rc;
  }
  // lengths without a fused kernel: the standalone update, then the z pass
  int rc = kind == 0   ? pfcs_hydro_psi_update_to(state_in, state_out, aux, aux2, n0, n1, n2, kx, ky, kz, c0, c1,
                                                  diag, stream)
           : kind == 1 ? pfcs_hydro_vel_update_to(state_in, state_out, aux, n0, n1, n2, kx, ky, kz, c0, c1, c2,
                                                  diag, stream)
                       : pfcs_ch_update_to(state_in, state_out, aux, aux2, n0, n1, n2, kx, ky, kz, c0, c1, c2, diag,
                                           stream);
  if (rc) return rc;
  return pfcs_fft_axis_c2c(state_out, zout, n0, n1, n2, 2, 0, stream);
}

int pfcs_update_zzinv(int kind, const void* state_in, void* aux, void* aux2, void* state_out, void* zout, int64_t n0,
                      int64_t n1, int64_t n2, const double* kx, const double* ky, const double* kz, double c0,
                      double c1, double c2, int flags, double* diag, void* stream) {
  if (kind < 0 || kind > 2) return fail(PFCS_E_ARG, "update kind must be 0 (psi), 1 (velocity) or 2 (composition)");
  if (!state_in || !aux || !state_out || !zout || !kx || !ky || !kz) return fail(PFCS_E_ARG, "null argument");
  if (zout == state_in || zout == state_out || zout == aux || (aux2 && zout == aux2))
    return fail(PFCS_E_ARG, "zout must not alias the state or the operands");
  if (n0 < 0 || n1 < 0 || n2 < 0) return fail(PFCS_E_ARG, "negative extent");
  if (n0 * n1 * n2 == 0) return PFCS_OK;
  if (kind == 1) aux2 = nullptr;
  const int rc = launch_upd_zz((const double2*)state_in, (const double2*)aux, (const double2*)aux2,
                               (double2*)state_out, (double2*)zout, n0 * n1, (int)n1, (int)n2, kx, ky, kz, kind, c0,
                               c1, c2, flags, diag, S(stream));
  if (rc != 1) return rc;
  // other z lengths: the operands' forward z passes in place, then the update + inverse z
  if (flags & 1)
    if (int r = pfcs_fft_axis_c2c(aux, aux, n0, n1, n2, 2, 1, stream)) return r;
  if (aux2 && (flags & 2))
    if (int r = pfcs_fft_axis_c2c(aux2, aux2, n0, n1, n2, 2, 1, stream)) return r;
  return pfcs_update_zinv(kind, state_in, aux, aux2, state_out, zout, n0, n1, n2, kx, ky, kz, c0, c1, c2, diag,
                          stream);
}

int pfcs_fft_axis_c2c_pro(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, int axis,
                          int forward, int pro, const void* aux, int aux_axis, void* stream) {
  if (pro == PRO_NONE) return pfcs_fft_axis_c2c(in, out, n0, n1, n2, axis, forward, stream);
  if (pro < PRO_CUBE || pro > PRO_DERIV) return fail(PFCS_E_ARG, "unknown prologue");
  if (axis < 0 || axis > 2 || aux_axis < 0 || aux_axis > 2) return fail(PFCS_E_ARG, "axis must be 0, 1 or 2");
  if (n0 < 0 || n1 < 0 || n2 < 0) return fail(PFCS_E_ARG, "negative extent");
  if (pro != PRO_CUBE && aux == nullptr) return fail(PFCS_E_ARG, "prologue needs aux");
  if (aux == out) return fail(PFCS_E_ARG, "aux must not alias out");
  const int64_t total = n0 * n1 * n2;
  if (total == 0) return PFCS_OK;
  const int64_t n = axis == 0 ? n0 : (axis == 1 ? n1 : n2);
  const int64_t outer = axis == 0 ? 1 : (axis == 1 ? n0 : n0 * n1);
  const int64_t inner = axis == 0 ? n1 * n2 : (axis == 1 ? n2 : 1);
  Pro p{pro, aux, aux_axis, (int)n1, (int)n2};
  p.pass = axis;
  if (n > 1 && n <= 4096) {
    // fused: contiguous lines (k_lines) or the TMA-staged strided pass
    // (B200, 512^3 multiphysics step: 105 -> 95 ms with cube, product and
    // derivative multipliers fused)
    const int rc = inner == 1 ? launch_lines_pro((const double2*)in, (double2*)out, outer, (int)n, p,
                                                 forward != 0, S(stream))
                   : (tma_enabled() ? launch_strided_tma((const double2*)in, (double2*)out, outer, (int)n, inner,
                                                         forward != 0, S(stream), nullptr, nullptr, &p)
                                    : 1);
    if (rc != 1) return rc;
  }
  // unfused: the standalone pointwise kernel into out, then the pass in place
  int rc = PFCS_OK;
  if (pro == PRO_CUBE) {
    if (in != out)
      rc = check_cuda(cudaMemcpyAsync(out, in, (size_t)total * 16, cudaMemcpyDeviceToDevice, S(stream)), "copy");
    if (!rc) rc = pfcs_pfc_cube(out, total, 0, nullptr, stream);
  } else if (pro == PRO_CMUL) {
    rc = pfcs_cmul(aux, in, out, total, stream);
  } else {
    rc = pfcs_mul_deriv(in, out, n0, n1, n2, (const double*)aux, aux_axis, stream);
  }
  if (rc) return rc;
  return pfcs_fft_axis_c2c(out, out, n0, n1, n2, axis, forward, stream);
}

int pfcs_fft_zlines(const void* in, void* out, int64_t nlines, int64_t nz, int g_in, int g_out,
                    int forward, void* stream) {
  if (nlines < 0 || nz < 1 || g_in < 1 || g_out < 1) return fail(PFCS_E_ARG, "bad z-line geometry");
  if (nlines == 0) return PFCS_OK;
  if (nz == 1) {
    if (in != out)
      return check_cuda(cudaMemcpyAsync(out, in, (size_t)nlines * 16, cudaMemcpyDeviceToDevice, S(stream)),
                        "copy");
    return PFCS_OK;
  }
  if (nz > 16384) return fail(PFCS_E_UNSUPPORTED, "line length > 16384");
  return launch_lines_c2c((const double2*)in, (double2*)out, nlines, (int)nz, g_in, g_out, forward != 0,
                          S(stream));
}

int pfcs_fft_lines(const void* in, void* out, int64_t outer, int64_t n, int64_t inner, int g_in, int g_out,
                   int forward, void* stream) {
  if (outer < 0 || n < 1 || inner < 0 || g_in < 1 || g_out < 1) return fail(PFCS_E_ARG, "bad line geometry");
  if (outer == 0 || inner == 0) return PFCS_OK;
  if (n == 1) {
    if (in != out)
      return check_cuda(cudaMemcpyAsync(out, in, (size_t)(outer * inner) * 16, cudaMemcpyDeviceToDevice,
                                        S(stream)),
                        "copy");
    return PFCS_OK;
  }
  return launch_strided_blocked((const double2*)in, (double2*)out, outer, (int)n, inner, g_in, g_out,
                                forward != 0, S(stream));
}

int pfcs_rfft_x_pro(const double* in, void* out, int64_t nx, int64_t inner, int kind, const double* aux,
                    double alpha, void* stream) {
  if (!in || !out) return fail(PFCS_E_ARG, "null argument");
  return launch_rfft_x_pro(in, out, nx, inner, kind, aux, alpha, S(stream));
}

int pfcs_xmul_x(void* data, const double* aux, int64_t nx, int64_t inner, void* stream) {
  if (!data) return fail(PFCS_E_ARG, "null argument");
  if (nx < 1 || inner < 0) return fail(PFCS_E_ARG, "bad shape");
  if ((const void*)aux == data) return fail(PFCS_E_ARG, "aux must not alias data");
  return launch_xmul(data, aux, nx, inner, S(stream));
}

int pfcs_hydro_mu_z(const void* nl_xy, const void* f_xy, void* mu, void* nl_out, int64_t n0, int64_t n1,
                    int64_t n2, const double* kx, const double* ky, const double* kz, double eps, void* stream) {
  return pfcs_hydro_mu_zgrad(nl_xy, f_xy, mu, nl_out, nullptr, nullptr, nullptr, n0, n1, n2, kx, ky, kz, eps, stream);
}

int pfcs_hydro_mu_zgrad(const void* nl_xy, const void* f_xy, void* mu, void* nl_out, void* t0_out, void* tz_out,
                        const double* dz, int64_t n0, int64_t n1, int64_t n2, const double* kx, const double* ky,
                        const double* kz, double eps, void* stream) {
  if (!nl_xy || !f_xy || !kx || !ky || !kz) return fail(PFCS_E_ARG, "null argument");
  if (!mu && !t0_out && !tz_out) return fail(PFCS_E_ARG, "no output");
  if (tz_out && !dz) return fail(PFCS_E_ARG, "tz_out needs the derivative vector dz");
  const void* outs[4] = {mu, nl_out, t0_out, tz_out};
  for (int i = 0; i < 4; ++i) {
    if (outs[i] && (outs[i] == nl_xy || outs[i] == f_xy)) return fail(PFCS_E_ARG, "an output aliases an operand");
    for (int k = 0; k < i; ++k)
      if (outs[i] && outs[i] == outs[k]) return fail(PFCS_E_ARG, "outputs alias each other");
  }
  if (n0 < 0 || n1 < 0 || n2 < 0) return fail(PFCS_E_ARG, "negative extent");
  if (n0 * n1 * n2 == 0) return PFCS_OK;
  const int rc = launch_mu_z((const double2*)nl_xy, (const double2*)f_xy, (double2*)mu, (double2*)nl_out, n0 * n1,
                             (int)n1, (int)n2, kx, ky, kz, eps, S(stream), (double2*)t0_out, (double2*)tz_out, dz);
  if (rc != 1) return rc;
  if (t0_out || tz_out || !mu)
    return fail(PFCS_E_UNSUPPORTED, "mu_hat with its gradient's z passes needs a power-of-two z length in [8, 4096]");
  // other z lengths: the two forward z passes, then the mu pass
  void* nlz = nl_out ? nl_out : (void*)nl_xy;
  if (int r = pfcs_fft_axis_c2c(nl_xy, nlz, n0, n1, n2, 2, 1, stream)) return r;
  if (int r = pfcs_fft_axis_c2c(f_xy, (void*)f_xy, n0, n1, n2, 2, 1, stream)) return r;
  return pfcs_hydro_mu(nlz, f_xy, mu, n0, n1, n2, kx, ky, kz, eps, stream);
}

int pfcs_xdot3_supported(int64_t nx, int64_t inner) { return xdot3_supported(nx, inner) ? 1 : 0; }

int pfcs_xdot3_x(const void* s0, const void* s1, const void* s2, const double* v0, const double* v1,
                 const double* v2, void* out, int64_t nx, int64_t inner, const double* dx, void* stream) {
  if (!s0 || !s1 || !s2 || !v0 || !v1 || !v2 || !out) return fail(PFCS_E_ARG, "null argument");
  if (out == s0 || out == s1 || out == s2) return fail(PFCS_E_ARG, "out must not alias the derivative spectra");
  const void* spec[3] = {s0, s1, s2};
  const int rc = launch_xdot3(spec, v0, v1, v2, out, nx, inner, dx, S(stream));
  if (rc == 1) return fail(PFCS_E_UNSUPPORTED, "fused advection x pass: nx 256 or 512 with TMA (pfcs_xdot3_supported)");
  return rc;
}

int pfcs_rfft_x(const double* in, void* out, int64_t nx, int64_t inner, void* stream) {
  if (nx < 1 || inner < 0) return fail(PFCS_E_ARG, "bad shape");
  return launch_real_x(in, out, nx, inner, 0, nullptr, S(stream));
}

int pfcs_irfft_x(const void* in, double* out, int64_t nx, int64_t inner, void* stream) {
  if (nx < 1 || inner < 0) return fail(PFCS_E_ARG, "bad shape");
  return launch_real_x(in, out, nx, inner, 1, nullptr, S(stream));
}

int pfcs_pfc_cube_x(void* data, int64_t nx, int64_t inner, int real, double* diag, void* stream) {
  if (nx < 1 || inner < 0) return fail(PFCS_E_ARG, "bad shape");
  if (real) return launch_real_x(data, data, nx, inner, 2, diag, S(stream));
  return launch_cube_c2c(data, nx, inner, diag, S(stream));
}

int pfcs_pfc_update_z(const void* nl, void* psi_hat, void* next_out, int64_t cx, int64_t ny,
                      int64_t nz, int g_in, int g_out, const double* kx, const double* ky,
                      const double* kz, double eps, double dt, double* diag, void* stream) {
  if (cx < 0 || ny < 1 || nz < 1 || g_in < 1 || g_out < 1) return fail(PFCS_E_ARG, "bad slab geometry");
  return launch_pfc_z((const double2*)nl, (double2*)psi_hat, (double2*)next_out, cx, ny, nz, g_in, g_out,
                      kx, ky, kz, eps, dt, diag, S(stream), nullptr);
}

// ------------------------------------------------------ fused exchanges ----

static int make_table(const uint64_t* dst, int g, PeerTable* t) {
  if (!dst || g < 1 || g > PFCS_MAX_PEERS) return fail(PFCS_E_ARG, "destination table needs 1..16 entries");
  *t = PeerTable{};
  for (int i = 0; i < g; ++i) t->p[i] = (double2*)(uintptr_t)dst[i];
  return PFCS_OK;
}

int pfcs_fft_zlines_to(const void* in, const uint64_t* dst, int64_t nlines, int64_t nz, int g_in, int g_out,
                       int forward, void* stream) {
  PeerTable t;
  if (int rc = make_table(dst, g_out, &t)) return rc;
  if (nlines <= 0) return PFCS_OK;
  return launch_lines_to((const double2*)in, nullptr, nlines, (int)nz, g_in, g_out, &t, forward != 0,
                         S(stream));
}

int pfcs_fft_lines_scatter(const void* in, const uint64_t* dst, int64_t outer, int64_t n, int64_t inner,
                           int g_in, int g_outer, int forward, void* stream) {
  PeerTable t;
  if (int rc = make_table(dst, g_outer, &t)) return rc;
  return launch_strided_to((const double2*)in, outer, (int)n, inner, g_in, &t, g_outer, forward != 0,
                           S(stream));
}

int pfcs_pfc_update_z_to(const void* nl, void* psi_hat, const uint64_t* dst, int64_t cx, int64_t ny, int64_t nz,
                         int g_in, int g_out, const double* kx, const double* ky, const double* kz, double eps,
                         double dt, double* diag, void* stream) {
  PeerTable t;
  if (int rc = make_table(dst, g_out, &t)) return rc;
  if (cx < 0 || ny < 1 || nz < 1 || g_in < 1) return fail(PFCS_E_ARG, "bad slab geometry");
  return launch_pfc_z((const double2*)nl, (double2*)psi_hat, nullptr, cx, ny, nz, g_in, g_out, kx, ky, kz, eps,
                      dt, diag, S(stream), &t);
}

int pfcs_enable_peer_access(int peer_device) {
  int dev = 0;
  if (int rc = check_cuda(cudaGetDevice(&dev), "cudaGetDevice")) return rc;
  if (peer_device == dev) return PFCS_OK;
  int can = 0;
  if (int rc = check_cuda(cudaDeviceCanAccessPeer(&can, dev, peer_device), "cudaDeviceCanAccessPeer")) return rc;
  if (!can) return fail(PFCS_E_UNSUPPORTED, "no peer access between these devices");
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return PFCS_OK;
  }
  return check_cuda(e, "cudaDeviceEnablePeerAccess");
}

int pfcs_malloc(int64_t bytes, void** ptr) {
  return check_cuda(cudaMalloc(ptr, (size_t)(bytes > 0 ? bytes : 16)), "cudaMalloc");
}

int pfcs_free(void* ptr) { return check_cuda(cudaFree(ptr), "cudaFree"); }

int pfcs_ipc_get_handle(const void* ptr, void* handle64) {
  cudaIpcMemHandle_t h;
  if (int rc = check_cuda(cudaIpcGetMemHandle(&h, (void*)ptr), "cudaIpcGetMemHandle")) return rc;
  memcpy(handle64, &h, sizeof(h));
  return PFCS_OK;
}

int pfcs_ipc_open_handle(const void* handle64, void** ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return check_cuda(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int pfcs_ipc_close(void* ptr) { return check_cuda(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle"); }

int pfcs_stream_sync(void* stream) { return check_cuda(cudaStreamSynchronize(S(stream)), "cudaStreamSynchronize"); }

// Interprocess events: device-side ordering of the fused exchanges between
// processes (peer.fence) — record on one process's stream, wait on another's.
int pfcs_ipc_event_create(void** event, void* handle64) {
  cudaEvent_t ev;
  if (int rc = check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess),
                          "cudaEventCreateWithFlags"))
    return rc;
  cudaIpcEventHandle_t h;
  if (int rc = check_cuda(cudaIpcGetEventHandle(&h, ev), "cudaIpcGetEventHandle")) {
    cudaEventDestroy(ev);
    return rc;
  }
  memcpy(handle64, &h, sizeof(h));
  *event = (void*)ev;
  return PFCS_OK;
}

int pfcs_ipc_event_open(const void* handle64, void** event) {
  cudaIpcEventHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaEvent_t ev;
  if (int rc = check_cuda(cudaIpcOpenEventHandle(&ev, h), "cudaIpcOpenEventHandle")) return rc;
  *event = (void*)ev;
  return PFCS_OK;
}

int pfcs_event_record(void* event, void* stream) {
  return check_cuda(cudaEventRecord((cudaEvent_t)event, S(stream)), "cudaEventRecord");
}

int pfcs_stream_wait_event(void* stream, void* event) {
  return check_cuda(cudaStreamWaitEvent(S(stream), (cudaEvent_t)event, 0), "cudaStreamWaitEvent");
}

int pfcs_event_destroy(void* event) { return check_cuda(cudaEventDestroy((cudaEvent_t)event), "cudaEventDestroy"); }

int pfcs_pfc_cube(void* data, int64_t n, int real, double* diag, void* stream) {
  if (n < 0) return fail(PFCS_E_ARG, "negative count");
  return launch_pfc_cube(data, n, real, diag, S(stream));
}

int pfcs_pfc_update(const void* nl_hat, void* psi_hat, int64_t cx, int64_t ny, int64_t nz,
                    const double* kx, const double* ky, const double* kz, double eps, double dt,
                    double* diag, void* stream) {
  if (cx < 0 || ny < 1 || nz < 1) return fail(PFCS_E_ARG, "bad slab geometry");
  return launch_pfc_update((const double2*)nl_hat, (double2*)psi_hat, cx, ny, nz, kx, ky, kz, eps, dt,
                           diag, S(stream));
}

int pfcs_energy_sum(const double* a, int64_t sa, const double* b, int64_t sb, int64_t n, double* out,
                    double* scratch, void* stream) {
  if (n < 0) return fail(PFCS_E_ARG, "negative count");
  return launch_energy_sum(a, sa, b, sb, n, out, scratch, S(stream));
}

int64_t pfcs_energy_scratch_bytes(int64_t n) { return energy_scratch_bytes(n); }

int pfcs_absmax(const double* a, int64_t sa, int64_t n, double* out, void* stream) {
  if (n < 0) return fail(PFCS_E_ARG, "negative count");
  return launch_absmax(a, sa, n, out, S(stream));
}

int pfcs_apply_op(const void* in, void* out, int64_t cx, int64_t ny, int64_t nz, const double* kx,
                  const double* ky, const double* kz, double eps, void* stream) {
  return launch_apply_op((const double2*)in, (double2*)out, cx, ny, nz, kx, ky, kz, eps, S(stream));
}

}  // extern "C"

// ------------------------------------------------------------ plan API ----
struct pfcs_plan {
  int64_t nx, ny, nz, nh;
};

extern "C" {

int pfcs_plan_create(int64_t nx, int64_t ny, int64_t nz, pfcs_plan** plan) {
  if (!plan) return fail(PFCS_E_ARG, "plan out-pointer is null");
  *plan = nullptr;
  if (nx < 4 || ny < 1 || nz < 1) return fail(PFCS_E_ARG, "bad grid");
  if (!is_pow2(nx) || nx > 8192) return fail(PFCS_E_UNSUPPORTED, "plan needs a power-of-two nx in [4, 8192]");
  if (!is_pow2(nz) || nz > 4096) return fail(PFCS_E_UNSUPPORTED, "plan needs a power-of-two nz <= 4096");
  *plan = new pfcs_plan{nx, ny, nz, nx / 2 + 1};
  return PFCS_OK;
}

int pfcs_plan_destroy(pfcs_plan* plan) {
  delete plan;
  return PFCS_OK;
}

int64_t pfcs_plan_spectral_elems(const pfcs_plan* p) { return p ? p->nh * p->ny * p->nz : -1; }

int pfcs_plan_fwd(const pfcs_plan* p, const double* in, void* out, void* stream) {
  if (!p || !in || !out) return fail(PFCS_E_ARG, "null argument");
  // x (R2C), y in place, z in place: distfft._forward_core at G = 1
  if (int rc = pfcs_rfft_x(in, out, p->nx, p->ny * p->nz, stream)) return rc;
  if (p->ny > 1)
    if (int rc = pfcs_fft_axis_c2c(out, out, p->nh, p->ny, p->nz, 1, 1, stream)) return rc;
  return pfcs_fft_zlines(out, out, p->nh * p->ny, p->nz, 1, 1, 1, stream);
}

int pfcs_plan_inv(const pfcs_plan* p, const void* in, double* out, void* work, void* stream) {
  if (!p || !in || !out || !work) return fail(PFCS_E_ARG, "null argument");
  // z (into work), y in place, x (C2R): distfft._inverse_core at G = 1
  if (int rc = pfcs_fft_zlines(in, work, p->nh * p->ny, p->nz, 1, 1, 0, stream)) return rc;
  if (p->ny > 1)
    if (int rc = pfcs_fft_axis_c2c(work, work, p->nh, p->ny, p->nz, 1, 0, stream)) return rc;
  return pfcs_irfft_x(work, out, p->nx, p->ny * p->nz, stream);
}

int pfcs_plan_pfc_steps(const pfcs_plan* p, void* psi_hat, const double* kx, const double* ky, const double* kz,
                        double eps, double dt, int64_t nsteps, double* diag, void* work, void* stream) {
  if (!p || !psi_hat || !kx || !ky || !kz || !work) return fail(PFCS_E_ARG, "null argument");
  if (nsteps < 0) return fail(PFCS_E_ARG, "negative step count");
  if (nsteps == 0) return PFCS_OK;
  const size_t per = (size_t)PFCS_DIAG_SLOTS * 4;
  if (diag)
    if (int rc = check_cuda(cudaMemsetAsync(diag, 0, (size_t)nsteps * per * sizeof(double), S(stream)), "memset"))
      return rc;
  // pfc._StepEngine.launch, fused G = 1: work holds the z-inverse of psi_hat
  // (the update kernel leaves the next step's in it)
  const int64_t lines = p->nh * p->ny;
  if (int rc = pfcs_fft_zlines(psi_hat, work, lines, p->nz, 1, 1, 0, stream)) return rc;
  for (int64_t s = 0; s < nsteps; ++s) {
    double* d = diag ? diag + s * per : nullptr;
    if (p->ny > 1)
      if (int rc = pfcs_fft_axis_c2c(work, work, p->nh, p->ny, p->nz, 1, 0, stream)) return rc;
    if (int rc = pfcs_pfc_cube_x(work, p->nx, p->ny * p->nz, 1, d, stream)) return rc;
    if (p->ny > 1)
      if (int rc = pfcs_fft_axis_c2c(work, work, p->nh, p->ny, p->nz, 1, 1, stream)) return rc;
    if (int rc = pfcs_pfc_update_z(work, psi_hat, work, p->nh, p->ny, p->nz, 1, 1, kx, ky, kz, eps, dt, d, stream))
      return rc;
  }
  return PFCS_OK;
}

}  // extern "C"

