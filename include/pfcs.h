/* pfcs.h — C ABI of libpfcs, the sm_100a pseudo-spectral hot path.
 *
 * Plain pointers and sizes only: every array argument is a DEVICE pointer
 * (fp64 / complex128 = interleaved {re, im} doubles, C order), every
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Calls are asynchronous on `stream` unless stated; the caller owns all
 * buffers.  Return value: PFCS_OK or a PFCS_E_* code; the message of the most
 * recent failure on the calling thread is available from pfcs_last_error().
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/pfcspectral/<file>:<line>).  The reference is a
 * pure-Python package with no FFI of its own; the Python layer of this repo
 * (paper_2603_26818_b200/) keeps the reference signatures and binds these
 * symbols with ctypes (INTEGRATION.md shows the binding).
 */
#ifndef PFCS_H
#define PFCS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFCS_OK 0
#define PFCS_E_ARG 1         /* bad shape / axis / layout  -> ValueError      */
#define PFCS_E_CUDA 2        /* CUDA runtime failure                           */
#define PFCS_E_UNSUPPORTED 3 /* size not supported by the kernels              */
#define PFCS_E_NONFINITE 4   /* non-finite field -> pfc.DivergenceError        */

#define PFCS_DIAG_SLOTS 64
#define PFCS_DIAG_VALS 4

/* Library version (major*10000 + minor*100 + patch). */
int pfcs_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* pfcs_last_error(void);
/* Number of CUDA devices visible to the library (sanity/probe). */
int pfcs_device_count(int* count);

/* ---- serial line transforms: fftcore.fft_axis (fftcore.py:31-40) ------------
 * 1D DFT of every line along `axis` (0, 1, 2) of a C-order (n0, n1, n2)
 * complex128 array.  forward != 0: unnormalised; forward == 0: inverse with
 * every output scaled by fl(1/n_axis) (numpy ifft convention).  in == out is
 * allowed (in-place).  Any length: power-of-two lengths <= 4096 take the
 * Stockham kernels, other lengths the direct DFT kernel. */
int pfcs_fft_axis_c2c(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, int axis,
                      int forward, void* stream);

/* ---- pfcs_fft_axis_c2c with a pointwise prologue fused into the pass: the
 * products of hydro.hydro_psi_step / hydro_velocity_step (hydro.py:83-86,
 * 100-103) that feed fftcore.fft_nd.  The pass reads `in`, applies
 *   pro = 0: nothing (plain pfcs_fft_axis_c2c)
 *   pro = 1: x*(x*x), complex, numpy order (psi**3, pfc.py:109 / hydro.py:86)
 *   pro = 2: aux[idx] * x, aux complex128 of the same (n0, n1, n2) shape
 *   pro = 3: i * d[k] * x, aux = float64 vector indexed by coordinate aux_axis
 * and writes the transformed result to `out` (out != aux).  Bit-identical to
 * pfcs_pfc_cube / pfcs_cmul / pfcs_mul_deriv into `out` followed by
 * pfcs_fft_axis_c2c(out, out, ...); that two-kernel form is also what runs
 * when no fused kernel applies (non-power-of-two lengths). */
int pfcs_fft_axis_c2c_pro(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, int axis,
                          int forward, int pro, const void* aux, int aux_axis, void* stream);

/* ---- slab-pipeline z-line transforms: distfft.dist_fft_forward/inverse
 * (distfft.py:150-173) fused with distfft._exchange's concatenate/slice
 * (distfft.py:110-124).  `nlines` contiguous-z lines of length nz.  When
 * g_in > 1 the input is "blocked": nz split into g_in balanced slabs
 * (grid.slab_layout, grid.py:103-111), slab g stored densely as
 * (nlines, cz_g) at element offset nlines*zoff_g — the all-to-all receive
 * buffer.  g_out > 1 writes the same blocked layout (the send buffer). */
int pfcs_fft_zlines(const void* in, void* out, int64_t nlines, int64_t nz, int g_in, int g_out,
                    int forward, void* stream);

/* ---- pencil-pipeline line transforms (new: pencil decomposition, north-star
 * item (2)).  Lines along the middle axis of an (outer, n, inner) array
 * (inner = 1: contiguous lines).  g_in / g_out > 1 select the "blocked"
 * layout of the line axis: n split into g balanced slabs, slab g stored
 * densely as (outer, cn_g, inner) at element offset outer*inner*noff_g —
 * what a pencil all-to-all over that axis delivers / needs.  Generalises
 * pfcs_fft_zlines (inner = 1). */
int pfcs_fft_lines(const void* in, void* out, int64_t outer, int64_t n, int64_t inner, int g_in, int g_out,
                   int forward, void* stream);

/* ---- fused exchanges (north-star item (2): the transpose fused into the
 * FFT epilogue over NVLink peer memory).  `dst` is a HOST array of g_out
 * device addresses — typically the receive buffers of the g_out ranks,
 * mapped with pfcs_enable_peer_access (threads) or pfcs_ipc_open_handle
 * (processes), each already offset to where this rank's block lands.  The
 * kernel stores every output element straight into its owner's buffer, so
 * there is no send buffer and no separate all-to-all; the caller only
 * orders the step with a barrier.
 * pfcs_fft_zlines_to:     as pfcs_fft_zlines; z block h of line l goes to
 *                         dst[h] + l*cz_h + (z - zoff_h).
 * pfcs_fft_lines_scatter: lines along the middle axis of (outer, n, inner)
 *                         (input plain or blocked over g_in); output row o
 *                         goes to dst[h] + ((o - ooff_h)*n + k)*inner + i,
 *                         h the owner of o in slab_layout(outer, g_outer).
 * pfcs_pfc_update_z_to:   pfcs_pfc_update_z with the next-step inverse
 *                         scattered like pfcs_fft_zlines_to. */
int pfcs_fft_zlines_to(const void* in, const uint64_t* dst, int64_t nlines, int64_t nz, int g_in, int g_out,
                       int forward, void* stream);
int pfcs_fft_lines_scatter(const void* in, const uint64_t* dst, int64_t outer, int64_t n, int64_t inner,
                           int g_in, int g_outer, int forward, void* stream);
int pfcs_pfc_update_z_to(const void* nl, void* psi_hat, const uint64_t* dst, int64_t cx, int64_t ny, int64_t nz,
                         int g_in, int g_out, const double* kx, const double* ky, const double* kz, double eps,
                         double dt, double* diag, void* stream);
/* Peer / IPC plumbing for the fused exchanges. */
int pfcs_enable_peer_access(int peer_device);
int pfcs_malloc(int64_t bytes, void** ptr);
int pfcs_free(void* ptr);
int pfcs_ipc_get_handle(const void* ptr, void* handle64);
int pfcs_ipc_open_handle(const void* handle64, void** ptr);
int pfcs_ipc_close(void* ptr);
int pfcs_stream_sync(void* stream);
/* Interprocess events (device-side ordering of the fused exchanges between
 * processes): create an interprocess event and its 64-byte IPC handle, open
 * a peer's handle, record on a stream, make a stream wait for an event. */
int pfcs_ipc_event_create(void** event, void* handle64);
int pfcs_ipc_event_open(const void* handle64, void** event);
int pfcs_event_record(void* event, void* stream);
int pfcs_stream_wait_event(void* stream, void* event);
int pfcs_event_destroy(void* event);

/* ---- real transforms along axis 0 (x) of a C-order array (new: R2C/C2R,
 * north-star item (1)).  rfft: real (nx, inner) -> complex (nx/2+1, inner),
 * unnormalised.  irfft: complex (nx/2+1, inner) -> real (nx, inner), scaled
 * by fl(1/nx); the imaginary parts of modes 0 and nx/2 are ignored (numpy
 * irfft convention).  nx must be an even power of two in [4, 8192]. */
int pfcs_rfft_x(const double* in, void* out, int64_t nx, int64_t inner, void* stream);
int pfcs_irfft_x(const void* in, double* out, int64_t nx, int64_t inner, void* stream);
/* rfft of f(in) with the pointwise f fused into the x pass (the R2C
 * multiphysics transforms of hydro.py:86, 96-98): kind 0 f(x) = (x*x)*x,
 * kind 1 f(x) = x*aux (aux: a real array of in's layout), kind 3
 * f(x) = alpha*(x*(x*x) - x) — pfcs_real_pointwise's arithmetic, so
 * bit-identical to that kernel followed by pfcs_rfft_x. */
int pfcs_rfft_x_pro(const double* in, void* out, int64_t nx, int64_t inner, int kind, const double* aux,
                    double alpha, void* stream);
/* The x pass of a pseudo-spectral product, in place: data (an (nx/2+1,
 * inner) x-halved spectrum whose y and z passes are done) <- R2C(C2R(data) *
 * aux), aux a real (nx, inner) field — the hydro force psi * F^-1(i k mu)
 * between the inverse and forward x stages (hydro.py:98), so neither factor
 * nor product reaches HBM.  Bit-identical to pfcs_irfft_x, then
 * pfcs_real_pointwise kind 1 with aux, then pfcs_rfft_x. */
int pfcs_xmul_x(void* data, const double* aux, int64_t nx, int64_t inner, void* stream);
/* The x pass of the advection term v . grad x (hydro.py:83-85) in one pass:
 * s0, s1, s2 = the three derivative spectra i d_a x_hat after their inverse
 * z and y passes ((nx/2+1, inner) each); v0..v2 real (nx, inner); out
 * (nx/2+1, inner) = R2C((v0 g0 + v1 g1) + v2 g2), g_a = C2R(s_a) —
 * bit-identical to three pfcs_irfft_x + pfcs_real_pointwise kind 2 +
 * pfcs_rfft_x.  dx (or NULL): s0 is the plain transform and its i d_x
 * multiplier (a function of the x mode only) is applied to the loaded modes
 * first, as pfcs_mul_deriv(axis 0) would.  nx 256 or 512 (TMA-staged);
 * pfcs_xdot3_supported(nx, inner) says whether this build / setting has the
 * fused kernel (PFCS_E_UNSUPPORTED otherwise). */
int pfcs_xdot3_supported(int64_t nx, int64_t inner);
/* mu_hat of hydro_velocity_step (hydro.py:99-101) fused with the forward z
 * passes of its operands: nl_xy, f_xy = F(psi^3) and F(psi) after their x
 * and y passes ((n0, n1, n2) complex, z contiguous); mu = nl + op(k) f with
 * op = eps + ((1-k2)^2)((4/3-k2)^2) — bit-identical to pfcs_fft_axis_c2c
 * (axis 2, forward) on both, then pfcs_hydro_mu.  nl_out (or NULL)
 * receives the finished F(psi^3) (the next step's density update reads the
 * same spectrum of the same psi).  Other z lengths run the unfused form
 * (transforming f_xy, and nl_xy when nl_out is NULL, in place). */
int pfcs_hydro_mu_z(const void* nl_xy, const void* f_xy, void* mu, void* nl_out, int64_t n0, int64_t n1,
                    int64_t n2, const double* kx, const double* ky, const double* kz, double eps, void* stream);
/* pfcs_hydro_mu_z that also runs the first inverse z passes of grad mu
 * (the x / y derivatives' shared plain pass -> t0_out, the z derivative's
 * pass with the i k_z multiplier dz -> tz_out; either may be NULL), so
 * mu_hat itself need not be stored (mu may be NULL).  Bit-identical to
 * pfcs_hydro_mu_z followed by pfcs_fft_axis_c2c(mu, t0, axis 2, inverse) and
 * pfcs_fft_axis_c2c_pro(mu, tz, axis 2, inverse, derivative dz, 2).  Power-of-
 * two z lengths in [8, 4096] only (PFCS_E_UNSUPPORTED otherwise). */
int pfcs_hydro_mu_zgrad(const void* nl_xy, const void* f_xy, void* mu, void* nl_out, void* t0_out, void* tz_out,
                        const double* dz, int64_t n0, int64_t n1, int64_t n2, const double* kx, const double* ky,
                        const double* kz, double eps, void* stream);
int pfcs_xdot3_x(const void* s0, const void* s1, const void* s2, const double* v0, const double* v1,
                 const double* v2, void* out, int64_t nx, int64_t inner, const double* dx, void* stream);

/* ---- fused PFC step kernels: pfc.pfc_step (pfc.py:96-128) ---------------
 * Diagnostics block `diag` (device, PFCS_DIAG_SLOTS x 4 doubles; the caller
 * zeroes it per step and max-reduces the slots): per slot
 *   [0] = max |Re psi|, [1] = max |Im psi|, [2] = max |psi|
 *   (of the physical field before the update, pfc.py:100-105,124),
 *   [3] = non-zero if a non-finite value was produced (pfc.py:122).
 * CTAs stripe their atomics over the slots (no same-address hot spot).
 * diag may be NULL (no diagnostics).
 *
 * pfcs_pfc_cube_x: x-line pass of the physical-space nonlinearity.  On a
 * (nxm, inner) spectral-in-x slab (y and z already physical) it performs
 *   inverse x-transform -> psi -> psi*(psi*psi) -> forward x-transform
 * in place.  real != 0: half-spectrum data (nxm = nx/2+1, C2R/R2C, psi real);
 * real == 0: full complex data (nxm = nx, C2C, complex cube as numpy's
 * `psi ** 3`, pfc.py:109). */
int pfcs_pfc_cube_x(void* data, int64_t nx, int64_t inner, int real, double* diag, void* stream);

/* pfcs_pfc_update_z: z-line pass of the semi-implicit update (pfc.py:114-124)
 * for an X-slab spectral field psi_hat (cx, ny, nz) (plain layout, updated
 * in place).  Reads N-hat's un-transformed z lines from `nl` (blocked over
 * g_in slabs), forward z-transform, then
 *     psi_hat <- (psi_hat + dt*(lap*N_hat)) / (1 - dt*lin)
 * with the symbols of grid.make_symbols (grid.py:155-208) evaluated from the
 * 1D wavenumber vectors kx (the cx rows owned, already offset), ky, kz with
 * numpy's operation order, finiteness check into diag[3]; then, if
 * `next_out` is non-NULL, the inverse z-transform of the new psi_hat written
 * to `next_out` in the layout blocked over g_out slabs (the first stage of
 * the next step's inverse transform). */
int pfcs_pfc_update_z(const void* nl, void* psi_hat, void* next_out, int64_t cx, int64_t ny,
                      int64_t nz, int g_in, int g_out, const double* kx, const double* ky,
                      const double* kz, double eps, double dt, double* diag, void* stream);

/* Unfused forms for grids the fused passes do not cover (any size):
 * pfcs_pfc_cube: in place psi <- psi**3 on a physical slab of n points
 * (real != 0: float64 data; else complex128 with numpy's complex power
 * psi*(psi*psi)), diagnostics as above.
 * pfcs_pfc_update: the pointwise update of pfcs_pfc_update_z on an already
 * transformed nl_hat (plain (cx, ny, nz) layout), psi_hat in place. */
int pfcs_pfc_cube(void* data, int64_t n, int real, double* diag, void* stream);
int pfcs_pfc_update(const void* nl_hat, void* psi_hat, int64_t cx, int64_t ny, int64_t nz,
                    const double* kx, const double* ky, const double* kz, double eps, double dt,
                    double* diag, void* stream);

/* ---- hydrodynamic PFC pointwise operators (hydro.py:77-107) on full-grid
 * C-order (n0, n1, n2) complex128 fields; numpy's evaluation order, so the
 * viscous decay is bit-exact and v = 0 reproduces the PFC update bit for bit.
 * pfcs_mul_deriv:        out = (i d_axis) * in   (sym.d1/d2/d3 * x, hydro.py:83-85,102)
 * pfcs_cmul:             out = a * b (complex; psi * F^-1(...), hydro.py:102)
 * pfcs_hydro_advect:     out = v1*x1 + v2*x2 + v3*x3 (hydro.py:83-85)
 * pfcs_hydro_psi_update: psi_hat <- (psi_hat + dt*(lap*nl_hat - adv_hat)) / (1 - dt*lin)
 *                        (hydro.py:86-88; adv_hat may be NULL = 0)
 * pfcs_hydro_mu:         out = nl_hat + op * f_hat (hydro.py:101)
 * pfcs_hydro_vel_update: v_hat <- (v_hat - (c_cg * exp(c_exp k^2)) * force) / (1 - c_den*lap)
 *                        with c_cg = dt/rho, c_den = (dt/rho)*gamma, c_exp = -0.5*a0**2
 *                        (hydro.py:103-106; force may be NULL = 0)
 * diag as for the PFC passes (value 3 = non-finite real part seen). */
int pfcs_mul_deriv(const void* in, void* out, int64_t n0, int64_t n1, int64_t n2, const double* d,
                   int axis, void* stream);
int pfcs_cmul(const void* a, const void* b, void* out, int64_t n, void* stream);
int pfcs_hydro_advect(const void* v1, const void* x1, const void* v2, const void* x2, const void* v3,
                      const void* x3, void* out, int64_t n, void* stream);
int pfcs_hydro_psi_update(void* psi_hat, const void* nl_hat, const void* adv_hat, int64_t n0, int64_t n1,
                          int64_t n2, const double* kx, const double* ky, const double* kz, double eps,
                          double dt, double* diag, void* stream);
int pfcs_hydro_mu(const void* nl_hat, const void* f_hat, void* out, int64_t n0, int64_t n1, int64_t n2,
                  const double* kx, const double* ky, const double* kz, double eps, void* stream);
int pfcs_hydro_vel_update(void* v_hat, const void* force, int64_t n0, int64_t n1, int64_t n2,
                          const double* kx, const double* ky, const double* kz, double c_cg, double c_den,
                          double c_exp, double* diag, void* stream);
/* Out-of-place forms of the three spectral updates (state_in read, state_out
 * written; in == out is the in-place form above): the Python steps return
 * new arrays without copying the state first. */
int pfcs_hydro_psi_update_to(const void* psi_in, void* psi_out, const void* nl_hat, const void* adv_hat, int64_t n0,
                             int64_t n1, int64_t n2, const double* kx, const double* ky, const double* kz,
                             double eps, double dt, double* diag, void* stream);
int pfcs_hydro_vel_update_to(const void* v_in, void* v_out, const void* force, int64_t n0, int64_t n1, int64_t n2,
                             const double* kx, const double* ky, const double* kz, double c_cg, double c_den,
                             double c_exp, double* diag, void* stream);
int pfcs_ch_update_to(const void* c_in, void* c_out, const void* f_hat, const void* adv_hat, int64_t n0, int64_t n1,
                      int64_t n2, const double* kx, const double* ky, const double* kz, double mobility,
                      double kappa, double dt, double* diag, void* stream);

/* ---- composition field of the multiphysics mode (new; no reference
 * counterpart — restated in oracle/ref_numpy.py): Cahn-Hilliard c advected
 * by v,  mu_c = alpha (c^3 - c) - kappa lap c,  dc/dt = M lap mu_c - v.grad c.
 * pfcs_ch_nonlin: out = alpha * (c*(c*c) - c)
 * pfcs_ch_update: c_hat <- (c_hat + dt (M lap f_hat - adv_hat)) / (1 + dt M kappa lap^2)
 * pfcs_ch_mu:     out = f_hat - kappa lap c_hat
 * pfcs_add3:      out = (a + b) + c      (advection assembled from per-rank products)
 * pfcs_axpy:      out = a + w * b        (velocity force with the composition term) */
int pfcs_ch_nonlin(const void* c, void* out, int64_t n, double alpha, void* stream);
int pfcs_ch_update(void* c_hat, const void* f_hat, const void* adv_hat, int64_t n0, int64_t n1, int64_t n2,
                   const double* kx, const double* ky, const double* kz, double mobility, double kappa,
                   double dt, double* diag, void* stream);
int pfcs_ch_mu(const void* f_hat, const void* c_hat, void* out, int64_t n0, int64_t n1, int64_t n2,
               const double* kx, const double* ky, const double* kz, double kappa, void* stream);
int pfcs_add3(const void* a, const void* b, const void* c, void* out, int64_t n, void* stream);
/* A spectral update fused into the first (z) pass of the inverse transform
 * that follows it (hydro.py:86-89, 103-105 and the composition update, as
 * k_pfc_z does for PFC): reads the old state, writes the new state to
 * state_out (may alias state_in) and the inverse z transform of the new
 * state to zout, one pass.  kind 0 psi: aux = nl_hat, aux2 = adv_hat (or
 * NULL), c0 = eps, c1 = dt; kind 1 velocity: aux = force, c0 = dt/rho,
 * c1 = (dt/rho) gamma, c2 = -a0^2/2; kind 2 composition: aux = f_hat,
 * aux2 = adv_hat, c0 = mobility, c1 = kappa, c2 = dt.  Arithmetic of
 * pfcs_hydro_psi_update_to / pfcs_hydro_vel_update_to / pfcs_ch_update_to
 * followed by pfcs_fft_axis_c2c(axis 2, inverse): bit-identical. */
int pfcs_update_zinv(int kind, const void* state_in, const void* aux, const void* aux2, void* state_out, void* zout,
                     int64_t n0, int64_t n1, int64_t n2, const double* kx, const double* ky, const double* kz,
                     double c0, double c1, double c2, double* diag, void* stream);
/* pfcs_update_zinv whose operands arrive before their forward z pass
 * (flags bit 0: aux, bit 1: aux2 — after only their x and y passes): the
 * z passes run in registers inside the update (the k_pfc_z pattern), so
 * the operand spectra never reach HBM.  Bit-identical to
 * pfcs_fft_axis_c2c(axis 2, forward) on the flagged operands, then
 * pfcs_update_zinv.  Other z lengths run that form, transforming the
 * flagged operands in place. */
int pfcs_update_zzinv(int kind, const void* state_in, void* aux, void* aux2, void* state_out, void* zout, int64_t n0,
                      int64_t n1, int64_t n2, const double* kx, const double* ky, const double* kz, double c0,
                      double c1, double c2, int flags, double* diag, void* stream);
/* Real-field pointwise operators of the R2C multiphysics path (physical
 * fields real: 8-byte samples), numpy evaluation order, no FMA; all operand
 * pointers 16-byte aligned, unused ones may be NULL:
 *   kind 0  out = (a*a)*a                        psi**3 (hydro.py:86, 96)
 *   kind 1  out = a*b                            psi * F^-1(i k mu) (hydro.py:98)
 *   kind 2  out = (a*b + c*d) + e*f              v . grad psi (hydro.py:83-85)
 *   kind 3  out = alpha*(a*(a*a) - a)            composition nonlinearity
 *   kind 4  out = (a + b) + c                    sum of the advection products */
int pfcs_real_pointwise(int kind, const double* a, const double* b, const double* c, const double* d,
                        const double* e, const double* f, double* out, int64_t n, double alpha, void* stream);
int pfcs_axpy(const void* a, const void* b, void* out, int64_t n, double w, void* stream);

/* ---- deterministic reductions (pfc._reduce_sum / free_energy,
 * pfc.py:131-162).  out[0] = sum_i f(a_i, b_i) in a fixed order,
 * independent of the launch: f = 0.5*a*b + 0.25*a^4 (free-energy density,
 * `b` the real part of F^-1(op*psi_hat)).  Real strided inputs: element i at
 * a[i*sa], b[i*sb] (sa = 2 reads the real part of a complex array). */
int pfcs_energy_sum(const double* a, int64_t sa, const double* b, int64_t sb, int64_t n,
                    double* out, double* scratch, void* stream);
/* out[0] = max_i |a_i| (strided like above); NaN propagates. */
int pfcs_absmax(const double* a, int64_t sa, int64_t n, double* out, void* stream);
/* Multiply complex x-slab data by the PFC operator symbol op = eps +
 * two_ring (grid.py:192-194), out = op*in, symbols from wavenumbers. */
int pfcs_apply_op(const void* in, void* out, int64_t cx, int64_t ny, int64_t nz, const double* kx,
                  const double* ky, const double* kz, double eps, void* stream);
/* Scratch bytes pfcs_energy_sum needs for n elements. */
int64_t pfcs_energy_scratch_bytes(int64_t n);

/* ---- single-GPU plan API: the whole hot path from C without Python.
 * A plan describes one real (nx, ny, nz) C-order fp64 grid on the current
 * device (2D grids: pass (nx, 1, ny)); the spectrum is the R2C half
 * spectrum (nx/2+1, ny, nz) complex128, C order, numpy's rfftn layout
 * along x.  Same arithmetic and launch sequence as distfft.forward/inverse
 * and pfc.pfc_run at one rank (distfft.py:150-173, pfc.py:96-128), so the
 * results are bit-identical to the Python path.  Needs power-of-two nx >= 4
 * and nz <= 4096 (else PFCS_E_UNSUPPORTED at create).
 *   fwd:  in (real, read only) -> out (spectrum)
 *   inv:  in (spectrum, read only) -> out (real); work >= spectral_elems
 *   pfc_steps: nsteps fused semi-implicit PFC steps on psi_hat in place;
 *         kx (nx/2+1), ky (ny), kz (nz) are the 1D wavenumbers
 *         (grid.wavenumbers), diag (nullable) receives nsteps x
 *         PFCS_DIAG_SLOTS x 4 per-step diagnostics (zeroed here), work >=
 *         spectral_elems complex128. */
typedef struct pfcs_plan pfcs_plan;
int pfcs_plan_create(int64_t nx, int64_t ny, int64_t nz, pfcs_plan** plan);
int pfcs_plan_destroy(pfcs_plan* plan);
int64_t pfcs_plan_spectral_elems(const pfcs_plan* plan);
int pfcs_plan_fwd(const pfcs_plan* plan, const double* in, void* out, void* stream);
int pfcs_plan_inv(const pfcs_plan* plan, const void* in, double* out, void* work, void* stream);
int pfcs_plan_pfc_steps(const pfcs_plan* plan, void* psi_hat, const double* kx, const double* ky,
                        const double* kz, double eps, double dt, int64_t nsteps, double* diag, void* work,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PFCS_H */
