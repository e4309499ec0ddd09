// pfcs_pfc2d.cu — the whole 2D PFC time loop in ONE thread-block cluster.
//
// Reference path: pfc.pfc_step (pfc.py:96-128) on a 2D grid (configs[0],
// 256^2), run as the fused single-rank engine of pfc.py (_StepEngine, G = 1,
// the (nx, 1, ny) view): per step the x pass (C2R -> psi^3 -> R2C on every
// y column, k_real_x MODE_CUBE) and the z pass (forward FFT of N_hat, the
// semi-implicit update, inverse FFT of the new psi_hat, k_pfc_z) — the same
// arithmetic, statement for statement, so the result is bit-identical to
// the two-kernel step.
//
// B200 mapping: the half spectrum (nx/2+1 rows x ny, 528 KB at 256^2) lives
// in the distributed shared memory of a 16-CTA cluster for the whole run.
// CTA c owns spectral rows kx = c, c+16, ... (psi_hat and the inverse-z
// "work" rows) and y columns [c*TC, (c+1)*TC) for the x pass.  A step is:
//   gather its columns from the row owners (ld.shared::cluster) -> x pass ->
//   scatter the columns back (st.shared::cluster) -> cluster barrier -> z
//   pass on its own rows -> cluster barrier.
// No HBM traffic and no kernel launches inside the loop: the step is bound
// by the cluster barriers and the per-CTA FFT latency, not by launches.
// Measured on the B200 at 256^2: 14.4 us/step, vs 10.5-11 us/step for the
// CUDA-graph-replayed two-kernel step that spreads each pass over all 148
// SMs — so the cluster loop is opt-in (pfc.py, PFCS_CLUSTER2D=1).
#include <cooperative_groups.h>

#include "pfcs_diag.cuh"
#include "pfcs_fft.cuh"
#include "pfcs_internal.h"

namespace cg = cooperative_groups;

namespace pfcs {

// W_N^k for k = j + P e with N = 2M = 16 P (R = 8): W_N^j * W_16^e (pfcs_x.cu twiddle_k)
__device__ __forceinline__ double2 w16c(int e) {
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

__device__ __forceinline__ double k2_2d(double kx, double ky, double kz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(kx, kx), __dmul_rn(ky, ky)), __dmul_rn(kz, kz));
}

template <int NX, int NY, int C>
struct Pfc2dCfg {
  static constexpr int M = NX / 2;         // x: M-point complex FFT per real line of NX
  static constexpr int NH = M + 1;         // spectral rows
  static constexpr int RC = (NH + C - 1) / C;  // rows per CTA (max)
  static constexpr int TC = NY / C;        // x-pass columns per CTA
  static constexpr int RX = 8, PX = M / RX;  // x-pass values / threads per column
  static constexpr int RZ = 8, PZ = NY / RZ;  // z-pass values / threads per row
  static constexpr int THREADS = (TC * PX > RC * PZ) ? TC * PX : RC * PZ;
  // every thread runs both passes' FFTs (they contain CTA barriers); threads
  // beyond a pass's real lines work on private dummy lines
  static constexpr int XL = (THREADS + PX - 1) / PX;  // x lines incl. dummies
  static constexpr int ZL = (THREADS + PZ - 1) / PZ;  // z lines incl. dummies
  static constexpr int LSX = tile_ls(M, TC, true) + 8;   // x workspace line stride
  static constexpr int LSZ = tile_ls(NY, RC, false);      // z workspace line stride
  // shared layout (double2): psi rows, work rows (z-inverse), N-hat rows
  // (x-pass results, double buffer so a step needs two cluster barriers),
  // x buffer [NH][TC], x ws, z ws
  static constexpr size_t PSI = (size_t)RC * NY, WORK = (size_t)RC * NY, XB = (size_t)NH * TC;
  static constexpr size_t XWS = (size_t)XL * LSX, ZWS = (size_t)ZL * LSZ;
  static constexpr size_t SMEM = (PSI + 2 * WORK + XB + XWS + ZWS) * 16;
};

template <int NX, int NY, int C>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(Pfc2dCfg<NX, NY, C>::THREADS, 1)
    k_pfc2d_cluster(double2* psi_hat, double2* work, const double* __restrict__ kx, const double* __restrict__ ky,
                    const double* __restrict__ kz, double eps, double dt, int nsteps, double* diag,
                    const double2* __restrict__ twN, const double2* __restrict__ twZ) {
  using Cf = Pfc2dCfg<NX, NY, C>;
  constexpr int M = Cf::M, NH = Cf::NH, TC = Cf::TC, RX = Cf::RX, PX = Cf::PX, RZ = Cf::RZ, PZ = Cf::PZ;
  cg::cluster_group cluster = cg::this_cluster();
  const int c = (int)cluster.block_rank();
  extern __shared__ double2 s2d[];
  double2* psi_s = s2d;
  double2* work_s = psi_s + Cf::PSI;
  double2* nl_s = work_s + Cf::WORK;  // x-pass results scattered by every CTA
  double2* xb = nl_s + Cf::WORK;
  double2* xws = xb + Cf::XB;
  double2* zws = xws + Cf::XWS;
  const int tid = threadIdx.x;
  const int nrows = (NH - c + C - 1) / C;  // rows kx = c + C*r owned here

  // load this CTA's rows of psi_hat and of the prepared z-inverse
  for (int idx = tid; idx < nrows * NY; idx += blockDim.x) {
    const int r = idx / NY, z = idx - r * NY;
    const size_t g = (size_t)(c + C * r) * NY + z;
    psi_s[idx] = psi_hat[g];
    work_s[idx] = work[g];
  }
  const double scale_x = 1.0 / (double)(2 * M);
  const double scale_z = 1.0 / (double)NY;
  const double kyy = __ldg(&ky[0]);
  cluster.sync();

  for (int step = 0; step < nsteps; ++step) {
    double* dstep = diag ? diag + (size_t)step * PFCS_DIAG_SLOTS * PFCS_DIAG_VALS : nullptr;
    // ---- gather this CTA's columns [c*TC, c*TC+TC) of every row into xb[kx][t]
    {
      constexpr int G = (NH * TC + Cf::THREADS - 1) / Cf::THREADS;
      double2 tmp[G];
#pragma unroll
      for (int q = 0; q < G; ++q) {  // all remote loads in flight before the stores
        const int idx = tid + q * Cf::THREADS;
        if (idx < NH * TC) {
          const int kxi = idx / TC, t = idx - kxi * TC;
          const double2* src = cluster.map_shared_rank(work_s, (unsigned)(kxi % C));
          tmp[q] = src[(kxi / C) * NY + c * TC + t];
        }
      }
#pragma unroll
      for (int q = 0; q < G; ++q) {
        const int idx = tid + q * Cf::THREADS;
        if (idx < NH * TC) xb[idx] = tmp[q];
      }
    }
    __syncthreads();
    // ---- x pass (k_real_x MODE_CUBE, mirror rows read from the buffer)
    double m_abs = 0.0;
    const bool xact = tid < TC * PX;
    const int xt = xact ? tid % TC : TC + (tid - TC * PX) / PX;  // dummy lines after the real ones
    const int xj = xact ? tid / TC : (tid - TC * PX) % PX;
    double2 xr[RX];
    double2 xm_out = make_double2(0.0, 0.0);
    {
      const int t = xt, jj = xj;
      double2* sl = xws + t * Cf::LSX;
      double2 v[RX];
#pragma unroll
      for (int e = 0; e < RX; ++e) v[e] = xact ? xb[(jj + PX * e) * TC + t] : make_double2(0.0, 0.0);
      const double2 wj = __ldg(&twN[jj]);
#pragma unroll
      for (int e = 0; e < RX; ++e) {
        const int k = jj + PX * e;
        double2 a = v[e];
        double2 bm = xact ? xb[(M - k) * TC + t] : make_double2(0.0, 0.0);
        if (k == 0) {
          a.y = 0.0;
          bm.y = 0.0;
        }
        const double2 b = make_double2(bm.x, -bm.y);
        const double2 s = cadd(a, b);
        const double2 d = csub(a, b);
        const double2 w = cmul(wj, w16c(e));
        const double2 wd = make_double2(fma(d.x, w.x, d.y * w.y), fma(d.y, w.x, -d.x * w.y));
        v[e] = make_double2(s.x - wd.y, s.y + wd.x);
      }
      fft_line<M, false, 2, PFCS_X_TWL, RX>(v, jj, sl, twN);
#pragma unroll
      for (int e = 0; e < RX; ++e) v[e] = make_double2(v[e].x * scale_x, v[e].y * scale_x);
#pragma unroll
      for (int e = 0; e < RX; ++e) {
        const double a = v[e].x, b = v[e].y;
        if (xact) m_abs = dmax_bits(m_abs, dmax_bits(fabs(a), fabs(b)));
        v[e] = make_double2(__dmul_rn(__dmul_rn(a, a), a), __dmul_rn(__dmul_rn(b, b), b));
      }
      fft_line<M, true, 2, PFCS_X_TWL, RX>(v, jj, sl, twN);
      // pairing Z_k with Z_{M-k} through xb (its last reads were the pre-step,
      // separated from here by the FFTs' barriers)
      if (xact) {
#pragma unroll
        for (int e = 0; e < RX; ++e) xb[(jj + PX * e) * TC + t] = v[e];
      }
      __syncthreads();
      if (xact) {
#pragma unroll
        for (int e = 0; e < RX; ++e) {
          const int k = jj + PX * e;
          const double2 zk = v[e];
          const double2 zm = xb[((M - k) & (M - 1)) * TC + t];
          double2 x;
          if (k == 0) {
            x = make_double2(zk.x + zk.y, 0.0);
          } else {
            const double2 s = make_double2(zk.x + zm.x, zk.y - zm.y);
            const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);
            const double2 w = cmul(wj, w16c(e));
            const double2 wd = make_double2(fma(d.x, w.x, -d.y * w.y), fma(d.x, w.y, d.y * w.x));
            x = make_double2(0.5 * (s.x + wd.y), 0.5 * (s.y - wd.x));
          }
          xr[e] = x;
        }
        if (jj == 0) {
          const double2 z0 = v[0];
          xm_out = make_double2(z0.x - z0.y, 0.0);
        }
      }
    }
    diag_block_max(dstep, m_abs, 0.0, m_abs);  // block-wide (contains __syncthreads)
    // ---- scatter the finished columns to the row owners' N-hat rows (a
    // buffer nobody gathers from, so no barrier is needed in front)
    if (xact) {
      const int t = tid % TC, jj = tid / TC;
#pragma unroll
      for (int e = 0; e < RX; ++e) {
        const int k = jj + PX * e;
        double2* dst = cluster.map_shared_rank(nl_s, (unsigned)(k % C));
        dst[(k / C) * NY + c * TC + t] = xr[e];
      }
      if (jj == 0) {
        double2* dst = cluster.map_shared_rank(nl_s, (unsigned)(M % C));
        dst[(M / C) * NY + c * TC + t] = xm_out;
      }
    }
    cluster.sync();
    // ---- z pass on the owned rows (k_pfc_z: fwd FFT, update, inverse FFT)
    bool bad = false;
    {
      const int line = tid / PZ, j = tid - line * PZ;
      const bool active = line < nrows;
      const int lrow = active ? line : 0;  // data row (dummies read row 0, never write)
      double2* sl = zws + line * Cf::LSZ;  // private workspace line, dummies included
      double2 v[RZ];
#pragma unroll
      for (int e = 0; e < RZ; ++e) v[e] = nl_s[lrow * NY + j + PZ * e];
      const int jj = opaque(j);
      fft_line<NY, true, 1, 1, RZ>(v, jj, sl, twZ);
      const double kxx = __ldg(&kx[c + C * lrow]);
#pragma unroll
      for (int e = 0; e < RZ; ++e) {
        const int z = jj + PZ * e;
        const double k2 = k2_2d(kxx, kyy, __ldg(&kz[z]));
        const double lap = -k2;
        const double a = __dsub_rn(1.0, k2);
        const double b = __dsub_rn(4.0 / 3.0, k2);
        const double two_ring = __dmul_rn(__dmul_rn(a, a), __dmul_rn(b, b));
        const double op = __dadd_rn(eps, two_ring);
        const double lin = __dmul_rn(lap, op);
        const double rden = __drcp_rn(__dsub_rn(1.0, __dmul_rn(dt, lin)));
        const double2 ph = psi_s[lrow * NY + z];
        const double nr = __dadd_rn(ph.x, __dmul_rn(dt, __dmul_rn(lap, v[e].x)));
        const double ni = __dadd_rn(ph.y, __dmul_rn(dt, __dmul_rn(lap, v[e].y)));
        const double2 nw = make_double2(__dmul_rn(nr, rden), __dmul_rn(ni, rden));
        bad |= active && !(isfinite(nw.x) && isfinite(nw.y));
        if (active) psi_s[lrow * NY + z] = nw;
        v[e] = nw;
      }
      const int j2 = opaque(jj);
      fft_line<NY, false, 1, 1, RZ>(v, j2, sl, twZ);
      if (active) {
#pragma unroll
        for (int e = 0; e < RZ; ++e)
          work_s[lrow * NY + j2 + PZ * e] = make_double2(v[e].x * scale_z, v[e].y * scale_z);
      }
    }
    diag_flag_nonfinite(dstep, bad);
    cluster.sync();
  }
  // write the state back: psi_hat rows and the prepared z-inverse of the last step
  for (int idx = tid; idx < nrows * NY; idx += blockDim.x) {
    const int r = idx / NY, z = idx - r * NY;
    const size_t g = (size_t)(c + C * r) * NY + z;
    psi_hat[g] = psi_s[idx];
    work[g] = work_s[idx];
  }
}

template <int NX, int NY, int C>
static int pfc2d_nc(double2* psi, double2* work, const double* kx, const double* ky, const double* kz, double eps,
                    double dt, int nsteps, double* diag, cudaStream_t st) {
  using Cf = Pfc2dCfg<NX, NY, C>;
  if constexpr (Cf::SMEM > 227 * 1024) {
    return 1;
  } else {
    const double2* twN = twiddles(NX);
    const double2* twZ = twiddles(NY);
    if (!twN || !twZ) return PFCS_E_CUDA;
    auto kern = k_pfc2d_cluster<NX, NY, C>;
    static bool attr = false;
    if (!attr) {
      if (int rc = check_cuda(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                              "cluster size attribute"))
        return rc;
      if (int rc = check_cuda(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)Cf::SMEM),
                              "smem attribute"))
        return rc;
      attr = true;
    }
    kern<<<C, Cf::THREADS, Cf::SMEM, st>>>(psi, work, kx, ky, kz, eps, dt, nsteps, diag, twN, twZ);
    return check_launch("k_pfc2d_cluster");
  }
}

// Returns 1 when the shape has no cluster kernel (caller keeps the two-kernel step).
int launch_pfc2d_cluster(void* psi_hat, void* work, long long nx, long long ny, const double* kx, const double* ky,
                         const double* kz, double eps, double dt, long long nsteps, double* diag, cudaStream_t st) {
  if (nsteps <= 0) return PFCS_OK;
  if (nx == 256 && ny == 256)
    return pfc2d_nc<256, 256, 16>((double2*)psi_hat, (double2*)work, kx, ky, kz, eps, dt, (int)nsteps, diag, st);
  return 1;
}

}  // namespace pfcs
