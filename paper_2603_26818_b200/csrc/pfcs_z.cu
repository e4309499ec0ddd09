// pfcs_z.cu — z-line (contiguous axis of the X-slab spectral layout) passes of
// the PFC step, and the deterministic diagnostic reductions.
//
// k_pfc_z fuses, per z-line of the X slab (cx, ny, nz):
//   (i)   the unpack of the all-to-all receive buffer (distfft._exchange's
//         np.concatenate along z, distfft.py:120) into the prologue,
//   (ii)  the forward z FFT (distfft.dist_fft_forward, distfft.py:158),
//   (iii) the semi-implicit update of pfc.pfc_step (pfc.py:116-121)
//             psi_hat <- (psi_hat + dt*(lap*N_hat)) / (1 - dt*linear)
//         with the multipliers of grid.make_symbols (grid.py:183-191)
//         rebuilt from the 1D wavenumbers in numpy's evaluation order
//         (no FMA contraction: k2 = (kx*kx + ky*ky) + kz*kz, lap = -k2,
//         two_ring = ((1-k2)*(1-k2)) * ((4/3-k2)*(4/3-k2)), op = eps + two_ring,
//         linear = lap*op; complex/real division as numpy does it: the
//         numerator times fl(1/den)) — so given identical N_hat the update is
//         bit-identical to the reference's,
//   (iv)  the non-finite check (pfc.py:122),
//   (v)   the inverse z FFT of the NEW psi_hat (first stage of the next
//         step's distfft.inverse, distfft.py:166) and the pack into the
//         per-destination send blocks (distfft.py:118).
// HBM traffic per mode: read N_hat, read+write psi_hat, write next = 4 x 16 B.
#include "pfcs_diag.cuh"
#include "pfcs_fft.cuh"
#include "pfcs_internal.h"
#include "pfcs_pfcmath.cuh"
#include "pfcs_tma.cuh"

namespace pfcs {

template <int R>
struct RegsZ {
  double2 v[R];  // N-hat z line (un-transformed)
  double2 p[R];  // psi_hat z line
};

#ifndef PFCS_Z_TARGET
#define PFCS_Z_TARGET 640  // resident threads per SM the register cap of k_pfc_z aims for (B200: 640 -> 96 regs, 5 CTAs; 1024^3 6.80 -> 6.46 ms)
#endif
#ifndef PFCS_Z_TMA_TARGET
#define PFCS_Z_TMA_TARGET 512
#endif
template <int N, int T, int ST, bool BIN, bool BOUT, bool NEXT>
__global__ void __launch_bounds__(T*(N / radix_R(N)),
                                  min_blocks(T*(N / radix_R(N)), ST == 3 ? PFCS_Z_TMA_TARGET : PFCS_Z_TARGET))
    k_pfc_z(const double2* nl, double2* psi_hat, double2* next, i64 nlines, int ny, SlabSplit sin,
            SlabSplit sout, const double* __restrict__ kx, const double* __restrict__ ky,
            const double* __restrict__ kz, PfcSym p, const double2* __restrict__ tw, double scale,
            double* diag, PeerTable tnext) {
  pdl_wait();
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  constexpr int LS = tile_ls(N, T, false);
  // TMA: psi_hat lines are bulk-copied into a shared stage (needed only after
  // the forward FFT of N-hat, so they cost no registers across it); N-hat is
  // loaded straight into registers.
  constexpr bool TMA = ST == 3;
  extern __shared__ unsigned char zraw[];
  unsigned char* zbase = TMA ? zraw + ((1024u - (smem_u32(zraw) & 1023u)) & 1023u) : zraw;
  double2* stage = (double2*)zbase;  // psi_hat stage: T x N
  double2* smem = TMA ? stage + (size_t)T * N : (double2*)zraw;  // FFT workspace
  unsigned long long* bar = (unsigned long long*)(smem + (size_t)T * LS);
  int it_cur = 0;
  const int tid = threadIdx.x;
  const int t = tid / P;
  const int j = tid - t * P;
  double2* sl = smem + t * LS;
  const i64 ntiles = (nlines + T - 1) / T;
  bool bad = false;
  auto load = [&](i64 tile, RegsZ<R>& r) {
    const i64 l = tile * T + t;
    const bool ok = l < nlines;
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int z = j + P * e;
      i64 a;
      if (BIN) {
        int zoff, cz;
        sin.locate(z, zoff, cz);
        a = nlines * zoff + l * cz + (z - zoff);
      } else {
        a = l * N + z;
      }
      r.v[e] = ok ? nl[a] : make_double2(0.0, 0.0);
      if constexpr (!TMA) r.p[e] = ok ? psi_hat[l * N + z] : make_double2(0.0, 0.0);
    }
  };
  auto issue = [&](i64 tile) {  // thread 0: psi_hat lines of `tile` -> stage
    const i64 l0 = tile * T;
    const i64 lines = (nlines - l0) < T ? (nlines - l0) : T;
    const unsigned bytes = (unsigned)(lines * N * 16);
    mbar_expect_tx(bar, bytes);
    bulk_load(stage, psi_hat + l0 * N, bytes, bar);
  };
  auto comp = [&](i64 tile, RegsZ<R>& r) {
    const i64 l = tile * T + t;
    const bool ok = l < nlines;
    const int jj = opaque(j);
    fft_line<N, true, 1, PFCS_Z_TWL>(r.v, jj, sl, tw);
    const i64 lx = ok ? l / ny : 0;
    const int ly = ok ? (int)(l - lx * ny) : 0;
    const double kxx = __ldg(&kx[lx]);
    const double kyy = __ldg(&ky[ly]);
    if constexpr (TMA) mbar_wait(bar, (unsigned)(it_cur & 1));
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int z = jj + P * e;
      const double k2 = k2_of(kxx, kyy, __ldg(&kz[z]));
      double lap, rden;
      pfc_symbols(k2, p.eps, p.dt, lap, rden);
      const double2 ph = TMA ? stage[(size_t)t * N + z] : r.p[e];
      const double nr = __dadd_rn(ph.x, __dmul_rn(p.dt, __dmul_rn(lap, r.v[e].x)));
      const double ni = __dadd_rn(ph.y, __dmul_rn(p.dt, __dmul_rn(lap, r.v[e].y)));
      const double2 nw = make_double2(__dmul_rn(nr, rden), __dmul_rn(ni, rden));
      bad |= ok && !(isfinite(nw.x) && isfinite(nw.y));
      if (ok) psi_hat[l * N + z] = nw;
      r.v[e] = nw;
    }
    if constexpr (TMA) {  // stage read by every thread: refill with the next tile
      __syncthreads();
      if (threadIdx.x == 0 && tile + gridDim.x < ntiles) {
        fence_proxy_async();
        issue(tile + gridDim.x);
      }
    }
    if (NEXT) {
      const int j2 = opaque(jj);
      fft_line<N, false, 1, PFCS_Z_TWL>(r.v, j2, sl, tw);
      if (ok) {
#pragma unroll
        for (int e = 0; e < R; ++e) {
          const int z = j2 + P * e;
          const double2 x = make_double2(r.v[e].x * scale, r.v[e].y * scale);
          if (BOUT) {  // z block h -> tnext.p[h]: local send slab or rank h's receive buffer
            int h, zoff, cz;
            sout.locate3(z, h, zoff, cz);
            tnext.p[h][l * cz + (z - zoff)] = x;
          } else {
            next[l * N + z] = x;
          }
        }
      }
    }
  };
  if constexpr (!TMA) {
    reg_tile_loop<ST, RegsZ<R>>(ntiles, load, comp);
  } else {
    if (tid == 0) {
      mbar_init(bar, 1);
      mbar_fence_init();
    }
    __syncthreads();
    i64 tile = blockIdx.x;
    if (tid == 0 && tile < ntiles) issue(tile);
    for (; tile < ntiles; ++it_cur, tile += gridDim.x) {
      RegsZ<R> r;
      load(tile, r);
      comp(tile, r);
    }
  }
  diag_flag_nonfinite(diag, bad);
}

template <int N>
static int pfc_z_n(const double2* nl, double2* psi_hat, double2* next, i64 cx, i64 ny,
                   SlabSplitH si, SlabSplitH so, const double* kx, const double* ky,
                   const double* kz, double eps, double dt, double* diag, const PeerTable* dst,
                   cudaStream_t st) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  const i64 nlines = cx * ny;
  SlabSplit a{si.G, si.base, si.extra}, b{so.G, so.base, so.extra};
  PfcSym p{eps, dt};
  if (so.G > PFCS_MAX_PEERS) return fail(PFCS_E_UNSUPPORTED, "more than 16 slabs");
  const bool bin = si.G > 1, bout = so.G > 1 || dst != nullptr, nx = next != nullptr || dst != nullptr;
  const PeerTable tab = dst ? *dst : local_table(next, nlines, so.G, so.base, so.extra);
  const double scale = 1.0 / (double)N;
  return with_variant_n<KIND_PFCZ, N>((nlines + TileCfg<N>::T_MIN - 1) / TileCfg<N>::T_MIN, [&](auto var) -> int {
    constexpr int V = decltype(var)::value;
    constexpr int T = TileCfg<N>::T_MIN << (V & 3);
    constexpr int ST = 1 + (V >> 2);
    constexpr int P = TileCfg<N>::P;
    if constexpr (T * P > 1024) {
      return fail(PFCS_E_UNSUPPORTED, "tile too large");
    } else {
      // (A TMA-staged form of this pass — psi_hat or N-hat bulk-copied into
      // shared memory — measured slower on the B200: 1024^3 6.80 ms
      // register-loaded vs 7.09 / 7.57 ms staged; the kernel keeps the ST == 3
      // code path but nothing launches it.)
      const size_t smem = (size_t)T * tile_ls(N, T, false) * sizeof(double2);
      const i64 ntiles = (nlines + T - 1) / T;
      int grid = 0;
#define PFCS_ZK(BI, BO, NX) k_pfc_z<N, T, ST, BI, BO, NX>
#define PFCS_ZL(BI, BO, NX)                                                                       \
  do {                                                                                            \
    if (int rc = persistent_grid((const void*)PFCS_ZK(BI, BO, NX), T * P, smem, ntiles, &grid))   \
      return rc;                                                                                  \
    launch_pdl(PFCS_ZK(BI, BO, NX), dim3(grid), dim3(T * P), smem, st, nl, psi_hat, next, nlines,     \
               (int)ny, a, b, kx, ky, kz, p, tw, scale, diag, tab);                               \
  } while (0)
      if (!nx) {
        if (bin) PFCS_ZL(true, false, false);
        else PFCS_ZL(false, false, false);
      } else if (bin && bout) PFCS_ZL(true, true, true);
      else if (bin) PFCS_ZL(true, false, true);
      else if (bout) PFCS_ZL(false, true, true);
      else PFCS_ZL(false, false, true);
#undef PFCS_ZL
#undef PFCS_ZK
      return check_launch("k_pfc_z");
    }
  });
}

int launch_pfc_z(const double2* nl, double2* psi_hat, double2* next, long long cx, long long ny,
                 long long nz, int g_in, int g_out, const double* kx, const double* ky,
                 const double* kz, double eps, double dt, double* diag, cudaStream_t st,
                 const PeerTable* dst) {
  if (cx * ny <= 0) return PFCS_OK;
  if (!is_pow2(nz) || nz < 2 || nz > 4096)
    return fail(PFCS_E_UNSUPPORTED, "fused z update needs a power-of-two nz in [2, 4096]");
  const SlabSplitH si = slab_split(nz, g_in), so = slab_split(nz, g_out);
  switch (nz) {
#define PFCS_CASE(NN) \
  case NN:            \
    return pfc_z_n<NN>(nl, psi_hat, next, cx, ny, si, so, kx, ky, kz, eps, dt, diag, dst, st);
    PFCS_CASE(2) PFCS_CASE(4) PFCS_CASE(8) PFCS_CASE(16) PFCS_CASE(32) PFCS_CASE(64)
    PFCS_CASE(128) PFCS_CASE(256) PFCS_CASE(512) PFCS_CASE(1024) PFCS_CASE(2048) PFCS_CASE(4096)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported nz");
}

// ------------------------------------------------------- unfused forms ----
__global__ void k_pfc_cube(void* data, i64 n, int real, double* diag) {
  double m_re = 0.0, m_im = 0.0, m_abs = 0.0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    if (real) {
      double* d = (double*)data;
      const double a = d[i];
      m_re = dmax_bits(m_re, fabs(a));
      d[i] = __dmul_rn(__dmul_rn(a, a), a);
    } else {
      double2* d = (double2*)data;
      const double a = d[i].x, b = d[i].y;
      m_re = dmax_bits(m_re, fabs(a));
      m_im = dmax_bits(m_im, fabs(b));
      m_abs = dmax_bits(m_abs, hypot(a, b));
      const double cr = __dsub_rn(__dmul_rn(a, a), __dmul_rn(b, b));
      const double ci = __dadd_rn(__dmul_rn(a, b), __dmul_rn(b, a));
      d[i] = make_double2(__dsub_rn(__dmul_rn(a, cr), __dmul_rn(b, ci)),
                          __dadd_rn(__dmul_rn(a, ci), __dmul_rn(b, cr)));
    }
  }
  if (real) m_abs = m_re;
  diag_block_max(diag, m_re, m_im, m_abs);
}

int launch_pfc_cube(void* data, long long n, int real, double* diag, cudaStream_t st) {
  if (n <= 0) return PFCS_OK;
  i64 blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_pfc_cube<<<(unsigned)blocks, 256, 0, st>>>(data, n, real, diag);
  return check_launch("k_pfc_cube");
}

__global__ void k_pfc_update(const double2* nl, double2* psi_hat, i64 n, int ny, int nz,
                             const double* __restrict__ kx, const double* __restrict__ ky,
                             const double* __restrict__ kz, PfcSym p, double* diag) {
  bool bad = false;
  const i64 stride = (i64)gridDim.x * blockDim.x;
  const i64 i0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  const i64 nround = ((n + stride - 1) / stride) * stride;  // keep warps converged for the ballot
  for (i64 i = i0; i < nround; i += stride) {
    if (i < n) {
      const i64 line = i / nz;
      const int z = (int)(i - line * nz);
      const i64 x = line / ny;
      const int y = (int)(line - x * ny);
      double lap, rden;
      pfc_symbols(k2_of(__ldg(&kx[x]), __ldg(&ky[y]), __ldg(&kz[z])), p.eps, p.dt, lap, rden);
      const double2 ph = psi_hat[i];
      const double2 v = nl[i];
      const double nr = __dadd_rn(ph.x, __dmul_rn(p.dt, __dmul_rn(lap, v.x)));
      const double ni = __dadd_rn(ph.y, __dmul_rn(p.dt, __dmul_rn(lap, v.y)));
      const double2 nw = make_double2(__dmul_rn(nr, rden), __dmul_rn(ni, rden));
      bad |= !(isfinite(nw.x) && isfinite(nw.y));
      psi_hat[i] = nw;
    }
  }
  diag_flag_nonfinite(diag, bad);
}

int launch_pfc_update(const double2* nl, double2* psi_hat, long long cx, long long ny, long long nz,
                      const double* kx, const double* ky, const double* kz, double eps, double dt,
                      double* diag, cudaStream_t st) {
  const i64 n = cx * ny * nz;
  if (n <= 0) return PFCS_OK;
  i64 blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_pfc_update<<<(unsigned)blocks, 256, 0, st>>>(nl, psi_hat, n, (int)ny, (int)nz, kx, ky, kz,
                                                 PfcSym{eps, dt}, diag);
  return check_launch("k_pfc_update");
}

// --------------------------------------------------------- symbol multiply --
// out = op * in over an X slab (cx, ny, nz) (complex * real, componentwise:
// numpy's real-array x complex-array product, grid.py:192 / pfc.py:156).
__global__ void k_apply_op(const double2* in, double2* out, i64 n, int ny, int nz,
                           const double* __restrict__ kx, const double* __restrict__ ky,
                           const double* __restrict__ kz, double eps) {
  for (i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (i64)gridDim.x * blockDim.x) {
    const i64 line = idx / nz;
    const int z = (int)(idx - line * nz);
    const i64 x = line / ny;
    const int y = (int)(line - x * ny);
    const double k2 = k2_of(__ldg(&kx[x]), __ldg(&ky[y]), __ldg(&kz[z]));
    const double a = __dsub_rn(1.0, k2);
    const double b = __dsub_rn(4.0 / 3.0, k2);
    const double op = __dadd_rn(eps, __dmul_rn(__dmul_rn(a, a), __dmul_rn(b, b)));
    const double2 v = in[idx];
    out[idx] = make_double2(__dmul_rn(op, v.x), __dmul_rn(op, v.y));
  }
}

int launch_apply_op(const double2* in, double2* out, long long cx, long long ny, long long nz,
                    const double* kx, const double* ky, const double* kz, double eps,
                    cudaStream_t st) {
  const i64 n = cx * ny * nz;
  if (n <= 0) return PFCS_OK;
  i64 blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_apply_op<<<(unsigned)blocks, 256, 0, st>>>(in, out, n, (int)ny, (int)nz, kx, ky, kz, eps);
  return check_launch("k_apply_op");
}

// ------------------------------------------------------------ reductions ----
// Deterministic two-stage sum: fixed grid (RED_BLOCKS CTAs, grid-stride with
// a launch-independent assignment), fixed-order tree inside each CTA, then
// one CTA sums the RED_BLOCKS partials in a fixed tree.  The result depends
// only on n and the data, never on timing (pfc._reduce_sum is rank-ordered
// for the same reason, pfc.py:131-137).
#define RED_BLOCKS 1184
#define RED_THREADS 256

__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = RED_THREADS / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

__global__ void k_energy_partial(const double* a, i64 sa, const double* b, i64 sb, i64 n,
                                 double* partial) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (i64 i = (i64)blockIdx.x * RED_THREADS + threadIdx.x; i < n; i += (i64)RED_BLOCKS * RED_THREADS) {
    const double x = a[i * sa];
    const double y = b[i * sb];
    const double x2 = __dmul_rn(x, x);
    acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(__dmul_rn(0.5, x), y), __dmul_rn(0.25, __dmul_rn(x2, x2))));
  }
  const double s = block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void k_sum_partials(const double* partial, int m, double* out) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += RED_THREADS) acc = acc + partial[i];
  const double s = block_sum_fixed(acc, sh);
  if (threadIdx.x == 0) out[0] = s;
}

int launch_energy_sum(const double* a, long long sa, const double* b, long long sb, long long n,
                      double* out, double* scratch, cudaStream_t st) {
  k_energy_partial<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, sa, b, sb, n, scratch);
  if (int rc = check_launch("k_energy_partial")) return rc;
  k_sum_partials<<<1, RED_THREADS, 0, st>>>(scratch, RED_BLOCKS, out);
  return check_launch("k_sum_partials");
}

long long energy_scratch_bytes(long long) { return (long long)RED_BLOCKS * sizeof(double); }

__global__ void k_absmax(const double* a, i64 sa, i64 n, double* out) {
  double m = 0.0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    m = dmax_bits(m, fabs(a[i * sa]));
  m = warp_max_bits(m);
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = m;
  __syncthreads();
  if (w == 0) {
    m = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    m = warp_max_bits(m);
    if (lane == 0) atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(m));
  }
}

int launch_absmax(const double* a, long long sa, long long n, double* out, cudaStream_t st) {
  if (cudaMemsetAsync(out, 0, sizeof(double), st) != cudaSuccess)
    return check_cuda(cudaGetLastError(), "memset absmax");
  if (n <= 0) return PFCS_OK;
  i64 blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_absmax<<<(unsigned)blocks, 256, 0, st>>>(a, sa, n, out);
  return check_launch("k_absmax");
}

}  // namespace pfcs
