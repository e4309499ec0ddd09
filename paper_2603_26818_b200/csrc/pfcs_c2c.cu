// pfcs_c2c.cu — batched complex-to-complex line transforms (fp64, sm_100a).
//
// Reference semantics: fftcore.fft_axis (pkg/src/pfcspectral/fftcore.py:31-40)
// for the three axes of a C-order (n0, n1, n2) complex128 buffer, plus the
// z-line transforms of the slab pipeline that read the all-to-all receive
// buffer / write the send buffer directly (distfft._exchange,
// distfft.py:110-124, whose concatenate/slice pack and unpack are fused into
// the z-line prologue/epilogue here).
//
//  * k_lines    : contiguous lines (axis 2).  Input and output addressing may
//                 each be "plain" (line*N + z) or "blocked": the z axis split
//                 into G balanced slabs, slab g stored as a dense
//                 (nlines, cz_g) block at offset nlines*zoff_g — exactly the
//                 layout an all-to-all of per-rank z-slabs produces/consumes.
//  * k_strided  : one transform axis with a contiguous "inner" extent
//                 (axes 0 and 1).  A CTA takes T adjacent inner columns so each
//                 row of the tile is one T*16-byte coalesced segment.
//  * k_dft      : direct O(N^2) DFT for non-power-of-two N (the reference
//                 accepts any N, SPEC sizes 1..16 and primes).
#include "pfcs_diag.cuh"
#include "pfcs_fft.cuh"
#include "pfcs_internal.h"
#include "pfcs_pro.cuh"

namespace pfcs {

template <int R>
struct Regs1 {
  double2 v[R];
};

// PRO: a pointwise prologue (pfcs_pro.cuh) applied to each loaded element
// before the transform (plain layouts only): 1 cube / cmul / deriv, 2 a
// spectral update (PRO_UPD_*; its own instantiation so the light prologues
// do not carry its registers).
#ifndef PFCS_LINES_TARGET2
#define PFCS_LINES_TARGET2 768  // register target of the 2-stage z-line kernel (B200 512^3: 0.360 -> 0.357 ms)
#endif
#ifndef PFCS_UPD_ST
#define PFCS_UPD_ST 1  // register stages of the update-fused z pass (A/B: profiles/r2_ab_kernels.txt)
#endif
#ifndef PFCS_UPD_TARGET
#define PFCS_UPD_TARGET 512  // resident-thread target of the update-fused z pass
#endif
template <int N, int T, int ST, bool FWD, bool BIN, bool BOUT, int PRO = 0>
__global__ void __launch_bounds__(T*(N / radix_R(N)), min_blocks(T*(N / radix_R(N)), PRO == 2 ? PFCS_UPD_TARGET
                                                                                   : ST == 2 ? PFCS_LINES_TARGET2
                                                                                             : 1024))
    k_lines(const double2* in, double2* out, i64 nlines, SlabSplit sin, SlabSplit sout, PeerTable tout,
            const double2* __restrict__ tw, double scale, Pro pro = Pro{}) {
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  constexpr int LS = tile_ls(N, T, false);
  extern __shared__ double2 smem[];
  const int tid = threadIdx.x;
  const int t = tid / P;
  const int j = tid - t * P;
  double2* sl = smem + t * LS;
  const i64 ntiles = (nlines + T - 1) / T;
  auto load = [&](i64 tile, Regs1<R>& r) {
    const i64 l = tile * T + t;
    const bool ok = l < nlines;
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int z = j + P * e;
      i64 a = 0;
      if (BIN) {
        int zoff, cz;
        sin.locate(z, zoff, cz);
        a = nlines * zoff + l * cz + (z - zoff);
      } else {
        a = l * N + z;
      }
      r.v[e] = ok ? in[a] : make_double2(0.0, 0.0);
    }
  };
  auto comp = [&](i64 tile, Regs1<R>& r) {
    const i64 l = tile * T + t;
    const int jj = opaque(j);
    if constexpr (PRO == 1) {  // lines run along z: (x, y) = (l / n1, l % n1)
      if (l < nlines) {  // (a partial last tile: no aux reads / state writes past the end)
        const i64 lx = l / pro.n1;
        const i64 ly = l - lx * pro.n1;
        const i64 cl = pro.axis == 0 ? lx : ly;
#pragma unroll
        for (int e = 0; e < R; ++e)
          r.v[e] = apply_pro(pro, r.v[e], l * N + jj + P * e, pro.axis == 2 ? (i64)(jj + P * e) : cl);
      }
    } else if constexpr (PRO == 2) {
      if (l < nlines) {
        const i64 lx = l / pro.n1;
        const i64 ly = l - lx * pro.n1;
        const double ka = __ldg(pro.kx + lx), kb = __ldg(pro.ky + ly);
        const double kxy = __dadd_rn(__dmul_rn(ka, ka), __dmul_rn(kb, kb));
        const double2* A = (const double2*)pro.aux + l * N;
        const double2* B = (const double2*)pro.aux2 + l * N;
        double2 a[R], b[R];
#pragma unroll
        for (int e = 0; e < R; ++e) {  // all operand loads in flight before the first use
          a[e] = __ldg(A + jj + P * e);
          b[e] = pro.aux2 ? __ldg(B + jj + P * e) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int e = 0; e < R; ++e) {
          const double kc = __ldg(pro.kz + jj + P * e);
          r.v[e] = apply_upd(pro, r.v[e], a[e], b[e], l * N + jj + P * e, __dadd_rn(kxy, __dmul_rn(kc, kc)));
        }
      }
    }
    fft_line<N, FWD, 1, PFCS_LINES_TWL>(r.v, jj, sl, tw);
    if (l < nlines) {
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int z = jj + P * e;
        double2 x = r.v[e];
        if (!FWD) x = make_double2(x.x * scale, x.y * scale);
        if (BOUT) {  // block h of z -> tout.p[h] (local send slab or the peer's buffer)
          int h, zoff, cz;
          sout.locate3(z, h, zoff, cz);
          tout.p[h][l * cz + (z - zoff)] = x;
        } else {
          out[l * N + z] = x;
        }
      }
    }
  };
  reg_tile_loop<ST, Regs1<R>>(ntiles, load, comp);
}

// Address of element (o, n, i) of an (outer, N, inner) array whose line axis
// n is either plain or "blocked": split into G balanced slabs, slab g stored
// densely as (outer, cn_g, inner) at element offset outer*inner*noff_g —
// the layout a pencil exchange over the line axis produces or consumes.
template <bool BLOCKED>
__device__ __forceinline__ i64 line_addr(i64 o, int n, i64 i, int N, i64 outer, i64 inner,
                                         const SlabSplit& s) {
  if (!BLOCKED) return (o * N + n) * inner + i;
  int noff, cn;
  s.locate(n, noff, cn);
  return outer * inner * noff + (o * cn + (n - noff)) * inner + i;
}

// OPEER: the output rows (outer index o) are scattered by owner — row o of
// the plain result goes to tout.p[h] + ((o - ooff_h) N + n) inner + i, h the
// slab of o under `souter` (fused forward exchange: the peer's receive
// buffer, written over NVLink from this epilogue).
template <int N, int T, int ST, bool FWD, bool BIN, bool BOUT, bool OPEER = false>
__global__ void __launch_bounds__(T*(N / radix_R(N)), min_blocks(T*(N / radix_R(N)), ST == 2 ? 640 : 1024))
    k_strided(const double2* in, double2* out, i64 outer, i64 inner, i64 tpo, SlabSplit sin,
              SlabSplit sout, const double2* __restrict__ tw, double scale, SlabSplit souter = SlabSplit{},
              PeerTable tout = PeerTable{}) {
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  constexpr int LS = tile_ls(N, T, true);
  extern __shared__ double2 smem[];
  const int tid = threadIdx.x;
  const int t = tid % T;
  const int j = tid / T;
  double2* sl = smem + t * LS;
  const i64 ntiles = outer * tpo;
  auto load = [&](i64 tile, Regs1<R>& r) {
    const i64 o = tile / tpo;
    const i64 i = (tile - o * tpo) * T + t;
    const bool ok = i < inner;
#pragma unroll
    for (int e = 0; e < R; ++e)
      r.v[e] = ok ? in[line_addr<BIN>(o, j + P * e, i, N, outer, inner, sin)] : make_double2(0.0, 0.0);
  };
  auto comp = [&](i64 tile, Regs1<R>& r) {
    const i64 o = tile / tpo;
    const i64 i = (tile - o * tpo) * T + t;
    const int jj = opaque(j);
    fft_line<N, FWD, 1, PFCS_Y_TWL>(r.v, jj, sl, tw);
    if (i < inner) {
      double2* dst = out;
      i64 orow = o;
      if (OPEER) {
        int h, ooff, co;
        souter.locate3((int)o, h, ooff, co);
        dst = tout.p[h];
        orow = o - ooff;
      }
#pragma unroll
      for (int e = 0; e < R; ++e) {
        double2 x = r.v[e];
        if (!FWD) x = make_double2(x.x * scale, x.y * scale);
        dst[line_addr<BOUT>(orow, jj + P * e, i, N, outer, inner, sout)] = x;
      }
    }
  };
  reg_tile_loop<ST, Regs1<R>>(ntiles, load, comp);
}

// Direct DFT for arbitrary N: a CTA loads a tile of T lines (T adjacent inner
// columns when inner > 1) into shared memory and every thread produces
// outputs X[k] = sum_n x[n] w[(n k) mod N] with the index advanced
// incrementally (no integer multiply in the inner loop).
__global__ void k_dft(const double2* in, double2* out, int N, i64 outer, i64 inner, int T,
                      i64 tpo, const double2* __restrict__ tw, int fwd, double scale) {
  extern __shared__ double2 sm[];
  const bool contig = inner == 1;
  i64 o0, i0;
  if (contig) {
    o0 = (i64)blockIdx.x * T;
    i0 = 0;
  } else {
    o0 = (i64)blockIdx.x / tpo;
    i0 = ((i64)blockIdx.x - o0 * tpo) * T;
  }
  const int tot = T * N;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int t, n;
    if (contig) {
      t = idx / N;
      n = idx - t * N;
    } else {
      n = idx / T;
      t = idx - n * T;
    }
    const i64 o = contig ? o0 + t : o0;
    const i64 i = contig ? 0 : i0 + t;
    double2 val = make_double2(0.0, 0.0);
    if (o < outer && i < inner) val = in[o * (i64)N * inner + (i64)n * inner + i];
    sm[t * N + n] = val;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int t, k;
    if (contig) {
      t = idx / N;
      k = idx - t * N;
    } else {
      k = idx / T;
      t = idx - k * T;
    }
    const i64 o = contig ? o0 + t : o0;
    const i64 i = contig ? 0 : i0 + t;
    const double2* x = sm + t * N;
    double ar = 0.0, ai = 0.0;
    int m = 0;
    for (int n = 0; n < N; ++n) {
      const double2 w = __ldg(&tw[m]);
      const double2 a = x[n];
      if (fwd) {
        ar = fma(a.x, w.x, fma(-a.y, w.y, ar));
        ai = fma(a.x, w.y, fma(a.y, w.x, ai));
      } else {
        ar = fma(a.x, w.x, fma(a.y, w.y, ar));
        ai = fma(a.y, w.x, fma(-a.x, w.y, ai));
      }
      m += k;
      if (m >= N) m -= N;
    }
    if (o < outer && i < inner) {
      if (!fwd) {
        ar *= scale;
        ai *= scale;
      }
      out[o * (i64)N * inner + (i64)k * inner + i] = make_double2(ar, ai);
    }
  }
}

// Copy between plain and blocked layouts of the line axis of an
// (outer, n, inner) array (the np.concatenate / slicing of
// distfft._exchange for sizes the fused kernels do not cover).
__global__ void k_reblock(const double2* in, double2* out, i64 outer, int n, i64 inner, SlabSplit a,
                          SlabSplit b) {
  const i64 total = outer * n * inner;
  for (i64 idx = (i64)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (i64)gridDim.x * blockDim.x) {
    const i64 o = idx / ((i64)n * inner);
    const i64 rem = idx - o * n * inner;
    const int z = (int)(rem / inner);
    const i64 i = rem - (i64)z * inner;
    int zo, cz;
    a.locate(z, zo, cz);
    const i64 ia = outer * inner * zo + (o * cz + (z - zo)) * inner + i;
    b.locate(z, zo, cz);
    const i64 ib = outer * inner * zo + (o * cz + (z - zo)) * inner + i;
    out[ib] = in[ia];
  }
}

static int reblock(const double2* in, double2* out, i64 outer, int n, i64 inner, SlabSplitH a,
                   SlabSplitH b, cudaStream_t st) {
  i64 blocks = (outer * n * inner + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) return PFCS_OK;
  k_reblock<<<(unsigned)blocks, 256, 0, st>>>(in, out, outer, n, inner, SlabSplit{a.G, a.base, a.extra},
                                              SlabSplit{b.G, b.base, b.extra});
  return check_launch("k_reblock");
}

// Any length with blocked layouts: re-block through a plain temporary
// around the direct DFT (non-power-of-two sizes are a parity path).
static int blocked_dft(const double2* in, double2* out, i64 outer, int n, i64 inner, SlabSplitH si,
                       SlabSplitH so, bool forward, cudaStream_t st) {
  if (si.G == 1 && so.G == 1) return launch_dft(in, out, outer, n, inner, forward, st);
  double2* tmp = nullptr;
  const size_t bytes = (size_t)outer * n * inner * sizeof(double2);
  if (int rc = check_cuda(cudaMallocAsync((void**)&tmp, bytes, st), "cudaMallocAsync")) return rc;
  int rc = reblock(in, tmp, outer, n, inner, si, slab_split(n, 1), st);
  if (!rc) rc = launch_dft(tmp, tmp, outer, n, inner, forward, st);
  if (!rc) rc = reblock(tmp, out, outer, n, inner, slab_split(n, 1), so, st);
  cudaFreeAsync(tmp, st);
  return rc;
}

// ---------------------------------------------------------------- dispatch --

template <int N, bool FWD>
static int lines_n(const double2* in, double2* out, i64 nlines, SlabSplitH si, SlabSplitH so,
                   const PeerTable* dst, cudaStream_t st, const Pro* pro = nullptr) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  SlabSplit a{si.G, si.base, si.extra}, b{so.G, so.base, so.extra};
  const double scale = 1.0 / (double)N;
  const bool bin = si.G > 1, bout = so.G > 1 || dst != nullptr;
  if (so.G > PFCS_MAX_PEERS) return fail(PFCS_E_UNSUPPORTED, "more than 16 slabs");
  const PeerTable tab = dst ? *dst : local_table(out, nlines, so.G, so.base, so.extra);
  return with_variant<KIND_LINES, N>([&](auto var) -> int {
    constexpr int V = decltype(var)::value;
    constexpr int T = TileCfg<N>::T_MIN << (V & 3);
    constexpr int ST = 1 + (V >> 2);
    constexpr int P = TileCfg<N>::P;
    if constexpr (T * P > 1024) {
      return fail(PFCS_E_UNSUPPORTED, "tile too large");
    } else {
    const size_t smem = (size_t)T * tile_ls(N, T, false) * sizeof(double2);
    const i64 ntiles = (nlines + T - 1) / T;
    if (pro) {
      if (bin || bout) return fail(PFCS_E_UNSUPPORTED, "prologue on a blocked line pass");
      int grid = 0;
      if (pro->kind >= PRO_UPD_PSI) {  // updates feed inverse transforms only
        if constexpr (FWD) {
          return fail(PFCS_E_UNSUPPORTED, "update prologue on a forward pass");
        } else {
          if (int rc = persistent_grid((const void*)k_lines<N, T, PFCS_UPD_ST, FWD, false, false, 2>, T * P, smem,
                                       ntiles, &grid))
            return rc;
          k_lines<N, T, PFCS_UPD_ST, FWD, false, false, 2><<<grid, T * P, smem, st>>>(in, out, nlines, a, b, tab,
                                                                                      tw, scale, *pro);
          return check_launch("k_lines(update)");
        }
      }
      if (int rc = persistent_grid((const void*)k_lines<N, T, ST, FWD, false, false, 1>, T * P, smem, ntiles, &grid))
        return rc;
      k_lines<N, T, ST, FWD, false, false, 1><<<grid, T * P, smem, st>>>(in, out, nlines, a, b, tab, tw, scale, *pro);
      return check_launch("k_lines(pro)");
    }
    const void* f;
    if (bin && bout) f = (const void*)k_lines<N, T, ST, FWD, true, true>;
    else if (bin) f = (const void*)k_lines<N, T, ST, FWD, true, false>;
    else if (bout) f = (const void*)k_lines<N, T, ST, FWD, false, true>;
    else f = (const void*)k_lines<N, T, ST, FWD, false, false>;
    int grid = 0;
    if (int rc = persistent_grid(f, T * P, smem, ntiles, &grid)) return rc;
    if (bin && bout) k_lines<N, T, ST, FWD, true, true><<<grid, T * P, smem, st>>>(in, out, nlines, a, b, tab, tw, scale);
    else if (bin) k_lines<N, T, ST, FWD, true, false><<<grid, T * P, smem, st>>>(in, out, nlines, a, b, tab, tw, scale);
    else if (bout) k_lines<N, T, ST, FWD, false, true><<<grid, T * P, smem, st>>>(in, out, nlines, a, b, tab, tw, scale);
    else k_lines<N, T, ST, FWD, false, false><<<grid, T * P, smem, st>>>(in, out, nlines, a, b, tab, tw, scale);
    return check_launch("k_lines");
    }
  });
}

template <int N, bool FWD>
static int strided_n(const double2* in, double2* out, i64 outer, i64 inner, SlabSplitH si, SlabSplitH so,
                     cudaStream_t st) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  SlabSplit a{si.G, si.base, si.extra}, b{so.G, so.base, so.extra};
  const bool bin = si.G > 1, bout = so.G > 1;
  // TMA staging up to N = 1024; 2048-point lines fit only 2 per TMA tile,
  // where 4 register-loaded lines per CTA win (B200 2048^3: 50.6 -> 44.3 ms)
  if (!bin && !bout && inner > 1 && N <= 1024 && tma_enabled()) {
    const int rc = launch_strided_tma(in, out, outer, N, inner, FWD, st);
    if (rc != 1) return rc;
  }
  return with_variant<KIND_STRIDED, N>([&](auto var) -> int {
    constexpr int V = decltype(var)::value;
    constexpr int T = TileCfg<N>::T_MIN << (V & 3);
    constexpr int ST = 1 + (V >> 2);
    constexpr int P = TileCfg<N>::P;
    if constexpr (T * P > 1024) {
      return fail(PFCS_E_UNSUPPORTED, "tile too large");
    } else {
      const size_t smem = (size_t)T * tile_ls(N, T, true) * sizeof(double2);
      const i64 tpo = (inner + T - 1) / T;
      const void* f;
      if (bin && bout) f = (const void*)k_strided<N, T, ST, FWD, true, true>;
      else if (bin) f = (const void*)k_strided<N, T, ST, FWD, true, false>;
      else if (bout) f = (const void*)k_strided<N, T, ST, FWD, false, true>;
      else f = (const void*)k_strided<N, T, ST, FWD, false, false>;
      int grid = 0;
      if (int rc = persistent_grid(f, T * P, smem, outer * tpo, &grid)) return rc;
      const double sc = 1.0 / (double)N;
      if (bin && bout)
        k_strided<N, T, ST, FWD, true, true><<<grid, T * P, smem, st>>>(in, out, outer, inner, tpo, a, b, tw, sc);
      else if (bin)
        k_strided<N, T, ST, FWD, true, false><<<grid, T * P, smem, st>>>(in, out, outer, inner, tpo, a, b, tw, sc);
      else if (bout)
        k_strided<N, T, ST, FWD, false, true><<<grid, T * P, smem, st>>>(in, out, outer, inner, tpo, a, b, tw, sc);
      else
        k_strided<N, T, ST, FWD, false, false><<<grid, T * P, smem, st>>>(in, out, outer, inner, tpo, a, b, tw, sc);
      return check_launch("k_strided");
    }
  });
}

#define PFCS_POW2_CASES(MACRO) \
  MACRO(2) MACRO(4) MACRO(8) MACRO(16) MACRO(32) MACRO(64) MACRO(128) MACRO(256) MACRO(512) \
      MACRO(1024) MACRO(2048) MACRO(4096)

int launch_lines_c2c(const double2* in, double2* out, long long nlines, int n, int g_in, int g_out,
                     bool forward, cudaStream_t st) {
  return launch_lines_to(in, out, nlines, n, g_in, g_out, nullptr, forward, st);
}

// As launch_lines_c2c; with `dst` the blocked output slab g goes to
// dst->p[g] instead of out + nlines*zoff_g (fused exchange: peer buffers).
int launch_lines_to(const double2* in, double2* out, long long nlines, int n, int g_in, int g_out,
                    const PeerTable* dst, bool forward, cudaStream_t st) {
  if (nlines <= 0) return PFCS_OK;
  const SlabSplitH si = slab_split(n, g_in), so = slab_split(n, g_out);
  if (!is_pow2(n) || n > 4096) {
    if (dst) return fail(PFCS_E_UNSUPPORTED, "peer-scattered z lines need a power-of-two length");
    return blocked_dft(in, out, nlines, n, 1, si, so, forward, st);
  }
  switch (n) {
#define PFCS_CASE(NN) \
  case NN:            \
    return forward ? lines_n<NN, true>(in, out, nlines, si, so, dst, st)  \
                   : lines_n<NN, false>(in, out, nlines, si, so, dst, st);
    PFCS_POW2_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported line length");
}

// mu_hat of hydro_velocity_step (hydro.py:99-101) fused with the forward z
// passes of its two operands: per z line, the x/y-transformed lines of
// F(psi^3) and F(psi) are z-transformed in registers (the standalone forward
// z pass's arithmetic) and combined as pfcs_hydro_mu does,
//   mu = nl + (eps + ((1-k2)(1-k2)) ((4/3-k2)(4/3-k2))) f,
// so neither operand spectrum reaches HBM: 2S read + S written instead of
// two z passes (4S) and the mu pass (3S).
#ifndef PFCS_MUZ_TARGET
#define PFCS_MUZ_TARGET 512  // resident threads per SM the register cap aims for (two line register sets)
#endif
template <int N>
__global__ void __launch_bounds__(N / radix_R(N), min_blocks(N / radix_R(N), PFCS_MUZ_TARGET))
    k_mu_z(const double2* __restrict__ nl, const double2* __restrict__ f, double2* mu, double2* nl_out, i64 nlines,
           int n1, const double* __restrict__ kx, const double* __restrict__ ky, const double* __restrict__ kz,
           double eps, const double2* __restrict__ tw, double2* t0_out, double2* tz_out,
           const double* __restrict__ dz, double scale) {
  pdl_wait();
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  extern __shared__ double2 smem[];
  const int j = threadIdx.x;
  for (i64 l = blockIdx.x; l < nlines; l += gridDim.x) {
    double2 a[R], b[R];
#pragma unroll
    for (int e = 0; e < R; ++e) {
      a[e] = nl[l * N + j + P * e];
      b[e] = f[l * N + j + P * e];
    }
    const int jj = opaque(j);
    fft_line<N, true, 1, PFCS_LINES_TWL>(a, jj, smem, tw);
    const int j2 = opaque(jj);
    fft_line<N, true, 1, PFCS_LINES_TWL>(b, j2, smem, tw);
    const i64 lx = l / n1;
    const int ly = (int)(l - lx * n1);
    const double ka = __ldg(kx + lx), kb = __ldg(ky + ly);
    const double kxy = __dadd_rn(__dmul_rn(ka, ka), __dmul_rn(kb, kb));
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int z = j2 + P * e;
      const double kc = __ldg(kz + z);
      const double k2 = __dadd_rn(kxy, __dmul_rn(kc, kc));
      const double p1 = __dsub_rn(1.0, k2);
      const double p2 = __dsub_rn(4.0 / 3.0, k2);
      const double op = __dadd_rn(eps, __dmul_rn(__dmul_rn(p1, p1), __dmul_rn(p2, p2)));
      const double2 m = make_double2(__dadd_rn(a[e].x, __dmul_rn(op, b[e].x)), __dadd_rn(a[e].y, __dmul_rn(op, b[e].y)));
      if (mu) mu[l * N + z] = m;
      if (nl_out) nl_out[l * N + z] = a[e];  // F(psi^3), for the next step's density update
      b[e] = m;
    }
    // the inverse z passes grad mu starts with (_Real3._grad_zy): plain (the
    // x / y derivatives' shared pass) and with the i k_z multiplier
    // (pfcs_fft_axis_c2c_pro's derivative prologue), so mu_hat itself need
    // not reach HBM
    if (t0_out) {
#pragma unroll
      for (int e = 0; e < R; ++e) a[e] = b[e];
      const int j3 = opaque(j2);
      fft_line<N, false, 1, PFCS_LINES_TWL>(a, j3, smem, tw);
#pragma unroll
      for (int e = 0; e < R; ++e) t0_out[l * N + j3 + P * e] = make_double2(a[e].x * scale, a[e].y * scale);
    }
    if (tz_out) {
      const int j4 = opaque(j2);
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const double dk = __ldg(dz + j4 + P * e);
        b[e] = make_double2(-__dmul_rn(dk, b[e].y), __dmul_rn(dk, b[e].x));
      }
      fft_line<N, false, 1, PFCS_LINES_TWL>(b, j4, smem, tw);
#pragma unroll
      for (int e = 0; e < R; ++e) tz_out[l * N + j4 + P * e] = make_double2(b[e].x * scale, b[e].y * scale);
    }
  }
}

template <int N>
static int mu_z_n(const double2* nl, const double2* f, double2* mu, double2* nl_out, i64 nlines, int n1,
                  const double* kx, const double* ky, const double* kz, double eps, cudaStream_t st,
                  double2* t0_out, double2* tz_out, const double* dz) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  constexpr int P = N / radix_R(N);
  const size_t smem = (size_t)tile_ls(N, 1, false) * sizeof(double2);
  int grid = 0;
  if (int rc = persistent_grid((const void*)k_mu_z<N>, P, smem, nlines, &grid)) return rc;
  launch_pdl(k_mu_z<N>, dim3(grid), dim3(P), smem, st, nl, f, mu, nl_out, nlines, n1, kx, ky, kz, eps, tw, t0_out,
             tz_out, dz, 1.0 / (double)N);
  return check_launch("k_mu_z");
}

// returns 1 when not applicable (z length not a power of two in [8, 4096])
int launch_mu_z(const double2* nl, const double2* f, double2* mu, double2* nl_out, long long nlines, int n1, int n,
                const double* kx, const double* ky, const double* kz, double eps, cudaStream_t st, double2* t0_out,
                double2* tz_out, const double* dz) {
  if (nlines <= 0) return PFCS_OK;
  switch (n) {
#define PFCS_MU_CASE(NN) \
  case NN:               \
    return mu_z_n<NN>(nl, f, mu, nl_out, nlines, n1, kx, ky, kz, eps, st, t0_out, tz_out, dz);
    PFCS_MU_CASE(8) PFCS_MU_CASE(16) PFCS_MU_CASE(32) PFCS_MU_CASE(64) PFCS_MU_CASE(128) PFCS_MU_CASE(256)
    PFCS_MU_CASE(512) PFCS_MU_CASE(1024) PFCS_MU_CASE(2048) PFCS_MU_CASE(4096)
#undef PFCS_MU_CASE
    default:
      return 1;
  }
}

// A spectral update with the forward z passes of its operands AND the
// inverse z pass of its result, per z line (the k_pfc_z pattern for the
// hydro / multiphysics updates): operands that arrive after only their x and
// y passes (flags bit 0: aux, bit 1: aux2) are z-transformed in registers
// (the standalone forward z pass's arithmetic), the old state is updated as
// pfcs_update_zinv does (pfcs_hydro_math.cuh), the new state is stored and
// its inverse z transform written to zout — bit-identical to the forward z
// passes, then pfcs_update_zinv.  Neither operand spectrum reaches HBM.
#ifndef PFCS_UPDZ_TARGET
#define PFCS_UPDZ_TARGET 512  // resident threads per SM the register cap aims for (all operands loaded up front: 122 registers)
#endif
template <int N>
__global__ void __launch_bounds__(N / radix_R(N), min_blocks(N / radix_R(N), PFCS_UPDZ_TARGET))
    k_upd_zz(const double2* __restrict__ state, const double2* __restrict__ aux, const double2* __restrict__ aux2,
             double2* state_out, double2* zout, i64 nlines, int n1, const double* __restrict__ kx,
             const double* __restrict__ ky, const double* __restrict__ kz, int kind, double c0, double c1, double c2,
             int flags, double* diag, const double2* __restrict__ tw, double scale) {
  pdl_wait();
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  extern __shared__ double2 smem[];
  const int j = threadIdx.x;
  bool bad = false;
  for (i64 l = blockIdx.x; l < nlines; l += gridDim.x) {
    double2 a[R], b[R];
    double2 s0[R];
#pragma unroll
    for (int e = 0; e < R; ++e) {  // every operand of the line in flight before the first FFT
      a[e] = aux[l * N + j + P * e];
      b[e] = aux2 ? aux2[l * N + j + P * e] : make_double2(0.0, 0.0);
      s0[e] = state[l * N + j + P * e];
    }
    int jj = opaque(j);
    if (flags & 1) fft_line<N, true, 1, PFCS_LINES_TWL>(a, jj, smem, tw);
    if (aux2 && (flags & 2)) {
      jj = opaque(jj);
      fft_line<N, true, 1, PFCS_LINES_TWL>(b, jj, smem, tw);
    }
    const i64 lx = l / n1;
    const int ly = (int)(l - lx * n1);
    const double ka = __ldg(kx + lx), kb = __ldg(ky + ly);
    const double kxy = __dadd_rn(__dmul_rn(ka, ka), __dmul_rn(kb, kb));
    double2 v[R];
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int z = jj + P * e;
      const double kc = __ldg(kz + z);
      const double k2 = __dadd_rn(kxy, __dmul_rn(kc, kc));
      const double2 old = s0[e];
      const double2 nw = kind == 0   ? psi_update(old, a[e], b[e], k2, c0, c1)
                         : kind == 1 ? vel_update(old, a[e], k2, c0, c1, c2)
                                     : ch_update(old, a[e], b[e], k2, c0, c1, c2);
      bad |= !isfinite(nw.x);
      state_out[l * N + z] = nw;
      v[e] = nw;
    }
    const int j3 = opaque(jj);
    fft_line<N, false, 1, PFCS_LINES_TWL>(v, j3, smem, tw);
#pragma unroll
    for (int e = 0; e < R; ++e) zout[l * N + j3 + P * e] = make_double2(v[e].x * scale, v[e].y * scale);
  }
  diag_flag_nonfinite(diag, bad);
}

template <int N>
static int upd_zz_n(const double2* state, const double2* aux, const double2* aux2, double2* state_out, double2* zout,
                    i64 nlines, int n1, const double* kx, const double* ky, const double* kz, int kind, double c0,
                    double c1, double c2, int flags, double* diag, cudaStream_t st) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  constexpr int P = N / radix_R(N);
  const size_t smem = (size_t)tile_ls(N, 1, false) * sizeof(double2);
  int grid = 0;
  if (int rc = persistent_grid((const void*)k_upd_zz<N>, P, smem, nlines, &grid)) return rc;
  launch_pdl(k_upd_zz<N>, dim3(grid), dim3(P), smem, st, state, aux, aux2, state_out, zout, nlines, n1, kx, ky, kz,
             kind, c0, c1, c2, flags, diag, tw, 1.0 / (double)N);
  return check_launch("k_upd_zz");
}

// returns 1 when not applicable (z length not a power of two in [8, 4096])
int launch_upd_zz(const double2* state, const double2* aux, const double2* aux2, double2* state_out, double2* zout,
                  long long nlines, int n1, int n, const double* kx, const double* ky, const double* kz, int kind,
                  double c0, double c1, double c2, int flags, double* diag, cudaStream_t st) {
  if (nlines <= 0) return PFCS_OK;
  switch (n) {
#define PFCS_UZ_CASE(NN) \
  case NN:               \
    return upd_zz_n<NN>(state, aux, aux2, state_out, zout, nlines, n1, kx, ky, kz, kind, c0, c1, c2, flags, diag, st);
    PFCS_UZ_CASE(8) PFCS_UZ_CASE(16) PFCS_UZ_CASE(32) PFCS_UZ_CASE(64) PFCS_UZ_CASE(128) PFCS_UZ_CASE(256)
    PFCS_UZ_CASE(512) PFCS_UZ_CASE(1024) PFCS_UZ_CASE(2048) PFCS_UZ_CASE(4096)
#undef PFCS_UZ_CASE
    default:
      return 1;
  }
}

// Plain contiguous lines with a fused prologue; returns 1 when not
// applicable (non-power-of-two length).
int launch_lines_pro(const double2* in, double2* out, long long nlines, int n, const Pro& pro, bool forward,
                     cudaStream_t st) {
  if (nlines <= 0) return PFCS_OK;
  if (!is_pow2(n) || n > 4096 || n < 2) return 1;
  const SlabSplitH one = slab_split(n, 1);
  switch (n) {
#define PFCS_CASE(NN) \
  case NN:            \
    return forward ? lines_n<NN, true>(in, out, nlines, one, one, nullptr, st, &pro)  \
                   : lines_n<NN, false>(in, out, nlines, one, one, nullptr, st, &pro);
    PFCS_POW2_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return 1;
}

int launch_strided_c2c(const double2* in, double2* out, long long outer, int n, long long inner,
                       bool forward, cudaStream_t st) {
  return launch_strided_blocked(in, out, outer, n, inner, 1, 1, forward, st);
}

template <int N, bool FWD>
static int strided_to_n(const double2* in, i64 outer, i64 inner, SlabSplitH si, SlabSplitH souter,
                        const PeerTable& dst, cudaStream_t st) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  SlabSplit a{si.G, si.base, si.extra}, so{souter.G, souter.base, souter.extra};
  const bool bin = si.G > 1;
  if (!bin && inner > 1 && N <= 1024 && tma_enabled()) {
    const int rc = launch_strided_tma(in, nullptr, outer, N, inner, FWD, st, &souter, &dst);
    if (rc != 1) return rc;
  }
  return with_variant<KIND_STRIDED, N>([&](auto var) -> int {
    constexpr int V = decltype(var)::value;
    constexpr int T = TileCfg<N>::T_MIN << (V & 3);
    constexpr int ST = 1 + (V >> 2);
    constexpr int P = TileCfg<N>::P;
    if constexpr (T * P > 1024) {
      return fail(PFCS_E_UNSUPPORTED, "tile too large");
    } else {
      const size_t smem = (size_t)T * tile_ls(N, T, true) * sizeof(double2);
      const i64 tpo = (inner + T - 1) / T;
      const void* f = bin ? (const void*)k_strided<N, T, ST, FWD, true, false, true>
                          : (const void*)k_strided<N, T, ST, FWD, false, false, true>;
      int grid = 0;
      if (int rc = persistent_grid(f, T * P, smem, outer * tpo, &grid)) return rc;
      const double sc = 1.0 / (double)N;
      if (bin)
        k_strided<N, T, ST, FWD, true, false, true><<<grid, T * P, smem, st>>>(
            in, nullptr, outer, inner, tpo, a, a, tw, sc, so, dst);
      else
        k_strided<N, T, ST, FWD, false, false, true><<<grid, T * P, smem, st>>>(
            in, nullptr, outer, inner, tpo, a, a, tw, sc, so, dst);
      return check_launch("k_strided(peer)");
    }
  });
}

int launch_strided_to(const double2* in, long long outer, int n, long long inner, int g_in,
                      const PeerTable* dst, int g_outer, bool forward, cudaStream_t st) {
  if (outer <= 0 || inner <= 0) return PFCS_OK;
  if (!dst || g_outer > PFCS_MAX_PEERS) return fail(PFCS_E_ARG, "bad destination table");
  if (!is_pow2(n) || n > 4096 || inner == 1)
    return fail(PFCS_E_UNSUPPORTED, "peer-scattered strided lines need a power-of-two length and inner > 1");
  const SlabSplitH si = slab_split(n, g_in), so = slab_split(outer, g_outer);
  switch (n) {
#define PFCS_CASE(NN)                                                             \
  case NN:                                                                        \
    return forward ? strided_to_n<NN, true>(in, outer, inner, si, so, *dst, st)   \
                   : strided_to_n<NN, false>(in, outer, inner, si, so, *dst, st);
    PFCS_POW2_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported line length");
}

int launch_strided_blocked(const double2* in, double2* out, long long outer, int n, long long inner, int g_in,
                           int g_out, bool forward, cudaStream_t st) {
  if (outer <= 0 || inner <= 0) return PFCS_OK;
  const SlabSplitH si = slab_split(n, g_in), so = slab_split(n, g_out);
  if (inner == 1) return launch_lines_c2c(in, out, outer, n, g_in, g_out, forward, st);
  if (!is_pow2(n) || n > 4096) {
    return blocked_dft(in, out, outer, n, inner, si, so, forward, st);
  }
  switch (n) {
#define PFCS_CASE(NN)                                                                  \
  case NN:                                                                             \
    return forward ? strided_n<NN, true>(in, out, outer, inner, si, so, st)            \
                   : strided_n<NN, false>(in, out, outer, inner, si, so, st);
    PFCS_POW2_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported line length");
}

int launch_mixed(const double2* in, double2* out, long long outer, int n, long long inner, bool forward,
                 cudaStream_t st);

int launch_dft(const double2* in, double2* out, long long outer, int n, long long inner, bool forward,
               cudaStream_t st) {
  if (outer <= 0 || inner <= 0) return PFCS_OK;
  // mixed-radix Stockham first (pfcs_mixed.cu); the O(N^2) sum only for
  // lengths with a prime factor > 64 or tiles beyond shared memory
  const int rc = launch_mixed(in, out, outer, n, inner, forward, st);
  if (rc != -1) return rc;
  if (n > 16384) return fail(PFCS_E_UNSUPPORTED, "direct DFT limited to N <= 16384");
  const double2* tw = twiddles(n);
  if (!tw) return PFCS_E_CUDA;
  int T = 2048 / n;
  if (T < 1) T = 1;
  if (T > 16) T = 16;
  const bool contig = inner == 1;
  const i64 tpo = contig ? 1 : (inner + T - 1) / T;
  const i64 blocks = contig ? (outer + T - 1) / T : outer * tpo;
  const size_t smem = (size_t)T * n * sizeof(double2);
  if (ensure_smem((const void*)k_dft, smem)) return PFCS_E_CUDA;
  int threads = T * n;
  if (threads > 256) threads = 256;
  if (threads < 32) threads = 32;
  k_dft<<<(unsigned)blocks, threads, smem, st>>>(in, out, n, outer, inner, T, tpo, tw, forward ? 1 : 0,
                                                 1.0 / (double)n);
  return check_launch("k_dft");
}

}  // namespace pfcs
