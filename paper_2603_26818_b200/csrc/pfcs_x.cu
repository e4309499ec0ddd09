// pfcs_x.cu — x-axis (slowest, strided) passes: real transforms and the fused
// physical-space nonlinearity of the PFC step.
//
// Reference path replaced: the x stage of fftcore.fft_2d (fftcore.py:43-45,
// forward axis order 0,1,2 pinned in fftcore.py:4-11) inside
// distfft.dist_fft_forward/inverse (distfft.py:150-173), and the pointwise
// `nl = psi.local ** 3` of pfc.pfc_step (pfc.py:109) with its realness /
// max|psi| diagnostics (pfc.py:100-105, 124).
//
// Real transforms use the half-length packing: a real x-line of length N = 2M
// is read as z[m] = x[2m] + i x[2m+1], transformed with an M-point complex
// FFT, and split into the N/2+1 = M+1 Hermitian modes
//     X[k] = 1/2 (Z_k + conj Z_{M-k}) - i/2 W_N^k (Z_k - conj Z_{M-k}),
// the inverse (C2R) runs the same relations backwards, so every x pass moves
// only the half spectrum through HBM.
//
// The fused cube pass (MODE_CUBE) keeps the whole x-line in shared memory:
//   C2R pre-twiddle -> M-point inverse FFT -> scale fl(1/N) -> x^3 per real
//   sample -> M-point forward FFT -> R2C post-twiddle
// so the physical field never reaches HBM (1 read + 1 write per mode).
//
// All kernels are persistent with register-pipelined loads (reg_tile_loop).
// A tile is T adjacent inner columns (the contiguous y*z extent), so each
// row of a tile is one T*16 (complex) or T*8 (real) byte segment.
#include <stdlib.h>

#include "pfcs_diag.cuh"
#include "pfcs_fft.cuh"
#include "pfcs_internal.h"
#include "pfcs_pfcmath.cuh"
#include "pfcs_tma.cuh"

namespace pfcs {

enum { MODE_R2C = 0, MODE_C2R = 1, MODE_CUBE = 2, MODE_R2C_PRO = 3, MODE_XMUL = 4 };
// MODE_XMUL: the x pass of a pseudo-spectral product, in place like the cube
// pass: C2R -> x * aux per real sample (pfcs_real_pointwise kind 1's
// arithmetic) -> R2C, so neither the physical factor F^-1(.) nor the
// product reaches HBM (the hydro force psi * F^-1(i k mu), hydro.py:98).
__host__ __device__ constexpr bool is_r2c(int mode) { return mode == MODE_R2C || mode == MODE_R2C_PRO; }

// Pointwise prologue of an R2C x pass (MODE_R2C_PRO): the real sample x of
// the transformed field is replaced by f(x) before the transform — the
// R2C multiphysics path's psi**3, psi * g and alpha (c^3 - c) (hydro.py:86,
// 96-98), in pfcs_real_pointwise's arithmetic (kinds 0, 1, 3), so fused and
// two-pass results are bit-identical and the product never reaches HBM.
struct RPro {
  int kind;           // 0 cube, 1 product with aux, 3 alpha (x^3 - x)
  double alpha;
  const double* aux;  // kind 1: the other factor, same (nx, inner) layout
};
// `a` = the kind-1 factor (loaded ahead of use by the caller: a product
// prologue that loads its factor when it needs it exposes a full DRAM latency
// per tile — 1.22 vs 0.44 ms per 512^3 launch)
__device__ __forceinline__ double rpro_apply(const RPro& p, double x, double a) {
  if (p.kind == 0) return __dmul_rn(__dmul_rn(x, x), x);
  if (p.kind == 1) return __dmul_rn(x, a);
  return __dmul_rn(p.alpha, __dsub_rn(__dmul_rn(x, __dmul_rn(x, x)), x));
}
// the kind-1 factors of rows 2m and 2m+1 of column i (zero outside the grid)
__device__ __forceinline__ double2 rpro_factor(const RPro& p, i64 m, i64 i, i64 inner, bool ok) {
  if (p.kind != 1 || !ok) return make_double2(0.0, 0.0);
  return make_double2(__ldg(p.aux + (2 * m) * inner + i), __ldg(p.aux + (2 * m + 1) * inner + i));
}

// values per thread of the fused cube pass (A/B experiments: -DPFCS_CUBE_R,
// -DPFCS_CUBE_TARGET = resident threads per SM the register cap aims for)
#ifndef PFCS_CUBE_R
#define PFCS_CUBE_R 8
#endif
#ifndef PFCS_CUBE_TARGET
#define PFCS_CUBE_TARGET 768
#endif
__host__ __device__ constexpr int real_R(int m, int mode) {
  return ((mode == 2 || mode == 4) && m >= 64) ? PFCS_CUBE_R : radix_R(m);
}

// Mirrored pre-step: the C2R pre-twiddle pairs X_k with X_{M-k}.  With
// PFCS_MIRROR=2 (default) the cube pass loads the mirror rows straight from
// global memory at the start of the tile's compute (the rows were just
// fetched by the partner threads, so they come from L1/L2) instead of
// exchanging them through shared memory: one smem round trip and one CTA
// barrier less per tile, no registers held across the prefetch window.
// PFCS_MIRROR=0 restores the shared-memory pairing (A/B).  The TMA-staged
// form reads the mirror rows from the stage instead (SMIR below).
#ifndef PFCS_MIRROR
#define PFCS_MIRROR 2
#endif
#ifndef PFCS_MIRROR_C2R
#define PFCS_MIRROR_C2R 0
#endif
__host__ __device__ constexpr bool late_mirror(int mode) {
  return PFCS_MIRROR == 2 && (mode == 2 || (PFCS_MIRROR_C2R && mode == 1));
}

template <int R, bool AX = false>
struct RegsX {
  double2 v[R];
  double2 xm;           // row M (half-spectrum Nyquist mode), used by thread j == 0
  double2 ax[AX ? R : 1];  // MODE_R2C_PRO: the prologue's factors of rows 2m, 2m+1
};

// Extra +8 keeps row M (index PAD(M)) inside the line when the bank rule
// gives no padding, without changing the line base's bank slot.
__host__ __device__ constexpr int real_ls(int m, int t) {
  return tile_ls(m, t, true) + (tile_ls(m, t, true) == pad_idx(m) ? 8 : 0);
}

// ST == 3: TMA-staged tiles.  Stage = the tile's input rows as TMA lands
// them, [row][t]: 2M real rows (R2C) or M+1 complex rows (C2R / cube), each
// T values wide; two stages (1024-byte aligned) + the FFT workspace + bars.
template <int M, int T, int MODE>
struct XStage {
  static constexpr size_t BYTES = is_r2c(MODE) ? (size_t)2 * M * T * 8 : (size_t)(M + 1) * T * 16;
  static constexpr size_t PADDED = (BYTES + 1023) / 1024 * 1024;
  static constexpr int ROWS = is_r2c(MODE) ? 2 * M : M;       // rows moved by the tiled map
  static constexpr int BR = ROWS < 256 ? ROWS : 256;          // rows per box
  static constexpr int NB = ROWS / BR;
  static constexpr size_t SMEM = 2 * PADDED + (size_t)T * real_ls(M, T) * 16 + 16 + 1024;
};

#ifndef PFCS_XMUL_TARGET
#define PFCS_XMUL_TARGET 256  // resident threads per SM of the TMA-staged product x pass (512: 128 registers, 120 B spills, 1.01 vs 0.88 ms)
#endif
template <int M, int T, int ST, int MODE>
__global__ void __launch_bounds__(T*(M / real_R(M, MODE)),
                                  min_blocks(T*(M / real_R(M, MODE)), ST == 3 ? (MODE == MODE_XMUL ? PFCS_XMUL_TARGET : 512) : (MODE == 2 ? PFCS_CUBE_TARGET : (ST == 2 ? 640 : 768))))
    k_real_x(const void* in_, void* out_, i64 inner, const double2* __restrict__ twN, double scale,
             double* diag, const __grid_constant__ TmaPair tm, RPro rp = RPro{}) {
  pdl_wait();
  constexpr int R = real_R(M, MODE);
  constexpr int P = M / R;
  constexpr int LS = real_ls(M, T);
  constexpr bool TMA = ST == 3;
  constexpr bool SMIR = TMA && !is_r2c(MODE);  // mirror rows read from the TMA stage
  constexpr bool LMIR = !TMA && late_mirror(MODE);
  using XS = XStage<M, T, MODE>;
  extern __shared__ unsigned char xraw[];
  unsigned char* xbase = TMA ? xraw + ((1024u - (smem_u32(xraw) & 1023u)) & 1023u) : xraw;
  double2* stage0 = (double2*)xbase;
  double2* stage1 = (double2*)(xbase + XS::PADDED);
  double2* smem = TMA ? (double2*)(xbase + 2 * XS::PADDED) : (double2*)xraw;  // FFT workspace
  const double2* cur = stage0;  // TMA stage holding the current tile
  const int tid = threadIdx.x;
  const int t = tid % T;
  const int j = tid / T;
  const i64 ntiles = (inner + T - 1) / T;
  double m_abs = 0.0;
  constexpr bool AXR = MODE == MODE_R2C_PRO || MODE == MODE_XMUL;  // Regs carry the product factors
  using Regs = RegsX<R, AXR>;

  auto load = [&](i64 tile, Regs& r) {
    const i64 i = tile * T + t;
    const bool ok = i < inner;
    if (is_r2c(MODE)) {
      const double* in = (const double*)in_;
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const i64 m = j + P * e;
        r.v[e] = ok ? make_double2(in[(2 * m) * inner + i], in[(2 * m + 1) * inner + i])
                    : make_double2(0.0, 0.0);
        if constexpr (MODE == MODE_R2C_PRO) r.ax[e] = rpro_factor(rp, m, i, inner, ok);  // applied in comp
      }
    } else {
      const double2* in = (const double2*)in_;
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const i64 k = j + P * e;
        r.v[e] = ok ? in[k * inner + i] : make_double2(0.0, 0.0);
        if constexpr (MODE == MODE_XMUL) r.ax[e] = rpro_factor(rp, k, i, inner, ok);  // applied in comp
      }
      r.xm = (ok && j == 0) ? in[(i64)M * inner + i] : make_double2(0.0, 0.0);
    }
  };

  auto comp = [&](i64 tile, Regs& r) {
    const unsigned tid_ = opaque_tid();
    const int t = tid_ % T;
    const int jj = tid_ / T;
    double2* sl = smem + t * LS;
    const i64 i = tile * T + t;
    const bool ok = i < inner;
    double2* v = r.v;
    if constexpr (MODE == MODE_R2C_PRO && !TMA) {
      if (ok) {
#pragma unroll
        for (int e = 0; e < R; ++e)
          v[e] = make_double2(rpro_apply(rp, v[e].x, r.ax[e].x), rpro_apply(rp, v[e].y, r.ax[e].y));
      }
    }
    // MODE_XMUL: the factors of rows 2m, 2m+1 (loaded with the tile, or
    // one tile ahead on the TMA path)
    double2 xf[MODE == MODE_XMUL ? R : 1];
    if constexpr (MODE == MODE_XMUL) {
#pragma unroll
      for (int e = 0; e < R; ++e) xf[e] = r.ax[e];
    }
    if (!is_r2c(MODE)) {
      // Z'[k] = (X_k + conj X_{M-k}) + i W_N^{-k} (X_k - conj X_{M-k});
      // Im X_0 and Im X_M are ignored (numpy irfft convention)
      double2 wl[LMIR ? R : 1];
      if constexpr (LMIR) {
        const double2* in = (const double2*)in_;
#pragma unroll
        for (int e = 0; e < R; ++e) {
          const i64 km = M - (jj + P * e);  // in [1, M]
          wl[e] = ok ? in[km * inner + i] : make_double2(0.0, 0.0);
        }
      }
      if constexpr (!LMIR && !SMIR) {
        stash_line<M, R>(r.v, jj, sl);
        if (jj == 0) sl[pad_idx(M)] = r.xm;
        __syncthreads();
      }
      const double2 wj = __ldg(&twN[jj]);
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int k = jj + P * e;
        double2 a = v[e];
        double2 bm;
        if constexpr (LMIR) {
          bm = wl[e];
        } else if constexpr (SMIR) {
          bm = cur[(M - k) * T + t];  // row M for k = 0
        } else {
          bm = sl[pad_idx(M - k)];
        }
        if (k == 0) {
          a.y = 0.0;
          bm.y = 0.0;
        }
        const double2 b = make_double2(bm.x, -bm.y);
        const double2 s = cadd(a, b);
        const double2 d = csub(a, b);
        const double2 w = twiddle_k<R>(twN, wj, jj, e, P);
        const double2 wd = make_double2(fma(d.x, w.x, d.y * w.y), fma(d.y, w.x, -d.x * w.y));
        v[e] = make_double2(s.x - wd.y, s.y + wd.x);
      }
      fft_line<M, false, 2, PFCS_X_TWL, R>(r.v, jj, sl, twN);
#pragma unroll
      for (int e = 0; e < R; ++e) v[e] = make_double2(v[e].x * scale, v[e].y * scale);
    }

    if (MODE == MODE_C2R) {
      if (ok) {
        double* out = (double*)out_;
#pragma unroll
        for (int e = 0; e < R; ++e) {
          const i64 m = jj + P * e;
          out[(2 * m) * inner + i] = v[e].x;
          out[(2 * m + 1) * inner + i] = v[e].y;
        }
      }
      return;
    }

    if (MODE == MODE_CUBE) {
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const double a = v[e].x, b = v[e].y;
        if (ok) m_abs = dmax_bits(m_abs, dmax_bits(fabs(a), fabs(b)));
        // psi**3 of a real sample, x*x*x in numpy's left-to-right order
        v[e] = make_double2(__dmul_rn(__dmul_rn(a, a), a), __dmul_rn(__dmul_rn(b, b), b));
      }
    }
    if constexpr (MODE == MODE_XMUL) {
#pragma unroll
      for (int e = 0; e < R; ++e) v[e] = make_double2(__dmul_rn(v[e].x, xf[e].x), __dmul_rn(v[e].y, xf[e].y));
    }

    // forward M-point FFT, then the R2C split
    const int j2 = opaque(jj);  // keep the forward FFT's index math out of the inverse's live range
    fft_line<M, true, 2, PFCS_X_TWL, R>(r.v, j2, sl, twN);
    const double2 wj = __ldg(&twN[jj]);
    // Pairing Z_k with Z_{M-k}.  TMA mode exchanges through the current stage
    // ([k][t] rows, conflict-free for t-fastest lanes): it was last read
    // before the FFT's barriers and is refilled only after the end-of-tile
    // barrier, so no barrier is needed in front of the stash.
    double2* stg = const_cast<double2*>(cur);
    if constexpr (TMA) {
#pragma unroll
      for (int e = 0; e < R; ++e) stg[(jj + P * e) * T + t] = v[e];
    } else {
      __syncthreads();
      stash_line<M, R>(r.v, jj, sl);
    }
    __syncthreads();
    double2* out = (double2*)out_;
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int k = jj + P * e;
      const double2 zk = v[e];
      const double2 zm = TMA ? stg[((M - k) & (M - 1)) * T + t] : sl[pad_idx((M - k) & (M - 1))];
      double2 x;
      if (k == 0) {
        x = make_double2(zk.x + zk.y, 0.0);
      } else {
        const double2 s = make_double2(zk.x + zm.x, zk.y - zm.y);  // Zk + conj Zm
        const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);  // Zk - conj Zm
        const double2 w = twiddle_k<R>(twN, wj, jj, e, P);
        const double2 wd = make_double2(fma(d.x, w.x, -d.y * w.y), fma(d.x, w.y, d.y * w.x));
        x = make_double2(0.5 * (s.x + wd.y), 0.5 * (s.y - wd.x));  // 1/2 (s - i wd)
      }
      if (ok) out[(i64)k * inner + i] = x;
    }
    if (jj == 0 && ok) {
      const double2 z0 = v[0];
      out[(i64)M * inner + i] = make_double2(z0.x - z0.y, 0.0);
    }
  };

  if constexpr (!TMA) {
    reg_tile_loop<ST, Regs>(ntiles, load, comp);
  } else {
    unsigned long long* bars = (unsigned long long*)(smem + (size_t)T * LS);
    auto issue = [&](i64 tile, int sidx) {
      const int i0 = (int)(tile * T);
      unsigned char* dst = (unsigned char*)(sidx ? stage1 : stage0);
      mbar_expect_tx(&bars[sidx], (unsigned)XS::BYTES);
      constexpr int W = is_r2c(MODE) ? 8 : 16;  // bytes per stage element
#pragma unroll
      for (int b = 0; b < XS::NB; ++b)
        tma_load_2d(dst + (size_t)b * XS::BR * T * W, &tm.a, &bars[sidx], (is_r2c(MODE) ? 1 : 2) * i0, b * XS::BR);
      if (!is_r2c(MODE)) tma_load_2d(dst + (size_t)M * T * W, &tm.b, &bars[sidx], 2 * i0, M);
    };
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      mbar_fence_init();
    }
    __syncthreads();
    i64 tile = blockIdx.x;
    if (tid == 0 && tile < ntiles) issue(tile, 0);
    // MODE_R2C_PRO / MODE_XMUL: the product factors of the tile, loaded one tile ahead
    double2 axn[AXR ? R : 1];
    auto aux_ahead = [&](i64 tl) {
      if constexpr (AXR) {
#pragma unroll
        for (int e = 0; e < R; ++e) axn[e] = rpro_factor(rp, j + P * e, tl * T + t, inner, tl * T + t < inner);
      }
    };
    aux_ahead(tile);
    for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
      const int sidx = it & 1;
      if (tid == 0) {
        const i64 nx = tile + gridDim.x;
        if (nx < ntiles) {
          fence_proxy_async();
          issue(nx, sidx ^ 1);
        }
      }
      mbar_wait(&bars[sidx], (unsigned)((it >> 1) & 1));
      cur = sidx ? stage1 : stage0;
      Regs r;
      if (is_r2c(MODE)) {
        // rows 2m and 2m+1 of a T-double stage row pair sit in opposite
        // halves of the 32 banks when T = 8: odd-j threads read their odd
        // row first, so each load instruction touches both halves (2
        // wavefronts per warp instead of 4)
        const double* sd = (const double*)cur;
        const int sw = j & 1;
#pragma unroll
        for (int e = 0; e < R; ++e) {
          const int m = j + P * e;
          const double a = sd[(2 * m + sw) * T + t];
          const double b = sd[(2 * m + 1 - sw) * T + t];
          r.v[e] = sw ? make_double2(b, a) : make_double2(a, b);
          if constexpr (MODE == MODE_R2C_PRO)
            r.v[e] = make_double2(rpro_apply(rp, r.v[e].x, axn[e].x), rpro_apply(rp, r.v[e].y, axn[e].y));
        }
        if constexpr (MODE == MODE_R2C_PRO) aux_ahead(tile + gridDim.x);  // in flight during comp
      } else {
#pragma unroll
        for (int e = 0; e < R; ++e) r.v[e] = cur[(j + P * e) * T + t];
        if constexpr (MODE == MODE_XMUL) {
#pragma unroll
          for (int e = 0; e < R; ++e) r.ax[e] = axn[e];
          aux_ahead(tile + gridDim.x);  // in flight during comp
        }
      }
      comp(tile, r);
      __syncthreads();
    }
  }
  if (MODE == MODE_CUBE) diag_block_max(diag, m_abs, 0.0, m_abs);
}

// ----------------------------------------------- advection dot product --
// v . grad x on the R2C path in ONE x pass (hydro.py:83-85 and the
// composition advection): the inputs are the three derivative spectra
// i d_a x_hat after their inverse z and y passes (three (M+1, inner) arrays;
// with dx, the first is the plain inverse z / y transform of x_hat and its
// i d_x multiplier — constant along y and z lines — is applied here, to the
// loaded modes, as pfcs_mul_deriv would);
// per tile the kernel runs three C2R sub-passes (TMA-staged, double-buffered
// across sub-passes) and accumulates v_a * g_a per real sample in registers
// in pfcs_real_pointwise kind 2's order ((v0 g0 + v1 g1) + v2 g2), then the
// R2C of the sum: the three physical derivatives and the product never
// reach HBM.  Arithmetic of k_real_x MODE_C2R / MODE_R2C (bit-identical to
// three pfcs_irfft_x + pfcs_real_pointwise kind 2 + pfcs_rfft_x).
#ifndef PFCS_XDOT_MINB
#define PFCS_XDOT_MINB 1  // CTAs per SM the register cap aims for (2: 128 registers with 284 B of spills, 2.80 vs 2.61 ms)
#endif
template <int M, int T>
__global__ void __launch_bounds__(T*(M / 8), PFCS_XDOT_MINB)
    k_xdot3(double2* out, i64 inner, const double2* __restrict__ twN, double scale,
            const __grid_constant__ TmaPair tm0, const __grid_constant__ TmaPair tm1,
            const __grid_constant__ TmaPair tm2, const double* __restrict__ v0, const double* __restrict__ v1,
            const double* __restrict__ v2, const double* __restrict__ dx) {
  pdl_wait();
  constexpr int R = 8;
  constexpr int P = M / R;
  constexpr int LS = real_ls(M, T);
  using XS = XStage<M, T, MODE_C2R>;
  extern __shared__ unsigned char draw[];
  unsigned char* dbase = draw + ((1024u - (smem_u32(draw) & 1023u)) & 1023u);
  double2* stage0 = (double2*)dbase;
  double2* stage1 = (double2*)(dbase + XS::PADDED);
  double2* smem = (double2*)(dbase + 2 * XS::PADDED);  // FFT workspace
  unsigned long long* bars = (unsigned long long*)(smem + (size_t)T * LS);
  const int tid = threadIdx.x;
  const int t = tid % T;
  const int j = tid / T;
  const i64 ntiles = (inner + T - 1) / T;

  auto issue = [&](i64 tile, int sub, int sidx) {
    const int i0 = (int)(tile * T);
    const TmaPair* tm = sub == 0 ? &tm0 : (sub == 1 ? &tm1 : &tm2);
    unsigned char* dst = (unsigned char*)(sidx ? stage1 : stage0);
    mbar_expect_tx(&bars[sidx], (unsigned)XS::BYTES);
#pragma unroll
    for (int b = 0; b < XS::NB; ++b)
      tma_load_2d(dst + (size_t)b * XS::BR * T * 16, &tm->a, &bars[sidx], 2 * i0, b * XS::BR);
    tma_load_2d(dst + (size_t)M * T * 16, &tm->b, &bars[sidx], 2 * i0, M);
  };
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < ntiles) issue(blockIdx.x, 0, 0);
  // velocity samples (rows 2m, 2m+1) of sub-pass `sub` of `tile`, loaded one
  // sub-pass ahead (a load consumed right after its FFT exposed its latency:
  // long_scoreboard was the top stall)
  auto load_v = [&](i64 tl, int sub, double2 (&dst)[R]) {
    const double* vp = sub == 0 ? v0 : (sub == 1 ? v1 : v2);
    const i64 ii = tl * T + t;
    const bool okk = tl < ntiles && ii < inner;
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const i64 m = j + P * e;
      dst[e] = okk ? make_double2(__ldg(vp + (2 * m) * inner + ii), __ldg(vp + (2 * m + 1) * inner + ii))
                   : make_double2(0.0, 0.0);
    }
  };
  double2 vf[R];
  load_v(blockIdx.x, 0, vf);
  int it = 0;
  for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const i64 i = tile * T + t;
    const bool ok = i < inner;
    double2 acc[R];
    const double2* cur = stage0;
#pragma unroll 1
    for (int sub = 0; sub < 3; ++sub, ++it) {
      const int sidx = it & 1;
      if (tid == 0) {
        const i64 ntile = sub < 2 ? tile : tile + gridDim.x;
        if (ntile < ntiles) {
          fence_proxy_async();  // the other stage was read by every thread before the last barrier
          issue(ntile, sub < 2 ? sub + 1 : 0, sidx ^ 1);
        }
      }
      mbar_wait(&bars[sidx], (unsigned)((it >> 1) & 1));
      cur = sidx ? stage1 : stage0;
      const int jj = opaque(j);
      double2* sl = smem + t * LS;
      double2 v[R];
#pragma unroll
      for (int e = 0; e < R; ++e) v[e] = cur[(jj + P * e) * T + t];
      double2 vn[R];  // the next sub-pass's velocities, in flight during this one
      if (sub < 2) load_v(tile, sub + 1, vn);
      else load_v(tile + gridDim.x, 0, vn);
      // C2R (k_real_x MODE_C2R, mirror rows from the stage)
      const double2 wj = __ldg(&twN[jj]);
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int k = jj + P * e;
        double2 a = v[e];
        double2 bm = cur[(M - k) * T + t];  // row M for k = 0
        if (sub == 0 && dx) {  // i d_x[k] (pfcs_mul_deriv's arithmetic) on both paired modes
          const double dk = __ldg(dx + k), dm = __ldg(dx + (M - k));
          a = make_double2(-__dmul_rn(dk, a.y), __dmul_rn(dk, a.x));
          bm = make_double2(-__dmul_rn(dm, bm.y), __dmul_rn(dm, bm.x));
        }
        if (k == 0) {
          a.y = 0.0;
          bm.y = 0.0;
        }
        const double2 b = make_double2(bm.x, -bm.y);
        const double2 sm = cadd(a, b);
        const double2 d = csub(a, b);
        const double2 w = twiddle_k<R>(twN, wj, jj, e, P);
        const double2 wd = make_double2(fma(d.x, w.x, d.y * w.y), fma(d.y, w.x, -d.x * w.y));
        v[e] = make_double2(sm.x - wd.y, sm.y + wd.x);
      }
      fft_line<M, false, 2, PFCS_X_TWL, R>(v, jj, sl, twN);
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const double gx = v[e].x * scale, gy = v[e].y * scale;
        if (sub == 0) {
          acc[e] = make_double2(__dmul_rn(vf[e].x, gx), __dmul_rn(vf[e].y, gy));
        } else {
          acc[e] = make_double2(__dadd_rn(acc[e].x, __dmul_rn(vf[e].x, gx)),
                                __dadd_rn(acc[e].y, __dmul_rn(vf[e].y, gy)));
        }
      }
#pragma unroll
      for (int e = 0; e < R; ++e) vf[e] = vn[e];
      if (sub < 2) __syncthreads();  // stage and workspace free for the next sub-pass
    }
    // R2C of the sum (k_real_x MODE_R2C's forward FFT and split; the last
    // sub-pass's stage pairs Z_k with Z_{M-k}: it is refilled only after the
    // end-of-tile barrier)
    const int j2 = opaque(j);
    double2* sl = smem + t * LS;
    fft_line<M, true, 2, PFCS_X_TWL, R>(acc, j2, sl, twN);
    const double2 wj = __ldg(&twN[j2]);
    double2* stg = const_cast<double2*>(cur);
#pragma unroll
    for (int e = 0; e < R; ++e) stg[(j2 + P * e) * T + t] = acc[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int k = j2 + P * e;
      const double2 zk = acc[e];
      const double2 zm = stg[((M - k) & (M - 1)) * T + t];
      double2 x;
      if (k == 0) {
        x = make_double2(zk.x + zk.y, 0.0);
      } else {
        const double2 sp = make_double2(zk.x + zm.x, zk.y - zm.y);
        const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);
        const double2 w = twiddle_k<R>(twN, wj, j2, e, P);
        const double2 wd = make_double2(fma(d.x, w.x, -d.y * w.y), fma(d.x, w.y, d.y * w.x));
        x = make_double2(0.5 * (sp.x + wd.y), 0.5 * (sp.y - wd.x));
      }
      if (ok) out[(i64)k * inner + i] = x;
    }
    if (j2 == 0 && ok) out[(i64)M * inner + i] = make_double2(acc[0].x - acc[0].y, 0.0);
    __syncthreads();
  }
}

template <int M>
static int xdot3_m(const double2* const* spec, const double* v0, const double* v1, const double* v2, double2* out,
                   i64 inner, const double* dx, cudaStream_t st) {
#ifndef PFCS_XDOT_T
#define PFCS_XDOT_T 8
#endif
  constexpr int T = PFCS_XDOT_T;  // lines per tile (8: 128-byte complex rows, as the cube pass at M = 256)
  using XS = XStage<M, T, MODE_C2R>;
  static_assert(XS::SMEM <= 227 * 1024, "stage + workspace fit");
  if (2 * inner >= (1LL << 31)) return 1;
  const double2* twN = twiddles(2 * M);
  if (!twN) return PFCS_E_CUDA;
  TmaPair tm[3] = {};
  const unsigned long long dims[2] = {(unsigned long long)(2 * inner), (unsigned long long)(M + 1)};
  const unsigned long long str[1] = {(unsigned long long)inner * 16};
  const unsigned box[2] = {(unsigned)(2 * T), (unsigned)XS::BR};
  const unsigned box1[2] = {(unsigned)(2 * T), 1u};
  for (int a = 0; a < 3; ++a) {
    if (((uintptr_t)spec[a] & 15) || !make_tmap(&tm[a].a, 2, spec[a], dims, str, box) ||
        !make_tmap(&tm[a].b, 2, spec[a], dims, str, box1))
      return 1;
  }
  const i64 ntiles = (inner + T - 1) / T;
  int grid = 0;
  auto kern = k_xdot3<M, T>;
  if (int rc = persistent_grid((const void*)kern, T * (M / 8), XS::SMEM, ntiles, &grid)) return rc;
  launch_pdl(kern, dim3(grid), dim3(T * (M / 8)), XS::SMEM, st, out, inner, twN, 1.0 / (double)(2 * M), tm[0], tm[1],
             tm[2], v0, v1, v2, dx);
  return check_launch("k_xdot3");
}

// returns 1 when not applicable (the caller runs the three C2R passes, the
// pointwise kernel and the R2C pass instead)
bool xdot3_supported(long long nx, long long inner) {
  return tma_enabled() && (nx == 256 || nx == 512) && inner >= 0 && 2 * inner < (1LL << 31);
}

int launch_xdot3(const void* const* spec, const double* v0, const double* v1, const double* v2, void* out,
                 long long nx, long long inner, const double* dx, cudaStream_t st) {
  if (inner <= 0) return PFCS_OK;
  if (!xdot3_supported(nx, inner)) return 1;
  const double2* s[3] = {(const double2*)spec[0], (const double2*)spec[1], (const double2*)spec[2]};
  switch (nx) {
    case 256: return xdot3_m<128>(s, v0, v1, v2, (double2*)out, inner, dx, st);
    case 512: return xdot3_m<256>(s, v0, v1, v2, (double2*)out, inner, dx, st);
    default: return 1;
  }
}

// ------------------------------------------- line-synchronous cube pass --
// Same arithmetic as k_real_x<M, T, 3, MODE_CUBE> (bit-identical), different
// execution: the CTA-wide barriers of the interleaved tile made all 16 warps
// alternate in lock step between butterflies (fp64 pipe) and exchanges
// (shared-memory pipe) — ncu: fp64 49.6 % + smem 48.9 % busy, issue 40 %,
// i.e. the two pipes never overlap.  Here
//   * a line's P threads are consecutive (line-major), exchange through that
//     line's own padded workspace and synchronise on a named barrier of P
//     threads only, so the T lines of a tile drift into different phases;
//   * the HBM tile still moves as T*16-byte rows: TMA loads it into a
//     swizzled stage (row r, column t at chunk t ^ f(r): the line-major
//     stage reads are conflict-free), results are written back into the same
//     stage column and leave through a TMA tensor STORE, so the global stores
//     stay full rows too;
//   * no CTA-wide barrier in the tile loop: each line's leader counts its line
//     in on the stage; the LAST line to finish a tile stores the stage and
//     refills it with the tile after next (no producer warp, so 16 warps keep
//     128 registers each), while the other lines already work on the other
//     stage.
template <int M, int T>
struct CubeLs {
  static constexpr int R = 8;
  static constexpr int P = M / R;
  static constexpr int ROWB = T * 16;                 // bytes per stage row (= swizzle span)
  static constexpr size_t STAGE = (size_t)(M + 1) * ROWB;
  static constexpr size_t PADDED = (STAGE + 1023) / 1024 * 1024;
  static constexpr int NS = 3;                        // pipeline stages (no separate FFT workspace)
  static constexpr int BR = M < 256 ? M : 256;        // rows per TMA box
  static constexpr int NB = M / BR;
  static constexpr int THREADS = T * P;
  static constexpr size_t SMEM = NS * PADDED + 64 + 1024;
  // stage element (row r, column t) under the TMA swizzle of a ROWB-byte row:
  // line t owns chunk t ^ f(r) of every row, and the 16-byte slot of any 8
  // rows with distinct r & 7 fall on distinct banks (ROWB = 128 or 64)
  __device__ __forceinline__ static int at(int r, int t) {
    return r * T + (t ^ ((r * ROWB >> 7) & (T - 1)));
  }
};

// The FFT exchanges of line t run inside the line's own stage column (the
// slots it owns in every row), with logical element n on row
// rho(n) = (n & ~7) | ((n ^ (n >> 3)) & 7): any 8 aligned consecutive
// elements and any 8 elements of stride 8 (the Stockham write pattern of the
// first radix-8 pass) land on rows with distinct r & 7, i.e. distinct banks.
// The inputs were consumed before the first exchange, so the padded
// per-line workspace is not needed and its 74 KB buy a third stage.
template <class C>
struct StageCol {
  double2* base;
  int t;
  __device__ __forceinline__ double2& ref(int n) const {
    const int r = (n & ~7) | ((n ^ (n >> 3)) & 7);
    return base[C::at(r, t)];
  }
};

// Results go back into the line's stage column and leave through a TMA
// tensor store; the stage is refilled once the store has read it.  (Storing
// straight from registers instead — 16 bytes per thread and row, so the stage
// could be refilled right after the reads — measured 3.2x slower on the
// B200: 5.18 -> 16.7 ms per 1024^3 launch.)
//
// Scale folding: the inverse transform's fl(1/N) is an exact power of two, so
// it commutes with every rounding of the cube, the forward FFT and the R2C
// split; it is applied once, as s^3 (0.5 s^3 where the split halves) on the
// final modes, and max|psi| is scaled once at the end — bit-identical to
// scaling each sample (no subnormal intermediates on this path).
template <int M, int T>
__global__ void __launch_bounds__(CubeLs<M, T>::THREADS, 1)
    k_cube_ls(double2* data, i64 inner, const double2* __restrict__ twN, double scale, double* diag,
              const __grid_constant__ TmaPair tm) {
  pdl_wait();
  using C = CubeLs<M, T>;
  constexpr int R = C::R;
  constexpr int P = C::P;
  constexpr int NS = C::NS;
  extern __shared__ unsigned char craw[];
  unsigned char* cbase = craw + ((1024u - (smem_u32(craw) & 1023u)) & 1023u);
  unsigned long long* full = (unsigned long long*)(cbase + NS * C::PADDED);
  unsigned* done = (unsigned*)(full + NS);  // lines finished with the stage's tile
  const int tid = threadIdx.x;
  const i64 ntiles = (inner + T - 1) / T;
  double m_abs = 0.0;

  // TMA transfer of one tile between global memory and stage s
  auto xfer = [&](i64 tile, int s, bool load) {
    const int c0 = (int)(2 * tile * T);
    unsigned char* buf = cbase + (size_t)s * C::PADDED;
#pragma unroll
    for (int b = 0; b < C::NB; ++b) {
      if (load) tma_load_2d(buf + (size_t)b * C::BR * C::ROWB, &tm.a, &full[s], c0, b * C::BR);
      else tma_store_2d(&tm.a, buf + (size_t)b * C::BR * C::ROWB, c0, b * C::BR);
    }
    if (load) tma_load_2d(buf + (size_t)M * C::ROWB, &tm.b, &full[s], c0, M);
    else tma_store_2d(&tm.b, buf + (size_t)M * C::ROWB, c0, M);
  };
  // line leader, once its line is done with stage s of `tile`: the last line
  // of the tile stores the stage and refills it with this CTA's tile NS later
  auto release = [&](i64 tile, int s) {
    __threadfence_block();
    const unsigned prev = atomicAdd(&done[s], 1u);
    if (prev == (unsigned)T - 1) {
      __threadfence_block();
      done[s] = 0;
      const i64 nxt = tile + NS * (i64)gridDim.x;
      fence_proxy_async();
      xfer(tile, s, false);
      bulk_commit();
      if (nxt < ntiles) {
        bulk_wait_read0();
        fence_proxy_async();
        mbar_expect_tx(&full[s], (unsigned)C::STAGE);
        xfer(nxt, s, true);
      }
    }
  };

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0;
    }
    mbar_fence_init();
    for (int s = 0; s < NS; ++s) {
      const i64 tile = blockIdx.x + (i64)s * gridDim.x;
      if (tile < ntiles) {
        mbar_expect_tx(&full[s], (unsigned)C::STAGE);
        xfer(tile, s, true);
      }
    }
  }
  __syncthreads();

  const int t = tid / P;  // line of the tile, position j = tid % P
  const BarSync lsync{1u + (unsigned)t, (unsigned)P};
  int it = 0, s = 0, ph = 0;  // stage s = it % NS, its phase parity ph = (it / NS) & 1
  for (i64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int jj = opaque((int)(opaque_tid() % P));
    double2* cur = (double2*)(cbase + (size_t)s * C::PADDED);
    mbar_wait(&full[s], (unsigned)ph);
    const double2 wj = __ldg(&twN[jj]);
    double2 v[R];
#pragma unroll
    for (int e = 0; e < R; ++e) v[e] = cur[C::at(jj + P * e, t)];
    // C2R pre-twiddle (as k_real_x MODE_CUBE), mirror rows from the stage
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int k = jj + P * e;
      double2 a = v[e];
      double2 bm = cur[C::at(M - k, t)];  // row M for k = 0
      if (k == 0) {
        a.y = 0.0;
        bm.y = 0.0;
      }
      const double2 b = make_double2(bm.x, -bm.y);
      const double2 sm = cadd(a, b);
      const double2 d = csub(a, b);
      const double2 w = twiddle_k<R>(twN, wj, jj, e, P);
      const double2 wd = make_double2(fma(d.x, w.x, d.y * w.y), fma(d.y, w.x, -d.x * w.y));
      v[e] = make_double2(sm.x - wd.y, sm.y + wd.x);
    }
    fft_line<M, false, 2, PFCS_X_TWL, R, false, BarSync>(v, jj, StageCol<C>{cur, t}, twN, lsync);
    const bool ok = (i64)opaque((int)(tile * T)) + t < inner;
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const double a = v[e].x, b = v[e].y;  // unscaled (see above)
      if (ok) m_abs = dmax_bits(m_abs, dmax_bits(fabs(a), fabs(b)));
      v[e] = make_double2(__dmul_rn(__dmul_rn(a, a), a), __dmul_rn(__dmul_rn(b, b), b));
    }
    const unsigned tid2 = opaque_tid();
    const int j2 = (int)(tid2 % P), t2 = (int)(tid2 / P);
    double2* col = (double2*)(cbase + (size_t)opaque(s) * C::PADDED);
    fft_line<M, true, 2, PFCS_X_TWL, R, false, BarSync>(v, j2, StageCol<C>{col, t2}, twN, lsync);
    // R2C split: pair Z_k with Z_{M-k} through the line's stage column (the
    // TMA-swizzle layout keeps any 8 consecutive rows on distinct banks, for
    // the stash and the mirrored reads alike)
    lsync();  // the last exchange's reads of the column are done
#pragma unroll
    for (int e = 0; e < R; ++e) col[C::at(j2 + P * e, t2)] = v[e];
    lsync();
    {
      double sc = scale;
      asm volatile("" : "+d"(sc));  // keep s^3 local (no loop-long registers)
      const double s3 = sc * sc * sc, hs3 = 0.5 * s3;
      const double2 wj2 = __ldg(&twN[j2]);
      const double2 xm = make_double2((v[0].x - v[0].y) * s3, 0.0);  // Nyquist mode (j == 0)
#pragma unroll
      for (int e = 0; e < R; ++e) {
        const int k = j2 + P * e;
        const int km = (M - k) & (M - 1);
        const double2 zk = v[e];
        const double2 zm = col[C::at(km, t2)];
        double2 x;
        if (k == 0) {
          x = make_double2((zk.x + zk.y) * s3, 0.0);
        } else {
          const double2 sp = make_double2(zk.x + zm.x, zk.y - zm.y);
          const double2 d = make_double2(zk.x - zm.x, zk.y + zm.y);
          const double2 w = twiddle_k<R>(twN, wj2, j2, e, P);
          const double2 wd = make_double2(fma(d.x, w.x, -d.y * w.y), fma(d.x, w.y, d.y * w.x));
          x = make_double2(hs3 * (sp.x + wd.y), hs3 * (sp.y - wd.x));
        }
        v[e] = x;
      }
      lsync();  // every mirror read of the column is done
#pragma unroll
      for (int e = 0; e < R; ++e) col[C::at(j2 + P * e, t2)] = v[e];
      if (j2 == 0) col[C::at(M, t2)] = xm;
      fence_proxy_async();  // my stage writes before the async-proxy store
      lsync();
      if (j2 == 0) release(tile, s);
    }
    if (++s == NS) {
      s = 0;
      ph ^= 1;
    }
  }
  if (threadIdx.x % P == 0) bulk_wait0();  // stores this thread issued have completed
  m_abs *= scale;  // exact (power of two)
  diag_block_max(diag, m_abs, 0.0, m_abs);
}

template <int M, int T>
static int cube_ls_m(void* data, i64 inner, double* diag, cudaStream_t st) {
  using C = CubeLs<M, T>;
  static_assert(C::ROWB == 128 || C::ROWB == 64, "stage rows of 64 or 128 bytes (TMA swizzle span)");
  if (2 * inner >= (1LL << 31) || ((uintptr_t)data & 15)) return 1;
  const double2* twN = twiddles(2 * M);
  if (!twN) return PFCS_E_CUDA;
  TmaPair tm{};
  const unsigned long long dims[2] = {(unsigned long long)(2 * inner), (unsigned long long)(M + 1)};
  const unsigned long long str[1] = {(unsigned long long)inner * 16};
  const unsigned box[2] = {(unsigned)(2 * T), (unsigned)C::BR};
  const unsigned box1[2] = {(unsigned)(2 * T), 1u};
  if (!make_tmap(&tm.a, 2, data, dims, str, box, C::ROWB) || !make_tmap(&tm.b, 2, data, dims, str, box1, C::ROWB))
    return 1;
  const i64 ntiles = (inner + T - 1) / T;
  int grid = 0;
  auto kern = k_cube_ls<M, T>;
  if (int rc = persistent_grid((const void*)kern, C::THREADS, C::SMEM, ntiles, &grid)) return rc;
  launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, st, (double2*)data, inner, twN, 1.0 / (double)(2 * M),
             diag, tm);
  return check_launch("k_cube_ls");
}

// PFCS_CUBE_LS=0 selects k_real_x MODE_CUBE instead (A/B; bit-identical)
static int cube_ls_mode() {
  static const int m = [] {
    const char* v = getenv("PFCS_CUBE_LS");
    return (v && *v) ? atoi(v) : 1;
  }();
  return m;
}

int launch_cube_ls(void* data, long long nx, long long inner, double* diag, cudaStream_t st) {
  const int mode = cube_ls_mode();
  if (mode == 0 || !tma_enabled()) return 1;
  // production tiles only: enough T-wide tiles to fill every SM
  // (T = 4 at M = 512 — two 256-thread CTAs per SM, 64-byte rows — measured
  // 5.15 -> 7.44 ms per 1024^3 launch: 128-byte rows stay)
  if (nx == 1024 && inner >= 8 * 148) return cube_ls_m<512, 8>(data, inner, diag, st);
  if (nx == 2048 && inner >= 4 * 148) return cube_ls_m<1024, 4>(data, inner, diag, st);
  return 1;
}

// Fused complex-data cube pass (C2C mode, reference-layout fields):
// inverse x FFT -> psi*(psi*psi) (numpy complex power, pfc.py:109) -> forward.
template <int N, int T, int ST>
__global__ void __launch_bounds__(T*(N / radix_R(N)), min_blocks(T*(N / radix_R(N)), 512))
    k_cube_c2c(double2* data, i64 inner, const double2* __restrict__ tw, double scale, double* diag) {
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  constexpr int LS = tile_ls(N, T, true);
  extern __shared__ double2 smem[];
  const int tid = threadIdx.x;
  const int t = tid % T;
  const int j = tid / T;
  const i64 ntiles = (inner + T - 1) / T;
  double m_re = 0.0, m_im = 0.0, m_abs = 0.0;
  auto load = [&](i64 tile, RegsX<R>& r) {
    const i64 i = tile * T + t;
    const bool ok = i < inner;
#pragma unroll
    for (int e = 0; e < R; ++e) r.v[e] = ok ? data[(i64)(j + P * e) * inner + i] : make_double2(0.0, 0.0);
  };
  auto comp = [&](i64 tile, RegsX<R>& r) {
    const unsigned tid_ = opaque_tid();
    const int t = tid_ % T;
    const int jj = tid_ / T;
    double2* sl = smem + t * LS;
    const i64 i = tile * T + t;
    const bool ok = i < inner;
    double2* v = r.v;
    fft_line<N, false>(r.v, jj, sl, tw);
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const double a = v[e].x * scale, b = v[e].y * scale;
      if (ok) {
        m_re = dmax_bits(m_re, fabs(a));
        m_im = dmax_bits(m_im, fabs(b));
        m_abs = dmax_bits(m_abs, hypot(a, b));
      }
      // c = psi*psi ; psi*c, no contraction (numpy cmul)
      const double cr = __dsub_rn(__dmul_rn(a, a), __dmul_rn(b, b));
      const double ci = __dadd_rn(__dmul_rn(a, b), __dmul_rn(b, a));
      v[e] = make_double2(__dsub_rn(__dmul_rn(a, cr), __dmul_rn(b, ci)),
                          __dadd_rn(__dmul_rn(a, ci), __dmul_rn(b, cr)));
    }
    const int j2 = opaque(jj);
    fft_line<N, true>(r.v, j2, sl, tw);
    if (ok) {
#pragma unroll
      for (int e = 0; e < R; ++e) data[(i64)(j2 + P * e) * inner + i] = v[e];
    }
  };
  reg_tile_loop<ST, RegsX<R>>(ntiles, load, comp);
  diag_block_max(diag, m_re, m_im, m_abs);
}

// ---------------------------------------------------------------- dispatch --

// tensor maps of the x-pass input: rows of `inner` contiguous values
template <int M, int T, int MODE>
static bool x_tmaps(TmaPair* tm, const void* in, i64 inner) {
  if (2 * inner >= (1LL << 31)) return false;
  using XS = XStage<M, T, MODE>;
  if (is_r2c(MODE)) {
    if (inner % 2) return false;  // row stride must be a multiple of 16 bytes
    const unsigned long long dims[2] = {(unsigned long long)inner, (unsigned long long)(2 * M)};
    const unsigned long long str[1] = {(unsigned long long)inner * 8};
    const unsigned box[2] = {(unsigned)T, (unsigned)XS::BR};
    return make_tmap(&tm->a, 2, in, dims, str, box);
  }
  const unsigned long long dims[2] = {(unsigned long long)(2 * inner), (unsigned long long)(M + 1)};
  const unsigned long long str[1] = {(unsigned long long)inner * 16};
  const unsigned box[2] = {(unsigned)(2 * T), (unsigned)XS::BR};
  const unsigned box1[2] = {(unsigned)(2 * T), 1u};
  return make_tmap(&tm->a, 2, in, dims, str, box) && make_tmap(&tm->b, 2, in, dims, str, box1);
}

template <int M, int MODE>
static int real_x_m(const void* in, void* out, i64 inner, double* diag, cudaStream_t st, RPro rp = RPro{}) {
  const double2* twN = twiddles(2 * M);
  if (!twN) return PFCS_E_CUDA;
  constexpr int PM = M / real_R(M, MODE);
  const long long tiles_min = (inner + (PM >= 32 ? 1 : 32 / PM) - 1) / (PM >= 32 ? 1 : 32 / PM);
  return with_variant_n<(MODE == MODE_CUBE || MODE == MODE_XMUL) ? KIND_CUBER : KIND_REALX, M>(tiles_min, [&](auto var) -> int {
    constexpr int V = decltype(var)::value;
    constexpr int P = M / real_R(M, MODE);
    // R2C/C2R at M = 256 (the 512^3 round trip) take 16 lines per tile:
    // 128-byte complex rows and real rows, one 512-thread CTA per SM (B200:
    // rfft_x 0.50 -> 0.42 ms, irfft_x 0.53 -> 0.43 ms; the cube pass stays
    // at 8 lines, 0.67 vs 0.71 ms)
    constexpr int TX = (MODE != MODE_CUBE && MODE != MODE_XMUL && M == 256) ? 1 : 0;
    constexpr int T = ((P >= 32 ? 1 : 32 / P) << (V & 3)) << TX;
    constexpr int ST = 1 + (V >> 2);
    if constexpr (T * P > 1024) {
      return fail(PFCS_E_UNSUPPORTED, "tile too large");
    } else {
      const i64 ntiles = (inner + T - 1) / T;
      TmaPair tm{};  // unused (zero) unless the TMA path is taken
      // TMA staging (B200 A/B, ms per launch, off -> on): cube 1024^3 7.02 -> 5.85,
      // 512^3 0.79 -> 0.67; C2R 1024^3 4.96 -> 4.75; R2C 512^3 0.57 -> 0.50 but
      // 1024^3 4.94 -> 5.58 (64-byte real rows, one CTA per SM), so R2C keeps
      // the register pipeline from M = 512 up.
      if constexpr (XStage<M, T, MODE>::SMEM <= 227 * 1024 && (!is_r2c(MODE) || (T >= 2 && M <= 256))) {
        // a product prologue (kind 1) streams a second real array: the
        // register pipeline prefetches it with the tile (512^3: 0.67 ms vs
        // 0.85 ms TMA-staged with the factor loaded one tile ahead)
        const bool reg_product = MODE == MODE_R2C_PRO && rp.kind == 1;
        if (!reg_product && tma_enabled() && x_tmaps<M, T, MODE>(&tm, in, inner)) {
          constexpr size_t smem = XStage<M, T, MODE>::SMEM;
          int grid = 0;
          if (int rc = persistent_grid((const void*)k_real_x<M, T, 3, MODE>, T * P, smem, ntiles, &grid)) return rc;
          launch_pdl(k_real_x<M, T, 3, MODE>, dim3(grid), dim3(T * P), smem, st, in, out, inner, twN,
                     1.0 / (double)(2 * M), diag, tm, rp);
          return check_launch("k_real_x(tma)");
        }
      }
      const size_t smem = (size_t)T * real_ls(M, T) * sizeof(double2);
      int grid = 0;
      if (int rc = persistent_grid((const void*)k_real_x<M, T, ST, MODE>, T * P, smem, ntiles, &grid)) return rc;
      launch_pdl(k_real_x<M, T, ST, MODE>, dim3(grid), dim3(T * P), smem, st, in, out, inner, twN,
                 1.0 / (double)(2 * M), diag, tm, rp);
      return check_launch("k_real_x");
    }
  });
}

template <int N>
static int cube_c2c_n(double2* data, i64 inner, double* diag, cudaStream_t st) {
  const double2* tw = twiddles(N);
  if (!tw) return PFCS_E_CUDA;
  return with_variant<KIND_CUBEC, N>([&](auto var) -> int {
    constexpr int V = decltype(var)::value;
    constexpr int T = TileCfg<N>::T_MIN << (V & 3);
    constexpr int ST = 1 + (V >> 2);
    constexpr int P = TileCfg<N>::P;
    if constexpr (T * P > 1024) {
      return fail(PFCS_E_UNSUPPORTED, "tile too large");
    } else {
      const size_t smem = (size_t)T * tile_ls(N, T, true) * sizeof(double2);
      const i64 ntiles = (inner + T - 1) / T;
      int grid = 0;
      if (int rc = persistent_grid((const void*)k_cube_c2c<N, T, ST>, T * P, smem, ntiles, &grid)) return rc;
      k_cube_c2c<N, T, ST><<<grid, T * P, smem, st>>>(data, inner, tw, 1.0 / (double)N, diag);
      return check_launch("k_cube_c2c");
    }
  });
}

#define PFCS_M_CASES(MACRO) \
  MACRO(2) MACRO(4) MACRO(8) MACRO(16) MACRO(32) MACRO(64) MACRO(128) MACRO(256) MACRO(512) \
      MACRO(1024) MACRO(2048) MACRO(4096)

int launch_real_x(const void* in, void* out, long long nx, long long inner, int mode, double* diag,
                  cudaStream_t st) {
  if (inner <= 0) return PFCS_OK;
  if (!is_pow2(nx) || nx < 4 || nx > 8192)
    return fail(PFCS_E_UNSUPPORTED, "real x transforms need a power-of-two nx in [4, 8192]");
  const int M = (int)(nx / 2);
  switch (M) {
#define PFCS_CASE(MM)                                                                   \
  case MM:                                                                              \
    if (mode == MODE_R2C) return real_x_m<MM, MODE_R2C>(in, out, inner, diag, st);     \
    if (mode == MODE_C2R) return real_x_m<MM, MODE_C2R>(in, out, inner, diag, st);     \
    if (in == out) {                                                                   \
      const int rc = launch_cube_ls(out, nx, inner, diag, st);                        \
      if (rc != 1) return rc;                                                         \
    }                                                                                 \
    return real_x_m<MM, MODE_CUBE>(in, out, inner, diag, st);
    PFCS_M_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported nx");
}

// x pass of a pseudo-spectral product (MODE_XMUL), in place
int launch_xmul(void* data, const double* aux, long long nx, long long inner, cudaStream_t st) {
  if (inner <= 0) return PFCS_OK;
  if (!aux) return fail(PFCS_E_ARG, "x-pass product needs aux");
  if (!is_pow2(nx) || nx < 4 || nx > 8192)
    return fail(PFCS_E_UNSUPPORTED, "real x transforms need a power-of-two nx in [4, 8192]");
  const RPro rp{1, 0.0, aux};
  switch (nx / 2) {
#define PFCS_CASE(MM) \
  case MM:            \
    return real_x_m<MM, MODE_XMUL>(data, data, inner, nullptr, st, rp);
    PFCS_M_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported nx");
}

// R2C x pass with a pointwise prologue (kinds of pfcs_real_pointwise 0, 1, 3)
int launch_rfft_x_pro(const double* in, void* out, long long nx, long long inner, int kind, const double* aux,
                      double alpha, cudaStream_t st) {
  if (inner <= 0) return PFCS_OK;
  if (kind != 0 && kind != 1 && kind != 3) return fail(PFCS_E_ARG, "rfft_x prologue kind must be 0, 1 or 3");
  if (kind == 1 && !aux) return fail(PFCS_E_ARG, "rfft_x product prologue needs aux");
  if (!is_pow2(nx) || nx < 4 || nx > 8192)
    return fail(PFCS_E_UNSUPPORTED, "real x transforms need a power-of-two nx in [4, 8192]");
  const RPro rp{kind, alpha, aux};
  switch (nx / 2) {
#define PFCS_CASE(MM) \
  case MM:            \
    return real_x_m<MM, MODE_R2C_PRO>(in, out, inner, nullptr, st, rp);
    PFCS_M_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported nx");
}

int launch_cube_c2c(void* data, long long nx, long long inner, double* diag, cudaStream_t st) {
  if (inner <= 0) return PFCS_OK;
  if (!is_pow2(nx) || nx < 2 || nx > 4096)
    return fail(PFCS_E_UNSUPPORTED, "fused complex cube pass needs a power-of-two nx in [2, 4096]");
  switch (nx) {
#define PFCS_CASE(NN) \
  case NN:            \
    return cube_c2c_n<NN>((double2*)data, inner, diag, st);
    PFCS_M_CASES(PFCS_CASE)
#undef PFCS_CASE
    default:
      break;
  }
  return fail(PFCS_E_UNSUPPORTED, "unsupported nx");
}

}  // namespace pfcs
