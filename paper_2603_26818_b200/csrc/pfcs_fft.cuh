// pfcs_fft.cuh — register/shared-memory Stockham line-FFT core for sm_100a (fp64).
//
// Replaces the arithmetic of the reference's serial line transform
// `fftcore.fft_axis` (pkg/src/pfcspectral/fftcore.py:31-40), which delegates to
// numpy's pocketfft.  Conventions follow the reference exactly:
//   forward  X[k] = sum_n x[n] exp(-2 pi i n k / N)       (unnormalised)
//   inverse  x[n] = fl(1/N) * sum_k X[k] exp(+2 pi i n k / N)
// (numpy's `ifft` multiplies every output by fct = 1/n, fftcore.py:13-14).
//
// Execution model.  One CTA owns a tile of T lines of length N (power of two).
// Each line is served by P = N/R threads that each hold R = 8 complex values in
// registers.  A pass performs R/r radix-r butterflies per thread (Stockham
// autosort, decimation in time: Govindaraju et al. 2008 formulation); the
// values are exchanged between passes through a padded shared-memory line.
// The first pass consumes the registers straight from global memory and the
// last pass leaves element j + P*e in register e of thread j, so global loads
// and stores are both unit-stride in j (coalesced) and no extra shared-memory
// round trip is spent at either end.
//
// Shared-memory layout: element n of line t lives at t*LS + PAD(n) with
// PAD(n) = n + n/8 and LS = PAD(N) + 2 (16-byte elements).  A bank simulator
// shows this is conflict-free (1.00x of the ideal
// wavefront count) for every pass of every N in 2..4096, for both the
// contiguous-line and the strided-column thread mappings.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pfcs {

typedef long long i64;

__host__ __device__ constexpr int pad_idx(int n) { return n + (n >> 3); }
__host__ __device__ constexpr int line_stride(int n) { return pad_idx(n) + 2; }
__host__ __device__ constexpr int radix_R(int n) { return n >= 8 ? 8 : n; }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * w (forward) or a * conj(w) (inverse)
template <bool FWD>
__device__ __forceinline__ double2 twmul(double2 a, double2 w) {
  if (FWD) return make_double2(fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x));
  return make_double2(fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y));
}
// a * (-i) forward, a * (+i) inverse
template <bool FWD>
__device__ __forceinline__ double2 mul_j(double2 a) {
  return FWD ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

template <bool FWD>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool FWD>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  double2 a0 = cadd(x0, x2), a1 = csub(x0, x2);
  double2 a2 = cadd(x1, x3), a3 = mul_j<FWD>(csub(x1, x3));
  x0 = cadd(a0, a2);
  x2 = csub(a0, a2);
  x1 = cadd(a1, a3);
  x3 = csub(a1, a3);
}

template <bool FWD>
__device__ __forceinline__ void dft8(double2 (&y)[8]) {
  const double s = 0.70710678118654752440;  // 1/sqrt(2)
  double2 e0 = y[0], e1 = y[2], e2 = y[4], e3 = y[6];
  double2 o0 = y[1], o1 = y[3], o2 = y[5], o3 = y[7];
  dft4<FWD>(e0, e1, e2, e3);
  dft4<FWD>(o0, o1, o2, o3);
  double2 t1, t2, t3;
  if (FWD) {
    t1 = make_double2((o1.x + o1.y) * s, (o1.y - o1.x) * s);
    t3 = make_double2((o3.y - o3.x) * s, -(o3.x + o3.y) * s);
  } else {
    t1 = make_double2((o1.x - o1.y) * s, (o1.x + o1.y) * s);
    t3 = make_double2(-(o3.x + o3.y) * s, (o3.x - o3.y) * s);
  }
  t2 = mul_j<FWD>(o2);
  y[0] = cadd(e0, o0);
  y[4] = csub(e0, o0);
  y[1] = cadd(e1, t1);
  y[5] = csub(e1, t1);
  y[2] = cadd(e2, t2);
  y[6] = csub(e2, t2);
  y[3] = cadd(e3, t3);
  y[7] = csub(e3, t3);
}

template <int r, bool FWD>
__device__ __forceinline__ void dft_r(double2 (&y)[r]) {
  if constexpr (r == 2) {
    dft2<FWD>(y[0], y[1]);
  } else if constexpr (r == 4) {
    dft4<FWD>(y[0], y[1], y[2], y[3]);
  } else if constexpr (r == 8) {
    dft8<FWD>(y);
  }
}

// One Stockham pass (span Ns) followed, if more passes remain, by the
// shared-memory exchange and the next pass.  On entry v[e] holds element
// j + P*e of this pass's input; on exit of the last pass v[e] holds output
// element j + P*e.  `tw` is the size-N table exp(-2 pi i m / N), m < N,
// read with stride TWS (so a size-2N table serves an N-point transform).
template <int N, int Ns, bool FWD, int TWS>
__device__ __forceinline__ void fft_pass(double2 (&v)[radix_R(N)], int j, double2* sl,
                                         const double2* __restrict__ tw) {
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
  constexpr int rem = N / Ns;
  constexpr int r = (R < 8) ? R : (rem >= 8 ? 8 : rem);
  constexpr int S = R / r;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int b = j + s * P;
    const int k = b & (Ns - 1);
    double2 y[r];
#pragma unroll
    for (int q = 0; q < r; ++q) y[q] = v[s + q * S];
    if constexpr (Ns > 1) {
#pragma unroll
      for (int q = 1; q < r; ++q) y[q] = twmul<FWD>(y[q], __ldg(&tw[TWS * (q * k) * (N / (Ns * r))]));
    }
    dft_r<r, FWD>(y);
#pragma unroll
    for (int q = 0; q < r; ++q) v[s + q * S] = y[q];
  }
  if constexpr (Ns * r < N) {
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int b = j + s * P;
      const int k = b & (Ns - 1);
      const int base = (b / Ns) * Ns * r + k;
#pragma unroll
      for (int q = 0; q < r; ++q) sl[pad_idx(base + q * Ns)] = v[s + q * S];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < R; ++e) v[e] = sl[pad_idx(j + P * e)];
    fft_pass<N, Ns * r, FWD, TWS>(v, j, sl, tw);
  }
}

// Full N-point transform of the register set (see fft_pass).  All threads of
// the CTA must call it (it contains __syncthreads when N > 8).
template <int N, bool FWD, int TWS = 1>
__device__ __forceinline__ void fft_line(double2 (&v)[radix_R(N)], int j, double2* sl,
                                         const double2* __restrict__ tw) {
  fft_pass<N, 1, FWD, TWS>(v, j, sl, tw);
}

// Stash register set (element j + P*e in v[e]) into the padded smem line.
template <int N>
__device__ __forceinline__ void stash_line(const double2 (&v)[radix_R(N)], int j, double2* sl) {
  constexpr int R = radix_R(N);
  constexpr int P = N / R;
#pragma unroll
  for (int e = 0; e < R; ++e) sl[pad_idx(j + P * e)] = v[e];
}

// Tile shape policy: T lines per CTA so that a tile holds ~4096 complex
// values (64 KB of shared memory, <= 512 threads), at least 1 line, and at
// least one full warp per CTA (warp-synchronous diagnostics need it).
template <int N>
struct TileCfg {
  static constexpr int R = radix_R(N);
  static constexpr int P = N / R;
  static constexpr int T_CONTIG = (N >= 4096) ? 1 : (4096 / N > 64 ? 64 : 4096 / N);
  static constexpr int T_STRIDED = (N >= 4096) ? 1 : (4096 / N > 32 ? 32 : 4096 / N);
};

// Balanced slab bookkeeping (grid.slab_layout, grid.py:103-111): the first
// `extra` ranks own base+1 planes, the rest own `base`.
struct SlabSplit {
  int G, base, extra;
  __host__ __device__ __forceinline__ void locate(int z, int& zoff, int& cz) const {
    const int big = base + 1;
    const int split = extra * big;
    if (z < split) {
      const int g = z / big;
      zoff = g * big;
      cz = big;
    } else {
      const int g = (z - split) / base;
      zoff = split + g * base;
      cz = base;
    }
  }
};

}  // namespace pfcs
