// pfcs_mixed.cu — mixed-radix Stockham line transforms for lengths that are
// not powers of two (the reference accepts any N: sizes 1..16 and primes in
// its tests, 750^3 and 1400^3 grids in the paper).
//
// N is factorised into radices 4, 2, 3, 5, 7 and any remaining primes; a CTA
// loads a tile of T lines into shared memory and runs one Stockham pass per
// radix (generalised span Ns = product of the previous radices) between two
// ping-pong shared buffers, then stores.  Radices 2..5 are closed-form
// butterflies; other primes use an O(r^2) DFT on the table twiddles, so a
// prime N degenerates gracefully to the direct DFT.  Twiddles come from the
// same exact size-N table as the power-of-two kernels.  This is the parity
// path for arbitrary sizes; the fused PFC passes stay power-of-two.
#include "pfcs_fft.cuh"
#include "pfcs_internal.h"

namespace pfcs {

#define PFCS_MAX_PASSES 24

struct RadixPlan {
  int n, np;
  int r[PFCS_MAX_PASSES];
};

template <bool FWD>
__device__ __forceinline__ double2 tw_at(const double2* __restrict__ tw, long long idx, int n) {
  const double2 w = __ldg(&tw[idx % n]);
  return FWD ? w : make_double2(w.x, -w.y);
}

// y[m] = sum_q x[q] W_r^{q m} (sign by FWD), generic r via the size-n table
template <bool FWD>
__device__ void dft_generic(double2* x, double2* y, int r, const double2* __restrict__ tw, int n) {
  const int step = n / r;
  if (r == 2) {
    y[0] = cadd(x[0], x[1]);
    y[1] = csub(x[0], x[1]);
  } else if (r == 3) {
    const double c = -0.5, s = FWD ? -0.86602540378443864676 : 0.86602540378443864676;
    const double2 a = cadd(x[1], x[2]), d = csub(x[1], x[2]);
    y[0] = cadd(x[0], a);
    const double2 m = make_double2(x[0].x + c * a.x, x[0].y + c * a.y);
    y[1] = make_double2(m.x - s * d.y, m.y + s * d.x);
    y[2] = make_double2(m.x + s * d.y, m.y - s * d.x);
  } else if (r == 4) {
    double2 a0 = x[0], a1 = x[1], a2 = x[2], a3 = x[3];
    dft4<FWD>(a0, a1, a2, a3);
    y[0] = a0;
    y[1] = a1;
    y[2] = a2;
    y[3] = a3;
  } else {
    for (int m = 0; m < r; ++m) {
      double ar = 0.0, ai = 0.0;
      for (int q = 0; q < r; ++q) {
        const double2 w = tw_at<FWD>(tw, (long long)step * ((q * m) % r), n);
        ar = fma(x[q].x, w.x, fma(-x[q].y, w.y, ar));
        ai = fma(x[q].x, w.y, fma(x[q].y, w.x, ai));
      }
      y[m] = make_double2(ar, ai);
    }
  }
}

#define PFCS_MIXED_MAXR 64

// One Stockham pass of radix RR (compile time): butterfly b reads
// A[b + q N/RR], twiddles by W_{Ns RR}^{q k} (k = b mod Ns), writes
// B[(b/Ns) Ns RR + k + q Ns].
template <bool FWD, int RR>
__device__ __forceinline__ void mixed_pass(const double2* A, double2* B, int T, int n, int Ns,
                                           const double2* __restrict__ tw) {
  const int nb = n / RR;
  for (int idx = threadIdx.x; idx < T * nb; idx += blockDim.x) {
    const int t = idx / nb;
    const int b = idx - t * nb;
    const int k = b % Ns;
    double2 x[RR], y[RR];
    const double2* src = A + t * n;
#pragma unroll
    for (int q = 0; q < RR; ++q) {
      double2 v = src[b + q * nb];
      if (q > 0 && Ns > 1) v = cmul(v, tw_at<FWD>(tw, (long long)q * k * (n / (Ns * RR)), n));
      x[q] = v;
    }
    if constexpr (RR == 5) {
      // closed-form radix 5 (cos/sin of 2 pi/5, 4 pi/5)
      const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
      const double s1 = FWD ? -0.95105651629515357212 : 0.95105651629515357212;
      const double s2 = FWD ? -0.58778525229247312917 : 0.58778525229247312917;
      const double2 a1 = cadd(x[1], x[4]), b1 = csub(x[1], x[4]);
      const double2 a2 = cadd(x[2], x[3]), b2 = csub(x[2], x[3]);
      y[0] = make_double2(x[0].x + a1.x + a2.x, x[0].y + a1.y + a2.y);
      const double2 m1 = make_double2(x[0].x + c1 * a1.x + c2 * a2.x, x[0].y + c1 * a1.y + c2 * a2.y);
      const double2 m2 = make_double2(x[0].x + c2 * a1.x + c1 * a2.x, x[0].y + c2 * a1.y + c1 * a2.y);
      const double2 n1 = make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
      const double2 n2 = make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
      // y_m = m + i n  for m = 1, 2 and conjugate pairs for 4, 3
      y[1] = make_double2(m1.x - n1.y, m1.y + n1.x);
      y[4] = make_double2(m1.x + n1.y, m1.y - n1.x);
      y[2] = make_double2(m2.x - n2.y, m2.y + n2.x);
      y[3] = make_double2(m2.x + n2.y, m2.y - n2.x);
    } else {
      dft_generic<FWD>(x, y, RR, tw, n);
    }
    double2* dst = B + t * n;
    const int base = (b / Ns) * Ns * RR + k;
#pragma unroll
    for (int q = 0; q < RR; ++q) dst[base + q * Ns] = y[q];
  }
}

template <bool FWD>
__device__ void mixed_pass_generic(const double2* A, double2* B, int T, int n, int Ns, int r,
                                   const double2* __restrict__ tw) {
  const int nb = n / r;
  for (int idx = threadIdx.x; idx < T * nb; idx += blockDim.x) {
    const int t = idx / nb;
    const int b = idx - t * nb;
    const int k = b % Ns;
    double2 x[PFCS_MIXED_MAXR], y[PFCS_MIXED_MAXR];
    const double2* src = A + t * n;
    for (int q = 0; q < r; ++q) {
      double2 v = src[b + q * nb];
      if (Ns > 1 && q > 0) v = cmul(v, tw_at<FWD>(tw, (long long)q * k * (n / (Ns * r)), n));
      x[q] = v;
    }
    dft_generic<FWD>(x, y, r, tw, n);
    double2* dst = B + t * n;
    const int base = (b / Ns) * Ns * r + k;
    for (int q = 0; q < r; ++q) dst[base + q * Ns] = y[q];
  }
}

template <bool FWD>
__global__ void k_mixed(const double2* in, double2* out, long long outer, long long inner, int T,
                        long long tpo, RadixPlan plan, const double2* __restrict__ tw, double scale) {
  extern __shared__ double2 sm[];
  const int n = plan.n;
  double2* A = sm;
  double2* B = sm + (size_t)T * n;
  const bool contig = inner == 1;
  long long o0, i0;
  if (contig) {
    o0 = (long long)blockIdx.x * T;
    i0 = 0;
  } else {
    o0 = (long long)blockIdx.x / tpo;
    i0 = ((long long)blockIdx.x - o0 * tpo) * T;
  }
  const int tot = T * n;
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int t, e;
    if (contig) {
      t = idx / n;
      e = idx - t * n;
    } else {
      e = idx / T;
      t = idx - e * T;
    }
    const long long o = contig ? o0 + t : o0;
    const long long i = contig ? 0 : i0 + t;
    double2 v = make_double2(0.0, 0.0);
    if (o < outer && i < inner) v = in[(o * n + e) * inner + i];
    A[t * n + e] = v;
  }
  __syncthreads();
  int Ns = 1;
  for (int p = 0; p < plan.np; ++p) {
    const int r = plan.r[p];
    switch (r) {  // register-resident butterflies for the common radices
      case 2: mixed_pass<FWD, 2>(A, B, T, n, Ns, tw); break;
      case 3: mixed_pass<FWD, 3>(A, B, T, n, Ns, tw); break;
      case 4: mixed_pass<FWD, 4>(A, B, T, n, Ns, tw); break;
      case 5: mixed_pass<FWD, 5>(A, B, T, n, Ns, tw); break;
      case 7: mixed_pass<FWD, 7>(A, B, T, n, Ns, tw); break;
      default: mixed_pass_generic<FWD>(A, B, T, n, Ns, r, tw); break;
    }
    __syncthreads();
    double2* tmp = A;
    A = B;
    B = tmp;
    Ns *= r;
  }
  for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    int t, e;
    if (contig) {
      t = idx / n;
      e = idx - t * n;
    } else {
      e = idx / T;
      t = idx - e * T;
    }
    const long long o = contig ? o0 + t : o0;
    const long long i = contig ? 0 : i0 + t;
    if (o < outer && i < inner) {
      double2 v = A[t * n + e];
      if (!FWD) v = make_double2(v.x * scale, v.y * scale);
      out[(o * n + e) * inner + i] = v;
    }
  }
}

static bool make_plan(int n, RadixPlan& pl) {
  pl.n = n;
  pl.np = 0;
  int m = n;
  while (m % 4 == 0) {
    pl.r[pl.np++] = 4;
    m /= 4;
  }
  while (m % 2 == 0) {
    pl.r[pl.np++] = 2;
    m /= 2;
  }
  for (int p = 3; m > 1;) {
    if (m % p == 0) {
      if (p > PFCS_MIXED_MAXR || pl.np >= PFCS_MAX_PASSES) return false;
      pl.r[pl.np++] = p;
      m /= p;
    } else {
      p += 2;
    }
  }
  return true;
}

int launch_mixed(const double2* in, double2* out, long long outer, int n, long long inner, bool forward,
                 cudaStream_t st) {
  RadixPlan plan;
  if (!make_plan(n, plan)) return -1;  // caller falls back to the direct DFT
  const double2* tw = twiddles(n);
  if (!tw) return PFCS_E_CUDA;
  int T = 1024 / n;
  if (T < 1) T = 1;
  if (T > 16) T = 16;
  const bool contig = inner == 1;
  const long long tpo = contig ? 1 : (inner + T - 1) / T;
  const long long blocks = contig ? (outer + T - 1) / T : outer * tpo;
  const size_t smem = 2 * (size_t)T * n * sizeof(double2);
  if (smem > 227 * 1024) return -1;
  const void* f = forward ? (const void*)k_mixed<true> : (const void*)k_mixed<false>;
  if (ensure_smem(f, smem)) return PFCS_E_CUDA;
  if (forward)
    k_mixed<true><<<(unsigned)blocks, 256, smem, st>>>(in, out, outer, inner, T, tpo, plan, tw, 1.0 / n);
  else
    k_mixed<false><<<(unsigned)blocks, 256, smem, st>>>(in, out, outer, inner, T, tpo, plan, tw, 1.0 / n);
  return check_launch("k_mixed");
}

}  // namespace pfcs
