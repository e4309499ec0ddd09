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

#include <type_traits>

namespace pfcs {

typedef long long i64;

#ifndef PFCS_TW_LOADS
#define PFCS_TW_LOADS 3  // twiddle-table loads per radix-8 butterfly (7, 3 or 1)
#endif
#ifndef PFCS_X_TWL
// twiddle loads per butterfly in the x passes (R2C / C2R / fused cube): one
// table load + products measured faster there on the B200 (cube 1024^3
// 5.83 -> 5.70 ms, R2C/C2R 512^3 -3 %); the y / z line passes keep 3
#define PFCS_X_TWL 1
#endif
#ifndef PFCS_LINES_TWL
// contiguous z-line passes (k_lines): one load + products measured faster
// (1024-point lines 3.38 -> 2.85 ms per 1024^3 pass, 512-point unchanged)
#define PFCS_LINES_TWL 1
#endif
#ifndef PFCS_Y_TWL
#define PFCS_Y_TWL PFCS_TW_LOADS  // strided y passes: 3 (1 measured 2 % slower)
#endif
#ifndef PFCS_Y_TWSMEM
#define PFCS_Y_TWSMEM 0  // 1: TMA y pass reads twiddles from a smem copy (A/B: 1024^3 3.83 -> 3.98 ms, slower)
#endif
#ifndef PFCS_DFT8_FMA
#define PFCS_DFT8_FMA 0  // A/B: fold the radix-8 1/sqrt(2) rotations into FMAs
#endif

__host__ __device__ constexpr int pad_idx(int n) { return n + (n >> 3); }
__host__ __device__ constexpr int line_stride(int n) { return pad_idx(n) + 2; }
// Line stride of a T-line tile.  Contiguous-line tiles put 8 consecutive j
// of one line in a quarter warp, so any stride is conflict-free; strided
// tiles put min(T, 8) columns side by side, so line bases must fall on
// distinct 16-byte bank slots: stride = PAD(N) + (8 / min(T, 8)) mod 8
// (bank simulator: 1.00x ideal wavefronts for every
// N in 16..4096 and T in 1..32).
__host__ __device__ constexpr int tile_ls(int n, int t, bool strided) {
  return pad_idx(n) + ((!strided || n <= 8) ? 0 : (8 / (t < 8 ? t : 8)) % 8);
}
#ifndef PFCS_R16
#define PFCS_R16 0  // lines of >= PFCS_R16 points hold 16 values per thread (radix-16 passes); 0 = off
#endif
__host__ __device__ constexpr int radix_R(int n) {
  return (PFCS_R16 > 0 && n >= PFCS_R16) ? 16 : (n >= 8 ? 8 : n);
}
// minBlocksPerSM for __launch_bounds__: enough CTAs for `target` resident
// threads per SM, which caps registers at 65536 / target per thread.
__host__ __device__ constexpr int min_blocks(int threads, int target) {
  return target / threads < 1 ? 1 : (target / threads > 16 ? 16 : target / threads);
}

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

// Opaque copy of an index: the compiler must assume it changes here, so the
// (thread-index-only) address arithmetic of the exchanges is recomputed
// where it is used instead of being hoisted out of the persistent tile loop
// or above the previous FFT of a fused pass, where it pinned ~60 registers
// (the fused cube pass went from 128 registers + spills to 64 without).
__device__ __forceinline__ int opaque(int x) {
  asm volatile("" : "+r"(x));
  return x;
}
// Programmatic dependent launch: wait until the stream predecessor grid has
// completed and its writes are visible, then let our own dependents launch.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// threadIdx.x read that cannot be hoisted (recomputing a tile's thread
// coordinates per tile keeps the whole index/pointer family loop-local)
// (unsigned, so tid % T and tid / T stay single AND/shift instructions)
__device__ __forceinline__ unsigned opaque_tid() {
  unsigned t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

// Twiddle load through the read-only path, as volatile asm so the compiler
// keeps it inside its pass instead of hoisting every pass's twiddles to the
// top of the kernel (which costs ~30 live registers in the fused passes).
__device__ __forceinline__ double2 ldg_tw(const double2* p) {
#ifdef PFCS_TW_HOIST
  return __ldg(p);
#else
  double2 w;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y) : "l"(p));
  return w;
#endif
}

// Twiddle load from a shared-memory copy of the table (kernels that stage it
// with `TSM`); volatile for the same no-hoisting reason as ldg_tw.
__device__ __forceinline__ double2 lds_tw(const double2* p) {
  double2 w;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w.x), "=d"(w.y)
               : "r"((unsigned)__cvta_generic_to_shared(p)));
  return w;
}
template <bool TSM>
__device__ __forceinline__ double2 ld_tw(const double2* p) {
  if constexpr (TSM) return lds_tw(p);
  else return ldg_tw(p);
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
#if PFCS_DFT8_FMA
  // the 1/sqrt(2) rotations folded into the final add/sub as FMAs (4 fewer
  // fp64 instructions per dft8)
  double2 u1, u3;
  if (FWD) {
    u1 = make_double2(o1.x + o1.y, o1.y - o1.x);
    u3 = make_double2(o3.y - o3.x, -(o3.x + o3.y));
  } else {
    u1 = make_double2(o1.x - o1.y, o1.x + o1.y);
    u3 = make_double2(-(o3.x + o3.y), o3.x - o3.y);
  }
  const double2 t2 = mul_j<FWD>(o2);
  y[0] = cadd(e0, o0);
  y[4] = csub(e0, o0);
  y[1] = make_double2(fma(s, u1.x, e1.x), fma(s, u1.y, e1.y));
  y[5] = make_double2(fma(-s, u1.x, e1.x), fma(-s, u1.y, e1.y));
  y[2] = cadd(e2, t2);
  y[6] = csub(e2, t2);
  y[3] = make_double2(fma(s, u3.x, e3.x), fma(s, u3.y, e3.y));
  y[7] = make_double2(fma(-s, u3.x, e3.x), fma(-s, u3.y, e3.y));
#else
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
#endif
}

// 16-point DFT as 4 x 4: dft4 over stride-4 columns, twiddles W16^(n2 k1),
// dft4 over rows; output index k1 + 4 k2 sits at 4 k1 + k2 before the final
// (compile-time) transpose.
template <bool FWD>
__device__ __forceinline__ void dft16(double2 (&y)[16]) {
  const double c = 0.92387953251128675613;  // cos(pi/8)
  const double s = 0.38268343236508977173;  // sin(pi/8)
  const double h = 0.70710678118654752440;  // 1/sqrt(2)
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) dft4<FWD>(y[n2], y[4 + n2], y[8 + n2], y[12 + n2]);
  // element (k1, n2) is y[4 k1 + n2]; multiply by W16^(n2 k1)
  const double sg = FWD ? -1.0 : 1.0;
  y[5] = cmul(y[5], make_double2(c, sg * s));            // k1=1 n2=1: W^1
  y[6] = cmul(y[6], make_double2(h, sg * h));            // W^2
  y[7] = cmul(y[7], make_double2(s, sg * c));            // W^3
  y[9] = cmul(y[9], make_double2(h, sg * h));            // k1=2 n2=1: W^2
  y[10] = mul_j<FWD>(y[10]);                             // W^4
  y[11] = cmul(y[11], make_double2(-h, sg * h));         // W^6
  y[13] = cmul(y[13], make_double2(s, sg * c));          // k1=3 n2=1: W^3
  y[14] = cmul(y[14], make_double2(-h, sg * h));         // W^6
  y[15] = cmul(y[15], make_double2(-c, -sg * s));        // W^9
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) dft4<FWD>(y[4 * k1], y[4 * k1 + 1], y[4 * k1 + 2], y[4 * k1 + 3]);
  double2 z[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) z[i] = y[i];
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) y[k1 + 4 * k2] = z[4 * k1 + k2];
}

template <int r, bool FWD>
__device__ __forceinline__ void dft_r(double2 (&y)[r]) {
  if constexpr (r == 2) {
    dft2<FWD>(y[0], y[1]);
  } else if constexpr (r == 4) {
    dft4<FWD>(y[0], y[1], y[2], y[3]);
  } else if constexpr (r == 8) {
    dft8<FWD>(y);
  } else if constexpr (r == 16) {
    dft16<FWD>(y);
  }
}

// Barrier flavours of the shared-memory exchanges: the whole CTA (tiles whose
// lines are interleaved across warps), or a named barrier over the `n`
// threads of one line group (line-major tiles: each line's warps exchange
// through their own workspace and synchronise only among themselves, so
// different lines drift into different phases and the fp64 and shared-memory
// pipes overlap instead of alternating CTA-wide).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct BarSync {
  unsigned id, n;  // barrier id (1..15; 0 is __syncthreads), participating threads
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
  }
};

// Exchange workspace of one line: a padded shared-memory line (double2*,
// element n at PAD(n)) or any accessor with ref(n) (e.g. the line's column
// of a swizzled TMA stage, pfcs_x.cu k_cube_ls).
__device__ __forceinline__ double2& ws_ref(double2* sl, int n) { return sl[pad_idx(n)]; }
template <class W>
__device__ __forceinline__ double2& ws_ref(const W& w, int n) { return w.ref(n); }

// One Stockham pass (span Ns) followed, if more passes remain, by the
// shared-memory exchange and the next pass.  On entry v[e] holds element
// j + P*e of this pass's input; on exit of the last pass v[e] holds output
// element j + P*e.  `tw` is the size-N table exp(-2 pi i m / N), m < N,
// read with stride TWS (so a size-2N table serves an N-point transform).
template <int N, int Ns, bool FWD, int TWS, int TWL = PFCS_TW_LOADS, int R = radix_R(N), bool TSM = false,
          class Sync = CtaSync, class WS = double2*>
__device__ __forceinline__ void fft_pass(double2 (&v)[R], int j, WS sl,
                                         const double2* __restrict__ tw, Sync sync = Sync{}) {
  // R = values per thread (8, or 4 for the register-heavy fused passes);
  // each pass uses radix min(R, remaining) and R/r butterflies per thread
  constexpr int P = N / R;
  constexpr int rem = N / Ns;
  constexpr int r = (rem >= R) ? R : rem;
  constexpr int S = R / r;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int b = j + s * P;
    const int k = b & (Ns - 1);
    double2 y[r];
#pragma unroll
    for (int q = 0; q < r; ++q) y[q] = v[s + q * S];
    if constexpr (Ns > 1) {
      // twiddles w^q, w = W_{r Ns}^k: TW_LOADS table loads (w, w^2, w^4 or
      // w alone) and the other powers by complex products — the L1/LSU path
      // they would otherwise occupy is shared with the smem exchanges
      // (7 loads -> 3 lifted z-line kernels from 4.3 to 5.9 TB/s on B200)
      const int t1 = TWS * k * (N / (Ns * r));
      double2 w[r];
      w[1] = ld_tw<TSM>(&tw[t1]);
      if constexpr (r >= 4) w[2] = (TWL >= 3) ? ld_tw<TSM>(&tw[2 * t1]) : cmul(w[1], w[1]);
      if constexpr (r == 4) w[3] = (TWL >= 7) ? ld_tw<TSM>(&tw[3 * t1]) : cmul(w[1], w[2]);
      if constexpr (r == 8) {
        w[4] = (TWL >= 3) ? ld_tw<TSM>(&tw[4 * t1]) : cmul(w[2], w[2]);
        if constexpr (TWL >= 7) {  // every power from the table: no fp64 products
          w[3] = ld_tw<TSM>(&tw[3 * t1]);
          w[5] = ld_tw<TSM>(&tw[5 * t1]);
          w[6] = ld_tw<TSM>(&tw[6 * t1]);
          w[7] = ld_tw<TSM>(&tw[7 * t1]);
        } else {
          w[3] = cmul(w[1], w[2]);
          w[5] = cmul(w[1], w[4]);
          w[6] = cmul(w[2], w[4]);
          w[7] = cmul(w[3], w[4]);
        }
      }
      if constexpr (r == 16) {
        w[4] = (TWL >= 3) ? ld_tw<TSM>(&tw[4 * t1]) : cmul(w[2], w[2]);
        w[8] = (TWL >= 3) ? ld_tw<TSM>(&tw[8 * t1]) : cmul(w[4], w[4]);
        w[3] = cmul(w[1], w[2]);
        w[5] = cmul(w[1], w[4]);
        w[6] = cmul(w[2], w[4]);
        w[7] = cmul(w[3], w[4]);
#pragma unroll
        for (int q = 9; q < 16; ++q) w[q] = cmul(w[q - 8], w[8]);
      }
#pragma unroll
      for (int q = 1; q < r; ++q) y[q] = twmul<FWD>(y[q], w[q]);
    }
    dft_r<r, FWD>(y);
#pragma unroll
    for (int q = 0; q < r; ++q) v[s + q * S] = y[q];
  }
  if constexpr (Ns * r < N) {
    sync();
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int b = j + s * P;
      const int k = b & (Ns - 1);
      const int base = (b / Ns) * Ns * r + k;
#pragma unroll
      for (int q = 0; q < r; ++q) {
        if constexpr (std::is_pointer_v<WS>) sl[pad_idx(base + q * Ns)] = v[s + q * S];
        else ws_ref(sl, base + q * Ns) = v[s + q * S];
      }
    }
    sync();
#pragma unroll
    for (int e = 0; e < R; ++e) {
      if constexpr (std::is_pointer_v<WS>) v[e] = sl[pad_idx(j + P * e)];
      else v[e] = ws_ref(sl, j + P * e);
    }
    fft_pass<N, Ns * r, FWD, TWS, TWL, R, TSM, Sync, WS>(v, j, sl, tw, sync);
  }
}

// Full N-point transform of the register set (see fft_pass).  All threads of
// the CTA must call it (it contains __syncthreads when N > 8).
template <int N, bool FWD, int TWS = 1, int TWL = PFCS_TW_LOADS, int R = radix_R(N), bool TSM = false,
          class Sync = CtaSync, class WS = double2*>
__device__ __forceinline__ void fft_line(double2 (&v)[R], int j, WS sl,
                                         const double2* __restrict__ tw, Sync sync = Sync{}) {
  fft_pass<N, 1, FWD, TWS, TWL, R, TSM, Sync, WS>(v, j, sl, tw, sync);
}

// Stash register set (element j + P*e in v[e]) into the padded smem line.
template <int N, int R = radix_R(N)>
__device__ __forceinline__ void stash_line(const double2 (&v)[R], int j, double2* sl) {
  constexpr int P = N / R;
#pragma unroll
  for (int e = 0; e < R; ++e) sl[pad_idx(j + P * e)] = v[e];
}

// ------------------------------------------------------ tile pipelines --
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// Register-pipelined persistent loop: `Regs` is the per-thread register set
// of one tile (its R elements, plus whatever the kernel needs).
//   load(tile, regs)  issues the global loads of `tile` into registers
//   comp(tile, regs)  runs the transform out of the registers and stores
// ST == 2 issues the loads of tile i+1 before computing tile i, so ~R*16
// bytes per thread stay in flight through the butterflies (no extra shared
// memory traffic, unlike a cp.async landing buffer); ST == 1 loads at the
// top of each tile and relies on the other resident CTAs for overlap.
template <int ST, class Regs, class Load, class Comp>
__device__ __forceinline__ void reg_tile_loop(long long ntiles, Load&& load, Comp&& comp) {
  if constexpr (ST == 1) {
    for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      Regs r;
      load(tile, r);
      comp(tile, r);
      __syncthreads();
    }
  } else {
    Regs nxt;
    long long tile = blockIdx.x;
    if (tile < ntiles) load(tile, nxt);
    for (; tile < ntiles; tile += gridDim.x) {
      Regs cur = nxt;
      const long long next = tile + gridDim.x;
      if (next < ntiles) load(next, nxt);
      comp(tile, cur);
      __syncthreads();
    }
  }
}

// Tile shape: T lines per CTA, T = T_MIN << shift.  Small N needs several
// lines to fill a warp (warp-synchronous diagnostics); the shift and the
// number of pipeline stages come from the tuning table (pfcs_internal.h).
template <int N>
struct TileCfg {
  static constexpr int R = radix_R(N);
  static constexpr int P = N / R;
  static constexpr int T_MIN = (P >= 32) ? 1 : 32 / P;
};

// Balanced slab bookkeeping (grid.slab_layout, grid.py:103-111): the first
// `extra` ranks own base+1 planes, the rest own `base`.
struct SlabSplit {
  int G, base, extra;
  __host__ __device__ __forceinline__ void locate(int z, int& zoff, int& cz) const {
    int g;
    locate3(z, g, zoff, cz);
  }
  __host__ __device__ __forceinline__ void locate3(int z, int& g, int& zoff, int& cz) const {
    const int big = base + 1;
    const int split = extra * big;
    if (z < split) {
      g = z / big;
      zoff = g * big;
      cz = big;
    } else {
      g = extra + (z - split) / base;
      zoff = split + (g - extra) * base;
      cz = base;
    }
  }
};

// Per-destination base pointers of a scattered ("blocked") output.  Block g
// of the split axis goes to p[g]: a slab of the local send buffer, or —
// for the fused exchange — the receive buffer of rank g itself, mapped
// through CUDA peer access / IPC, so the FFT epilogue stores straight over
// NVLink (no separate all-to-all).  Passed by value (kernel parameter).
#define PFCS_MAX_PEERS 16
struct PeerTable {
  double2* p[PFCS_MAX_PEERS];
};

// Table of the local blocked layout: slab g of `out` at nlines * zoff_g.
inline PeerTable local_table(double2* out, long long nlines, int G, int base, int extra) {
  PeerTable t{};
  long long off = 0;
  for (int g = 0; g < G && g < PFCS_MAX_PEERS; ++g) {
    t.p[g] = out + nlines * off;
    off += base + (g < extra ? 1 : 0);
  }
  return t;
}

}  // namespace pfcs
