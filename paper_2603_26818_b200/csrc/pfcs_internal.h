// pfcs_internal.h — host-side helpers shared by the libpfcs translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <type_traits>
#include <utility>

#include "../../include/pfcs.h"

namespace pfcs {

// thread-local last error (pfcs_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_cuda(cudaError_t e, const char* what);
int check_launch(const char* what);

// exp(-2 pi i m / N) table for m < N on the current device (cached per
// device and N; built once with octant symmetry in long double).
const double2* twiddles(int N);
// same table for an arbitrary N (used by the direct-DFT path)
inline bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }
inline int ilog2(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

// TMA-staged strided pass (pfcs_tma.cu): default on, PFCS_TMA=0 disables; returns 1
// when it does not apply to the call.
bool tma_enabled();
bool make_tmap(CUtensorMap* map, int rank, const void* base, const unsigned long long* dims,
               const unsigned long long* strides_bytes, const unsigned* box, int swizzle_bytes = 0);
// Line-synchronous TMA cube pass (pfcs_cube.cu); returns 1 when it does not
// apply (the caller then runs k_real_x MODE_CUBE)
int launch_cube_ls(void* data, long long nx, long long inner, double* diag, cudaStream_t st);
struct SlabSplitH;
struct PeerTable;
struct Pro;
int launch_strided_tma(const double2* in, double2* out, long long outer, int n, long long inner, bool forward,
                       cudaStream_t st, const SlabSplitH* souter = nullptr, const PeerTable* dst = nullptr,
                       const Pro* pro = nullptr);
int launch_lines_pro(const double2* in, double2* out, long long nlines, int n, const Pro& pro, bool forward,
                     cudaStream_t st);

// Programmatic dependent launch (Hopper/Blackwell): the kernel may be
// scheduled while its stream predecessor drains; it calls pdl_wait() (device)
// before touching the predecessor's output.  Cuts the launch gap between the
// small back-to-back passes of launch-bound steps (2D PFC) and is a no-op
// cost for the large ones.  PFCS_PDL=0 disables it (A/B).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}


// Opt a kernel in to > 48 KB dynamic shared memory once.
int ensure_smem(const void* func, size_t bytes);

// Persistent launch size: min(ntiles, resident CTAs per SM x SM count),
// from the occupancy calculator (cached per kernel/config and device).
// Also performs the shared-memory opt-in.
int persistent_grid(const void* func, int threads, size_t smem, long long ntiles, int* grid);

// ----------------------------------------------------------- tile tuning ----
// Launch variant V = shift + 4 * (stages - 1): tile width T = T_MIN << shift,
// 1 or 2 cp.async pipeline stages.  The production build bakes the measured
// best variant per kernel kind and length (default_variant, from
// tools/tune.py on a B200); a build with -DPFCS_TUNE instantiates all eight
// and reads PFCS_VARIANT_<kind>_<N> from the environment.
enum { KIND_LINES = 0, KIND_STRIDED = 1, KIND_REALX = 2, KIND_CUBEC = 3, KIND_PFCZ = 4, KIND_CUBER = 5 };

// Measured on B200 (tools/tune.py, profiles/r1_tune.json): contiguous z
// lines like one line per CTA with the next tile's loads in flight; strided
// passes want >= 128-byte row segments (T*16 B) even at one CTA per SM.
#ifndef PFCS_CUBER_512
#define PFCS_CUBER_512 7  // A/B hook: cube pass tile at M = 512 (1024^3)
#endif
#ifndef PFCS_CUBER_1024
#define PFCS_CUBER_1024 2  // A/B hook: cube pass tile at M = 1024 (2048^3)
#endif
#ifndef PFCS_STRIDED_2048
#define PFCS_STRIDED_2048 2  // A/B hook: strided y pass tile at N = 2048
#endif
constexpr int default_variant(int kind, int n) {
  // n: transform length (REALX / CUBER: the half length M)
  return kind == KIND_LINES   ? (n <= 256 ? 5 : (n == 512 ? 4 : 0))
       : kind == KIND_STRIDED ? (n <= 512 ? 3 : (n == 1024 ? 6 : (n == 2048 ? PFCS_STRIDED_2048 : 4)))
       : kind == KIND_REALX   ? (n == 256 ? 3 : (n <= 512 ? 7 : (n == 1024 ? 6 : (n == 2048 ? 5 : 4))))
       : kind == KIND_CUBER   ? (n <= 256 ? 3 : (n == 512 ? PFCS_CUBER_512 : (n == 1024 ? PFCS_CUBER_1024 : (n == 2048 ? 1 : 0))))
       : kind == KIND_CUBEC   ? (n <= 512 ? 3 : (n == 1024 ? 2 : (n == 2048 ? 1 : 0)))
       : /* KIND_PFCZ */        (n <= 256 ? 1 : 0);
}

int tune_variant(int kind, int n, int dflt);

template <int KIND, int N, class F>
int with_variant(F&& f) {
  constexpr int d = default_variant(KIND, N);
#ifdef PFCS_TUNE
  switch (tune_variant(KIND, N, d)) {
    case 0: return f(std::integral_constant<int, 0>{});
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    case 5: return f(std::integral_constant<int, 5>{});
    case 6: return f(std::integral_constant<int, 6>{});
    default: return f(std::integral_constant<int, 7>{});
  }
#else
  return f(std::integral_constant<int, d>{});
#endif
}

// As with_variant, for launches whose default tile is too coarse for the
// problem: when the default tile width would give fewer tiles than SMs
// (`tiles_at_tmin` = tiles at the minimum width), the narrowest,
// single-stage variant 0 runs instead, so small grids (the 2D 256^2 step)
// spread over the whole GPU.
constexpr long long SMALL_TILE_THRESHOLD = 148;
template <int KIND, int N, class F>
int with_variant_n(long long tiles_at_tmin, F&& f) {
#ifdef PFCS_TUNE
  (void)tiles_at_tmin;
  return with_variant<KIND, N>(f);
#else
  constexpr int d = default_variant(KIND, N);
  if constexpr ((d & 3) != 0) {
    if ((tiles_at_tmin >> (d & 3)) < SMALL_TILE_THRESHOLD) return f(std::integral_constant<int, 0>{});
  }
  return f(std::integral_constant<int, d>{});
#endif
}

// Balanced-slab split descriptor for a line of length n over g ranks.
struct SlabSplitH {
  int G, base, extra;
};
inline SlabSplitH slab_split(long long n, int g) {
  SlabSplitH s;
  s.G = g;
  s.base = (int)(n / g);
  s.extra = (int)(n % g);
  return s;
}

// Internal launchers (pfcs_c2c.cu)
int launch_lines_c2c(const double2* in, double2* out, long long nlines, int n, int g_in,
                     int g_out, bool forward, cudaStream_t st);
int launch_strided_c2c(const double2* in, double2* out, long long outer, int n, long long inner,
                       bool forward, cudaStream_t st);
int launch_strided_blocked(const double2* in, double2* out, long long outer, int n, long long inner, int g_in,
                           int g_out, bool forward, cudaStream_t st);
int launch_dft(const double2* in, double2* out, long long outer, int n, long long inner,
               bool forward, cudaStream_t st);
struct PeerTable;
int launch_lines_to(const double2* in, double2* out, long long nlines, int n, int g_in, int g_out,
                    const PeerTable* dst, bool forward, cudaStream_t st);
int launch_strided_to(const double2* in, long long outer, int n, long long inner, int g_in,
                      const PeerTable* dst, int g_outer, bool forward, cudaStream_t st);

}  // namespace pfcs
