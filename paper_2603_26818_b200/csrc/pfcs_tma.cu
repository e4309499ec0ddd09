// pfcs_tma.cu — TMA-staged strided line pass (sm_100a bulk tensor copies).
//
// Same transform as k_strided (pfcs_c2c.cu) for the plain (unblocked) layout
// data[o][y][i], lines along y with the contiguous i extent tiled T at a
// time: reference path fftcore.fft_2d axis-1 stage (fftcore.py:43-45) inside
// distfft.dist_fft_forward/inverse (distfft.py:150-173).
//
// Instead of register-pipelined loads, one thread arms an mbarrier and issues
// cp.async.bulk.tensor.3d copies of the NEXT tile (N rows x T*16 bytes) into
// a second shared-memory stage while the CTA transforms the current one, so
// the in-flight HBM data costs no registers and no load instructions.  The
// stage is read into registers in the exact order k_strided loads them and
// the FFT code is shared, so results are bit-identical to k_strided.
#include "pfcs_internal.h"
#include "pfcs_pro.cuh"
#include "pfcs_tma.cuh"

namespace pfcs {

template <int N, int T>
struct TmaCfg {
  static constexpr int R = radix_R(N);
  static constexpr int P = N / R;
  static constexpr int LS = tile_ls(N, T, true);
  static constexpr int BR = N < 256 ? N : 256;  // rows per TMA box (box dims <= 256)
  static constexpr int NB = N / BR;
  static constexpr unsigned STAGE = (unsigned)N * T * 16u;  // bytes per stage
  // two stages + FFT workspace + 2 mbarriers (+ the twiddle table), plus
  // alignment slack
  static constexpr size_t BASE = 2 * (size_t)STAGE + (size_t)T * LS * 16 + 16 + 1024;
  static constexpr bool TSM = PFCS_Y_TWSMEM && BASE + (size_t)N * 16 <= 227 * 1024;
  static constexpr size_t SMEM = BASE + (TSM ? (size_t)N * 16 : 0);
};

// OPEER: outer row o goes to tout.p[h][(o - ooff_h) ...] (the fused
// transpose of the slab pipeline: souter splits the outer axis over ranks).
// PRO: pointwise prologue (pfcs_pro.cuh) on each element read from the stage.
template <int N, int T, bool FWD, bool OPEER = false, bool PRO = false>
__global__ void __launch_bounds__(T*(N / radix_R(N)), 1)
    k_strided_tma(const __grid_constant__ CUtensorMap map, double2* out, i64 outer, i64 inner, i64 tpo,
                  const double2* __restrict__ tw, double scale, SlabSplit souter = SlabSplit{},
                  PeerTable tout = PeerTable{}, Pro pro = Pro{}) {
  using C = TmaCfg<N, T>;
  constexpr int R = C::R;
  constexpr int P = C::P;
  extern __shared__ unsigned char sraw[];
  // 1024-byte aligned stages (TMA destinations), then the workspace, then bars
  unsigned char* base = sraw + ((1024u - (smem_u32(sraw) & 1023u)) & 1023u);
  double2* stage0 = (double2*)base;
  double2* stage1 = stage0 + (size_t)N * T;
  double2* ws = stage1 + (size_t)N * T;
  unsigned long long* bars = (unsigned long long*)(ws + (size_t)T * C::LS);
  // twiddle table copy (C::TSM, A/B only): L1 holds only what the ~200 KB of
  // shared memory leave and 1024-point lines miss it on a quarter of the
  // loads, but the pass is bound by shared-memory instruction issue
  // (mio_throttle), so moving the loads there made it slower
  double2* tws = (double2*)(bars + 2);
  if constexpr (C::TSM) {
    for (int k = threadIdx.x; k < N; k += blockDim.x) tws[k] = tw[k];
  }
  const double2* twp = C::TSM ? (const double2*)tws : tw;

  const int tid = threadIdx.x;
  const int t = tid % T;
  const int j = tid / T;
  double2* sl = ws + t * C::LS;
  const i64 ntiles = outer * tpo;

  auto issue = [&](i64 tile, int s) {
    const i64 o = tile / tpo;
    const int i0 = (int)((tile - o * tpo) * T);
    double2* dst = s ? stage1 : stage0;
    mbar_expect_tx(&bars[s], C::STAGE);
#pragma unroll
    for (int b = 0; b < C::NB; ++b) tma_load_3d(dst + (size_t)b * C::BR * T, &map, &bars[s], 2 * i0, b * C::BR, (int)o);
  };

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  i64 tile = blockIdx.x;
  if (tid == 0 && tile < ntiles) issue(tile, 0);
  // PRO_DERIV along the line: the multipliers of this thread's elements are
  // the same in every tile
  double dline[PRO ? R : 1];
  if constexpr (PRO) {
#pragma unroll
    for (int e = 0; e < R; ++e)
      dline[e] = (pro.kind == PRO_DERIV && pro.axis == pro.pass) ? __ldg((const double*)pro.aux + j + P * e) : 0.0;
  }
  for (int it = 0; tile < ntiles; ++it, tile += gridDim.x) {
    const int s = it & 1;
    if (tid == 0) {
      const i64 nx = tile + gridDim.x;
      if (nx < ntiles) {
        fence_proxy_async();  // stage s^1 was read by every thread before the last barrier
        issue(nx, s ^ 1);
      }
    }
    mbar_wait(&bars[s], (unsigned)((it >> 1) & 1));
    const double2* src = s ? stage1 : stage0;
    double2 v[R];
#pragma unroll
    for (int e = 0; e < R; ++e) v[e] = src[(j + P * e) * T + t];
    const i64 o = tile / tpo;
    const i64 i = (tile - o * tpo) * T + t;
    const int jj = opaque(j);
    if constexpr (PRO) {
      if (i < inner) {
        // element (o, n, i) of the (outer, N, inner) view of the (n0, n1, n2)
        // grid.  PRO_DERIV: the multiplier's coordinate is n itself when it
        // runs along the line, else fixed for the thread's column — decoded
        // once per tile (a per-element 64-bit decode made the y pass with
        // an x / y derivative 1.5-2x slower than the plain pass)
        if (pro.kind == PRO_DERIV) {  // i d[c] v, apply_pro's arithmetic
          const i64 cfix = pro.pass == 1 ? (pro.axis == 0 ? o : i) : (pro.axis == 1 ? i / pro.n2 : i % pro.n2);
          const double dfix = pro.axis == pro.pass ? 0.0 : __ldg((const double*)pro.aux + cfix);
#pragma unroll
          for (int e = 0; e < R; ++e) {
            const double dk = pro.axis == pro.pass ? dline[e] : dfix;
            v[e] = make_double2(-__dmul_rn(dk, v[e].y), __dmul_rn(dk, v[e].x));
          }
        } else {
#pragma unroll
          for (int e = 0; e < R; ++e) v[e] = apply_pro(pro, v[e], (o * N + jj + P * e) * inner + i, 0);
        }
      }
    }
    fft_line<N, FWD, 1, PFCS_Y_TWL, R, C::TSM>(v, jj, sl, twp);
    if (i < inner) {
      double2* dst;
      if constexpr (OPEER) {
        int h, ooff, co;
        souter.locate3((int)o, h, ooff, co);
        dst = tout.p[h] + (o - ooff) * (i64)N * inner + i;
      } else {
        dst = out + o * (i64)N * inner + i;
      }
#pragma unroll
      for (int e = 0; e < R; ++e) {
        double2 x = v[e];
        if (!FWD) x = make_double2(x.x * scale, x.y * scale);
        dst[(i64)(jj + P * e) * inner] = x;
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ host ----
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn();

// Tiled FLOAT64 tensor map (rank <= 3); false when the driver rejects it or
// the entry point is unavailable (callers then take the non-TMA kernels).
bool make_tmap(CUtensorMap* map, int rank, const void* base, const unsigned long long* dims,
               const unsigned long long* strides_bytes, const unsigned* box, int swizzle_bytes) {
  EncodeTiledFn enc = encode_fn();
  if (!enc || ((uintptr_t)base & 15)) return false;
  cuuint64_t d[3], s[2];
  cuuint32_t b[3], e[3] = {1, 1, 1};
  for (int k = 0; k < rank; ++k) {
    d[k] = dims[k];
    b[k] = box[k];
    if (k + 1 < rank) s[k] = strides_bytes[k];
  }
  const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : swizzle_bytes == 64  ? CU_TENSOR_MAP_SWIZZLE_64B
                                : swizzle_bytes == 32  ? CU_TENSOR_MAP_SWIZZLE_32B
                                                       : CU_TENSOR_MAP_SWIZZLE_NONE;
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, (void*)base, d, s, b, e,
             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// On by default (B200 A/B: 512^3 y pass 0.469 -> 0.385 ms, 1024^3 4.36 ->
// 3.83 ms); PFCS_TMA=0 selects the register-pipelined k_strided.
bool tma_enabled() {
  static const bool on = [] {
    const char* v = getenv("PFCS_TMA");
    return !(v && *v && atoi(v) == 0);
  }();
  return on;
}

static int tma_tile_width(int dflt) {
  const char* v = getenv("PFCS_TMA_T");
  if (!v || !*v) return dflt;
  const int t = atoi(v);
  return (t == 1 || t == 2 || t == 4 || t == 8) ? t : dflt;
}

template <int N, int T, bool FWD>
static int strided_tma_nt(const double2* in, double2* out, i64 outer, i64 inner, cudaStream_t st,
                          const SlabSplitH* souter = nullptr, const PeerTable* dst = nullptr,
                          const Pro* pro = nullptr) {
  using C = TmaCfg<N, T>;
  if constexpr (C::SMEM > 227 * 1024 || T * C::P > 1024) {
    return 1;  // not applicable
  } else {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return 1;
    CUtensorMap map;
    const cuuint64_t dims[3] = {(cuuint64_t)(2 * inner), (cuuint64_t)N, (cuuint64_t)outer};
    const cuuint64_t strides[2] = {(cuuint64_t)inner * 16, (cuuint64_t)inner * 16 * N};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * T), (cuuint32_t)C::BR, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)in, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 1;
    const double2* tw = twiddles(N);
    if (!tw) return PFCS_E_CUDA;
    const i64 tpo = (inner + T - 1) / T;
    int grid = 0;
    if (pro) {
      if (int rc = persistent_grid((const void*)k_strided_tma<N, T, FWD, false, true>, T * C::P, C::SMEM,
                                   outer * tpo, &grid))
        return rc;
      k_strided_tma<N, T, FWD, false, true><<<grid, T * C::P, C::SMEM, st>>>(
          map, out, outer, inner, tpo, tw, 1.0 / (double)N, SlabSplit{}, PeerTable{}, *pro);
      return check_launch("k_strided_tma(pro)");
    }
    if (dst) {
      const SlabSplit so{souter->G, souter->base, souter->extra};
      if (int rc = persistent_grid((const void*)k_strided_tma<N, T, FWD, true>, T * C::P, C::SMEM, outer * tpo, &grid))
        return rc;
      k_strided_tma<N, T, FWD, true><<<grid, T * C::P, C::SMEM, st>>>(map, nullptr, outer, inner, tpo, tw,
                                                                      1.0 / (double)N, so, *dst);
      return check_launch("k_strided_tma(peer)");
    }
    if (int rc = persistent_grid((const void*)k_strided_tma<N, T, FWD>, T * C::P, C::SMEM, outer * tpo, &grid))
      return rc;
    k_strided_tma<N, T, FWD><<<grid, T * C::P, C::SMEM, st>>>(map, out, outer, inner, tpo, tw, 1.0 / (double)N);
    return check_launch("k_strided_tma");
  }
}

template <int N, bool FWD>
static int strided_tma_n(const double2* in, double2* out, i64 outer, i64 inner, cudaStream_t st,
                         const SlabSplitH* so = nullptr, const PeerTable* dst = nullptr, const Pro* pro = nullptr) {
  switch (tma_tile_width(N >= 1024 ? 4 : 8)) {
    case 1: return strided_tma_nt<N, 1, FWD>(in, out, outer, inner, st, so, dst, pro);
    case 2: return strided_tma_nt<N, 2, FWD>(in, out, outer, inner, st, so, dst, pro);
    case 4: return strided_tma_nt<N, 4, FWD>(in, out, outer, inner, st, so, dst, pro);
    default: return strided_tma_nt<N, 8, FWD>(in, out, outer, inner, st, so, dst, pro);
  }
}

// Returns PFCS_OK / an error code, or 1 when the TMA path does not apply
// (the caller then runs k_strided).
int launch_strided_tma(const double2* in, double2* out, long long outer, int n, long long inner, bool forward,
                       cudaStream_t st, const SlabSplitH* souter, const PeerTable* dst, const Pro* pro) {
  if (((uintptr_t)in & 15) || inner < 1 || 2 * inner >= (1LL << 31) || outer >= (1LL << 31)) return 1;
  switch (n) {
#define PFCS_TMA_CASE(NN)                                                            \
  case NN:                                                                           \
    return forward ? strided_tma_n<NN, true>(in, out, outer, inner, st, souter, dst, pro) \
                   : strided_tma_n<NN, false>(in, out, outer, inner, st, souter, dst, pro);
    PFCS_TMA_CASE(64)
    PFCS_TMA_CASE(128)
    PFCS_TMA_CASE(256)
    PFCS_TMA_CASE(512)
    PFCS_TMA_CASE(1024)
    PFCS_TMA_CASE(2048)
#undef PFCS_TMA_CASE
    default:
      return 1;
  }
}

}  // namespace pfcs
