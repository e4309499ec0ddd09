// TMA row-width probe: how fast can a persistent kernel stream an
// (outer, N, inner) complex128 array through shared memory when each TMA
// box row is T*16 bytes (T adjacent inner columns) — the access pattern of
// the strided y passes and the x passes.  Copies in place (load box, store
// box back), no arithmetic.  Usage: tma_rows <T> [outer N inner]
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../paper_2603_26818_b200/csrc/pfcs_tma.cuh"

using namespace pfcs;
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ void st3(const CUtensorMap* m, const void* src, int a, int b, int c) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   (unsigned long long)m), "r"(smem_u32(src)), "r"(a), "r"(b), "r"(c) : "memory");
}

// one thread per CTA moves boxes of ROWS rows; NBUF buffers in flight
template <int T, int ROWS, int NBUF>
__global__ void k_probe(const __grid_constant__ CUtensorMap map, long long outer, long long tpo, int nrow_boxes,
                        int store, int grp) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ unsigned long long bar[NBUF];
  const unsigned bytes = ROWS * T * 16;
  if (threadIdx.x != 0) return;
  for (int i = 0; i < NBUF; ++i) mbar_init(&bar[i], 1);
  mbar_fence_init();
  const long long nboxes = outer * tpo * nrow_boxes;
  long long k = 0;
  unsigned ph[NBUF] = {0};
  // box enumeration: (o, tile, rb) with `grp` adjacent column tiles kept on
  // one CTA back to back (same rows, neighbouring 16T-byte segments)
  auto decode = [&](long long q, long long& o, int& tile, int& rb) {
    const long long g = q / grp, w = q % grp;  // group g, member w
    const long long per_o = (tpo / grp) * nrow_boxes;
    o = g / per_o;
    const long long rem = g % per_o;
    rb = (int)(rem % nrow_boxes);
    tile = (int)((rem / nrow_boxes) * grp + w);
  };
  const long long ngroups = nboxes / grp;
  for (long long b = 0; b < nboxes; ++k) {
    // CTA-major: CTA c takes groups c, c + grid, ... (each group = grp boxes)
    const long long gi = blockIdx.x + (k / grp) * gridDim.x;
    if (gi >= ngroups) break;
    b = gi * grp + (k % grp);
    const int s = (int)(k % NBUF);
    if (k >= NBUF) {  // buffer s: wait for its load, store it back
      mbar_wait(&bar[s], ph[s]);
      ph[s] ^= 1;
      const long long kk = k - NBUF;
      const long long pb = (blockIdx.x + (kk / grp) * gridDim.x) * grp + (kk % grp);
      long long o; int tile, rb;
      decode(pb, o, tile, rb);
      if (store) {
        fence_proxy_async();
        st3(&map, base + (size_t)s * bytes, 2 * T * tile, rb * ROWS, (int)o);
        bulk_commit();
        bulk_wait_read0();
      }
    }
    long long o; int tile, rb;
    decode(b, o, tile, rb);
    mbar_expect_tx(&bar[s], bytes);
    tma_load_3d(base + (size_t)s * bytes, &map, &bar[s], 2 * T * tile, rb * ROWS, (int)o);
  }
  for (int s = 0; s < NBUF; ++s) {
    if (k > s) { mbar_wait(&bar[(k - 1 - s) % NBUF], ph[(k - 1 - s) % NBUF]); }
  }
  bulk_wait0();
}

template <int T>
static void run(long long outer, long long N, long long inner, int store, int grp = 1) {
  constexpr int ROWS = 256, NBUF = 6;
  double2* d;
  const size_t bytes = (size_t)outer * N * inner * 16;
  cudaMalloc(&d, bytes);
  cudaMemset(d, 0, bytes);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[3] = {(cuuint64_t)(2 * inner), (cuuint64_t)N, (cuuint64_t)outer};
  cuuint64_t str[2] = {(cuuint64_t)inner * 16, (cuuint64_t)inner * 16 * N};
  cuuint32_t box[3] = {2 * T, ROWS, 1}, e[3] = {1, 1, 1};
  ((Enc)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = (size_t)NBUF * ROWS * T * 16 + 1024;
  cudaFuncSetAttribute(k_probe<T, ROWS, NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_probe<T, ROWS, NBUF>, 32, smem);
  const long long tpo = inner / T;
  const int grid = 148 * per;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) k_probe<T, ROWS, NBUF><<<grid, 32, smem>>>(map, outer, tpo, (int)(N / ROWS), store, grp);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) k_probe<T, ROWS, NBUF><<<grid, 32, smem>>>(map, outer, tpo, (int)(N / ROWS), store, grp);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double moved = (double)bytes * (store ? 2 : 1);
  printf("grp=%d T=%2d (%3d-byte rows) %s: %.3f ms  %.1f GB/s  (%d CTAs/SM, err=%s)\n", grp, T, T * 16,
         store ? "load+store" : "load only ", ms, moved / (ms * 1e-3) / 1e9, per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main(int argc, char** argv) {
  long long outer = 513, N = 1024, inner = 1024;
  for (int store = 0; store < 2; ++store) {
    run<4>(outer, N, inner, store, 1);
    run<4>(outer, N, inner, store, 2);
    run<4>(outer, N, inner, store, 4);
    run<8>(outer, N, inner, store, 1);
    run<8>(outer, N, inner, store, 2);
  }
  return 0;
}
