// pfcs_internal.h — host-side helpers shared by the libpfcs translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

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

// Opt a kernel in to > 48 KB dynamic shared memory once.
int ensure_smem(const void* func, size_t bytes);

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
int launch_dft(const double2* in, double2* out, long long outer, int n, long long inner,
               bool forward, cudaStream_t st);

}  // namespace pfcs
