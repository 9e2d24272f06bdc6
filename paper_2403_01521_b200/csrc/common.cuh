// common.cuh -- shared helpers for the sm_100a slab-Ewald kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fastmath.cuh"

#define SLAB_CUDA_CHECK(expr)                              \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return slab_record_cuda(_e);    \
  } while (0)

// Checked build (make variant NAME=checked DEFS=-DSLAB_CHECKED): device-side bounds
// asserts on the arena indexing of the hot kernels (compute-sanitizer is not
// available on this pool); a violation prints its site and traps.
#ifdef SLAB_CHECKED
#include <cstdio>
#define SLAB_BOUND(i, n)                                                               \
  do {                                                                                 \
    if ((unsigned long long)(i) >= (unsigned long long)(n)) {                          \
      printf("slab bound violated %s:%d: %lld >= %lld\n", __FILE__, __LINE__,           \
             (long long)(i), (long long)(n));                                          \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define SLAB_BOUND(i, n) ((void)0)
#endif

namespace slab {

constexpr double kPi = 3.141592653589793;
constexpr double kSqrtPi = 1.7724538509055159;        // np.sqrt(np.pi)
constexpr double kTwoOverSqrtPi = 2.0 / 1.7724538509055159;
constexpr double kSingularTol = 2e-6;                 // reference soe.py:49
constexpr int kMaxPairs = 12;                         // M <= 24 SOE terms
constexpr int SLAB_STATUS_COINCIDENT_DEV = 1;         // mirrors SLAB_STATUS_* in the C ABI
constexpr int SLAB_STATUS_SINGULAR_DEV = 2;
constexpr int SLAB_STATUS_NBR_OVERFLOW_DEV = 4;
constexpr int SLAB_STATUS_NONFINITE_DEV = 8;          // a z coordinate is NaN / inf
constexpr int SLAB_STATUS_WALL_DEV = 16;              // a particle at or beyond a wall (md.py:72)

// Per-mode coefficient record (doubles), built by mode_table_kernel.
//   [0]=kx [1]=ky [2]=|k| [3]=ck=(pi/A)C_t/k [4]=cz=(pi/A)C_t [5]=kappa (real)
//   [6]=singular flag (0/1) [7]=unused
//   [8 + 2l .. ]        C_l  = 2 c_l           (re, im), l < Mh
//   [8 + 2Mh + 2l .. ]  CB_l = 2 c_l b_l       (re, im)
__host__ __device__ constexpr int mode_stride(int mh) { return 8 + 4 * mh; }

struct C2 {
  double re, im;
};
__device__ __forceinline__ C2 cmul(C2 a, C2 b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
__device__ __forceinline__ C2 cexp_neg(double xr, double xi) {
  // exp(-(xr + i xi)) for xr >= 0 (every caller: Re(b) > 0 times a z distance >= 0)
  const double e = exp_neg(xr);
  double s, c;
  sincos_fast(xi, &s, &c);
  return {e * c, -e * s};
}

// order-preserving uint64 image of a double, with -0.0 folded onto +0.0 so that
// the radix order equals the reference comparison order (core.py:196 uses '>').
__device__ __forceinline__ uint64_t z_key(double z) {
  if (z == 0.0) z = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(z);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace slab

// error bookkeeping shared by every C-ABI entry point (capi.cu)
int slab_record_cuda(cudaError_t e);
