// fastmath.cuh -- branch-light fp64 transcendentals for the hot loops.
//
// B200 has no fp64 SFU, so libdevice's exp / sincos / erfcx are long FMA
// sequences wrapped in special-case handling (profiled: sincos ~85, exp ~54,
// erfcx ~100 instructions per call in the sweep / pair kernels).  The hot
// loops only ever see a restricted domain, so these keep the ~1 ulp accuracy
// and drop the generality:
//   exp_neg(t)      e^{-t} for t >= 0 (0 beyond t = 700): Cody-Waite ln2 split,
//                   degree-13 Taylor on |r| <= ln2/2, exponent built directly.
//   sincos_fast(th) 3-constant FMA Cody-Waite reduction by pi/2 (|th| < 1e15),
//                   degree-15/16 Taylor on |r| <= pi/4.
//   erfc_gauss(x)   erfc(x) and e^{-x^2} for x >= 0 sharing one exp: e^{-x^2}
//                   with the exact x^2 = hi + lo split, erfc = erfcx * e^{-x^2}
//                   with erfcx from a piecewise degree-14 table on [0, 6)
//                   (erfcx_table.cuh, rel. err 2e-16), libdevice beyond.
// Parity is still checked end to end against the reference (1e-10 / 1e-9).
#pragma once
#include <cuda_runtime.h>

#include "erfcx_table.cuh"

namespace slab {

__device__ __forceinline__ double exp_neg(double t) {
  // branch-free: t >= 700 (and +inf) returns 0 through the final select
  const bool tiny = !(t < 700.0);
  t = tiny ? 0.0 : t;
  const double kL2e = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;  // 32 significant bits
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double n = rint(-t * kL2e);  // in [-1010, 0]
  double r = fma(n, -kLn2Hi, -t);
  r = fma(n, -kLn2Lo, r);
  double p = 1.6059043836821613e-10;  // 1/13!
  p = fma(p, r, 2.08767569878681e-09);
  p = fma(p, r, 2.505210838544172e-08);
  p = fma(p, r, 2.755731922398589e-07);
  p = fma(p, r, 2.7557319223985893e-06);
  p = fma(p, r, 2.48015873015873e-05);
  p = fma(p, r, 0.0001984126984126984);
  p = fma(p, r, 0.001388888888888889);
  p = fma(p, r, 0.008333333333333333);
  p = fma(p, r, 0.041666666666666664);
  p = fma(p, r, 0.16666666666666666);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const long long e = (long long)((int)n + 1023) << 52;
  return tiny ? 0.0 : p * __longlong_as_double(e);
}

// Branch-free.  The FMA reduction keeps ~1 ulp in r for |th| up to ~1e15 (the
// products n*P_i are exact inside the FMAs, th - n*P1 is exact by Sterbenz and
// pi/2 - (P1+P2+P3) ~ 1e-49); physical phases are |th| < 1e4.
__device__ __forceinline__ void sincos_fast(double th, double* s, double* c) {
  const double n = rint(th * 0.6366197723675814);
  double r = fma(n, -1.5707963267948966, th);
  r = fma(n, -6.123233995736766e-17, r);
  r = fma(n, 1.4973849048591698e-33, r);
  const double z = r * r;
  double ps = -7.647163731819816e-13;  // -1/15!
  ps = fma(ps, z, 1.6059043836821613e-10);
  ps = fma(ps, z, -2.505210838544172e-08);
  ps = fma(ps, z, 2.7557319223985893e-06);
  ps = fma(ps, z, -0.0001984126984126984);
  ps = fma(ps, z, 0.008333333333333333);
  ps = fma(ps, z, -0.16666666666666666);
  const double sr = fma(ps * z, r, r);
  double pc = 4.779477332387385e-14;  // 1/16!
  pc = fma(pc, z, -1.1470745597729725e-11);
  pc = fma(pc, z, 2.08767569878681e-09);
  pc = fma(pc, z, -2.755731922398589e-07);
  pc = fma(pc, z, 2.48015873015873e-05);
  pc = fma(pc, z, -0.001388888888888889);
  pc = fma(pc, z, 0.041666666666666664);
  pc = fma(pc, z, -0.5);
  const double cr = fma(pc, z, 1.0);
  const int q = ((int)(long long)n) & 3;
  const double ss = (q & 1) ? cr : sr;
  const double cc = (q & 1) ? sr : cr;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}

// tab: shared-memory copy of kErfcxCoef with row stride 17 (bank-conflict free)
constexpr int kErfcxStride = 17;

__device__ __forceinline__ void erfc_gauss(double x, const double* __restrict__ tab,
                                           double* erfc_out, double* g_out) {
  const double hi = x * x;
  const double lo = fma(x, x, -hi);
  double g = exp_neg(hi);
  g = fma(-lo, g, g);  // e^{-(hi+lo)} = e^{-hi} (1 - lo)
  double ex;
  if (x < 6.0) {
    const int i = (int)(x * 2.0);
    const double u = fma(4.0, x, -(double)(2 * i + 1));
    const double* cf = tab + i * kErfcxStride;
    ex = cf[SLAB_ERFCX_NCOEF - 1];
#pragma unroll
    for (int k = SLAB_ERFCX_NCOEF - 2; k >= 0; --k) ex = fma(ex, u, cf[k]);
  } else {
    ex = erfcx(x);
  }
  *erfc_out = ex * g;
  *g_out = g;
}

__device__ __forceinline__ void load_erfcx_table(double* tab) {
  for (int e = threadIdx.x; e < SLAB_ERFCX_NINT * SLAB_ERFCX_NCOEF; e += blockDim.x) {
    const int i = e / SLAB_ERFCX_NCOEF, k = e - i * SLAB_ERFCX_NCOEF;
    tab[i * kErfcxStride + k] = kErfcxCoef[e];
  }
}

}  // namespace slab
