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
//                   with erfcx from a piecewise degree-10 table on [0, 6)
//                   (erfcx_table.cuh, 24 rows, rel. err 3.4e-16), libdevice beyond.
// Parity is still checked end to end against the reference (1e-10 / 1e-9).
#pragma once
#include <cuda_runtime.h>

#include "erfcx_table.cuh"

namespace slab {

// SLAB_MINIMAX: near-minimax polynomials of lower degree on the same reduced
// ranges (Chebyshev fits, tools/fit_minimax.py): exp to r^11, sin to r^13, cos
// to r^14, max relative error 1.2e-16 evaluated in double -- 4 fewer DFMA and 4
// fewer constants per (exp, sincos) than the Taylor forms.
#ifndef SLAB_MINIMAX
#define SLAB_MINIMAX 1  // cfg4 step 8.75 -> 8.62 ms (sweep 3.31 -> 3.25, aggregate 1.11 -> 1.07)
#endif
#if SLAB_MINIMAX
constexpr int kExpTerms = 12, kSinTerms = 6, kCosTerms = 8;
#else
constexpr int kExpTerms = 14, kSinTerms = 7, kCosTerms = 9;
#endif
// e^r on |r| <= ln2/2 (highest degree first; the last two are 1, 1), sin: P(z)
// with sin r = r + r z P(z); cos: 1 + z Q(z) (Q's coefficients then the 1)
__device__ __forceinline__ constexpr double exp_coef(int i) {
#if SLAB_MINIMAX
  constexpr double c[12] = {2.5100375832561234e-08, 2.7620075879983367e-07,
                            2.7557268480310024e-06, 2.4801521322368692e-05,
                            0.00019841269863040545, 0.0013888888917196719,
                            0.008333333333330065,   0.041666666666624164,
                            0.16666666666666669,    0.5000000000000001,
                            1.0,                    1.0};
#else
  constexpr double c[14] = {1.6059043836821613e-10, 2.08767569878681e-09,  2.505210838544172e-08,
                            2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05,
                            0.0001984126984126984,  0.001388888888888889,  0.008333333333333333,
                            0.041666666666666664,   0.16666666666666666,   0.5,
                            1.0,                    1.0};
#endif
  return c[i];
}
__device__ __forceinline__ constexpr double sin_coef(int i) {
#if SLAB_MINIMAX
  constexpr double c[6] = {1.5918129294866608e-10, -2.5051131845003624e-08, 2.755731610255244e-06,
                           -0.00019841269836758574, 0.008333333333330948, -0.16666666666666666};
#else
  constexpr double c[7] = {-7.647163731819816e-13, 1.6059043836821613e-10, -2.505210838544172e-08,
                           2.7557319223985893e-06, -0.0001984126984126984, 0.008333333333333333,
                           -0.16666666666666666};
#endif
  return c[i];
}
__device__ __forceinline__ constexpr double cos_coef(int i) {
#if SLAB_MINIMAX
  constexpr double c[8] = {-1.1367998654022494e-11, 2.0875886738047052e-09, -2.7557315566341895e-07,
                           2.480158729369346e-05,   -0.0013888888888880775, 0.04166666666666664,
                           -0.5,                    1.0};
#else
  constexpr double c[9] = {4.779477332387385e-14, -1.1470745597729725e-11, 2.08767569878681e-09,
                           -2.755731922398589e-07, 2.48015873015873e-05,   -0.001388888888888889,
                           0.041666666666666664,  -0.5,                    1.0};
#endif
  return c[i];
}

__device__ __forceinline__ double exp_neg(double t) {
  // t >= 700 (and +inf) returns 0
  const bool tiny = !(t < 700.0);
  t = tiny ? 0.0 : t;
  const double kL2e = 1.4426950408889634;
  const double kLn2Hi = 6.93147180369123816490e-01;  // 32 significant bits
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double n = rint(-t * kL2e);  // in [-1010, 0]
  double r = fma(n, -kLn2Hi, -t);
  r = fma(n, -kLn2Lo, r);
  double p = exp_coef(0);
#pragma unroll
  for (int i = 1; i < kExpTerms; ++i) p = fma(p, r, exp_coef(i));
  const long long e = tiny ? 0ll : (long long)((int)n + 1023) << 52;
  return p * __longlong_as_double(e);  // zero exponent factor: no branch around the polynomial
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
  double ps = sin_coef(0);
#pragma unroll
  for (int i = 1; i < kSinTerms; ++i) ps = fma(ps, z, sin_coef(i));
  const double sr = fma(ps * z, r, r);
  double pc = cos_coef(0);
#pragma unroll
  for (int i = 1; i < kCosTerms; ++i) pc = fma(pc, z, cos_coef(i));
  const double cr = pc;
  const int q = ((int)(long long)n) & 3;
  const double ss = (q & 1) ? cr : sr;
  const double cc = (q & 1) ? sr : cr;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}

// *_cb variants: the same polynomials with the constants in the constant bank.
// sm_100a DFMA takes no c[][] operand, so they are fetched with LDCU.128 into
// uniform registers (two constants per load instead of four UMOVs per literal
// pair).  Faster where registers are plentiful (fourier_aggregate: 1.59 ->
// 1.41 ms at cfg4); slower in the 128-register sweep, where the extra live
// values spill (4.75 -> 6.0 ms) -- hence both forms.
#if SLAB_MINIMAX
static __constant__ double kFmExp[kExpTerms + 2] = {
    2.5100375832561234e-08, 2.7620075879983367e-07, 2.7557268480310024e-06,
    2.4801521322368692e-05, 0.00019841269863040545, 0.0013888888917196719,
    0.008333333333330065,   0.041666666666624164,   0.16666666666666669,
    0.5000000000000001,     1.0,                    1.0,
    6.93147180369123816490e-01,  // ln2 hi (32 significant bits)
    1.90821492927058770002e-10,  // ln2 lo
};
static __constant__ double kFmSin[kSinTerms + 1] = {
    1.5918129294866608e-10, -2.5051131845003624e-08, 2.755731610255244e-06,
    -0.00019841269836758574, 0.008333333333330948,   -0.16666666666666666,
    0.6366197723675814,  // 2/pi
};
static __constant__ double kFmCos[kCosTerms + 3] = {
    -1.1367998654022494e-11, 2.0875886738047052e-09, -2.7557315566341895e-07,
    2.480158729369346e-05,   -0.0013888888888880775, 0.04166666666666664,
    -0.5,                    1.0,
    -1.5707963267948966,  // -pi/2 split in three
    -6.123233995736766e-17,  1.4973849048591698e-33,
};
#else
static __constant__ double kFmExp[kExpTerms + 2] = {
    1.6059043836821613e-10,  // 1/13!
    2.08767569878681e-09,  2.505210838544172e-08, 2.755731922398589e-07,
    2.7557319223985893e-06, 2.48015873015873e-05, 0.0001984126984126984,
    0.001388888888888889,  0.008333333333333333,  0.041666666666666664,
    0.16666666666666666,   0.5,                   1.0,
    1.0,
    6.93147180369123816490e-01,  // ln2 hi (32 significant bits)
    1.90821492927058770002e-10,  // ln2 lo
};
static __constant__ double kFmSin[kSinTerms + 1] = {
    -7.647163731819816e-13,  // -1/15!
    1.6059043836821613e-10, -2.505210838544172e-08, 2.7557319223985893e-06,
    -0.0001984126984126984, 0.008333333333333333,   -0.16666666666666666,
    0.6366197723675814,      // 2/pi
};
static __constant__ double kFmCos[kCosTerms + 3] = {
    4.779477332387385e-14,  // 1/16!
    -1.1470745597729725e-11, 2.08767569878681e-09, -2.755731922398589e-07,
    2.48015873015873e-05,    -0.001388888888888889, 0.041666666666666664,
    -0.5,                    1.0,
    -1.5707963267948966,     // -pi/2 split in three
    -6.123233995736766e-17,  1.4973849048591698e-33,
};
#endif

__device__ __forceinline__ double exp_neg_cb(double t) {
  // branch-free: t >= 700 (and +inf) returns 0 by zeroing the exponent factor
  const bool tiny = !(t < 700.0);
  t = tiny ? 0.0 : t;
  const double n = rint(-t * 1.4426950408889634);  // in [-1010, 0]
  double r = fma(n, -kFmExp[kExpTerms], -t);
  r = fma(n, -kFmExp[kExpTerms + 1], r);
  double p = kFmExp[0];
#pragma unroll
  for (int i = 1; i < kExpTerms; ++i) p = fma(p, r, kFmExp[i]);
  const long long e = tiny ? 0ll : (long long)((int)n + 1023) << 52;
  return p * __longlong_as_double(e);
}

// Branch-free.  The FMA reduction keeps ~1 ulp in r for |th| up to ~1e15 (the
// products n*P_i are exact inside the FMAs, th - n*P1 is exact by Sterbenz and
// pi/2 - (P1+P2+P3) ~ 1e-49); physical phases are |th| < 1e4.
__device__ __forceinline__ void sincos_fast_cb(double th, double* s, double* c) {
  const double n = rint(th * kFmSin[kSinTerms]);
  double r = fma(n, kFmCos[kCosTerms], th);
  r = fma(n, kFmCos[kCosTerms + 1], r);
  r = fma(n, kFmCos[kCosTerms + 2], r);
  const double z = r * r;
  double ps = kFmSin[0];
#pragma unroll
  for (int i = 1; i < kSinTerms; ++i) ps = fma(ps, z, kFmSin[i]);
  const double sr = fma(ps * z, r, r);
  double pc = kFmCos[0];
#pragma unroll
  for (int i = 1; i < kCosTerms; ++i) pc = fma(pc, z, kFmCos[i]);
  const double cr = pc;
  const int q = ((int)(long long)n) & 3;
  const double ss = (q & 1) ? cr : sr;
  const double cc = (q & 1) ? sr : cr;
  *s = (q & 2) ? -ss : ss;
  *c = ((q + 1) & 2) ? -cc : cc;
}

// tab: shared-memory copy of kErfcxCoef, coefficient-major (tab[k * NINT + i]):
// the lanes of a warp evaluate different intervals i, and with consecutive
// intervals in consecutive 8-byte words only rows 16 apart share a bank (pair
// distances put x = alpha r in ~14 adjacent rows of width 1/4, so most loads
// see no such collision).  Interval-major rows read as
// 16-byte pairs measured 5% slower on the pair kernel (8 lanes per LDS.128
// phase over 8 bank groups collide).
#ifndef SLAB_ERFC_CB
#define SLAB_ERFC_CB 1  // constant-bank exp in the pair kernel: 2.34 -> 2.27 ms at cfg4
#endif
// kTabOnly: the caller guarantees x < 6 (alpha r_c < 6): no branch around the
// table (the libdevice arm costs ~8 branch-control instructions per pair even
// when never taken)
template <bool kTabOnly = false>
__device__ __forceinline__ void erfc_gauss(double x, const double* __restrict__ tab,
                                           double* erfc_out, double* g_out) {
  const double hi = x * x;
  const double lo = fma(x, x, -hi);
#if SLAB_ERFC_CB
  double g = exp_neg_cb(hi);
#else
  double g = exp_neg(hi);
#endif
  g = fma(-lo, g, g);  // e^{-(hi+lo)} = e^{-hi} (1 - lo)
  double ex;
  if (kTabOnly || x < SLAB_ERFCX_NINT / SLAB_ERFCX_INV_W) {
    const int i = (int)(x * SLAB_ERFCX_INV_W);
    const double u = fma(2.0 * SLAB_ERFCX_INV_W, x, -(double)(2 * i + 1));
    const double* cf = tab + i;
    ex = cf[(SLAB_ERFCX_NCOEF - 1) * SLAB_ERFCX_NINT];
#pragma unroll
    for (int k = SLAB_ERFCX_NCOEF - 2; k >= 0; --k) ex = fma(ex, u, cf[k * SLAB_ERFCX_NINT]);
  } else {
    ex = erfcx(x);
  }
  *erfc_out = ex * g;
  *g_out = g;
}

// erfcx(x) on [0, 6] with no table: one degree-19 polynomial in the rational
// map u = (7/3 x - 4) / (x + 4) (= (t + 0.4) / 0.6, t = (x - 4)/(x + 4)), max
// relative error 6e-16 (tools/gen_erfcx_rational.py).  Every lane uses the same
// coefficients, so they come from uniform registers / the constant bank -- a
// per-lane table in shared memory costs >= 2 wavefronts per coefficient load,
// which made the table forms of this kernel shared-memory bound.
__device__ __forceinline__ double rcp_fast(double x) {  // 1/x, x normal > 0, ~1 ulp
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// constant bank: LDCU.128 brings two coefficients into uniform registers per
// instruction (literals cost two UMOVs each, re-issued for every pair)
static __constant__ __align__(16) double kErfcxRat[20] = {
    2.89722116323464229e-01,  -3.30725380025229221e-01, 2.07401177991509089e-01,
    -1.06646031140752912e-01, 4.50108550943799507e-02,  -1.54181897135370650e-02,
    4.16094898189511321e-03,  -8.24498405499286065e-04, 9.61294917405419497e-05,
    2.04972504298114117e-06,  -2.99897570926783762e-06, 3.49340377437571895e-07,
    5.58422862486972409e-08,  -1.64955693655007643e-08, -8.63453257340785243e-10,
    6.39416928898986440e-10,  1.46431537907270747e-11,  -2.48249270445082579e-11,
    -4.86601666694534958e-13, 8.44604731366168551e-13};

__device__ __forceinline__ double erfcx_rat(double x) {
  const double u = fma(7.0 / 3.0, x, -4.0) * rcp_fast(x + 4.0);
  double p = kErfcxRat[19];
#pragma unroll
  for (int j = 18; j >= 0; --j) p = fma(p, u, kErfcxRat[j]);
  return p;
}

constexpr double kErfcxRatMax = 6.0;

// erfc(x) and e^{-x^2} sharing one exp (as fastmath.cuh's erfc_gauss)
template <bool kTabOnly>
__device__ __forceinline__ void erfc_gauss_rat(double x, double* erfc_out, double* g_out) {
  const double hi = x * x;
  const double lo = fma(x, x, -hi);
  double g = exp_neg_cb(hi);
  g = fma(-lo, g, g);
  const double ex = (kTabOnly || x <= kErfcxRatMax) ? erfcx_rat(x) : erfcx(x);
  *erfc_out = ex * g;
  *g_out = g;
}

constexpr int kErfcxTabSize = SLAB_ERFCX_NINT * SLAB_ERFCX_NCOEF;

__device__ __forceinline__ void load_erfcx_table(double* tab) {
  for (int e = threadIdx.x; e < kErfcxTabSize; e += blockDim.x) {
    const int i = e / SLAB_ERFCX_NCOEF, k = e - i * SLAB_ERFCX_NCOEF;
    tab[k * SLAB_ERFCX_NINT + i] = kErfcxCoef[e];
  }
}

}  // namespace slab
