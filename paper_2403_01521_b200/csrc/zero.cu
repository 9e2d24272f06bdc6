// zero.cu -- the k = 0 (in-plane averaged) mode on device.
//
// Replaces reference soewald2d.py:211-296 (_zero_mode_soe_sweep).  The code's
// kernel split G(z) = z - z erfc_SOE(a z) + g_SOE(z)/(a sqrt(pi)) (docstring
// soewald2d.py:22-27) gives, per SOE pair l (conjugate partner folded in as
// 2 Re(.)), with REAL input q:
//   A_{l,a} = sum_{j<a} q_j e^{-b_l (z_a - z_j)}
//   B_{l,a} = sum_{j<a} q_j (z_a - z_j) e^{-b_l (z_a - z_j)}
//   S0_a = sum_{j<a} q_j,  S1_a = sum_{j<a} q_j z_j
//   u_pair = sum q_a (z_a S0 - S1) - (2/sqrt pi) sum q_a Re sum (w/s) B
//            + 1/(alpha sqrt pi) sum q_a Re sum w A                    (soewald2d.py:249)
//   fz_a  += S0 - (2/sqrt pi) Re sum [(w/s + w s/2) A - alpha w B]   (forward, 264-277)
//   fz_a  -= suffix mirror                                             (backward, 282-295)
// Same 3-phase chunked scan as the Fourier path, one thread per (chunk, dir);
// (A, B) compose as the affine pair  A' = D A + X_A,  B' = D (B + dz A) + X_B.
#include "common.cuh"
#include "kernels.cuh"

namespace slab {

template <int MH>
__global__ void zero_aggregate_kernel(const double* __restrict__ zs, const double* __restrict__ qs,
                                      const double2* __restrict__ dtab, int64_t n, int R, int nch,
                                      double2* __restrict__ zagg) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * nch) return;
  const int c = e >> 1, dir = e & 1;
  const int64_t a0 = (int64_t)c * R, a1 = a0 + R < n ? a0 + R : n;
  C2 TA[MH], TB[MH];
#pragma unroll
  for (int l = 0; l < MH; ++l) TA[l] = TB[l] = C2{0.0, 0.0};
  double S0 = 0.0, S1 = 0.0;
  for (int64_t s = 0; s < a1 - a0; ++s) {
    const int64_t a = dir == 0 ? a0 + s : a1 - 1 - s;
    const double q = qs[a];
    if (s > 0) {
      const int64_t ad = dir == 0 ? a : a + 1;           // decay row
      const double dz = zs[ad] - zs[ad - 1];
#pragma unroll
      for (int l = 0; l < MH; ++l) {
        const double2 d = dtab[ad * MH + l];
        C2 bt{fma(dz, TA[l].re, TB[l].re), fma(dz, TA[l].im, TB[l].im)};
        TB[l] = cmul(bt, C2{d.x, d.y});
        TA[l] = cmul(TA[l], C2{d.x, d.y});
      }
    }
#pragma unroll
    for (int l = 0; l < MH; ++l) TA[l].re += q;
    S0 += q;
    S1 = fma(q, zs[a], S1);
  }
  double2* out = zagg + ((size_t)c * 2 + dir) * (2 * MH + 1);
#pragma unroll
  for (int l = 0; l < MH; ++l) {
    out[l] = make_double2(TA[l].re, TA[l].im);
    out[MH + l] = make_double2(TB[l].re, TB[l].im);
  }
  out[2 * MH] = make_double2(S0, S1);
}

// in-place: aggregates -> carried-in states.  thread per (dir, pair) + (dir, S)
template <int MH>
__global__ void zero_carry_kernel(const double* __restrict__ zs, int64_t n, int R, int nch,
                                  BVec b, double2* __restrict__ zagg) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * (MH + 1)) return;
  const int dir = e / (MH + 1), l = e % (MH + 1);
  const size_t rec = 2 * MH + 1;
  if (l == MH) {  // plain prefix / suffix sums of q and q z
    double S0 = 0.0, S1 = 0.0;
    for (int s = 0; s < nch; ++s) {
      const int c = dir == 0 ? s : nch - 1 - s;
      double2* p = zagg + ((size_t)c * 2 + dir) * rec + 2 * MH;
      const double2 X = *p;
      *p = make_double2(S0, S1);
      S0 += X.x;
      S1 += X.y;
    }
    return;
  }
  C2 TA{0.0, 0.0}, TB{0.0, 0.0};
  for (int s = 0; s < nch; ++s) {
    const int c = dir == 0 ? s : nch - 1 - s;
    double2* p = zagg + ((size_t)c * 2 + dir) * rec;
    const double2 XA = p[l], XB = p[MH + l];
    p[l] = make_double2(TA.re, TA.im);
    p[MH + l] = make_double2(TB.re, TB.im);
    const int64_t a0 = (int64_t)c * R, a1 = a0 + R < n ? a0 + R : n;
    double dz;  // distance from the carried state's z to this chunk's far end
    if (dir == 0) dz = c > 0 ? zs[a1 - 1] - zs[a0 - 1] : 0.0;
    else dz = c + 1 < nch ? zs[a1] - zs[a0] : 0.0;
    const C2 D = cexp_neg(b.re[l] * dz, b.im[l] * dz);
    C2 nb = cmul(D, C2{fma(dz, TA.re, TB.re), fma(dz, TA.im, TB.im)});
    C2 na = cmul(D, TA);
    TA = C2{na.re + XA.x, na.im + XA.y};
    TB = C2{nb.re + XB.x, nb.im + XB.y};
  }
}

template <int MH>
__global__ void zero_sweep_kernel(const double* __restrict__ zs, const double* __restrict__ qs,
                                  const double2* __restrict__ dtab, int64_t n, int R, int nch,
                                  const double2* __restrict__ zagg, ZCoef zc, int want_forces,
                                  double* __restrict__ fzf, double* __restrict__ fzb,
                                  double* __restrict__ zep) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * nch) return;
  const int c = e >> 1, dir = e & 1;
  const int64_t a0 = (int64_t)c * R, a1 = a0 + R < n ? a0 + R : n;
  const double2* cin = zagg + ((size_t)c * 2 + dir) * (2 * MH + 1);
  C2 TA[MH], TB[MH];
#pragma unroll
  for (int l = 0; l < MH; ++l) {
    TA[l] = C2{cin[l].x, cin[l].y};
    TB[l] = C2{cin[MH + l].x, cin[MH + l].y};
  }
  double S0 = cin[2 * MH].x, S1 = cin[2 * MH].y;
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  for (int64_t s = 0; s < a1 - a0; ++s) {
    const int64_t a = dir == 0 ? a0 + s : a1 - 1 - s;
    const int64_t ad = dir == 0 ? a : a + 1;  // decay row d_a (fwd) / d_{a+1} (bwd)
    const double q = qs[a], z = zs[a];
    if (ad > 0 && ad < n) {
      const double dz = zs[ad] - zs[ad - 1];
#pragma unroll
      for (int l = 0; l < MH; ++l) {
        const double2 d = dtab[ad * MH + l];
        C2 bt{fma(dz, TA[l].re, TB[l].re), fma(dz, TA[l].im, TB[l].im)};
        TB[l] = cmul(bt, C2{d.x, d.y});
        TA[l] = cmul(TA[l], C2{d.x, d.y});
      }
    } else {
      // a = 0 forward / a = n-1 backward: nothing below / above
#pragma unroll
      for (int l = 0; l < MH; ++l) TA[l] = TB[l] = C2{0.0, 0.0};
    }
    double sw = 0.0;  // Re sum_l [(w/s + w s/2) A - alpha w B] (pair-doubled)
#pragma unroll
    for (int l = 0; l < MH; ++l) {
      sw = fma(zc.f2[2 * l], TA[l].re, fma(-zc.f2[2 * l + 1], TA[l].im, sw));
      sw = fma(-zc.aw2[2 * l], TB[l].re, fma(zc.aw2[2 * l + 1], TB[l].im, sw));
    }
    if (dir == 0) {
      double sb = 0.0, sa = 0.0;
#pragma unroll
      for (int l = 0; l < MH; ++l) {
        sb = fma(zc.ws2[2 * l], TB[l].re, fma(-zc.ws2[2 * l + 1], TB[l].im, sb));
        sa = fma(zc.w2[2 * l], TA[l].re, fma(-zc.w2[2 * l + 1], TA[l].im, sa));
      }
      t0 = fma(q, fma(z, S0, -S1), t0);
      t1 = fma(q, sb, t1);
      t2 = fma(q, sa, t2);
      if (want_forces) fzf[a] = S0 - kTwoOverSqrtPi * sw;
      S1 = fma(q, z, S1);
    } else if (want_forces) {
      fzb[a] = S0 - kTwoOverSqrtPi * sw;
    }
#pragma unroll
    for (int l = 0; l < MH; ++l) TA[l].re += q;
    S0 += q;
  }
  if (dir == 0) {
    zep[3 * c + 0] = t0;
    zep[3 * c + 1] = t1;
    zep[3 * c + 2] = t2;
  }
}

__global__ void zero_energy_kernel(const double* __restrict__ zep, int nch, double alpha,
                                   double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double t0 = 0.0, t1 = 0.0, t2 = 0.0;
  for (int c = 0; c < nch; ++c) {
    t0 += zep[3 * c];
    t1 += zep[3 * c + 1];
    t2 += zep[3 * c + 2];
  }
  out[0] = t0 - kTwoOverSqrtPi * t1 + t2 / (alpha * kSqrtPi);
}

ZeroPlan zero_plan(int64_t n, int mh) {
  ZeroPlan p{};
  p.n = n;
  p.mh = mh;
  int R = 32;
  while (R * 2 <= 512 && (int64_t)R * 2 * 4096 <= n) R *= 2;
  p.R = R;
  p.nch = (int)((n + R - 1) / R);
  return p;
}

size_t zero_work_doubles(const ZeroPlan& p) {
  return 2 * (size_t)p.nch * 2 * (2 * p.mh + 1) + 3 * (size_t)p.nch + 8;
}

template <int MH>
static void zero_launch(const ZeroPlan& p, double* work, const double* zs, const double* qs,
                        const double2* dtab, const ZCoef& zc, const BVec& b, double alpha,
                        int want_forces, double* fzf, double* fzb, double* upair,
                        cudaStream_t st) {
  double2* zagg = reinterpret_cast<double2*>(work);
  double* zep = work + 2 * (size_t)p.nch * 2 * (2 * MH + 1);
  const int nthr = 2 * p.nch;
  zero_aggregate_kernel<MH><<<(nthr + 63) / 64, 64, 0, st>>>(zs, qs, dtab, p.n, p.R, p.nch, zagg);
  zero_carry_kernel<MH><<<1, 64, 0, st>>>(zs, p.n, p.R, p.nch, b, zagg);
  zero_sweep_kernel<MH><<<(nthr + 63) / 64, 64, 0, st>>>(zs, qs, dtab, p.n, p.R, p.nch, zagg, zc,
                                                         want_forces, fzf, fzb, zep);
  zero_energy_kernel<<<1, 32, 0, st>>>(zep, p.nch, alpha, upair);
}

cudaError_t zero_run_b(const ZeroPlan& p, double* work, const double* zs, const double* qs,
                       const double2* dtab, const ZCoef& zc, const BVec& b, double alpha,
                       int want_forces, double* fzf, double* fzb, double* upair,
                       cudaStream_t st) {
  if (p.n < 2) return cudaMemsetAsync(upair, 0, sizeof(double), st);
  switch (p.mh) {
#define ZCASE(K) \
  case K: zero_launch<K>(p, work, zs, qs, dtab, zc, b, alpha, want_forces, fzf, fzb, upair, st); break;
    ZCASE(2) ZCASE(3) ZCASE(4) ZCASE(5) ZCASE(6) ZCASE(7) ZCASE(8) ZCASE(9) ZCASE(10) ZCASE(11)
    ZCASE(12)
#undef ZCASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace slab
