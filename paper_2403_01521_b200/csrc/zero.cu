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
// Same 3-phase chunked scan as the Fourier path, one thread per (chunk, dir)
// for phases 1 and 3.  (A, B) compose as the affine map
//   A' = D A + X_A,  B' = D (B + dz A) + X_B,   D = e^{-b dz},
// closed under composition as (D, dz, X_A, X_B); phase 2 is a warp-cooperative
// scan of those maps (one warp per (direction, pair) chain).
#include "common.cuh"
#include "kernels.cuh"

namespace slab {

#ifndef SLAB_ZERO_LANES
#define SLAB_ZERO_LANES 1
#endif

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
      const int64_t ad = dir == 0 ? a : a + 1;  // decay row
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

// zdz[dir*nch + c] = distance from the carried state's z to chunk c's far end;
// zD[(dir*nch + c)*mh + l] = e^{-b_l zdz}
__global__ void zero_chunk_decay_kernel(const double* __restrict__ zs, int64_t n, int R, int nch,
                                        int mh, BVec b, double* __restrict__ zdz,
                                        double2* __restrict__ zD) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * nch * mh) return;
  const int l = e % mh, dc = e / mh, dir = dc / nch, c = dc % nch;
  const int64_t a0 = (int64_t)c * R, a1 = a0 + R < n ? a0 + R : n;
  double dz;
  if (dir == 0) dz = c > 0 ? zs[a1 - 1] - zs[a0 - 1] : 0.0;
  else dz = c + 1 < nch ? zs[a1] - zs[a0] : 0.0;
  if (l == 0) zdz[dc] = dz;
  const C2 D = cexp_neg(b.re[l] * dz, b.im[l] * dz);
  zD[e] = make_double2(D.re, D.im);
}

struct ZMap {
  C2 D, XA, XB;
  double dz;
};
// apply `first`, then `then`
__device__ __forceinline__ ZMap zcompose(const ZMap& first, const ZMap& then) {
  ZMap r;
  r.D = cmul(then.D, first.D);
  r.dz = first.dz + then.dz;
  const C2 xa = cmul(then.D, first.XA);
  r.XA = C2{xa.re + then.XA.re, xa.im + then.XA.im};
  const C2 xb = cmul(then.D, C2{fma(then.dz, first.XA.re, first.XB.re),
                                fma(then.dz, first.XA.im, first.XB.im)});
  r.XB = C2{xb.re + then.XB.re, xb.im + then.XB.im};
  return r;
}
__device__ __forceinline__ ZMap zshfl_up(const ZMap& m, int o) {
  ZMap r;
  r.D = C2{__shfl_up_sync(0xffffffffu, m.D.re, o), __shfl_up_sync(0xffffffffu, m.D.im, o)};
  r.XA = C2{__shfl_up_sync(0xffffffffu, m.XA.re, o), __shfl_up_sync(0xffffffffu, m.XA.im, o)};
  r.XB = C2{__shfl_up_sync(0xffffffffu, m.XB.re, o), __shfl_up_sync(0xffffffffu, m.XB.im, o)};
  r.dz = __shfl_up_sync(0xffffffffu, m.dz, o);
  return r;
}

// in place: aggregates -> carried-in states.  One 256-thread block per
// (dir, chain), chain = SOE pair l < mh, or mh for the (S0, S1) prefix sums:
// thread blocks of chunks composed serially, then a shuffle + shared-memory scan.
constexpr int kZCarryThreads = 256;

__global__ void __launch_bounds__(kZCarryThreads) zero_carry_kernel(
    int nch, int mh, const double* __restrict__ zdz, const double2* __restrict__ zD,
    double2* __restrict__ zagg) {
  __shared__ ZMap wagg[kZCarryThreads / 32];
  const int w = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int dir = w / (mh + 1), l = w % (mh + 1);
  const size_t rec = 2 * mh + 1;
  const int per = (nch + kZCarryThreads - 1) / kZCarryThreads;
  const int s0 = tid * per, s1 = min(nch, s0 + per);
  const ZMap ident{C2{1.0, 0.0}, C2{0.0, 0.0}, C2{0.0, 0.0}, 0.0};
  // the (S0, S1) chain is the same machinery with D = 1, dz = 0: X_A = S0, X_B = S1
  const bool sums = l == mh;
  auto element = [&](int c) {
    const double2* p = zagg + ((size_t)c * 2 + dir) * rec;
    if (sums) return ZMap{C2{1.0, 0.0}, C2{p[2 * mh].x, 0.0}, C2{p[2 * mh].y, 0.0}, 0.0};
    const double2 d = zD[((size_t)dir * nch + c) * mh + l];
    return ZMap{C2{d.x, d.y}, C2{p[l].x, p[l].y}, C2{p[mh + l].x, p[mh + l].y},
                zdz[(size_t)dir * nch + c]};
  };
  ZMap M = ident;
  for (int sb = s0; sb < s1; sb += 8) {
    ZMap es[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (sb + j < s1) es[j] = element(dir == 0 ? sb + j : nch - 1 - (sb + j));
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (sb + j < s1) M = zcompose(M, es[j]);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const ZMap u = zshfl_up(M, o);
    if (lane >= o) M = zcompose(u, M);
  }
  if (lane == 31) wagg[warp] = M;
  __syncthreads();
  ZMap pre = ident;
  for (int q = 0; q < warp; ++q) pre = zcompose(pre, wagg[q]);
  ZMap ex = zshfl_up(M, 1);
  if (lane == 0) ex = ident;
  const ZMap in = zcompose(pre, ex);
  C2 TA = in.XA, TB = in.XB;
  constexpr int B = 8;  // loads of a batch issued ahead of its stores
  for (int sb = s0; sb < s1; sb += B) {
    ZMap es[B];
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (sb + j < s1) es[j] = element(dir == 0 ? sb + j : nch - 1 - (sb + j));
#pragma unroll
    for (int j = 0; j < B; ++j) {
      if (sb + j >= s1) break;
      const int c = dir == 0 ? sb + j : nch - 1 - (sb + j);
      const ZMap& e = es[j];
      double2* p = zagg + ((size_t)c * 2 + dir) * rec;
      if (sums) {
        p[2 * mh] = make_double2(TA.re, TB.re);
        TA.re += e.XA.re;
        TB.re += e.XB.re;
      } else {
        p[l] = make_double2(TA.re, TA.im);
        p[mh + l] = make_double2(TB.re, TB.im);
        const C2 nb = cmul(e.D, C2{fma(e.dz, TA.re, TB.re), fma(e.dz, TA.im, TB.im)});
        const C2 na = cmul(e.D, TA);
        TA = C2{na.re + e.XA.re, na.im + e.XA.im};
        TB = C2{nb.re + e.XB.re, nb.im + e.XB.im};
      }
    }
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
  // the next step's charge and z values are loaded one step ahead (this kernel
  // runs a few warps per SM, mostly in the scan's tail; the decay rows stay
  // in-step: prefetching them too spills)
  const int64_t len = a1 - a0;
  double nq, nz, nz1, nz0;
  auto fetch = [&](int64_t s) {
    const int64_t ss = s < len ? s : len - 1;
    const int64_t a = dir == 0 ? a0 + ss : a1 - 1 - ss;
    const int64_t ad = dir == 0 ? a : a + 1;  // decay row d_a (fwd) / d_{a+1} (bwd)
    const int64_t adc = ad > 0 && ad < n ? ad : 1;
    nq = qs[a];
    nz = zs[a];
    nz1 = zs[adc];
    nz0 = zs[adc - 1];
  };
  fetch(0);
  for (int64_t s = 0; s < len; ++s) {
    const int64_t a = dir == 0 ? a0 + s : a1 - 1 - s;
    const int64_t ad = dir == 0 ? a : a + 1;
    const double q = nq, z = nz, dz = nz1 - nz0;
    fetch(s + 1);
    if (ad > 0 && ad < n) {
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
    zep[c] = t0;
    zep[nch + c] = t1;
    zep[2 * nch + c] = t2;
  }
}

// ---- lane-per-pair aggregate (default): the (chunk, direction) work is spread
// over G = pow2 >= MH lanes, lane l < MH carrying pair l (4 doubles of state
// instead of 4 MH per thread; the thread-per-chunk kernel runs at 10%
// occupancy): 0.106 -> 0.066 ms at cfg4.  Lane reads of the decay rows are
// contiguous; the (S0, S1) prefix sums are carried redundantly by every lane.
// (The same split of the sweep needs a per-particle shuffle reduction over the
// pairs and measured slower, 0.154 against 0.124 ms.)
template <int MH>
__host__ __device__ constexpr int zlanes() {
  return MH <= 2 ? 2 : MH <= 4 ? 4 : MH <= 8 ? 8 : 16;
}

template <int MH>
__global__ void __launch_bounds__(128) zero_aggregate_lane_kernel(
    const double* __restrict__ zs, const double* __restrict__ qs,
    const double2* __restrict__ dtab, int64_t n, int R, int nch, double2* __restrict__ zagg) {
  constexpr int G = zlanes<MH>();
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t grp = e / G;
  const int l = (int)(e - grp * G);
  if (grp >= 2 * (int64_t)nch) return;
  const int c = (int)(grp >> 1), dir = (int)(grp & 1);
  const int64_t a0 = (int64_t)c * R, a1 = a0 + R < n ? a0 + R : n;
  const bool act = l < MH;
  C2 TA{0.0, 0.0}, TB{0.0, 0.0};
  double S0 = 0.0, S1 = 0.0;
  for (int64_t s = 0; s < a1 - a0; ++s) {
    const int64_t a = dir == 0 ? a0 + s : a1 - 1 - s;
    const double q = qs[a];
    if (s > 0 && act) {
      const int64_t ad = dir == 0 ? a : a + 1;
      const double dz = zs[ad] - zs[ad - 1];
      const double2 d = dtab[ad * MH + l];
      const C2 bt{fma(dz, TA.re, TB.re), fma(dz, TA.im, TB.im)};
      TB = cmul(bt, C2{d.x, d.y});
      TA = cmul(TA, C2{d.x, d.y});
    }
    TA.re += q;
    S0 += q;
    S1 = fma(q, zs[a], S1);
  }
  double2* out = zagg + ((size_t)c * 2 + dir) * (2 * MH + 1);
  if (act) {
    out[l] = make_double2(TA.re, TA.im);
    out[MH + l] = make_double2(TB.re, TB.im);
  }
  if (l == 0) out[2 * MH] = make_double2(S0, S1);
}

// three fixed-order block sums over chunks (one block per term), then combine
__global__ void __launch_bounds__(256) zero_energy_kernel(const double* __restrict__ zep, int nch,
                                                          double* __restrict__ tsum) {
  __shared__ double red[256];
  double s = 0.0;
  for (int c = threadIdx.x; c < nch; c += 256) s += zep[(size_t)blockIdx.x * nch + c];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) tsum[blockIdx.x] = red[0];
}

__global__ void zero_upair_kernel(const double* __restrict__ tsum, double alpha,
                                  double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  out[0] = tsum[0] - kTwoOverSqrtPi * tsum[1] + tsum[2] / (alpha * kSqrtPi);
}

ZeroPlan zero_plan(int64_t n, int mh) {
  ZeroPlan p{};
  p.n = n;
  p.mh = mh;
#ifndef SLAB_ZERO_RMAX
#define SLAB_ZERO_RMAX 128
#endif
  int R = 32;
  while (R * 2 <= SLAB_ZERO_RMAX && (int64_t)R * 2 * 8192 <= n) R *= 2;
  p.R = R;
  p.nch = (int)((n + R - 1) / R);
  return p;
}

size_t zero_work_doubles(const ZeroPlan& p) {
  const size_t nch = (size_t)p.nch;
  return 2 * nch * 2 * (2 * p.mh + 1)   // zagg (double2)
         + 2 * 2 * nch * p.mh           // zD (double2)
         + 2 * nch                      // zdz
         + 3 * nch + 8;                 // zep, tsum
}

template <int MH>
static void zero_launch(const ZeroPlan& p, double* work, const double* zs, const double* qs,
                        const double2* dtab, const ZCoef& zc, const BVec& b, double alpha,
                        int want_forces, double* fzf, double* fzb, double* upair,
                        cudaStream_t st) {
  const size_t nch = (size_t)p.nch;
  double2* zagg = reinterpret_cast<double2*>(work);
  double2* zD = zagg + 2 * nch * (2 * MH + 1);
  double* zdz = reinterpret_cast<double*>(zD + 2 * nch * MH);
  double* zep = zdz + 2 * nch;
  double* tsum = zep + 3 * nch;
  const int nthr = 2 * p.nch;
#if SLAB_ZERO_LANES
  const int64_t nlane = (int64_t)nthr * zlanes<MH>();
  zero_aggregate_lane_kernel<MH><<<(unsigned)((nlane + 127) / 128), 128, 0, st>>>(
      zs, qs, dtab, p.n, p.R, p.nch, zagg);
#else
  zero_aggregate_kernel<MH><<<(nthr + 63) / 64, 64, 0, st>>>(zs, qs, dtab, p.n, p.R, p.nch, zagg);
#endif
  const int nd = 2 * p.nch * MH;
  zero_chunk_decay_kernel<<<(nd + 255) / 256, 256, 0, st>>>(zs, p.n, p.R, p.nch, MH, b, zdz, zD);
  zero_carry_kernel<<<2 * (MH + 1), kZCarryThreads, 0, st>>>(p.nch, MH, zdz, zD, zagg);
  zero_sweep_kernel<MH><<<(nthr + 63) / 64, 64, 0, st>>>(zs, qs, dtab, p.n, p.R, p.nch, zagg, zc,
                                                         want_forces, fzf, fzb, zep);
  zero_energy_kernel<<<3, 256, 0, st>>>(zep, p.nch, tsum);
  zero_upair_kernel<<<1, 1, 0, st>>>(tsum, alpha, upair);
}

cudaError_t zero_run_b(const ZeroPlan& p, double* work, const double* zs, const double* qs,
                       const double2* dtab, const ZCoef& zc, const BVec& b, double alpha,
                       int want_forces, double* fzf, double* fzb, double* upair,
                       cudaStream_t st) {
  if (p.n < 2) return cudaMemsetAsync(upair, 0, sizeof(double), st);
  switch (p.mh) {
#define ZCASE(K) \
  case K: zero_launch<K>(p, work, zs, qs, dtab, zc, b, alpha, want_forces, fzf, fzb, upair, st); break;
    ZCASE(1) ZCASE(2) ZCASE(3) ZCASE(4) ZCASE(5) ZCASE(6) ZCASE(7) ZCASE(8) ZCASE(9) ZCASE(10) ZCASE(11)
    ZCASE(12)
#undef ZCASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace slab
