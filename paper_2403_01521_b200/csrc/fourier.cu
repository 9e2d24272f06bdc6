// fourier.cu -- the SOE Fourier sweep (the hot path), B200 layout.
//
// Replaces reference soewald2d.py:85-208 (_fourier_soe_sweep) and the per-call
// decay table soewald2d.py:76-82.  Math, per mode t and
// SOE term l with b_l = alpha s_l:
//   forward   G_{l,a} = (G_{l,a-1} + u_{a-1}) e^{-b_l dz_a},  u = q e^{-i theta}
//   backward  mirror with v = q e^{+i theta}
//   p = kappa g - 2k sum_l c_l G_l,  zeta = 2 sum_l c_l b_l G_l - kappa g
//   U_t += ck q Re(e^{i theta} p);  F += ... (soewald2d.py:158-202)
//
// B200 design:
//  * Conjugate pairing.  s_{M-1-l} = conj(s_l) bitwise, so per pair one keeps two
//    complex recurrences with REAL inputs (R: q cos theta, I: -+ q sin theta) and
//    c_l G_l + conj = 2Re(c_l R_l) + 2i Re(c_l I_l).  kappa is real.
//  * Lanes = (mode, direction) work items, particles in sequence (a force plan's
//    warp: 16 modes forward in lanes 0-15, the same modes backward in 16-31).
//    Forward lanes walk the chunk from its start and backward lanes from its
//    end, each half-warp one particle per step, so the k-independent decays
//    e^{-b_l dz} are BROADCAST from shared memory: they are computed once per
//    step (decay_table_kernel) and reused by all 2P items -- the kernel is FP64
//    bound, not HBM bound.
//  * Particle axis split into chunks of R particles (one CTA each) with a 3-phase
//    affine scan: (1) chunk aggregates X_c = sum_j u_j e^{-b (z_end - z_j)} using
//    k-independent weights staged in smem, (2) a carry scan over chunks,
//    (3) the exact recurrence from the carried-in state with the fused
//    sincos/exp/energy/force epilogue.  All exponents stay <= 0 (stable in Lz).
//  * Forces: per particle the lanes' contributions are staged transposed in smem
//    and row-summed (forward and backward halves separately, spread through the
//    next particles' steps) into per-warp partial buffers, then summed over
//    warps in fixed order: deterministic, no atomics.
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace slab {

#ifndef SLAB_SWEEP_CB
#define SLAB_SWEEP_CB 0
#endif
#ifndef SLAB_SWEEP_CREG
#define SLAB_SWEEP_CREG 0
#endif
#ifndef SLAB_SWEEP_GDECAY
#define SLAB_SWEEP_GDECAY 0
#endif
#ifndef SLAB_SWEEP_REM
#define SLAB_SWEEP_REM 1
#endif
constexpr bool kSweepRem = SLAB_SWEEP_REM;
#ifndef SLAB_SWEEP_REM_MAX
#define SLAB_SWEEP_REM_MAX 8  // cfg3 (16 left over of 400) ran 2.21 -> 2.37 ms with it
#endif
constexpr int kSweepRemMax = SLAB_SWEEP_REM_MAX;
#ifndef SLAB_SWEEP_PIPE
#define SLAB_SWEEP_PIPE 1  // next particle's sincos/exp one iteration ahead: 3.57 -> 3.52 ms at 168 registers (2.5% slower at 128)
#endif
#ifndef SLAB_SWEEP_MAXT
#define SLAB_SWEEP_MAXT 256
#endif
// sweep CTA size cap: 2 CTAs/SM at 65536 / (2 * cap) registers per thread
constexpr int kSweepMaxThreads = SLAB_SWEEP_MAXT;  // force staging batch (particles)
#ifndef SLAB_SWEEP_MAXT_2CTA
#define SLAB_SWEEP_MAXT_2CTA 192
#endif
// CTA size cap of the two-CTAs-per-SM sweep: 192 threads (6 warps) lets the
// allocator use 168 registers (2 x 6 warps x 32 x 168 <= 64K; 3 warps per SM
// sub-partition) instead of 128 -- no spills, cfg4 sweep 3.77 -> 3.57 ms.  With
// the remainder sweep a P = 100 chunk's main items are exactly 192.  The
// one-CTA form (12 pairs) keeps 256-thread groups (cfg3: 192 -> 3 groups per
// chunk restaging the chunk, 2.20 -> 2.79 ms).
// force staging rows: 32 lanes, the backward half-warp shifted one column so
// that the row-summing lanes (8 rows x 2 halves per 16-lane phase) hit distinct
// banks; two buffers per warp (one batch staged while the previous one is summed)
constexpr int kStageStride = 34;
constexpr int kStageBuf = 3 * 4 * kStageStride;  // 4 particles x 3 components
// CTAs per SM the sweep is compiled for: 2 (<= 168 registers at 192 threads) up to
// SLAB_SWEEP_BIG_MH pairs; 1 above it, where two CTAs' budget spills hundreds of
// bytes per lane
#ifndef SLAB_SWEEP_BIG_MH
#define SLAB_SWEEP_BIG_MH 10  // cfg3 (M = 24, 12 pairs): sweep 1.90 -> 1.31 ms; 8 pairs stay at 2 CTAs (4.14 vs 4.86 ms)
#endif
__host__ __device__ constexpr int sweep_min_blocks(int mh) { return mh >= SLAB_SWEEP_BIG_MH ? 1 : 2; }
__host__ __device__ constexpr int sweep_max_threads(int mh) {
  return mh >= SLAB_SWEEP_BIG_MH ? SLAB_SWEEP_MAXT : SLAB_SWEEP_MAXT_2CTA;
}
constexpr int kMaxR = 256;
constexpr size_t kSmemPerSM = 227 * 1024;  // usable shared memory per SM (B200)
constexpr int kAggRegs = 72;               // fourier_aggregate_mma_kernel (ptxas)

__host__ __device__ inline int ncomp_of(int mh) { return 2 * mh + 1; }

// ---------------------------------------------------------------------------
// k-independent tables
// ---------------------------------------------------------------------------
// dtab[a*mh + l] = exp(-b_l (z_a - z_{a-1})), row 0 = 1, row n = 0 (backward guard)
// one thread per (row a, pair l), l fastest: coalesced 16-byte stores; MH a
// template parameter, so the row index is a multiply-shift instead of the
// 64-bit division of the round-1 form (a thread per row storing its 8 pairs
// measured slower: 0.071 against 0.061 ms, strided stores)
template <int MH>
__global__ void decay_table_kernel(const double* __restrict__ zs, int64_t n, BVec b,
                                   double2* __restrict__ dtab, int64_t a_lo, int64_t a_hi) {
  const int64_t e = a_lo * MH + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (a_hi + 1) * MH) return;
  const int64_t a = e / MH;
  const int l = (int)(e - a * MH);
  double2 d;
  if (a == 0) {
    d = make_double2(1.0, 0.0);
  } else if (a == n) {
    d = make_double2(0.0, 0.0);
  } else {
    const double dz = zs[a] - zs[a - 1];
    const C2 v = cexp_neg(b.re[l] * dz, b.im[l] * dz);
    d = make_double2(v.re, v.im);
  }
  dtab[e] = d;
}

// zbound[c] = z_end(c), zbound[nch + c] = z_start(c);
// Df[c*mh+l] = e^{-b_l (z_end(c) - z_end(c-1))}, Db[c*mh+l] = e^{-b_l (z_start(c+1) - z_start(c))}
__global__ void chunk_bounds_kernel(const double* __restrict__ zs, int64_t n, int R, int nch,
                                    int mh, BVec b, double* __restrict__ zbound,
                                    double2* __restrict__ Df, double2* __restrict__ Db) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nch * mh) return;
  int c = e / mh, l = e - c * mh;
  int64_t a0 = (int64_t)c * R;
  int64_t a1 = a0 + R < n ? a0 + R : n;
  double zend = zs[a1 - 1], zst = zs[a0];
  if (l == 0) {
    zbound[c] = zend;
    zbound[nch + c] = zst;
  }
  double2 df = make_double2(0.0, 0.0), db = make_double2(0.0, 0.0);
  if (c > 0) {
    double dz = zend - zs[a0 - 1];
    C2 v = cexp_neg(b.re[l] * dz, b.im[l] * dz);
    df = make_double2(v.re, v.im);
  }
  if (c + 1 < nch) {
    double dz = zs[a1] - zst;
    C2 v = cexp_neg(b.re[l] * dz, b.im[l] * dz);
    db = make_double2(v.re, v.im);
  }
  Df[e] = df;
  Db[e] = db;
}

// Per-mode coefficients (soewald2d.py:113-126), one thread per mode.
__global__ void mode_table_kernel(const double* __restrict__ modes,
                                  const double* __restrict__ commonv, double commonv_scalar,
                                  int P, int mh, double area, BVec b, WVec w,
                                  double* __restrict__ tab, int* __restrict__ status) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P) return;
  const double kx = modes[3 * t + 0], ky = modes[3 * t + 1], k = modes[3 * t + 2];
  const double ct = commonv ? commonv[t] : commonv_scalar;
  double* r = tab + (size_t)t * mode_stride(mh);
  double kappa = 0.0;
  double wsing = 0.0;  // W_s: weights of the singular terms (a pair carries w + conj w)
  for (int l = 0; l < mh; ++l) {
    const double br = b.re[l], bi = b.im[l];
    double cr = 0.0, ci = 0.0;
    if (hypot(br - k, bi) < kSingularTol * k) {
      wsing += 2.0 * w.re[l];  // analytic-limit branch (soewald2d.py:116-124): c_l = 0
    } else {
      // c = w / (b^2 - k^2)
      const double dr = br * br - bi * bi - k * k, di = 2.0 * br * bi;
      const double den = dr * dr + di * di;
      cr = (w.re[l] * dr + w.im[l] * di) / den;
      ci = (w.im[l] * dr - w.re[l] * di) / den;
    }
    // C = 2c, CB = 2 c b; kappa = sum over all M terms of 2 c b = sum_pairs 2 Re(CB)
    r[8 + 2 * l] = 2.0 * cr;
    r[8 + 2 * l + 1] = 2.0 * ci;
    const double cbr = 2.0 * (cr * br - ci * bi), cbi = 2.0 * (cr * bi + ci * br);
    r[8 + 2 * mh + 2 * l] = cbr;
    r[8 + 2 * mh + 2 * l + 1] = cbi;
    kappa += 2.0 * cbr;
  }
  const double pref = kPi / area;
  r[0] = kx;
  r[1] = ky;
  r[2] = k;
  r[3] = pref * ct / k;
  r[4] = pref * ct;
  r[5] = kappa;
  r[6] = wsing;  // consumed by fourier_singular_kernel
  r[7] = 0.0;
  (void)status;
}

// ---------------------------------------------------------------------------
// the singular-term correction (soewald2d.py:116-124, 146-149, 162-170)
// ---------------------------------------------------------------------------
// A term with |b_l - k| < 2e-6 k leaves the G recurrences (c_l = 0) and its
// weight W_s enters through an extra chain h_a = (h_{a-1} + dz_a (g_{a-1} +
// u_{a-1})) e^{-k dz_a}: p += W_s (g / k + h), zeta -= W_s h.  Everything is
// linear in (p, zeta), so the main sweep runs without the term and this pass
// adds its contribution.  Singular terms only exist for (near-)real exponents
// -- never in built contours; the host launches this only for tables that have
// such a term.  One block: per singular item, each thread composes the affine
// map of (g, h) over its contiguous particle segment, a block scan gives each
// segment its state, and the segment is re-walked with the readout.  Items run
// in sequence and each particle's force belongs to one thread: deterministic.
struct SingMap {  // (g, h) -> D [[1, 0], [del, 1]] (g, h) + (Xg, Xh)
  double D, del;
  C2 Xg, Xh;
};
__device__ __forceinline__ SingMap sing_compose(const SingMap& a, const SingMap& b) {  // b after a
  SingMap r;
  r.D = a.D * b.D;
  r.del = a.del + b.del;
  r.Xg = C2{b.D * a.Xg.re + b.Xg.re, b.D * a.Xg.im + b.Xg.im};
  r.Xh = C2{b.D * (b.del * a.Xg.re + a.Xh.re) + b.Xh.re,
            b.D * (b.del * a.Xg.im + a.Xh.im) + b.Xh.im};
  return r;
}
constexpr int kSingThreads = 512;
__global__ void __launch_bounds__(kSingThreads) fourier_singular_kernel(
    const double* __restrict__ xs, const double* __restrict__ ys, const double* __restrict__ zs,
    const double* __restrict__ qs, int64_t n, const double* __restrict__ modetab, int mh, int P,
    int items, int want_forces, double* __restrict__ esing, double* __restrict__ forces) {
  __shared__ SingMap sm[kSingThreads];
  __shared__ double red[kSingThreads];
  const int tid = threadIdx.x;
  const int64_t per = (n + kSingThreads - 1) / kSingThreads;
  for (int item = 0; item < items; ++item) {
    const bool fwd = item < P;
    const int t = fwd ? item : item - P;
    const double* mt = modetab + (size_t)t * mode_stride(mh);
    const double ws = mt[6];
    if (fwd && tid == 0) esing[t] = 0.0;
    if (ws == 0.0) continue;  // block-uniform
    const double kx = mt[0], ky = mt[1], k = mt[2], ck = mt[3], cz = mt[4];
    // positions s = 0 .. n-1 along the sweep direction
    const int64_t s0 = tid * per, s1 = min(n, s0 + per);
    auto idx = [&](int64_t sidx) { return fwd ? sidx : n - 1 - sidx; };
    // the step INTO position sidx (sidx >= 1) from sidx - 1
    auto step = [&](int64_t sidx, C2 u_prev) {
      const int64_t a = idx(sidx), ap = idx(sidx - 1);
      const double dz = fwd ? zs[a] - zs[ap] : zs[ap] - zs[a];
      const double D = exp(-k * dz);
      return SingMap{D, dz, C2{D * u_prev.re, D * u_prev.im},
                     C2{D * dz * u_prev.re, D * dz * u_prev.im}};
    };
    auto input = [&](int64_t sidx) {  // u (forward) or v (backward) of the particle at sidx
      const int64_t a = idx(sidx);
      double sn, cs;
      sincos(kx * xs[a] + ky * ys[a], &sn, &cs);
      return C2{qs[a] * cs, fwd ? -qs[a] * sn : qs[a] * sn};
    };
    SingMap M{1.0, 0.0, C2{0.0, 0.0}, C2{0.0, 0.0}};
    for (int64_t si = s0; si < s1; ++si)
      if (si >= 1) M = sing_compose(M, step(si, input(si - 1)));
    sm[tid] = M;
    __syncthreads();
    for (int o = 1; o < kSingThreads; o <<= 1) {  // inclusive scan (Hillis-Steele)
      const SingMap prev = tid >= o ? sm[tid - o] : SingMap{1.0, 0.0, C2{0, 0}, C2{0, 0}};
      __syncthreads();
      if (tid >= o) sm[tid] = sing_compose(prev, sm[tid]);
      __syncthreads();
    }
    // state at position s0 - 1 = the previous segments' composed map applied to (0, 0)
    C2 g{0.0, 0.0}, hh{0.0, 0.0};
    if (tid > 0) {
      g = sm[tid - 1].Xg;
      hh = sm[tid - 1].Xh;
    }
    __syncthreads();
    double e = 0.0;
    for (int64_t si = s0; si < s1; ++si) {
      const int64_t a = idx(si);
      if (si >= 1) {  // the state at position si from the one at si - 1
        const SingMap st1 = step(si, input(si - 1));
        const C2 g0 = g;
        g = C2{st1.D * g0.re + st1.Xg.re, st1.D * g0.im + st1.Xg.im};
        hh = C2{st1.D * (st1.del * g0.re + hh.re) + st1.Xh.re,
                st1.D * (st1.del * g0.im + hh.im) + st1.Xh.im};
      }
      // p_x = W_s (g / k + h), zeta_x = -W_s h; phase e^{+-i theta}
      const C2 px{ws * (g.re / k + hh.re), ws * (g.im / k + hh.im)};
      const C2 zx{-ws * hh.re, -ws * hh.im};
      double sn, cs;
      sincos(kx * xs[a] + ky * ys[a], &sn, &cs);
      const double ps = fwd ? sn : -sn;
      const double epr = cs * px.re - ps * px.im, epi = cs * px.im + ps * px.re;
      const double q = qs[a];
      if (fwd) e += q * epr;
      if (want_forces) {
        const double zr = cs * zx.re - ps * zx.im;
        const double sgn = fwd ? 1.0 : -1.0;
        forces[3 * a + 0] += sgn * ck * q * kx * epi;
        forces[3 * a + 1] += sgn * ck * q * ky * epi;
        forces[3 * a + 2] -= sgn * cz * q * zr;
      }
    }
    if (fwd) {
      red[tid] = e;
      __syncthreads();
      for (int w2 = kSingThreads / 2; w2 > 0; w2 >>= 1) {
        if (tid < w2) red[tid] += red[tid + w2];
        __syncthreads();
      }
      if (tid == 0) esing[t] = ck * red[0];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// phase 1 on the FP64 tensor cores (DMMA m8n8k4)
// ---------------------------------------------------------------------------
// For chunk c the pair aggregates are a GEMM over the chunk's particles j:
//   X[row][col] = sum_j U[row][j] W[j][col]
// rows (mode t, part s): U = q cos(theta) (s = 0, the R recurrence) or
//   -q sin(theta) (s = 1, I);
// cols (direction, pair l, re/im): the k-independent weights
//   W^f_l(j) = e^{-b_l (z_end - z_j)},  W^b_l(j) = e^{-b_l (z_j - z_start)}.
// A warp owns an m-tile of 8 modes.  Per 4-particle k-step each lane computes
// ONE sincos -- for (mode lane>>2, particle lane&3), exactly its A-fragment
// slot -- which feeds both the cos and the sin fragment, then issues 2 x NT
// DMMAs against NT B fragments read from the shared weight table (column-major,
// K stride R+4: conflict-free).  DMMA and DFMA share the FP64 pipe on B200
// (measured: 37 TF/s DMMA alone, 33 TF/s mixed), so the gain is issue
// efficiency: one instruction per 256 FMAs.  The k-dependent e^{-k dist}
// aggregates (the kappa g term) stay on DFMA, four lanes per mode, reduced by
// shuffles.  Carry layout identical to fourier_aggregate_kernel.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

#ifndef SLAB_AGG_MMA_MAXW
#define SLAB_AGG_MMA_MAXW 13  // m-tiles (warps) per CTA: P <= 104 in one CTA per chunk
#endif
__host__ __device__ constexpr int mma_mhp(int mh) { return (mh + 3) / 4 * 4; }
static size_t agg_mma_smem(int R, int mh) {
  return sizeof(double) * ((size_t)4 * mma_mhp(mh) * (R + 4) + 4 * (size_t)R +
                           4 * 32 * (size_t)SLAB_AGG_MMA_MAXW + 32);
}

#ifndef SLAB_AGG_RCP
#define SLAB_AGG_RCP 1
#endif
constexpr bool kAggRcp = SLAB_AGG_RCP;
// 1/x for a normal, finite x > 0 without the IEEE division's special-case
// branch: the hardware estimate refined by two Newton steps (~1 ulp)
__device__ __forceinline__ double rcp_normal(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// a per-lane constant re-read from shared memory at every use (volatile: kept
// out of the register file of the 72-register aggregate, which spilled its
// accumulators around the transcendentals)
__device__ __forceinline__ double lds_volatile(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}

constexpr int kAggMaxWarps = SLAB_AGG_MMA_MAXW;
#ifndef SLAB_AGG_MMA_CB
#define SLAB_AGG_MMA_CB 1  // constant-bank polynomial coefficients in the main loop
#endif
template <int MH>
#ifndef SLAB_AGG_MINB
#define SLAB_AGG_MINB 2
#endif
__global__ void __launch_bounds__(32 * SLAB_AGG_MMA_MAXW, SLAB_AGG_MINB) fourier_aggregate_mma_kernel(
    const double* __restrict__ xs, const double* __restrict__ ys, const double* __restrict__ zs,
    const double* __restrict__ qs, int64_t n, int R, const double* __restrict__ modetab, int P,
    int tiles_per_cta, BVec b, double2* __restrict__ carry, int c0, int swap) {
  constexpr int MHP = mma_mhp(MH);  // pairs padded to whole n-tiles of 4 pairs
  constexpr int NT = MHP / 2;       // n-tiles: 2 directions x MHP/4
  constexpr int NCOL = 8 * NT;      // (dir, l, re/im) columns
  extern __shared__ double4 smem4[];
  const int RP = R + 4;
  double* wt = reinterpret_cast<double*>(smem4);  // [NCOL][RP]
  double* sx = wt + (size_t)NCOL * RP;
  double* sy = sx + R;
  double* sz = sy + R;  // z_end - z_j
  double* sq = sz + R;
  double* sk = sq + R;   // per-lane (kx, ky, k): [3][blockDim]
  const int c = c0 + blockIdx.x;
  const int64_t a0 = (int64_t)c * R;
  const int len = (int)(a0 + R < n ? R : n - a0);
  const double z_end = zs[a0 + len - 1], z_start = zs[a0];
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    sx[i] = xs[a0 + i];
    sy[i] = ys[a0 + i];
    sz[i] = z_end - zs[a0 + i];
    sq[i] = qs[a0 + i];
  }
  // weights, column (dir * MHP + l) * 2 + e: W^b_j = e^{-b (z_j - z_start)} and
  // W^f_j = e^{-b (z_end - z_j)} of one particle together, the forward phase by
  // angle subtraction from the chunk's b.im * span (one sincos per (j, l)
  // instead of two)
  double* sspan = sk + 4 * 32 * kAggMaxWarps;  // (cos, sin) of b.im * span per pair
  const double span_w = z_end - z_start;
  if (threadIdx.x < MHP) {
    double sn = 0.0, cs = 1.0;
    if (threadIdx.x < MH) sincos_fast_cb(b.im[threadIdx.x] * span_w, &sn, &cs);
    sspan[2 * threadIdx.x] = cs;
    sspan[2 * threadIdx.x + 1] = sn;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < R * MHP; e += blockDim.x) {
    const int j = e % R, l = e / R;
    double fr = 0.0, fi = 0.0, br = 0.0, bi = 0.0;
    if (j < len && l < MH) {
      const double z = zs[a0 + j];
      const double db = z - z_start, df = z_end - z;
      const double eb = exp_neg_cb(b.re[l] * db), ef = exp_neg_cb(b.re[l] * df);
      double snb, csb;
      sincos_fast_cb(b.im[l] * db, &snb, &csb);
      const double css = sspan[2 * l], sns = sspan[2 * l + 1];
      const double csf = fma(css, csb, sns * snb), snf = fma(sns, csb, -css * snb);
      fr = ef * csf;
      fi = -ef * snf;
      br = eb * csb;
      bi = -eb * snb;
    }
    const int cf = l * 2, cb = (MHP + l) * 2;
    wt[cf * RP + j] = fr;
    wt[(cf + 1) * RP + j] = fi;
    wt[cb * RP + j] = br;
    wt[(cb + 1) * RP + j] = bi;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.y * tiles_per_cta + warp;
  if (tile * 8 >= P) return;  // no barrier below
  const int kk = lane & 3, nn = lane >> 2;
  const int t = tile * 8 + nn;
  const bool tv = t < P;
  const double* mt = modetab + (size_t)(tv ? t : 0) * mode_stride(MH);
  const double k = mt[2];
  sk[threadIdx.x] = mt[0];
  sk[blockDim.x + threadIdx.x] = mt[1];
  sk[2 * blockDim.x + threadIdx.x] = k;
  __syncwarp();
  double acc[2][NT][2];
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int u = 0; u < NT; ++u) acc[s][u][0] = acc[s][u][1] = 0.0;
  double gfr = 0.0, gfi = 0.0, gbr = 0.0, gbi = 0.0;
  const double* wk = wt + nn * RP + kk;
  const double span = z_end - z_start;
  // e^{-k span} per lane in shared memory too (0 when k span >= 600: the
  // reciprocal form's guard); re-read at each use, registers being the limit
  sk[3 * blockDim.x + threadIdx.x] = k * span < 600.0 ? exp_neg(k * span) : 0.0;
  __syncwarp();
  const double* skl = sk + threadIdx.x;
  // (the lane's particle bound folded with the mode's validity into one
  // loop-invariant: the round-1 form spilled j and reloaded it from local
  // memory at every iteration)
  const int jend = tv ? len : 0;
  for (int k0 = 0; k0 < len; k0 += 4) {
    const int j = k0 + kk;
    double ur = 0.0, ui = 0.0;
    if (j < jend) {
      const double th = __dadd_rn(__dmul_rn(lds_volatile(skl), sx[j]),
                                  __dmul_rn(lds_volatile(skl + blockDim.x), sy[j]));
      double sn, cs;
      const double q = sq[j], ze = sz[j];  // ze = z_end - z_j
      const double kj = lds_volatile(skl + 2 * blockDim.x);
#if SLAB_AGG_MMA_CB
      sincos_fast_cb(th, &sn, &cs);
      // e^{-k (z - z_start)} = e^{-k (z_end - z_start)} / e^{-k (z_end - z)} (one exp
      // and a reciprocal instead of two exps) while both factors stay normal
      const double wf = exp_neg_cb(kj * ze);
      // (Newton reciprocal vs IEEE division: register allocation decides --
      // measured 1.18 -> 1.10 ms for 8 pairs, 0.36 -> 0.39 ms for 12)
      double wb;
      const double ekspan = lds_volatile(skl + 3 * blockDim.x);
      const bool span_ok = ekspan != 0.0;
      if constexpr (kAggRcp && MH <= 8)
        wb = span_ok ? ekspan * rcp_normal(wf) : exp_neg_cb(kj * (span - ze));
      else
        wb = span_ok ? ekspan / wf : exp_neg_cb(kj * (span - ze));
#else
      sincos_fast(th, &sn, &cs);
      const double wf = exp_neg(kj * ze), wb = exp_neg(kj * (span - ze));
#endif
      ur = q * cs;
      ui = -q * sn;
      gfr = fma(ur, wf, gfr);
      gfi = fma(ui, wf, gfi);
      gbr = fma(ur, wb, gbr);
      gbi = fma(-ui, wb, gbi);
    }
#pragma unroll
    for (int u = 0; u < NT; ++u) {
      const double bf = wk[(size_t)u * 8 * RP + k0];
      dmma_8x8x4(acc[0][u][0], acc[0][u][1], ur, bf);
      dmma_8x8x4(acc[1][u][0], acc[1][u][1], ui, bf);
    }
  }
  // g aggregates: the four lanes of a mode hold disjoint particle subsets
#pragma unroll
  for (int o = 1; o < 4; o <<= 1) {
    gfr += __shfl_xor_sync(0xffffffffu, gfr, o);
    gfi += __shfl_xor_sync(0xffffffffu, gfi, o);
    gbr += __shfl_xor_sync(0xffffffffu, gbr, o);
    gbi += __shfl_xor_sync(0xffffffffu, gbi, o);
  }
  if (!tv) return;
  const int nitems = 2 * P, nc = ncomp_of(MH);
  double2* out = carry + (size_t)c * nc * nitems;
  // accumulator (row t, cols 2kk, 2kk+1 of n-tile u) = (re, im) of pair l
#pragma unroll
  for (int u = 0; u < NT; ++u) {
    const int dir = u / (MHP / 4);
    const int l = (u % (MHP / 4)) * 4 + kk;
    if (l < MH) {
      const int item = dir == 0 ? t : P + t;
      const double sgn = dir == 0 ? 1.0 : -1.0;  // backward I input is +q sin = -ui
      SLAB_BOUND((size_t)c * nc * nitems + (size_t)(MH + l) * nitems + item,
                 (size_t)(c + 1) * nc * nitems);
      // R slot <- row 0 (q cos), I slot <- row 1 (-+ q sin); swapped pass:
      // R slot <- the I input, I slot <- minus the R input
      const double2 rs = make_double2(acc[0][u][0], acc[0][u][1]);
      const double2 is = make_double2(sgn * acc[1][u][0], sgn * acc[1][u][1]);
      out[(size_t)l * nitems + item] = swap ? is : rs;
      out[(size_t)(MH + l) * nitems + item] = swap ? make_double2(-rs.x, -rs.y) : is;
    }
  }
  if (kk == 0) {  // the g chain's input is u itself: swapped, -i u
    out[(size_t)(2 * MH) * nitems + t] = swap ? make_double2(gfi, -gfr) : make_double2(gfr, gfi);
    out[(size_t)(2 * MH) * nitems + P + t] =
        swap ? make_double2(gbi, -gbr) : make_double2(gbr, gbi);
  }
}

// ---------------------------------------------------------------------------
// phase 2: carry scan over chunks (in place: aggregates -> carried-in states)
// ---------------------------------------------------------------------------
// Lanes are 32 consecutive items of one component (contiguous in the carry
// array: every load / store is a 512-byte coalesced row); the chunk axis is cut
// into T = G * kCarrySegs segments, one warp each (grid.z = G).  Three kernels:
//   A  compose each segment's affine maps T -> D T + X          (segment maps)
//   M  exclusive scan of the T segment maps per (item, comp)     (carried-in X)
//   B  rewrite each segment's chunks with the exclusive carries
// G is chosen per plan so that few-item plans (a multi-GPU rank's mode slice)
// still expose thousands of warps.
constexpr int kCarrySegs = 32;  // warps per CTA
#ifndef SLAB_CARRY_BATCH
#define SLAB_CARRY_BATCH 4
#endif
constexpr int kCarryBatch = SLAB_CARRY_BATCH;  // loads in flight per thread (2 / 8: slower at cfg4)

__device__ __forceinline__ C2 carry_decay(bool isg, bool fwd, int c, int nch, int l, int mh,
                                          double k, const double2* __restrict__ Df,
                                          const double2* __restrict__ Db,
                                          const double* __restrict__ zbound) {
  if (isg) {
    const double dz = fwd ? (c > 0 ? zbound[c] - zbound[c - 1] : 0.0)
                          : (c + 1 < nch ? zbound[nch + c + 1] - zbound[nch + c] : 0.0);
    return C2{exp_neg(k * dz), 0.0};
  }
  const double2 d = fwd ? Df[(size_t)c * mh + l] : Db[(size_t)c * mh + l];
  return C2{d.x, d.y};
}

struct AffC {
  C2 D, X;
};
// apply a first, then b
__device__ __forceinline__ AffC acompose(const AffC& a, const AffC& b) {
  const C2 x = cmul(b.D, a.X);
  return AffC{cmul(b.D, a.D), C2{x.re + b.X.re, x.im + b.X.im}};
}

// chunk ranges: this plan scans chunks [c0, c1) of the nch global chunks (a
// z-split multi-GPU rank owns a contiguous range); segment position s maps to
// chunk c0 + s (forward items) or c1 - 1 - s (backward items)
struct CarryLane {
  int item, comp, l, t, s0, s1, c0, c1;
  bool valid, fwd, isg;
  double k;
  __device__ __forceinline__ int chunk(int s) const { return fwd ? c0 + s : c1 - 1 - s; }
};

__device__ __forceinline__ CarryLane carry_lane(int c0, int c1, int P, int items, int mh,
                                                int nseg, const double* __restrict__ modetab) {
  CarryLane c;
  const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
  c.comp = blockIdx.y;
  const int item_raw = blockIdx.x * 32 + lane;
  c.valid = item_raw < items;
  c.item = c.valid ? item_raw : items - 1;
  c.fwd = c.item < P;
  c.t = c.fwd ? c.item : c.item - P;
  c.isg = c.comp == 2 * mh;
  c.l = c.comp < mh ? c.comp : c.comp - mh;
  c.k = modetab[(size_t)c.t * mode_stride(mh) + 2];
  const int sg = blockIdx.z * kCarrySegs + seg;
  const int len = c1 - c0;
  const int per = (len + nseg - 1) / nseg;
  c.s0 = min(len, sg * per);
  c.s1 = min(len, c.s0 + per);
  c.c0 = c0;
  c.c1 = c1;
  return c;
}

__global__ void __launch_bounds__(32 * kCarrySegs) fourier_carry_compose_kernel(
    const double2* __restrict__ carry, int nch, int c0, int c1, int P, int items, int mh,
    int nseg, const double* __restrict__ modetab, const double2* __restrict__ Df,
    const double2* __restrict__ Db, const double* __restrict__ zbound, AffC* __restrict__ segmap) {
  const CarryLane c = carry_lane(c0, c1, P, items, mh, nseg, modetab);
  const int nitems = 2 * P, nc = ncomp_of(mh);
  const size_t cstride = (size_t)nc * nitems;
  const double2* base = carry + (size_t)c.comp * nitems + c.item;
  AffC M{C2{1.0, 0.0}, C2{0.0, 0.0}};
  for (int sb = c.s0; sb < c.s1; sb += kCarryBatch) {
    double2 xs[kCarryBatch];
    C2 ds[kCarryBatch];
#pragma unroll
    for (int j = 0; j < kCarryBatch; ++j) {
      const int s = sb + j;
      if (s < c.s1) {
        const int ch = c.chunk(s);
        xs[j] = base[(size_t)ch * cstride];
        ds[j] = carry_decay(c.isg, c.fwd, ch, nch, c.l, mh, c.k, Df, Db, zbound);
      }
    }
#pragma unroll
    for (int j = 0; j < kCarryBatch; ++j)
      if (sb + j < c.s1) M = acompose(M, AffC{ds[j], C2{xs[j].x, xs[j].y}});
  }
  if (c.valid) {
    const int sg = blockIdx.z * kCarrySegs + (threadIdx.x >> 5);
    segmap[((size_t)sg * nc + c.comp) * items + c.item] = M;
  }
}

// one warp per (item, comp) chain: segmap[s].X <- exclusive prefix X (T0 = 0).
// Lane j composes a contiguous run of segments, a shuffle scan composes the
// lanes, then each lane rewrites its run.
// mode 0: exclusive prefixes with carried-in state tin[chain] (NULL = 0);
// mode 1: only the range's total map -> total[chain] (z-split phase 1).
__global__ void __launch_bounds__(128) fourier_carry_segscan_kernel(
    AffC* __restrict__ segmap, int items, int nc, int nseg, const double2* __restrict__ tin,
    AffC* __restrict__ total, int mode) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // chain
  const int lane = threadIdx.x & 31;
  if (e >= items * nc) return;
  const size_t stride = (size_t)nc * items;
  AffC* m = segmap + e;
  const int per = (nseg + 31) / 32;
  const int s0 = min(nseg, lane * per), s1 = min(nseg, s0 + per);
  AffC M{C2{1.0, 0.0}, C2{0.0, 0.0}};
  for (int s = s0; s < s1; ++s) M = acompose(M, m[(size_t)s * stride]);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    AffC u;
    u.D = C2{__shfl_up_sync(0xffffffffu, M.D.re, o), __shfl_up_sync(0xffffffffu, M.D.im, o)};
    u.X = C2{__shfl_up_sync(0xffffffffu, M.X.re, o), __shfl_up_sync(0xffffffffu, M.X.im, o)};
    if (lane >= o) M = acompose(u, M);
  }
  if (mode == 1) {  // lane 31 holds the inclusive composition of every segment
    if (lane == 31) total[e] = M;
    return;
  }
  AffC pre;
  pre.D = C2{__shfl_up_sync(0xffffffffu, M.D.re, 1), __shfl_up_sync(0xffffffffu, M.D.im, 1)};
  pre.X = C2{__shfl_up_sync(0xffffffffu, M.X.re, 1), __shfl_up_sync(0xffffffffu, M.X.im, 1)};
  if (lane == 0) pre = AffC{C2{1.0, 0.0}, C2{0.0, 0.0}};
  if (tin) {  // state entering the range: X <- D T_in + X
    const double2 t2 = tin[e];
    const C2 dx = cmul(pre.D, C2{t2.x, t2.y});
    pre.X = C2{dx.re + pre.X.re, dx.im + pre.X.im};
  }
  for (int s = s0; s < s1; ++s) {
    AffC* ms = m + (size_t)s * stride;
    const AffC cur = *ms;
    ms->X = pre.X;
    pre = acompose(pre, cur);
  }
}

// The same scan with one THREAD per chain, segments in sequence: used when
// there are few segments (nseg <= kSegSeqMax) and many chains (small systems,
// full mode sums), where the warp form's per-lane segment rows are uncoalesced
// (cfg1: 0.079 ms).  Consecutive chains are consecutive in each segment row.
constexpr int kSegSeqMax = 64;
__global__ void __launch_bounds__(128) fourier_carry_segscan_seq_kernel(
    AffC* __restrict__ segmap, int items, int nc, int nseg, const double2* __restrict__ tin,
    AffC* __restrict__ total, int mode) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // chain
  if (e >= items * nc) return;
  const size_t stride = (size_t)nc * items;
  AffC* m = segmap + e;
  AffC pre{C2{1.0, 0.0}, C2{0.0, 0.0}};
  if (mode == 0 && tin) {
    const double2 t2 = tin[e];
    pre.X = C2{t2.x, t2.y};
  }
  constexpr int B = 4;
  for (int s0 = 0; s0 < nseg; s0 += B) {
    AffC cur[B];
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (s0 + j < nseg) cur[j] = m[(size_t)(s0 + j) * stride];
#pragma unroll
    for (int j = 0; j < B; ++j)
      if (s0 + j < nseg) {
        if (mode == 0) m[(size_t)(s0 + j) * stride].X = pre.X;
        pre = acompose(pre, cur[j]);
      }
  }
  if (mode == 1) total[e] = pre;
}

__global__ void __launch_bounds__(32 * kCarrySegs) fourier_carry_rewrite_kernel(
    double2* __restrict__ carry, int nch, int c0, int c1, int P, int items, int mh, int nseg,
    const double* __restrict__ modetab, const double2* __restrict__ Df,
    const double2* __restrict__ Db, const double* __restrict__ zbound,
    const AffC* __restrict__ segmap) {
  const CarryLane c = carry_lane(c0, c1, P, items, mh, nseg, modetab);
  if (!c.valid) return;
  const int nitems = 2 * P, nc = ncomp_of(mh);
  const size_t cstride = (size_t)nc * nitems;
  double2* base = carry + (size_t)c.comp * nitems + c.item;
  const int sg = blockIdx.z * kCarrySegs + (threadIdx.x >> 5);
  C2 T = segmap[((size_t)sg * nc + c.comp) * items + c.item].X;
  for (int sb = c.s0; sb < c.s1; sb += kCarryBatch) {
    double2 xs[kCarryBatch];
    C2 ds[kCarryBatch];
#pragma unroll
    for (int j = 0; j < kCarryBatch; ++j) {
      const int s = sb + j;
      if (s < c.s1) {
        const int ch = c.chunk(s);
        xs[j] = base[(size_t)ch * cstride];
        ds[j] = carry_decay(c.isg, c.fwd, ch, nch, c.l, mh, c.k, Df, Db, zbound);
      }
    }
#pragma unroll
    for (int j = 0; j < kCarryBatch; ++j) {
      const int s = sb + j;
      if (s < c.s1) {
        const int ch = c.chunk(s);
        base[(size_t)ch * cstride] = make_double2(T.re, T.im);
        const C2 nt = cmul(ds[j], T);
        T = C2{nt.re + xs[j].x, nt.im + xs[j].y};
      }
    }
  }
}

// z-split phase 2: state entering rank r's chunk range, per (comp, item) chain,
// from every rank's total map (gathered [W][nc][items]): forward items compose
// ranks 0 .. r-1, backward items ranks W-1 .. r+1 (their chunk order runs down).
__global__ void fourier_zsplit_tin_kernel(const AffC* __restrict__ totals, int W, int r,
                                          int items, int nc, int P, double2* __restrict__ tin) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= items * nc) return;
  const int item = e % items;
  const bool fwd = item < P;
  AffC pre{C2{1.0, 0.0}, C2{0.0, 0.0}};
  if (fwd) {
    for (int q = 0; q < r; ++q) pre = acompose(pre, totals[(size_t)q * nc * items + e]);
  } else {
    for (int q = W - 1; q > r; --q) pre = acompose(pre, totals[(size_t)q * nc * items + e]);
  }
  tin[e] = make_double2(pre.X.re, pre.X.im);
}

// segment groups: enough CTAs to fill the GPU, at least ~16 chunks per segment
static int carry_groups(int nch, int items, int mh) {
  if (items <= 0) return 1;
  const int ctas = ((items + 31) / 32) * ncomp_of(mh);
  int g = (2 * 148 + ctas - 1) / ctas;
  const int gmax = nch / (kCarrySegs * 16);
  if (g > gmax) g = gmax;
  return g < 1 ? 1 : g;
}

// ---------------------------------------------------------------------------
// phase 3: exact recurrence from the carried-in state + fused epilogue
// ---------------------------------------------------------------------------
// Scaled state: per pair l the lane keeps H^R_l = C_l R_l and H^I_l = C_l I_l
// (C_l = 2 c_l, k-dependent), so
//   sum_l 2Re(c_l R_l) = sum_l Re(H^R_l)               (no C in the loop body)
//   sum_l 2Re(c_l b_l R_l) = sum_l Re(b_l H^R_l)        (b_l k-independent: kernel param)
// and the real input enters as H += C_l u.  C_l lives in shared memory
// (per-lane column), which keeps the 8-pair kernel at <= 168 registers: two
// 6-warp CTAs per SM (3 warps per sub-partition) without spills.
// Lanes (force plans, `paired`): a warp holds 16 modes, forward in lanes 0-15
// and backward in 16-31, so every warp has the same shape.  Energy-only plans
// (forward items only) keep consecutive items per lane.
// Forces: lanes stage (Fx, Fy, Fz) of each particle transposed in shared memory
// (one row per component, one column per lane); a batch of 4 particles is 12
// rows, and while the next batch is computed 24 lanes sum the previous batch's
// rows, one (row, half-warp) each and 4 columns per particle step, so the
// transposed reduction is spread through the recurrence instead of stalling the
// warp every 4 particles (measured: the batched flush cost 12% of the sweep).
// Each warp writes its forward and backward sums to two partial buffers of its
// own, reduced in fixed order afterwards: deterministic, no atomics.
template <int MH, bool kSwap>
__global__ void __launch_bounds__(sweep_max_threads(MH), sweep_min_blocks(MH)) fourier_sweep_kernel(
    const double* __restrict__ xs, const double* __restrict__ ys, const double* __restrict__ zs,
    const double* __restrict__ qs, const double2* __restrict__ dtab, int64_t n, int R,
    const double* __restrict__ modetab, int P, int units, int upg, int paired, BVec b,
    const double2* __restrict__ carry, double* __restrict__ epart, double* __restrict__ fpart,
    int want_forces, int c0) {
  extern __shared__ double4 smem4[];
  const int nwarps = blockDim.x >> 5;
  double2* sC = reinterpret_cast<double2*>(smem4);         // [MH][blockDim]
  double2* sd = sC + MH * blockDim.x;                      // (R + 1) * MH
  double* sx = reinterpret_cast<double*>(sd + (R + 1) * MH);
  double* sy = sx + R;
  double* sq = sy + R;
  double* sz = sq + R;                                     // R + 2 (halo below / above)
  double* stage = sz + R + 2;                              // nwarps * 2 * kStageBuf

  const int c = c0 + blockIdx.x, g = blockIdx.y;
  const int64_t a0 = (int64_t)c * R;
  const int len = (int)(a0 + R < n ? R : n - a0);
  const int64_t a1 = a0 + len;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    sx[i] = xs[a0 + i];
    sy[i] = ys[a0 + i];
    sq[i] = qs[a0 + i];
    sz[i + 1] = zs[a0 + i];
  }
  if (threadIdx.x == 0) {
    sz[0] = zs[a0 > 0 ? a0 - 1 : 0];
    sz[len + 1] = zs[a1 < n ? a1 : a1 - 1];
  }
  for (int e = threadIdx.x; e < nwarps * 2 * kStageBuf; e += blockDim.x) stage[e] = 0.0;
#if !SLAB_SWEEP_GDECAY
  for (int e = threadIdx.x; e < (len + 1) * MH; e += blockDim.x) sd[e] = dtab[a0 * MH + e];
#endif

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nitems = 2 * P;
  const int gend = min(units, (g + 1) * upg);  // units: modes (paired) or items
  int item;
  bool active, fwd;
  if (paired) {
    const int tm = g * upg + 16 * warp + (lane & 15);
    fwd = lane < 16;
    active = tm < gend;
    item = fwd ? tm : P + tm;
  } else {
    item = g * upg + threadIdx.x;
    active = item < gend;
    fwd = item < P;
  }
  const int t = active ? (fwd ? item : item - P) : 0;
  const unsigned fmask = __ballot_sync(0xffffffffu, active && fwd);
  const unsigned bmask = __ballot_sync(0xffffffffu, active && !fwd);

  const double* mt = modetab + (size_t)t * mode_stride(MH);
  const double kx = mt[0], ky = mt[1], k = mt[2];
  const double sigma = fwd ? 1.0 : -1.0;
  const double fxy_c = active ? sigma * mt[3] : 0.0;  // +-ck
  const double fz_c = active ? -sigma * mt[4] : 0.0;  // -+cz
  const double kappa = mt[5];
  const double two_k = 2.0 * k;
  const int nc = ncomp_of(MH);
  C2 HR[MH], HI[MH];
#if SLAB_SWEEP_CREG
  C2 CR[MH];  // C_l per lane in registers (168-register budget)
#endif
  C2 gk{0.0, 0.0};
  {
    const double2* cin = carry + (size_t)c * nc * nitems + (active ? item : 0);
#pragma unroll
    for (int l = 0; l < MH; ++l) {
      const C2 cl{mt[8 + 2 * l], mt[9 + 2 * l]};
#if SLAB_SWEEP_CREG
      CR[l] = cl;
#else
      sC[l * blockDim.x + threadIdx.x] = make_double2(cl.re, cl.im);
#endif
      const double2 r = cin[(size_t)l * nitems], im = cin[(size_t)(MH + l) * nitems];
      HR[l] = cmul(cl, C2{r.x, r.y});
      HI[l] = cmul(cl, C2{im.x, im.y});
    }
    const double2 gg = cin[(size_t)(2 * MH) * nitems];
    gk = C2{gg.x, gg.y};
  }
  __syncthreads();
  if ((fmask | bmask) == 0u) return;  // no items in this warp (its buffer is skipped)

  // partial force buffers: two per (group, warp), forward and backward half
  const int gw = g * nwarps + warp;
  const double2* sCl = sC + threadIdx.x;
  double* st = stage + warp * 2 * kStageBuf;
  const int scol = lane + (lane >> 4);  // staging column of this lane
  // the summing role of this lane: row r (slot r / 3, component r % 3) of half h
  const int rr = lane < 16 ? (lane & 7) : 8 + (lane & 3);
  const int rh = lane < 16 ? (lane >> 3) : ((lane - 16) >> 2) & 1;
  const bool rsum = lane < 24;
  const int rslot = rr / 3;
  const int roff = rr * kStageStride + 17 * rh;
  // destination of the row sum for chunk particle p: forward p, backward len-1-p
  double* const rdst = fpart + (size_t)(2 * gw + rh) * n * 3 +
                       (rh ? (a0 + len - 1) * 3 : a0 * 3) + (rr - 3 * rslot);
  const int rstep = rh ? -3 : 3;
  double facc = 0.0;
  double E = 0.0;
  // Software pipeline: the k-dependent transcendentals of the NEXT particle
  // (sincos of theta, e^{-k dz}) are issued in the same basic block as this
  // particle's recurrence, so their dependency chains interleave.
  auto phase = [&](int i, double& cs_, double& sn_, double& dk_, double& q_) {
    const int ia = fwd ? i : len - 1 - i;
    const double dz = fwd ? (sz[ia + 1] - sz[ia]) : (sz[ia + 2] - sz[ia + 1]);
    const double th = __dadd_rn(__dmul_rn(kx, sx[ia]), __dmul_rn(ky, sy[ia]));
#if SLAB_SWEEP_CB == 1
    dk_ = exp_neg_cb(k * dz);
    sincos_fast_cb(th, &sn_, &cs_);
#else
    dk_ = exp_neg(k * dz);
    sincos_fast(th, &sn_, &cs_);
#endif
    q_ = sq[ia];
  };
  double cs, sn, dk, q;
#if SLAB_SWEEP_PIPE
  phase(0, cs, sn, dk, q);
#endif
  for (int i = 0; i < len; ++i) {
#if SLAB_SWEEP_PIPE
    double cs_n, sn_n, dk_n, q_n;
    phase(i + 1 < len ? i + 1 : i, cs_n, sn_n, dk_n, q_n);
#else
    phase(i, cs, sn, dk, q);
#endif
    const int ia = fwd ? i : len - 1 - i;
    const int id = fwd ? ia : ia + 1;
    // S_a = T_{a-1} * d_a  (forward) / T'_{a+1} * d_{a+1} (backward)
#pragma unroll
    for (int l = 0; l < MH; ++l) {
#if SLAB_SWEEP_GDECAY  // experiment: decays straight from global memory (L1), not staged
      const double2 d = __ldg(dtab + (a0 + id) * MH + l);
#else
      const double2 d = sd[id * MH + l];
#endif
      HR[l] = cmul(HR[l], C2{d.x, d.y});
      HI[l] = cmul(HI[l], C2{d.x, d.y});
    }
    gk.re *= dk;
    gk.im *= dk;
    double sgr = 0.0, sgi = 0.0, sbr = 0.0, sbi = 0.0;
#pragma unroll
    for (int l = 0; l < MH; ++l) {
      sgr += HR[l].re;
      sgi += HI[l].re;
#if SLAB_SWEEP_NOB  // timing probe only (wrong results): the b-weighted readouts without b
      sbr += HR[l].re - HR[l].im;
      sbi += HI[l].re - HI[l].im;
#else
      sbr = fma(b.re[l], HR[l].re, fma(-b.im[l], HR[l].im, sbr));
      sbi = fma(b.re[l], HI[l].re, fma(-b.im[l], HI[l].im, sbi));
#endif
    }
    const double ps = sigma * sn;  // phase e^{+-i theta} = (cs, ps)
    const double pr = fma(kappa, gk.re, -two_k * sgr);
    const double pi = fma(kappa, gk.im, -two_k * sgi);
    const double er = fma(cs, pr, -ps * pi);
    const double ei = fma(cs, pi, ps * pr);
    E = fma(q, er, E);
    if (want_forces) {
      const double ztr = fma(2.0, sbr, -kappa * gk.re);
      const double zti = fma(2.0, sbi, -kappa * gk.im);
      const double fxy = fxy_c * q * ei;
      const int slot = i & 3;
      double* cur = st + ((i >> 2) & 1) * kStageBuf;
      const double* prv = st + (((i >> 2) & 1) ^ 1) * kStageBuf + roff + 4 * slot;
      __syncwarp();  // orders the previous batch's rows before their sums (and
                     // those sums' reads before this buffer's reuse)
      facc += prv[0];
      facc += prv[1];
      facc += prv[2];
      facc += prv[3];
      cur[(slot * 3 + 0) * kStageStride + scol] = fxy * kx;
      cur[(slot * 3 + 1) * kStageStride + scol] = fxy * ky;
      cur[(slot * 3 + 2) * kStageStride + scol] = fz_c * q * fma(cs, ztr, -ps * zti);
      if (slot == 3) {  // the previous batch (particles i - 7 .. i - 4) is summed
        if (rsum && i >= 7) {
          SLAB_BOUND(a0 + i - 7 + rslot, n);
          rdst[rstep * (i - 7 + rslot)] = facc;
        }
        facc = 0.0;
      }
    }
    // T_a = S_a + u_a: real input scaled by C_l into the scaled state
    const double ur0 = q * cs, ui0 = -sigma * q * sn;
    const double ur = kSwap ? ui0 : ur0, ui = kSwap ? -ur0 : ui0;
#pragma unroll
    for (int l = 0; l < MH; ++l) {
#if SLAB_SWEEP_CREG
      const double2 cl = make_double2(CR[l].re, CR[l].im);
#else
      const double2 cl = sCl[l * blockDim.x];
#endif
      HR[l].re = fma(cl.x, ur, HR[l].re);
      HR[l].im = fma(cl.y, ur, HR[l].im);
      HI[l].re = fma(cl.x, ui, HI[l].re);
      HI[l].im = fma(cl.y, ui, HI[l].im);
    }
    gk.re += ur;
    gk.im += ui;
#if SLAB_SWEEP_PIPE
    cs = cs_n;
    sn = sn_n;
    dk = dk_n;
    q = q_n;
#endif
  }
  if (want_forces && len > 0) {
    // the batch before the last one (unless the last, full batch summed it) and
    // the last batch (ns particles) -- columns in the same order as in the loop
    const int bl = (len - 1) >> 2, ns = len - 4 * bl;
    if (ns < 4 && bl >= 1) {
      const double* prv = st + ((bl & 1) ^ 1) * kStageBuf + roff;
      for (int j = 4 * ns; j < 16; ++j) facc += prv[j];
      if (rsum) {
        SLAB_BOUND(a0 + 4 * (bl - 1) + rslot, n);
        rdst[rstep * (4 * (bl - 1) + rslot)] = facc;
      }
    }
    __syncwarp();
    const double* lst = st + (bl & 1) * kStageBuf + roff;
    double a = 0.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) a += lst[j];
    if (rsum && rslot < ns) {
      SLAB_BOUND(a0 + 4 * bl + rslot, n);
      rdst[rstep * (4 * bl + rslot)] = a;
    }
  }
  if (active && fwd) epart[(size_t)c * P + t] = E;
}

// ---------------------------------------------------------------------------
// the remainder sweep: the last (items mod 32) items of every chunk
// ---------------------------------------------------------------------------
// A partial warp costs the fp64 pipe as much as a full one (measured at cfg4:
// P = 100 -> 200 items = 6 full warps + 8 lanes took 4.18 ms, P = 112 -> 7 full
// warps 4.16 ms, P = 96 -> 6 warps 3.63 ms).  So the main sweep runs the full
// warps only and this kernel packs the leftover L <= 16 items of G = 32 / L
// consecutive chunks into one warp: lane group g (L lanes) walks chunk
// c0 + G w + g.  The groups walk different particles, so nothing is staged in
// shared memory: particle data and decay rows come straight from global memory
// (read once per group; small next to the main sweep).  Same recurrence and
// epilogue as fourier_sweep_kernel; a group's force contributions are summed
// in fixed order over its lanes of each direction into the remainder's own
// forward / backward partial buffers (each particle has one remainder group):
// deterministic.
constexpr int kRemWarps = 4;
constexpr int kRemSB = 4;  // steps per force flush
#ifndef SLAB_REM_MINB
#define SLAB_REM_MINB 1
#endif
#ifndef SLAB_REM_MINB2
#define SLAB_REM_MINB2 3  // (3 x 4 warps x 168 registers fill the register file)
#endif
constexpr int kRemMinB2 = SLAB_REM_MINB2;
// SPL = 2 (opt-in, SLAB_REM_SPL=2, from 4 pairs): an item's pairs are split
// over two lanes (half h carries pairs [h MS, h MS + MS)); their readout sums
// are combined with one shuffle per sum, the transcendentals and the g chain
// run on both lanes, and half 0 alone stages forces and writes the energy.
// Twice the warps and half the state per lane -- measured slower (section
// 4.1 of DESIGN.md), kept as the experiment's switch.
template <int MH, bool kSwap, int SPL>
__global__ void __launch_bounds__(32 * kRemWarps, SPL == 2 ? (MH <= 8 ? kRemMinB2 : 2) : SLAB_REM_MINB) fourier_sweep_rem_kernel(
    const double* __restrict__ xs, const double* __restrict__ ys, const double* __restrict__ zs,
    const double* __restrict__ qs, const double2* __restrict__ dtab, int64_t n, int R,
    const double* __restrict__ modetab, int P, int unit0, int L, int paired, int G, BVec b,
    const double2* __restrict__ carry, double* __restrict__ epart, double* __restrict__ frem,
    int want_forces, int c0, int c1) {
  constexpr int MS = (MH + SPL - 1) / SPL;  // pairs per lane
  __shared__ double stg[kRemWarps][kRemSB * 32 * 3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wg = blockIdx.x * kRemWarps + warp;
  const int LS = L * SPL;  // lanes per chunk group
  const int grp = lane / LS;
  const int hs = (lane % LS) / L;  // pair half of this lane
  const int c = c0 + wg * G + grp;
  const bool active = lane < G * LS && c < c1;
  // paired: the group's first L/2 lanes (of each half) are modes unit0..
  // forward, the rest the same modes backward; otherwise L consecutive
  // (forward) items
  const int Ld = paired ? L / 2 : L;
  const int jl = lane % L;
  const int item = jl < Ld ? unit0 + jl : P + unit0 + (jl - Ld);
  const bool fwd = item < P;
  const int t = fwd ? item : item - P;
  const int nitems = 2 * P;
  const int64_t a0 = active ? (int64_t)c * R : 0;
  const int len = active ? (int)(a0 + R < n ? R : n - a0) : 0;
  const double* mt = modetab + (size_t)t * mode_stride(MH);
  const double kx = mt[0], ky = mt[1], k = mt[2];
  const double sigma = fwd ? 1.0 : -1.0;
  const bool owner = active && hs == 0;  // stages forces, writes the energy
  const double fxy_c = owner ? sigma * mt[3] : 0.0;
  const double fz_c = owner ? -sigma * mt[4] : 0.0;
  const double kappa = mt[5];
  const double two_k = 2.0 * k;
  const int nc = ncomp_of(MH);
  const int lb = hs * MS;  // first pair of this lane
  C2 HR[MS], HI[MS], CL[MS];
  double bre[MS], bim[MS];
  C2 gk{0.0, 0.0};
  {
    const double2* cin = carry + (size_t)(active ? c : c0) * nc * nitems + item;
#pragma unroll
    for (int ll = 0; ll < MS; ++ll) {
      const bool on = lb + ll < MH;  // (odd MH: the last half is one pair short)
      const int l = on ? lb + ll : 0;
      CL[ll] = on ? C2{mt[8 + 2 * l], mt[9 + 2 * l]} : C2{0.0, 0.0};
      bre[ll] = 0.0;
      bim[ll] = 0.0;
#pragma unroll
      for (int h = 0; h < SPL; ++h)
        if (h * MS + ll < MH && hs == h) {
          bre[ll] = b.re[h * MS + ll];
          bim[ll] = b.im[h * MS + ll];
        }
      const double2 r = cin[(size_t)l * nitems], im = cin[(size_t)(MH + l) * nitems];
      HR[ll] = cmul(CL[ll], C2{r.x, r.y});
      HI[ll] = cmul(CL[ll], C2{im.x, im.y});
    }
    const double2 gg = cin[(size_t)(2 * MH) * nitems];
    gk = C2{gg.x, gg.y};
  }
  double E = 0.0;
  // Positions, charge and the two z values of the step's dz are loaded TWO
  // steps ahead and only combined (dz, sincos, e^{-k dz}) one step ahead: a
  // warp stalls at the first use of a pending load, and this kernel has only
  // a few warps per SM to hide it (round 1 formed dz and the transcendentals
  // right after the loads: a quarter of its stall samples waited there).
  // Decay rows one step ahead.  Forces are staged for kRemSB steps and summed
  // per group in one pass.
  double px = 0.0, py = 0.0, pq = 0.0, pz1 = 0.0, pz0 = 0.0;  // step i + 2 (in flight)
  double2 nd[MS];                                              // step i + 1
  auto fetch_xyz = [&](int i) {
    const bool live = i < len;
    const int ia = fwd ? i : len - 1 - i;
    const int64_t ag = live ? a0 + ia : 0;
    // dz = z[hi] - z[lo]: forward (a - 1, a), backward (a, a + 1); 0 at the
    // ends (the forward chunk start is the carry's, the global end has none)
    const int64_t hi = fwd ? ag : (ag + 1 < n ? ag + 1 : ag);
    const int64_t lo = fwd ? (ag > 0 ? ag - 1 : ag) : ag;
    px = __ldg(xs + ag);
    py = __ldg(ys + ag);
    pq = live ? __ldg(qs + ag) : 0.0;
    pz1 = __ldg(zs + hi);
    pz0 = __ldg(zs + lo);
  };
  auto fetch_d = [&](int i) {
    const bool live = i < len;
    const int ia = fwd ? i : len - 1 - i;
    const int64_t ag = live ? a0 + ia : 0;
    const int64_t drow = live ? (fwd ? ag : ag + 1) : 0;
#pragma unroll
    for (int ll = 0; ll < MS; ++ll)
      nd[ll] = lb + ll < MH ? __ldg(dtab + drow * MH + lb + ll) : make_double2(0.0, 0.0);
  };
  double ncs, nsn, ndk, nq;
  auto trans = [&]() {  // transcendentals of the step whose data is in p*
    ndk = exp_neg(k * (pz1 - pz0));
    sincos_fast(__dadd_rn(__dmul_rn(kx, px), __dmul_rn(ky, py)), &nsn, &ncs);
    nq = pq;
  };
  fetch_xyz(0);
  fetch_d(0);
  trans();
  fetch_xyz(1);
  double* st = stg[warp];
  for (int i = 0; i < R; ++i) {
    const bool live = i < len;
    const double q = nq, cs = ncs, sn = nsn, dk = ndk;
    double2 dd[MS];
#pragma unroll
    for (int ll = 0; ll < MS; ++ll) dd[ll] = nd[ll];
    if (i + 1 < R) {
      fetch_d(i + 1);
      trans();
      fetch_xyz(i + 2);
    }
#pragma unroll
    for (int ll = 0; ll < MS; ++ll) {
      HR[ll] = cmul(HR[ll], C2{dd[ll].x, dd[ll].y});
      HI[ll] = cmul(HI[ll], C2{dd[ll].x, dd[ll].y});
    }
    gk.re *= dk;
    gk.im *= dk;
    // readout sums as two interleaved chains each (dependent-latency bound)
    double sgr = 0.0, sgi = 0.0, sbr = 0.0, sbi = 0.0;
    double sgr1 = 0.0, sgi1 = 0.0, sbr1 = 0.0, sbi1 = 0.0;
#pragma unroll
    for (int ll = 0; ll < MS; ll += 2) {
      sgr += HR[ll].re;
      sgi += HI[ll].re;
      sbr = fma(bre[ll], HR[ll].re, fma(-bim[ll], HR[ll].im, sbr));
      sbi = fma(bre[ll], HI[ll].re, fma(-bim[ll], HI[ll].im, sbi));
      if (ll + 1 < MS) {
        sgr1 += HR[ll + 1].re;
        sgi1 += HI[ll + 1].re;
        sbr1 = fma(bre[ll + 1], HR[ll + 1].re, fma(-bim[ll + 1], HR[ll + 1].im, sbr1));
        sbi1 = fma(bre[ll + 1], HI[ll + 1].re, fma(-bim[ll + 1], HI[ll + 1].im, sbi1));
      }
    }
    sgr += sgr1;
    sgi += sgi1;
    sbr += sbr1;
    sbi += sbi1;
    if constexpr (SPL == 2) {  // the item's other half (lane -+ L), fixed order
      const int pl = hs ? lane - L : lane + L;
      const double o0 = __shfl_sync(0xffffffffu, sgr, pl);
      const double o1 = __shfl_sync(0xffffffffu, sgi, pl);
      const double o2 = __shfl_sync(0xffffffffu, sbr, pl);
      const double o3 = __shfl_sync(0xffffffffu, sbi, pl);
      sgr = hs ? o0 + sgr : sgr + o0;
      sgi = hs ? o1 + sgi : sgi + o1;
      sbr = hs ? o2 + sbr : sbr + o2;
      sbi = hs ? o3 + sbi : sbi + o3;
    }
    const double ps = sigma * sn;
    const double pr = fma(kappa, gk.re, -two_k * sgr);
    const double pi = fma(kappa, gk.im, -two_k * sgi);
    const double er = fma(cs, pr, -ps * pi);
    const double ei = fma(cs, pi, ps * pr);
    E = fma(q, er, E);
    if (want_forces) {
      const double ztr = fma(2.0, sbr, -kappa * gk.re);
      const double zti = fma(2.0, sbi, -kappa * gk.im);
      const double fxy = fxy_c * q * ei;
      const int slot = i % kRemSB;
      double* row = st + slot * 32 * 3;
      row[lane * 3 + 0] = live ? fxy * kx : 0.0;
      row[lane * 3 + 1] = live ? fxy * ky : 0.0;
      row[lane * 3 + 2] = live ? fz_c * q * fma(cs, ztr, -ps * zti) : 0.0;
      if (slot == kRemSB - 1 || i == R - 1) {
        __syncwarp();
        // (slot, group, direction, comp) sums in fixed order over the group's
        // half-0 lanes of that direction, forward / backward into frem's two buffers
        const int ibase = i - slot;
        const int nd = paired ? 2 : 1;
        // one slot at a time, lanes over its (group, direction, comp) entries:
        // no run-time integer divisions
        for (int sl = 0; sl <= slot; ++sl)
        for (int e = lane; e < G * nd * 3; e += 32) {
          const int gd = e / 3, comp = e - 3 * gd;
          const int gg = paired ? gd >> 1 : gd, d = paired ? gd & 1 : 0;
          const int cg = c0 + wg * G + gg;
          const int64_t a0g = (int64_t)cg * R;
          const int leng = cg < c1 ? (int)(a0g + R < n ? R : n - a0g) : 0;
          const int ii = ibase + sl;
          if (ii < leng) {
            const double* rs = st + sl * 32 * 3;
            double sum = 0.0;
            for (int j = 0; j < Ld; ++j) sum += rs[(gg * LS + d * Ld + j) * 3 + comp];
            const bool dfwd = paired ? d == 0 : true;
            SLAB_BOUND(a0g + (dfwd ? ii : leng - 1 - ii), n);
            frem[(size_t)d * n * 3 + (a0g + (dfwd ? ii : leng - 1 - ii)) * 3 + comp] = sum;
          }
        }
        __syncwarp();
      }
    }
    const double ur0 = q * cs, ui0 = -sigma * q * sn;
    const double ur = kSwap ? ui0 : ur0, ui = kSwap ? -ur0 : ui0;
#pragma unroll
    for (int ll = 0; ll < MS; ++ll) {
      HR[ll].re = fma(CL[ll].re, ur, HR[ll].re);
      HR[ll].im = fma(CL[ll].im, ur, HR[ll].im);
      HI[ll].re = fma(CL[ll].re, ui, HI[ll].re);
      HI[ll].im = fma(CL[ll].im, ui, HI[ll].im);
    }
    gk.re += ur;
    gk.im += ui;
  }
  if (owner && fwd) epart[(size_t)c * P + t] = E;
}

// per-mode sums over chunks (one block per mode, fixed-order tree), then Kahan
// over modes in mode order exactly like soewald2d.py:204-207
__global__ void __launch_bounds__(256) fourier_mode_energy_kernel(
    const double* __restrict__ epart, int c0, int c1, int P, int mh,
    const double* __restrict__ modetab, const double* __restrict__ esing,
    double* __restrict__ se) {
  __shared__ double red[256];
  const int t = blockIdx.x;
  double s = 0.0;
  for (int c = c0 + threadIdx.x; c < c1; c += 256) s += epart[(size_t)c * P + t];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0)
    se[t] = modetab[(size_t)t * mode_stride(mh) + 3] * red[0] + (esing ? esing[t] : 0.0);
}

// Kahan over modes in mode order exactly like soewald2d.py:204-207, one thread
// per segment of seg_len consecutive modes (one segment = the whole sum)
// Compensated sum of each segment of per-mode energies: one block per segment,
// each thread a Kahan sum over a strided subset, then a fixed-order tree of
// (sum, error) pairs combined with TwoSum -- deterministic, and as accurate as
// the reference's sequential Kahan loop (a single thread walking 792 modes of
// the cfg1 full sum in sequence took 0.029 ms).
constexpr int kKahanThreads = 128;
__device__ __forceinline__ void two_sum_acc(double& s, double& e, double s2, double e2) {
  const double t = s + s2;
  const double bp = t - s;
  const double err = (s - (t - bp)) + (s2 - bp);
  s = t;
  e = e + e2 + err;
}
__global__ void __launch_bounds__(kKahanThreads) kahan_modes_kernel(
    const double* __restrict__ se, int nseg, int seg_len, double* __restrict__ out) {
  __shared__ double rs[kKahanThreads], re[kKahanThreads];
  const int s = blockIdx.x;
  double u = 0.0, comp = 0.0;
  for (int t = threadIdx.x; t < seg_len; t += kKahanThreads) {
    const double y = se[(size_t)s * seg_len + t] - comp;
    const double tt = u + y;
    comp = (tt - u) - y;
    u = tt;
  }
  rs[threadIdx.x] = u;
  re[threadIdx.x] = -comp;
  __syncthreads();
  for (int w = kKahanThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      double a = rs[threadIdx.x], b = re[threadIdx.x];
      two_sum_acc(a, b, rs[threadIdx.x + w], re[threadIdx.x + w]);
      rs[threadIdx.x] = a;
      re[threadIdx.x] = b;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[s] = rs[0] + re[0];
}

// forces_sorted += sum of the per-warp partial buffers (fixed order)
// Buffers b < 2 * ngroups * nwarps: (forward, backward) of warp (b / 2) % nwarps
// of group b / (2 nwarps), written only if that warp holds modes; the rest are
// the remainder sweep's.
// NS > 1 (few particles, many buffers: small systems with full mode sums): NS
// lanes per element take the buffers round robin and combine by a fixed
// xor-shuffle tree (deterministic).
template <int NS>
__global__ void fourier_force_reduce_kernel(const double* __restrict__ fpart, int b_lo,
                                            int nbuf, int ngroups, int nwarps, int upg,
                                            int units, int64_t n3, double* __restrict__ out,
                                            int64_t e0, int64_t e1) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int sub = (int)(t % NS);
  const int64_t e = e0 + t / NS;
  const bool live = e < e1;
  auto written = [&](int b) {
    if (b >= 2 * ngroups * nwarps) return true;  // the remainder's
    const int g = b / (2 * nwarps), w = (b >> 1) - g * nwarps;
    return 16 * w < min(units, (g + 1) * upg) - g * upg;
  };
  // four independent loads in flight per thread (one at a time left the kernel
  // latency-bound at ~45% of HBM bandwidth); the adds keep buffer order
  double v = 0.0;
  if (live) {
    int b = b_lo + sub;
    for (; b + 3 * NS < nbuf; b += 4 * NS) {
      double x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        x[u] = written(b + u * NS) ? fpart[(size_t)(b + u * NS) * n3 + e] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) v += x[u];
    }
    for (; b < nbuf; b += NS)
      if (written(b)) v += fpart[(size_t)b * n3 + e];
  }
#pragma unroll
  for (int o = 1; o < NS; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (live && sub == 0) out[e] += v;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t sweep_smem(int R, int mh, int warps) {
  return sizeof(double2) * (size_t)mh * warps * 32 + sizeof(double2) * (size_t)(R + 1) * mh +
         sizeof(double) * (3 * (size_t)R + R + 2) +
         sizeof(double) * (size_t)warps * 2 * kStageBuf;
}

FourierPlan fourier_plan(int64_t n, int P, int mh, int dirs, int ranks) {
  FourierPlan p{};
  p.n = n;
  p.P = P;
  p.mh = mh;
  // energy-only evaluations need only the forward sweep (the reference's energy
  // is the forward sum, soewald2d.py:138-170; the backward sweep only adds the
  // j-side forces, 172-202): active items = dirs * P, carry layout stays 2P
  p.items = (dirs == 1 ? 1 : 2) * P;
  // force plans pair the directions: a warp = 16 modes x (forward, backward);
  // energy-only plans: a warp = 32 consecutive forward items
  p.paired = dirs == 1 ? 0 : 1;
  const int upw = p.paired ? 16 : 32;          // units (modes / items) per warp
  const int units = p.paired ? P : p.items;
  // leftover units (units mod upw, <= 8 items) go to the remainder sweep,
  // several chunks per warp; the main sweep then runs whole warps only
  p.rem = 0;
  p.rem_g = 0;
  p.rem_spl = 1;
  {
    const int left = units % upw;
    const int left_items = left * (p.paired ? 2 : 1);
    if (kSweepRem && units >= upw && left > 0 && left_items <= kSweepRemMax) {
      p.rem = left_items;
      // one lane per item; SLAB_REM_SPL=2 splits an item's pairs over two lanes
      // (from 4 pairs up): twice the warps, but measured slower at cfg4 (the
      // remainder 0.46 -> 0.65 ms in the tail, step 8.31 -> 8.42 ms)
      p.rem_spl = 1;
      if (const char* env = getenv("SLAB_REM_SPL"))
        p.rem_spl = (atoi(env) == 2 && mh >= 4 && 2 * left_items <= 32) ? 2 : 1;
      p.rem_g = 32 / (p.rem_spl * left_items);
      if (const char* env = getenv("SLAB_REM_G")) {  // tuning knob
        const int gg = atoi(env);
        if (gg >= 1 && gg <= 32 / (p.rem_spl * left_items)) p.rem_g = gg;
      }
    }
  }
  p.units_main = units - (p.rem ? units % upw : 0);
  p.items_main = p.units_main * (p.paired ? 2 : 1);
  const int maxt = sweep_max_threads(mh);
  p.ngroups = (p.items_main + maxt - 1) / maxt;
  if (p.ngroups < 1) p.ngroups = 1;
  p.upg = (p.units_main + p.ngroups - 1) / p.ngroups;
  if (p.rem || p.paired) p.upg = (p.upg + upw - 1) / upw * upw;  // groups of whole warps
  if (p.upg < 1) p.upg = 1;
  p.warps = (p.upg + upw - 1) / upw;
  if (p.warps < 1) p.warps = 1;
  // >= 4 CTAs per SM of chunks in each rank's range (a z-split rank scans 1/ranks
  // of the chunks: shorter chunks keep its sweep grid from ending on a partial wave)
  const int64_t target_ctas = 4 * 148 * (int64_t)(ranks > 1 ? ranks : 1);
  int64_t rf = n * p.ngroups / target_ctas;
  int R = 16;
  while (R * 2 <= rf && R * 2 <= kMaxR) R *= 2;
  // Few items per chunk (a multi-GPU rank's mode slice, small P) means small
  // CTAs whose shared memory -- dominated by the R-particle decay and weight
  // tables -- would cap the SM at a handful of warps: shrink R until both the
  // sweep and the aggregate reach their register-limited occupancy.
  {
    const int tiles = P > 0 ? (P + 7) / 8 : 1;
    const int ngy = (tiles + kAggMaxWarps - 1) / kAggMaxWarps;
    const int tpc = (tiles + ngy - 1) / ngy;
    auto ctas = [](size_t smem, int threads, int regs) {
      const int by_smem = (int)(kSmemPerSM / (smem + 1024));
      const int by_regs = 65536 / (regs * threads);
      return by_smem < by_regs ? (by_smem < 32 ? by_smem : 32) : (by_regs < 32 ? by_regs : 32);
    };
    const int sw_regs = sweep_min_blocks(mh) == 1 ? 255 : 65536 / (2 * maxt) / 8 * 8;
    const int sw_full = 65536 / (sw_regs * 32 * p.warps) > 0 ? 65536 / (sw_regs * 32 * p.warps) : 1;
    const int ag_full = 65536 / (kAggRegs * 32 * tpc);
    // ... but not below 64 particles: shorter chunks multiply the chunk count and
    // with it the carry scan's traffic (cfg4 at 13 modes per rank: R = 16 ->
    // 64 took the rank from 2.72 to 2.30 ms, the carries from 0.51 to 0.10 ms)
    const int r_floor = R < 64 ? R : 64;
    while (R > r_floor && (ctas(sweep_smem(R, mh, p.warps), 32 * p.warps, sw_regs) < sw_full ||
                      ctas(agg_mma_smem(R, mh), 32 * tpc, kAggRegs) < ag_full))
      R /= 2;
  }
  if (const char* env = getenv("SLAB_CHUNK_R")) {  // tuning knob (multiple of 4, 16..256)
    const int r = atoi(env);
    if (r >= 16 && r <= kMaxR && r % 4 == 0) R = r;
  }
  p.R = R;
  p.nch = (int)((n + R - 1) / R);
  p.c0 = 0;
  p.c1 = p.nch;
  p.smem_sweep = sweep_smem(R, mh, p.warps);
  // partial force buffers: forward and backward per (group, warp), then the
  // remainder's forward and backward ones
  p.nbuf = 2 * p.ngroups * p.warps;
  p.rem_buf = p.nbuf;
  if (p.rem) p.nbuf += 2;
  return p;
}

size_t fourier_work_doubles(const FourierPlan& p) {
  const size_t nitems = 2 * (size_t)p.P;
  size_t d = (size_t)p.P * mode_stride(p.mh);
  d += 2 * (size_t)p.nch * ncomp_of(p.mh) * nitems;  // carry (double2)
  d += 2 * 2 * (size_t)p.nch * p.mh;                 // Df, Db (double2)
  d += 2 * (size_t)p.nch;                            // zbound
  d += (size_t)p.nch * p.P + 2 * (size_t)p.P;        // epart + per-mode sums + singular terms
  d += (size_t)(p.nbuf + 1) * p.n * 3;               // fpart
  d += 4 * (size_t)carry_groups(p.nch, p.items, p.mh) * 32 * ncomp_of(p.mh) * p.items;  // segmap
  d += 8 * (size_t)ncomp_of(p.mh) * p.items;  // z-split carried-in states (double2) + spare
  return d + 64;
}

void fourier_work_carve(const FourierPlan& p, double* base, FourierWork& w) {
  const size_t nitems = 2 * (size_t)p.P;
  double* q = base;
  w.modetab = q;
  q += (size_t)p.P * mode_stride(p.mh);
  q += (reinterpret_cast<uintptr_t>(q) / 8) & 1;  // 16-byte align for double2
  w.carry = reinterpret_cast<double2*>(q);
  q += 2 * (size_t)p.nch * ncomp_of(p.mh) * nitems;
  w.dchunk = reinterpret_cast<double2*>(q);
  q += 4 * (size_t)p.nch * p.mh;
  w.zbound = q;
  q += 2 * (size_t)p.nch;
  w.epart = q;
  q += (size_t)p.nch * p.P + 2 * (size_t)p.P;
  w.fpart = q;
  q += (size_t)(p.nbuf + 1) * p.n * 3;
  q += (reinterpret_cast<uintptr_t>(q) / 8) & 1;
  w.segmap = q;
  q += 4 * (size_t)carry_groups(p.nch, p.items, p.mh) * 32 * ncomp_of(p.mh) * p.items;
  w.tin = q;
}

cudaError_t decay_table(const double* zs, int64_t n, int mh, const BVec& b, double2* dtab,
                        cudaStream_t st, int64_t a_lo, int64_t a_hi) {
  if (a_hi < 0 || a_hi > n) a_hi = n;
  if (a_lo < 0) a_lo = 0;
  if (a_lo > a_hi) return cudaGetLastError();
  const int64_t tot = (a_hi - a_lo + 1) * mh;
  const unsigned grid = (unsigned)((tot + 255) / 256);
  switch (mh) {
#define DCASE(K) \
  case K: decay_table_kernel<K><<<grid, 256, 0, st>>>(zs, n, b, dtab, a_lo, a_hi); break;
    DCASE(1) DCASE(2) DCASE(3) DCASE(4) DCASE(5) DCASE(6) DCASE(7) DCASE(8) DCASE(9) DCASE(10)
    DCASE(11) DCASE(12)
#undef DCASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <int MH>
static void set_attrs() {
  // function attributes are per device context: one bit per device
  static unsigned long long done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (done & bit) return;
  // largest shared-memory carveout so two CTAs of each fit per SM
  for (auto fn : {fourier_sweep_kernel<MH, false>, fourier_sweep_kernel<MH, true>}) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sweep_smem(kMaxR, MH, 8));
    cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  }
  cudaFuncSetAttribute(fourier_aggregate_mma_kernel<MH>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)agg_mma_smem(kMaxR, MH));
  cudaFuncSetAttribute(fourier_aggregate_mma_kernel<MH>,
                       cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  done |= bit;
}

static dim3 carry_grid(const FourierPlan& p) {
  return dim3((p.items + 31) / 32, ncomp_of(p.mh), carry_groups(p.c1 - p.c0, p.items, p.mh));
}

// phase 1: aggregates of chunks [c0, c1) and their segment maps; with `totals`,
// also the range's total map per (comp, item) chain (z-split exchange payload)
// identity maps T -> 1 T + 0: the exchange payload of a rank whose chunk range is
// empty or a single-chunk plan (composing it leaves the other ranks' carries intact)
__global__ void affc_identity_kernel(AffC* __restrict__ out, int count) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < count) out[e] = AffC{C2{1.0, 0.0}, C2{0.0, 0.0}};
}

template <int MH>
static cudaError_t phase1_mh(const FourierPlan& p, const FourierWork& w, const double* xs,
                             const double* ys, const double* zs, const double* qs,
                             const BVec& b, double* totals, cudaStream_t st) {
  set_attrs<MH>();
  const int nch_r = p.c1 - p.c0;
  const int nchain = p.items * ncomp_of(MH);
  if (nch_r <= 0 || p.nch <= 1) {
    if (totals)
      affc_identity_kernel<<<(nchain + 127) / 128, 128, 0, st>>>(reinterpret_cast<AffC*>(totals),
                                                                  nchain);
    if (nch_r <= 0) return cudaGetLastError();
  }
  if (p.nch > 1) {
    const int tiles = (p.P + 7) / 8;
    const int ngy = (tiles + kAggMaxWarps - 1) / kAggMaxWarps;
    const int tpc = (tiles + ngy - 1) / ngy;
    fourier_aggregate_mma_kernel<MH><<<dim3(nch_r, ngy), tpc * 32, agg_mma_smem(p.R, MH), st>>>(
        xs, ys, zs, qs, p.n, p.R, w.modetab, p.P, tpc, b, w.carry, p.c0, p.swap);
    const dim3 cg = carry_grid(p);
    const int nseg = cg.z * kCarrySegs;
    fourier_carry_compose_kernel<<<cg, 32 * kCarrySegs, 0, st>>>(
        w.carry, p.nch, p.c0, p.c1, p.P, p.items, MH, nseg, w.modetab, w.dchunk,
        w.dchunk + (size_t)p.nch * MH, w.zbound, reinterpret_cast<AffC*>(w.segmap));
    if (totals) {
      if (nseg <= kSegSeqMax)
        fourier_carry_segscan_seq_kernel<<<(nchain + 127) / 128, 128, 0, st>>>(
            reinterpret_cast<AffC*>(w.segmap), p.items, ncomp_of(MH), nseg, nullptr,
            reinterpret_cast<AffC*>(totals), 1);
      else
        fourier_carry_segscan_kernel<<<(nchain + 3) / 4, 128, 0, st>>>(
            reinterpret_cast<AffC*>(w.segmap), p.items, ncomp_of(MH), nseg, nullptr,
            reinterpret_cast<AffC*>(totals), 1);
    }
  } else {  // one chunk: carried-in state 0 (its total map was written above)
    cudaMemsetAsync(w.carry, 0, sizeof(double2) * ncomp_of(MH) * 2 * (size_t)p.P, st);
  }
  return cudaGetLastError();
}

// phase 2: carried-in states (optionally entering the range with tin), the sweep
// The remainder sweep runs on a side stream beside the main sweep (it is a
// handful of latency-bound warps: alone after the main sweep it cost the whole
// of its serial walk; beside it, it fills the SMs the main sweep leaves idle).
// One high-priority stream and a fork / join event pair per device, created on
// first use (before any graph capture: the evaluators warm up first).
struct RemSide {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static RemSide& rem_side() {
  static RemSide sides[64];
  int dev = 0;
  cudaGetDevice(&dev);
  RemSide& r = sides[dev & 63];
  if (!r.s) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&r.s, cudaStreamNonBlocking, greatest);
    cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&r.join, cudaEventDisableTiming);
  }
  return r;
}

// out[e] += sum of the partial force buffers [b_lo, b_hi) of the plan's chunk
// range, in buffer order
static void force_reduce(const FourierPlan& p, const FourierWork& w, int b_hi, int b_lo,
                         double* out, cudaStream_t st) {
  const int64_t n3 = p.n * 3;
  const int64_t e0 = (int64_t)p.c0 * p.R * 3;
  int64_t e1 = (int64_t)p.c1 * p.R * 3;
  e1 = e1 < n3 ? e1 : n3;
  if (e1 <= e0 || b_hi <= b_lo) return;
  if ((e1 - e0) < (int64_t)148 * 2048 && b_hi - b_lo >= 16)
    fourier_force_reduce_kernel<8><<<(unsigned)((8 * (e1 - e0) + 255) / 256), 256, 0, st>>>(
        w.fpart, b_lo, b_hi, p.ngroups, p.warps, p.upg, p.units_main, n3, out, e0, e1);
  else
    fourier_force_reduce_kernel<1><<<(unsigned)((e1 - e0 + 255) / 256), 256, 0, st>>>(
        w.fpart, b_lo, b_hi, p.ngroups, p.warps, p.upg, p.units_main, n3, out, e0, e1);
}

template <int MH>
static cudaError_t phase2_mh(const FourierPlan& p, const FourierWork& w, const double* xs,
                             const double* ys, const double* zs, const double* qs,
                             const double2* dtab, const BVec& b, int want_forces,
                             const double2* tin, double* forces_sorted, cudaStream_t st) {
  const int nch_r = p.c1 - p.c0;
  if (nch_r <= 0) return cudaGetLastError();
  // forces need both directions in the paired lane layout (plans with dirs = 2)
  if (want_forces && !p.paired) return cudaErrorInvalidValue;
  if (p.nch > 1) {
    const dim3 cg = carry_grid(p);
    const int nseg = cg.z * kCarrySegs;
    const int nchain = p.items * ncomp_of(MH);
    AffC* segmap = reinterpret_cast<AffC*>(w.segmap);
    if (nseg <= kSegSeqMax)
      fourier_carry_segscan_seq_kernel<<<(nchain + 127) / 128, 128, 0, st>>>(
          segmap, p.items, ncomp_of(MH), nseg, tin, nullptr, 0);
    else
      fourier_carry_segscan_kernel<<<(nchain + 3) / 4, 128, 0, st>>>(
          segmap, p.items, ncomp_of(MH), nseg, tin, nullptr, 0);
    fourier_carry_rewrite_kernel<<<cg, 32 * kCarrySegs, 0, st>>>(
        w.carry, p.nch, p.c0, p.c1, p.P, p.items, MH, nseg, w.modetab, w.dchunk,
        w.dchunk + (size_t)p.nch * MH, w.zbound, segmap);
  }
  if (p.rem) {  // the remainder sweep, forked beside the main one
    RemSide& rs = rem_side();
    cudaEventRecord(rs.fork, st);
    cudaStreamWaitEvent(rs.s, rs.fork, 0);
    const int rwarps = (nch_r + p.rem_g - 1) / p.rem_g;
    const int rblocks = (rwarps + kRemWarps - 1) / kRemWarps;
    double* frem = w.fpart + (size_t)p.rem_buf * p.n * 3;
    constexpr int kSpl = MH >= 4 ? 2 : 1;
    auto fn = p.rem_spl == 2 ? (p.swap ? fourier_sweep_rem_kernel<MH, true, kSpl>
                                       : fourier_sweep_rem_kernel<MH, false, kSpl>)
                             : (p.swap ? fourier_sweep_rem_kernel<MH, true, 1>
                                       : fourier_sweep_rem_kernel<MH, false, 1>);
    fn<<<rblocks, 32 * kRemWarps, 0, rs.s>>>(xs, ys, zs, qs, dtab, p.n, p.R, w.modetab, p.P,
                                             p.units_main, p.rem, p.paired, p.rem_g, b, w.carry,
                                             w.epart, frem, want_forces, p.c0, p.c1);
    cudaEventRecord(rs.join, rs.s);
  }
  if (p.items_main > 0) {
    if (p.swap)
      fourier_sweep_kernel<MH, true><<<dim3(nch_r, p.ngroups), p.warps * 32, p.smem_sweep, st>>>(
          xs, ys, zs, qs, dtab, p.n, p.R, w.modetab, p.P, p.units_main, p.upg, p.paired, b,
          w.carry, w.epart, w.fpart, want_forces, p.c0);
    else
      fourier_sweep_kernel<MH, false><<<dim3(nch_r, p.ngroups), p.warps * 32, p.smem_sweep, st>>>(
          xs, ys, zs, qs, dtab, p.n, p.R, w.modetab, p.P, p.units_main, p.upg, p.paired, b,
          w.carry, w.epart, w.fpart, want_forces, p.c0);
  }
  if (p.rem) {
    cudaStreamWaitEvent(st, rem_side().join, 0);
  }
  return cudaGetLastError();
}

cudaError_t fourier_phase1(const FourierPlan& p, const FourierWork& w, const double* xs,
                           const double* ys, const double* zs, const double* qs,
                           const double* modes, const double* commonv, double commonv_scalar,
                           double area, const BVec& b, const WVec& wv, int* status,
                           double* totals, cudaStream_t st) {
  if (p.P <= 0 || p.n < 2) return cudaSuccess;
  mode_table_kernel<<<(p.P + 127) / 128, 128, 0, st>>>(modes, commonv, commonv_scalar, p.P, p.mh,
                                                       area, b, wv, w.modetab, status);
  const int nb = p.nch * p.mh;
  chunk_bounds_kernel<<<(nb + 127) / 128, 128, 0, st>>>(zs, p.n, p.R, p.nch, p.mh, b, w.zbound,
                                                        w.dchunk, w.dchunk + (size_t)p.nch * p.mh);
  switch (p.mh) {
#define FCASE(K) \
  case K: return phase1_mh<K>(p, w, xs, ys, zs, qs, b, totals, st);
    FCASE(1) FCASE(2) FCASE(3) FCASE(4) FCASE(5) FCASE(6) FCASE(7) FCASE(8) FCASE(9) FCASE(10) FCASE(11)
    FCASE(12)
#undef FCASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t fourier_zsplit_tin(const FourierPlan& p, const double* totals, int W, int r,
                               double* tin, cudaStream_t st) {
  if (p.P <= 0 || p.n < 2) return cudaSuccess;
  const int nchain = p.items * ncomp_of(p.mh);
  fourier_zsplit_tin_kernel<<<(nchain + 127) / 128, 128, 0, st>>>(
      reinterpret_cast<const AffC*>(totals), W, r, p.items, ncomp_of(p.mh), p.P,
      reinterpret_cast<double2*>(tin));
  return cudaGetLastError();
}

cudaError_t fourier_phase2(const FourierPlan& p, const FourierWork& w, const double* xs,
                           const double* ys, const double* zs, const double* qs,
                           const double2* dtab, const BVec& b, int want_forces,
                           double* energy_out, double* forces_sorted, const double* tin,
                           cudaStream_t st, int seg_len) {
  if (p.P <= 0 || p.n < 2) return cudaSuccess;
  if (seg_len <= 0 || p.P % seg_len != 0) seg_len = p.P;
  const double2* tin2 = reinterpret_cast<const double2*>(tin);
  cudaError_t e = cudaErrorInvalidValue;
  switch (p.mh) {
#define FCASE(K) \
  case K: e = phase2_mh<K>(p, w, xs, ys, zs, qs, dtab, b, want_forces, tin2, forces_sorted, st); break;
    FCASE(1) FCASE(2) FCASE(3) FCASE(4) FCASE(5) FCASE(6) FCASE(7) FCASE(8) FCASE(9) FCASE(10) FCASE(11)
    FCASE(12)
#undef FCASE
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  double* se = w.epart + (size_t)p.nch * p.P;  // P scratch doubles after the partials
  double* esing = se + p.P;                    // and P for the singular-term energies
  // tables with a (near-)real exponent can put a term within 2e-6 k of a mode
  // (soewald2d.py:116-124); complex pairs with |Im b| >= 1e-5 Re b never can
  bool near_real = false;
  for (int l = 0; l < p.mh; ++l) near_real |= fabs(b.im[l]) < 1e-5 * b.re[l];
  const bool sing = near_real && p.c0 == 0 && p.c1 == p.nch;
  if (sing)
    fourier_singular_kernel<<<1, kSingThreads, 0, st>>>(xs, ys, zs, qs, p.n, w.modetab, p.mh,
                                                         p.P, p.items, want_forces, esing,
                                                         forces_sorted);
  fourier_mode_energy_kernel<<<p.P, 256, 0, st>>>(w.epart, p.c0, p.c1, p.P, p.mh, w.modetab,
                                                  sing ? esing : nullptr, se);
  const int nseg = p.P / seg_len;
  if (nseg > 0) kahan_modes_kernel<<<nseg, kKahanThreads, 0, st>>>(se, nseg, seg_len, energy_out);
  // (summing the main sweep's buffers before the remainder's join, beside it in
  // the scan's tail, measured slower: cfg4 8.31 -> 8.33 ms)
  if (want_forces) force_reduce(p, w, p.nbuf, 0, forces_sorted, st);
  return cudaGetLastError();
}

// dst[i] += src[i] (the lone-term pass's energies into the main pass's)
__global__ void add_into_kernel(double* __restrict__ dst, const double* __restrict__ src, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) dst[i] += src[i];
}
cudaError_t add_into(double* dst, const double* src, int count, cudaStream_t st) {
  if (count > 0) add_into_kernel<<<(count + 255) / 256, 256, 0, st>>>(dst, src, count);
  return cudaGetLastError();
}

cudaError_t fourier_run(const FourierPlan& p, const FourierWork& w, const double* xs,
                        const double* ys, const double* zs, const double* qs,
                        const double2* dtab, const double* modes, const double* commonv,
                        double commonv_scalar, double area, const BVec& b, const WVec& wv,
                        int want_forces, double* energy_out, int* status, double* forces_sorted,
                        cudaStream_t st, int seg_len) {
  cudaError_t e = fourier_phase1(p, w, xs, ys, zs, qs, modes, commonv, commonv_scalar, area, b,
                                 wv, status, nullptr, st);
  if (e != cudaSuccess) return e;
  return fourier_phase2(p, w, xs, ys, zs, qs, dtab, b, want_forces, energy_out, forces_sorted,
                        nullptr, st, seg_len);
}

}  // namespace slab
