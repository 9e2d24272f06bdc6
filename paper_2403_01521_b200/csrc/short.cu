// short.cu -- erfc(alpha r)/r short-range sum on device.
//
// Replaces reference ewald2d.py:280-303 (short_range_energy_forces) with its
// cell list (build_cell_list 141-157, _cell_index 126-138) and pair kernels
// (_pair_kernel_cells 160-231, _pair_kernel_brute 234-277).  Same pair set:
// minimum image in x,y (dx -= lx rint(dx/lx), round-half-even), no wrap in z,
// pairs with d2 <= r_c^2, coincident (d2 < 1e-24) pairs flagged and skipped;
// cells of edge >= r_c, all pairs when ncx < 3 or ncy < 3.
//
// Device layout: stable radix sort of the cell ids (deterministic order inside
// each cell) -> cell-sorted SoA (fp64 + an fp32 copy) + cell_start.  One thread
// per home particle (cell-sorted, so a warp walks the same 27 cells and every
// candidate load is a broadcast).  Candidates are screened with a conservative
// fp32 distance test and the survivors queued per thread in shared memory; when
// any lane's queue fills, the warp drains all queues through the exact fp64
// pair kernel (so the erfc/exp work runs on full warps instead of the ~15% of
// lanes whose candidate happens to be in range).  Each force is accumulated by
// exactly one thread over the full shell: deterministic, no atomics;
// u_s = 1/2 of the full-shell sum.
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace slab {

struct PairAcc {
  double fx, fy, fz, e;
};

// exact reference pair term (ewald2d.py:199-230).  The minimum image uses the
// reference's rint(dx/lx); dx * (1/lx) only differs from dx/lx at exact
// half-box ties, i.e. |dx| = L/2 >= r_c, outside the cutoff.
__device__ __forceinline__ void pair_accumulate(double xi, double yi, double zi, double qi,
                                                double xj, double yj, double zj, double qj,
                                                double lx, double ly, double ilx, double ily,
                                                double alpha, double rc2, double c,
                                                const double* __restrict__ etab, PairAcc& acc,
                                                int& flag) {
  double dx = __dsub_rn(xi, xj), dy = __dsub_rn(yi, yj);
  const double dz = __dsub_rn(zi, zj);
  dx = __dsub_rn(dx, __dmul_rn(lx, rint(__dmul_rn(dx, ilx))));
  dy = __dsub_rn(dy, __dmul_rn(ly, rint(__dmul_rn(dy, ily))));
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  if (d2 > rc2) return;
  if (d2 < 1e-24) {
    flag = 1;
    return;
  }
  const double inv_d = rsqrt(d2);  // one MUFU.RSQ64H + Newton instead of sqrt and a divide
  const double d = d2 * inv_d;
  const double qq = qi * qj;
  const double x = alpha * d;
  double e, g;  // erfc(x) and the force Gaussian e^{-x^2} share one exp
  erfc_gauss(x, etab, &e, &g);
  acc.e = fma(qq * e, inv_d, acc.e);
  const double fmag = qq * (e * inv_d + c * g) * (inv_d * inv_d);
  acc.fx = fma(fmag, dx, acc.fx);
  acc.fy = fma(fmag, dy, acc.fy);
  acc.fz = fma(fmag, dz, acc.fz);
}

// Branch-free form of pair_accumulate for the neighbour-list kernel: list
// entries already passed the conservative screen, so nearly every pair is in
// range and the out-of-range / coincident ones are masked (charge product 0,
// finite stand-in distance) instead of branched around.  Without the early
// returns the four pairs in flight become independent dependency chains the
// scheduler can interleave.  Masked pairs add exact zeros.  (Measured slower:
// carrying the image shift in the row entries instead of rint(dx / lx), +5%;
// a warp-vote guard instead of the branch around the table, +4%; every extra table row costs: the per-block smem fill is ~7% of the kernel.)
// d - l rint(d / l), with the reciprocal product (a compare/select form for the
// shifts -1, 0, 1 measured 3% slower on the pair kernel: FRND is full rate)
__device__ __forceinline__ double min_image(double d, double l, double il) {
  return __dsub_rn(d, __dmul_rn(l, rint(__dmul_rn(d, il))));
}

#ifndef SLAB_PAIR_RAT
#define SLAB_PAIR_RAT 0  // table-free erfcx: pair_list 2.2 -> 2.97 ms at cfg4 (fp64-bound once L1 is not)
#endif
template <bool kTabOnly>
__device__ __forceinline__ void pair_accumulate_masked(double xi, double yi, double zi, double qi,
                                                       double xj, double yj, double zj, double qj,
                                                       double lx, double ly, double ilx, double ily,
                                                       double alpha, double rc2, double c,
                                                       const double* __restrict__ etab,
                                                       PairAcc& acc, int& flag) {
  double dx = __dsub_rn(xi, xj), dy = __dsub_rn(yi, yj);
  const double dz = __dsub_rn(zi, zj);
  dx = min_image(dx, lx, ilx);
  dy = min_image(dy, ly, ily);
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const bool in = d2 <= rc2;
  const bool coincident = d2 < 1e-24;
  flag |= (in && coincident) ? 1 : 0;
  const bool use = in && !coincident;
  const double d2u = use ? d2 : rc2;
  const double inv_d = rsqrt(d2u);
  const double d = d2u * inv_d;
  const double qq = use ? qi * qj : 0.0;
  double e, g;
#if SLAB_PAIR_RAT
  // table-free erfcx (fastmath.cuh): uniform coefficients, no per-lane
  // shared-memory reads on this L1-bound kernel
  if constexpr (kTabOnly)
    erfc_gauss_rat<true>(alpha * d, &e, &g);
  else
    erfc_gauss<false>(alpha * d, etab, &e, &g);
#else
  erfc_gauss<kTabOnly>(alpha * d, etab, &e, &g);
#endif
  acc.e = fma(qq * e, inv_d, acc.e);
  const double fmag = qq * (e * inv_d + c * g) * (inv_d * inv_d);
  acc.fx = fma(fmag, dx, acc.fx);
  acc.fy = fma(fmag, dy, acc.fy);
  acc.fz = fma(fmag, dz, acc.fz);
}

// WCA core (ewald2d.py:218-221 with shifted_lj = 1, used by md.py:34-56):
// 4 eps [(s/r)^12 - (s/r)^6] + eps and its force, for d2 <= rc2 = (2^(1/6) s)^2.
// Same minimum image, cutoff and coincidence rules as the Coulomb term.
// (Two explicit forms: a shared body with `use ? d2 : rc2` selects after the
// unmasked early return was miscompiled -- the selects took the masked arm.)
template <bool kMasked>
__device__ __forceinline__ void wca_accumulate(double xi, double yi, double zi, double xj,
                                               double yj, double zj, double lx, double ly,
                                               double ilx, double ily, double rc2, double eps,
                                               double sig2, PairAcc& acc, int& flag) {
  double dx = __dsub_rn(xi, xj), dy = __dsub_rn(yi, yj);
  const double dz = __dsub_rn(zi, zj);
  dx = __dsub_rn(dx, __dmul_rn(lx, rint(__dmul_rn(dx, ilx))));
  dy = __dsub_rn(dy, __dmul_rn(ly, rint(__dmul_rn(dy, ily))));
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const bool in = d2 <= rc2;
  const bool coincident = d2 < 1e-24;
  double inv_d2, e;
  if constexpr (kMasked) {
    flag |= (in && coincident) ? 1 : 0;
    const bool use = in && !coincident;
    inv_d2 = 1.0 / (use ? d2 : rc2);
    e = use ? eps : 0.0;
  } else {
    if (!in) return;
    if (coincident) {
      flag = 1;
      return;
    }
    inv_d2 = 1.0 / d2;
    e = eps;
  }
  const double s2 = sig2 * inv_d2;
  const double s6 = s2 * s2 * s2;
  acc.e += 4.0 * e * (s6 * s6 - s6) + e;
  const double fmag = 24.0 * e * (2.0 * s6 * s6 - s6) * inv_d2;
  acc.fx = fma(fmag, dx, acc.fx);
  acc.fy = fma(fmag, dy, acc.fy);
  acc.fz = fma(fmag, dz, acc.fz);
}

// Periodic image of x in [0, l): floor-based, with the rounding case x - l
// floor(x / l) == l folded to 0.  The search structure (cells and the fp32
// screen copy) uses this image so that a particle given outside the primary
// cell (x == lx from np.mod(-tiny, lx), an MD floor-wrap, or make_system without
// a box) still sits inside the cell it is filed under; the exact fp64 pair term
// keeps the raw coordinates and the reference's rint minimum image, so its
// values do not depend on the wrap.
__device__ __forceinline__ double wrap_periodic(double x, double l) {
  double w = x - l * floor(x / l);
  return (w >= l || w < 0.0) ? 0.0 : w;
}

// cells: as ewald2d.py:126-138 (x, y periodic, z clamped), on the wrapped image
__global__ void cell_index_kernel(const double* __restrict__ pos, int64_t n, double lx, double ly,
                                  double lz, int ncx, int ncy, int ncz, uint32_t* __restrict__ key,
                                  int32_t* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long cx = (long long)(wrap_periodic(pos[3 * i + 0], lx) / lx * ncx);
  long long cy = (long long)(wrap_periodic(pos[3 * i + 1], ly) / ly * ncy);
  long long cz = (long long)(pos[3 * i + 2] / lz * ncz);
  cx = cx < 0 ? 0 : (cx >= ncx ? ncx - 1 : cx);
  cy = cy < 0 ? 0 : (cy >= ncy ? ncy - 1 : cy);
  cz = cz < 0 ? 0 : (cz >= ncz ? ncz - 1 : cz);
  key[i] = (uint32_t)((cx * ncy + cy) * ncz + cz);
  val[i] = (int32_t)i;
}

__global__ void cell_start_kernel(const uint32_t* __restrict__ skey, int64_t n, int64_t ncell,
                                  int32_t* __restrict__ start) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c > ncell) return;
  int64_t lo = 0, hi = n;  // first index with key >= c
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (skey[mid] < (uint32_t)c) lo = mid + 1;
    else hi = mid;
  }
  start[c] = (int32_t)lo;
}

// cp: raw fp64 record (the pair term); cpf: the fp32 screen copy of the wrapped image
__global__ void cell_gather_kernel(const double* __restrict__ pos, const double* __restrict__ q,
                                   const int32_t* __restrict__ order, int64_t n, double lx,
                                   double ly, double4* __restrict__ cp, float4* __restrict__ cpf) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  int64_t i = order[a];
  const double x = pos[3 * i], y = pos[3 * i + 1], z = pos[3 * i + 2];
  cp[a] = make_double4(x, y, z, q[i]);
  // fp32 rounding of an image just below l may land on l: keep it below l, in
  // the top cell the index kernel files it under (cell_index_kernel clamps
  // x / l * nc == nc to nc - 1), not at 0
  const float xf = fminf((float)wrap_periodic(x, lx), nextafterf((float)lx, 0.0f));
  const float yf = fminf((float)wrap_periodic(y, ly), nextafterf((float)ly, 0.0f));
  cpf[a] = make_float4(xf, yf, (float)z, 0.0f);
}

constexpr int kSRThreads = 128;
#ifndef SLAB_NBR_WIDE
#define SLAB_NBR_WIDE 1
#endif
struct __align__(32) F8 {
  float v[8];
};
constexpr int kRing = 16;  // staged neighbour indices per thread (two 32-byte sectors)

// Pass 1: neighbour rows.  One thread per home particle in cell order.  Cells
// are ordered z-fastest, so the z cells of one (x, y) column are one contiguous
// range: at most (2S+1)^2 ranges per particle, each trimmed to the z extent the
// r_c sphere has over that column (corner columns often drop out).  Mean
// candidates per home at uniform density (sphere = 1): 2.3x for S = 2 (cells of
// edge >= r_c/2), 1.8x for S = 3 (the default), 6.4x for the reference's
// 27 cells of edge >= r_c.  Conservative fp32 distance screen; hits go to a
// per-thread ring in shared memory (slot-major: conflict-free) and are written
// as whole 32-byte sectors into the row nbr[(a - a_begin) * kcap + k].
template <int S>
__global__ void __launch_bounds__(kSRThreads) nbr_build_kernel(
    const float4* __restrict__ cpf, const uint32_t* __restrict__ skey,
    const int32_t* __restrict__ start, int64_t a_begin, int64_t a_end, int ncx, int ncy, int ncz,
    float lxf, float lyf, float lzf, float rc2f, int kcap, int32_t* __restrict__ nbr,
    int32_t* __restrict__ nn, int* __restrict__ maxnn, int* __restrict__ status) {
  __shared__ int32_t ring[kRing][kSRThreads];
  const int64_t a = a_begin + blockIdx.x * (int64_t)kSRThreads + threadIdx.x;
  if (a >= a_end) return;
  const int cid = (int)skey[a];
  const int cy = (cid / ncz) % ncy, cx = cid / (ncz * ncy);
  const float4 pi = cpf[a];
  const int self = (int)a;
  int32_t* st = &ring[0][threadIdx.x];
  int32_t* row = nbr + (a - a_begin) * (int64_t)kcap;
  int cnt = 0, done = 0;  // hits found / hits already written to the row
  const float ex = lxf / ncx, ey = lyf / ncy, izc = ncz / lzf;
  auto flush8 = [&]() {
    if (done + 8 <= kcap) {
      const int s0 = done & (kRing - 1);
      const int4 v0 = make_int4(st[(s0 + 0) * kSRThreads], st[(s0 + 1) * kSRThreads],
                                st[(s0 + 2) * kSRThreads], st[(s0 + 3) * kSRThreads]);
      const int4 v1 = make_int4(st[(s0 + 4) * kSRThreads], st[(s0 + 5) * kSRThreads],
                                st[(s0 + 6) * kSRThreads], st[(s0 + 7) * kSRThreads]);
      SLAB_BOUND(done + 7, kcap);
      int4* dst = reinterpret_cast<int4*>(row + done);
      dst[0] = v0;
      dst[1] = v1;
    }
    done += 8;
  };
  auto test = [&](int jj, const float4& pj, float px, float py) {
    const float dx = px - pj.x, dy = py - pj.y, dz = pi.z - pj.z;
    const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const bool hit = d2 <= rc2f && jj != self;
    if (hit) st[(cnt & (kRing - 1)) * kSRThreads] = jj;
    cnt += hit ? 1 : 0;
  };
#pragma unroll 1
  for (int ox = -S; ox <= S; ++ox) {
    // periodic image of the neighbour column folded into the home position (the
    // 2S+1 columns per axis are distinct cells: ncx, ncy >= 2S+1), a conservative
    // superset screen; the exact reference minimum image is applied in pair_list_kernel
    const int ux = cx + ox;
    const int nx = ux < 0 ? ux + ncx : (ux >= ncx ? ux - ncx : ux);
    const float px = pi.x + (ux < 0 ? lxf : (ux >= ncx ? -lxf : 0.0f));
#pragma unroll 1
    for (int oy = -S; oy <= S; ++oy) {
      const int uy = cy + oy;
      const int ny = uy < 0 ? uy + ncy : (uy >= ncy ? uy - ncy : uy);
      const float py = pi.y + (uy < 0 ? lyf : (uy >= ncy ? -lyf : 0.0f));
      // trim the column to the part of the r_c sphere it can hold: skip it when
      // its xy rectangle is out of reach, else scan only the z cells within
      // h = sqrt(rc2f - d_xy^2) of the home height (a superset of every pair:
      // rc2f is inflated, the cell bounds are widened by 1e-3 cells)
      const float dxr = fmaxf(0.0f, fmaxf(nx * ex - px, px - (nx + 1) * ex));
      const float dyr = fmaxf(0.0f, fmaxf(ny * ey - py, py - (ny + 1) * ey));
      const float dxy2 = fmaf(dxr, dxr, dyr * dyr);
      if (dxy2 > rc2f) continue;
      const float h = sqrtf(rc2f - dxy2);
      int zlo = (int)floorf((pi.z - h) * izc - 1e-3f);
      int zhi = (int)floorf((pi.z + h) * izc + 1e-3f);
      zlo = zlo < 0 ? 0 : (zlo >= ncz ? ncz - 1 : zlo);
      zhi = zhi < 0 ? 0 : (zhi >= ncz ? ncz - 1 : zhi);
      const int col = (nx * ncy + ny) * ncz;
      const int b1 = start[col + zhi + 1];
      int jj = start[col + zlo];
      // (scanning the warp-union of the lanes' ranges instead -- broadcast
      // loads, no idle lanes -- measured 1.51 ms against 1.13 ms per lane;
      // round 2: loading the next 4 candidates before testing the current 4,
      // 1.08 -> 1.15 ms -- this loop is issue-bound, not latency-bound)
#if SLAB_NBR_WIDE
      // two candidates per 256-bit load (32-byte aligned pairs): half the L1
      // requests of this L1-throughput-bound screen
      if ((jj & 1) && jj < b1) {
        test(jj, cpf[jj], px, py);
        ++jj;
      }
      for (; jj + 4 <= b1; jj += 4) {
        const F8 q0 = *reinterpret_cast<const F8*>(cpf + jj);
        const F8 q1 = *reinterpret_cast<const F8*>(cpf + jj + 2);
        test(jj, make_float4(q0.v[0], q0.v[1], q0.v[2], q0.v[3]), px, py);
        test(jj + 1, make_float4(q0.v[4], q0.v[5], q0.v[6], q0.v[7]), px, py);
        test(jj + 2, make_float4(q1.v[0], q1.v[1], q1.v[2], q1.v[3]), px, py);
        test(jj + 3, make_float4(q1.v[4], q1.v[5], q1.v[6], q1.v[7]), px, py);
        if (cnt - done >= 8) flush8();  // pending <= 7 + 4 < kRing
      }
#else
      for (; jj + 4 <= b1; jj += 4) {
        const float4 p0 = cpf[jj], p1 = cpf[jj + 1], p2 = cpf[jj + 2], p3 = cpf[jj + 3];
        test(jj, p0, px, py);
        test(jj + 1, p1, px, py);
        test(jj + 2, p2, px, py);
        test(jj + 3, p3, px, py);
        if (cnt - done >= 8) flush8();  // pending <= 7 + 4 < kRing
      }
#endif
      for (; jj < b1; ++jj) {
        test(jj, cpf[jj], px, py);
        if (cnt - done >= 8) flush8();
      }
    }
  }
  if (cnt <= kcap)
    for (int k = done; k < cnt; ++k) {
      SLAB_BOUND(k, kcap);
      row[k] = st[(k & (kRing - 1)) * kSRThreads];
    }
  nn[a - a_begin] = cnt <= kcap ? cnt : -1;  // -1: overflowed, evaluated by overflow_pairs_kernel
  if (cnt > kcap) {
    atomicOr(status, SLAB_STATUS_NBR_OVERFLOW_DEV);
    atomicMax(maxnn, cnt);
  }
}

// Pass 1, cell form (small systems): one warp per home cell, LANES = CANDIDATES.
// The homes of the cell (up to kCellHomes per pass, held warp-uniformly in
// registers) share one trimmed z range per neighbour column -- trimmed to the
// r_c sphere around the homes' bounding box -- so every candidate is loaded
// once per cell (coalesced along the column's z-sorted range) instead of once
// per home, and the lanes stay converged.  The columns' ranges are concatenated
// (warp prefix sum) and walked 32 candidates at a time; each home tests the
// batch, and the hits are appended to its row with a ballot (lanes in order:
// the row lists the columns in (ox, oy) order and each range in z order, as
// the per-lane form does).  Mean candidates per home at uniform density: 2.2x
// the sphere for S = 3 (the per-lane form: 1.8x, loaded per home, at 58% lane
// utilisation and L1-throughput bound).
constexpr int kCellHomes = 8;
// Used for small home sets only: it exposes a warp per cell where the per-lane
// form has too few warps to cover its load latency (cfg2, N = 1e4: 0.115 ->
// 0.057 ms); at N >= 1e5 it is latency-bound on its serial batch chain (owner
// search -> gather -> tests) and loses (cfg4: 3.36 against 1.02 ms for S = 3).
#ifndef SLAB_NBR_CELLS_MAX_HOMES
#define SLAB_NBR_CELLS_MAX_HOMES 32768
#endif
constexpr int64_t kNbrCellsMaxHomes = SLAB_NBR_CELLS_MAX_HOMES;

template <int S>
__global__ void __launch_bounds__(kSRThreads) nbr_cells_kernel(
    const float4* __restrict__ cpf, const int32_t* __restrict__ start, int64_t ncell,
    int64_t a_begin, int64_t a_end, int ncx, int ncy, int ncz, float lxf, float lyf, float lzf,
    float rc2f, int kcap, int32_t* __restrict__ nbr, int32_t* __restrict__ nn,
    int* __restrict__ maxnn, int* __restrict__ status) {
  constexpr int W = 2 * S + 1, NCOL = W * W;
  const int lane = threadIdx.x & 31;
  const int64_t c = blockIdx.x * (int64_t)(kSRThreads / 32) + (threadIdx.x >> 5);
  if (c >= ncell) return;
  const int64_t hb0 = start[c] > a_begin ? start[c] : a_begin;
  const int64_t he = start[c + 1] < a_end ? start[c + 1] : a_end;
  if (hb0 >= he) return;  // warp-uniform
  const int cz = (int)(c % ncz), cy = (int)((c / ncz) % ncy), cx = (int)(c / ((int64_t)ncz * ncy));
  (void)cz;
  const float ex = lxf / ncx, ey = lyf / ncy, izc = ncz / lzf;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t g0 = hb0; g0 < he; g0 += kCellHomes) {
    const int ng = (int)(he - g0 < kCellHomes ? he - g0 : kCellHomes);
    const float4 hl = lane < ng ? cpf[g0 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    float hx[kCellHomes], hy[kCellHomes], hz[kCellHomes];
    int cnt[kCellHomes];
#pragma unroll
    for (int h = 0; h < kCellHomes; ++h) {
      hx[h] = __shfl_sync(0xffffffffu, hl.x, h);
      hy[h] = __shfl_sync(0xffffffffu, hl.y, h);
      hz[h] = __shfl_sync(0xffffffffu, hl.z, h);
      cnt[h] = 0;
    }
    float x0 = hx[0], x1 = hx[0], y0 = hy[0], y1 = hy[0], z0 = hz[0], z1 = hz[0];
#pragma unroll
    for (int h = 1; h < kCellHomes; ++h)
      if (h < ng) {
        x0 = fminf(x0, hx[h]);
        x1 = fmaxf(x1, hx[h]);
        y0 = fminf(y0, hy[h]);
        y1 = fmaxf(y1, hy[h]);
        z0 = fminf(z0, hz[h]);
        z1 = fmaxf(z1, hz[h]);
      }
#pragma unroll 1
    for (int q0 = 0; q0 < NCOL; q0 += 32) {
      // lane -> one neighbour column: its periodic image shift (applied to the
      // homes, as in the per-lane form) and its trimmed candidate range
      const int q = q0 + lane;
      int j0 = 0, len = 0;
      float shx = 0.f, shy = 0.f;
      if (q < NCOL) {
        const int ux = cx + q / W - S, uy = cy + q % W - S;
        const int nx = ux < 0 ? ux + ncx : (ux >= ncx ? ux - ncx : ux);
        const int ny = uy < 0 ? uy + ncy : (uy >= ncy ? uy - ncy : uy);
        shx = ux < 0 ? lxf : (ux >= ncx ? -lxf : 0.0f);
        shy = uy < 0 ? lyf : (uy >= ncy ? -lyf : 0.0f);
        const float dxr = fmaxf(0.0f, fmaxf(nx * ex - (x1 + shx), (x0 + shx) - (nx + 1) * ex));
        const float dyr = fmaxf(0.0f, fmaxf(ny * ey - (y1 + shy), (y0 + shy) - (ny + 1) * ey));
        const float dxy2 = fmaf(dxr, dxr, dyr * dyr);
        if (dxy2 <= rc2f) {
          const float h = sqrtf(rc2f - dxy2);
          int zlo = (int)floorf((z0 - h) * izc - 1e-3f);
          int zhi = (int)floorf((z1 + h) * izc + 1e-3f);
          zlo = zlo < 0 ? 0 : (zlo >= ncz ? ncz - 1 : zlo);
          zhi = zhi < 0 ? 0 : (zhi >= ncz ? ncz - 1 : zhi);
          const int64_t col = ((int64_t)nx * ncy + ny) * ncz;
          j0 = start[col + zlo];
          len = start[col + zhi + 1] - j0;
        }
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      const int excl = incl - len;
#pragma unroll 1
      for (int f0 = 0; f0 < total; f0 += 32) {
        const int f = f0 + lane;
        // owner column: the number of columns whose inclusive end is <= f
        int k = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int v = __shfl_sync(0xffffffffu, incl, k + step - 1);
          if (v <= f) k += step;
        }
        const int jk = __shfl_sync(0xffffffffu, j0, k & 31);
        const int ek = __shfl_sync(0xffffffffu, excl, k & 31);
        const float sx = __shfl_sync(0xffffffffu, shx, k & 31);
        const float sy = __shfl_sync(0xffffffffu, shy, k & 31);
        const bool valid = f < total;
        const int j = jk + (f - ek);
        float4 pj = make_float4(3e30f, 3e30f, 3e30f, 0.f);
        if (valid) pj = cpf[j];
        const float xj = pj.x - sx, yj = pj.y - sy;
#pragma unroll
        for (int h = 0; h < kCellHomes; ++h) {
          if (h < ng) {  // warp-uniform
            const float dx = hx[h] - xj, dy = hy[h] - yj, dz = hz[h] - pj.z;
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            const bool hit = valid && d2 <= rc2f && (int64_t)j != g0 + h;
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (hit) {
              const int pos = cnt[h] + __popc(m & lt);
              if (pos < kcap) nbr[(g0 + h - a_begin) * (int64_t)kcap + pos] = j;
            }
            cnt[h] += __popc(m);
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < kCellHomes; ++h)
      if (h < ng && lane == h) {
        nn[g0 + h - a_begin] = cnt[h] <= kcap ? cnt[h] : -1;
        if (cnt[h] > kcap) {
          atomicOr(status, SLAB_STATUS_NBR_OVERFLOW_DEV);
          atomicMax(maxnn, cnt[h]);
        }
      }
  }
}

// Pass 2: one thread per home particle over its own row (rows have ~equal
// length, so the fp64 pair work runs on nearly full warps); four neighbours in
// flight per iteration (measured: 2 or 8 in flight, a generic unrolled loop, or
// a min-blocks launch bound are all 5-20% slower).  Each force is owned by one
// thread: deterministic.
// KIND 0: erfc Coulomb (alpha); KIND 2: the same with alpha r_c inside the erfcx table
// (branch-free); KIND 1: WCA core (eps, sig2 = sigma^2).
#ifndef SLAB_PAIR_WIDE
#define SLAB_PAIR_WIDE 1
#endif
struct __align__(32) Idx8 {
  int32_t a0, a1, a2, a3, a4, a5, a6, a7;
};
struct __align__(32) Rec4 {
  double x, y, z, w;
};
__device__ __forceinline__ double4 ld_rec(const double4* p) {  // one 256-bit load
  const Rec4 r = *reinterpret_cast<const Rec4*>(p);
  return make_double4(r.x, r.y, r.z, r.w);
}
// SPLIT > 1 (small systems, fewer homes than one resident wave of threads):
// SPLIT consecutive lanes share a home, taking its row's 4-entry blocks round
// robin, and combine their partial forces with a fixed xor-shuffle tree
// (deterministic).
#ifndef SLAB_PAIR_PFIDX
#define SLAB_PAIR_PFIDX 1
#endif
#ifndef SLAB_PAIR_CTAS
// resident CTAs per SM the pair kernel is compiled and gridded for (cfg4, 24-row
// erfcx table: 5 -> 1.95 ms; 6 / 7 / 8 cap the registers at 80 / 72 / 64 and
// spill: 2.08 / 1.99 / 2.19 ms).  Round 2, with the row entries loaded one block
// ahead (SLAB_PAIR_PFIDX): 4 -> 1.91 ms (5: 2.00, 3: 2.02; without the
// prefetch 4: 1.95; all 8 records loaded before the first term: 2.02 / 2.04)
#define SLAB_PAIR_CTAS 4
#endif
constexpr int kPairCtas = SLAB_PAIR_CTAS;
template <int KIND, int SPLIT>
__global__ void __launch_bounds__(kSRThreads, kPairCtas) pair_list_kernel(
    const double4* __restrict__ cp, const int32_t* __restrict__ order,
    const int32_t* __restrict__ nbr, const int32_t* __restrict__ nn, int64_t a_begin,
    int64_t a_end, int kcap, double lx, double ly, double alpha, double rc2, double eps,
    double sig2, double* __restrict__ forces, double* __restrict__ eblk,
    int* __restrict__ status, int accumulate) {
  constexpr bool kTable = KIND == 0 || (KIND == 2 && !SLAB_PAIR_RAT);
  __shared__ double etab[kTable ? kErfcxTabSize : 1];
  __shared__ double red[kSRThreads];
  if constexpr (kTable) load_erfcx_table(etab);
  __syncthreads();
  const double c = kTwoOverSqrtPi * alpha;
  const double ilx = 1.0 / lx, ily = 1.0 / ly;
  PairAcc acc{0.0, 0.0, 0.0, 0.0};
  int flag = 0;
#define PAIR(pi, pj)                                                                          \
  do {                                                                                        \
    if constexpr (KIND != 1)                                                                  \
      pair_accumulate_masked<KIND == 2>(pi.x, pi.y, pi.z, pi.w, pj.x, pj.y, pj.z, pj.w, lx, ly, ilx, ily, \
                             alpha, rc2, c, etab, acc, flag);                                 \
    else                                                                                      \
      wca_accumulate<true>(pi.x, pi.y, pi.z, pj.x, pj.y, pj.z, lx, ly, ilx, ily, rc2, eps,    \
                           sig2, acc, flag);                                                  \
  } while (0)
  // grid-stride over home particles (warp-uniform bound: the SPLIT lanes of a
  // home shuffle together): the smem erfcx fill is paid once per CTA
  const int sub = threadIdx.x % SPLIT;
  constexpr int kHomesPerCta = kSRThreads / SPLIT;
  const int64_t warp_first = (int64_t)(threadIdx.x & ~31) / SPLIT;
  for (int64_t base = a_begin + blockIdx.x * (int64_t)kHomesPerCta; base + warp_first < a_end;
       base += (int64_t)gridDim.x * kHomesPerCta) {
    const int64_t a = base + threadIdx.x / SPLIT;
    const bool active = a < a_end;
    const double4 pi = active ? cp[a] : make_double4(0.0, 0.0, 0.0, 0.0);
    const int cnt_raw = active ? nn[a - a_begin] : 0;
    const bool own = active && cnt_raw >= 0;  // overflowed homes: overflow_pairs_kernel
    const int cnt = cnt_raw > 0 ? cnt_raw : 0;
    const int32_t* row = nbr + (active ? a - a_begin : 0) * (int64_t)kcap;
    acc.fx = acc.fy = acc.fz = 0.0;
#if SLAB_PAIR_WIDE
    // 8 row entries per 256-bit load (rows are 32-byte aligned: kcap is a
    // multiple of 8) and one 256-bit load per neighbour record: half the L1
    // requests of 128-bit loads on this L1-bound kernel
    int k = 8 * sub;
#if SLAB_PAIR_PFIDX
    // the next block's 8 row entries are loaded one block ahead: the record
    // addresses no longer wait on the row load (round 2: 10% of this kernel's
    // stall samples sat on that dependency)
    Idx8 jn{};
    if (k + 8 <= cnt) jn = *reinterpret_cast<const Idx8*>(row + k);
#endif
    for (; k + 8 <= cnt; k += 8 * SPLIT) {
#if SLAB_PAIR_PFIDX
      const Idx8 j8 = jn;
      if (k + 8 * SPLIT + 8 <= cnt) jn = *reinterpret_cast<const Idx8*>(row + k + 8 * SPLIT);
#else
      const Idx8 j8 = *reinterpret_cast<const Idx8*>(row + k);
#endif
      {
        const double4 p0 = ld_rec(cp + j8.a0), p1 = ld_rec(cp + j8.a1), p2 = ld_rec(cp + j8.a2),
                      p3 = ld_rec(cp + j8.a3);
        PAIR(pi, p0);
        PAIR(pi, p1);
        PAIR(pi, p2);
        PAIR(pi, p3);
      }
      {
        const double4 p0 = ld_rec(cp + j8.a4), p1 = ld_rec(cp + j8.a5), p2 = ld_rec(cp + j8.a6),
                      p3 = ld_rec(cp + j8.a7);
        PAIR(pi, p0);
        PAIR(pi, p1);
        PAIR(pi, p2);
        PAIR(pi, p3);
      }
    }
    if (sub == 0)
      for (k = cnt & ~7; k < cnt; ++k) {
        const double4 pj = ld_rec(cp + row[k]);
        PAIR(pi, pj);
      }
#else
    int k = 4 * sub;
    for (; k + 4 <= cnt; k += 4 * SPLIT) {
      const int4 j4 = *reinterpret_cast<const int4*>(row + k);
      const double4 p0 = cp[j4.x], p1 = cp[j4.y], p2 = cp[j4.z], p3 = cp[j4.w];
      PAIR(pi, p0);
      PAIR(pi, p1);
      PAIR(pi, p2);
      PAIR(pi, p3);
    }
    if (sub == 0)
      for (k = cnt & ~3; k < cnt; ++k) {
        const double4 pj = cp[row[k]];
        PAIR(pi, pj);
      }
#endif
#pragma unroll
    for (int o = 1; o < SPLIT; o <<= 1) {
      acc.fx += __shfl_xor_sync(0xffffffffu, acc.fx, o);
      acc.fy += __shfl_xor_sync(0xffffffffu, acc.fy, o);
      acc.fz += __shfl_xor_sync(0xffffffffu, acc.fz, o);
    }
    if (own && sub == 0) {
      const int64_t i = order[a];
      if (accumulate) {  // one thread owns particle i: += is race-free and deterministic
        acc.fx += forces[3 * i + 0];
        acc.fy += forces[3 * i + 1];
        acc.fz += forces[3 * i + 2];
      }
      forces[3 * i + 0] = acc.fx;
      forces[3 * i + 1] = acc.fy;
      forces[3 * i + 2] = acc.fz;
    }
  }
#undef PAIR
  if (flag) atomicOr(status, SLAB_STATUS_COINCIDENT_DEV);
  red[threadIdx.x] = acc.e;
  __syncthreads();
  for (int w = kSRThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[blockIdx.x] = red[0];
}

// Homes whose neighbour row overflowed its capacity (nn = -1): one thread per
// such home searches its (2S+1)^2 trimmed columns again and evaluates every
// pair directly (same fp32 screen and exact fp64 term as the row path), writing
// the home's force and a per-block energy partial.  Always launched, in-stream
// and graph-safe; a run without overflow just scans nn.  The home's pair order
// (columns, then z) is fixed, so results stay deterministic.
constexpr int kOvfBlocks = 148;
template <int S, int KIND>
__global__ void __launch_bounds__(kSRThreads) overflow_pairs_kernel(
    const double4* __restrict__ cp, const float4* __restrict__ cpf,
    const uint32_t* __restrict__ skey, const int32_t* __restrict__ start,
    const int32_t* __restrict__ order, const int32_t* __restrict__ nn, int64_t a_begin,
    int64_t a_end, int ncx, int ncy, int ncz, float lxf, float lyf, float lzf, float rc2f,
    double lx, double ly, double alpha, double rc2, double eps, double sig2,
    double* __restrict__ forces, double* __restrict__ eblk, int* __restrict__ status,
    int accumulate) {
  __shared__ double etab[KIND != 1 ? kErfcxTabSize : 1];
  __shared__ double red[kSRThreads];
  if constexpr (KIND != 1) load_erfcx_table(etab);
  __syncthreads();
  const double c = kTwoOverSqrtPi * alpha, ilx = 1.0 / lx, ily = 1.0 / ly;
  const float ex = lxf / ncx, ey = lyf / ncy, izc = ncz / lzf;
  double e_sum = 0.0;
  int flag = 0;
  for (int64_t a = a_begin + blockIdx.x * (int64_t)kSRThreads + threadIdx.x; a < a_end;
       a += (int64_t)gridDim.x * kSRThreads) {
    if (nn[a - a_begin] >= 0) continue;
    const int cid = (int)skey[a];
    const int cy = (cid / ncz) % ncy, cx = cid / (ncz * ncy);
    const float4 pi = cpf[a];
    const double4 pd = cp[a];
    PairAcc acc{0.0, 0.0, 0.0, 0.0};
    for (int ox = -S; ox <= S; ++ox) {
      const int ux = cx + ox;
      const int nx = ux < 0 ? ux + ncx : (ux >= ncx ? ux - ncx : ux);
      const float px = pi.x + (ux < 0 ? lxf : (ux >= ncx ? -lxf : 0.0f));
      for (int oy = -S; oy <= S; ++oy) {
        const int uy = cy + oy;
        const int ny = uy < 0 ? uy + ncy : (uy >= ncy ? uy - ncy : uy);
        const float py = pi.y + (uy < 0 ? lyf : (uy >= ncy ? -lyf : 0.0f));
        const float dxr = fmaxf(0.0f, fmaxf(nx * ex - px, px - (nx + 1) * ex));
        const float dyr = fmaxf(0.0f, fmaxf(ny * ey - py, py - (ny + 1) * ey));
        const float dxy2 = fmaf(dxr, dxr, dyr * dyr);
        if (dxy2 > rc2f) continue;
        const float h = sqrtf(rc2f - dxy2);
        int zlo = (int)floorf((pi.z - h) * izc - 1e-3f);
        int zhi = (int)floorf((pi.z + h) * izc + 1e-3f);
        zlo = zlo < 0 ? 0 : (zlo >= ncz ? ncz - 1 : zlo);
        zhi = zhi < 0 ? 0 : (zhi >= ncz ? ncz - 1 : zhi);
        const int col = (nx * ncy + ny) * ncz;
        for (int jj = start[col + zlo]; jj < start[col + zhi + 1]; ++jj) {
          if (jj == (int)a) continue;
          const float4 pj = cpf[jj];
          const float dx = px - pj.x, dy = py - pj.y, dz = pi.z - pj.z;
          if (fmaf(dx, dx, fmaf(dy, dy, dz * dz)) > rc2f) continue;
          const double4 q = cp[jj];
          if constexpr (KIND != 1)
            pair_accumulate(pd.x, pd.y, pd.z, pd.w, q.x, q.y, q.z, q.w, lx, ly, ilx, ily, alpha,
                            rc2, c, etab, acc, flag);
          else
            wca_accumulate<false>(pd.x, pd.y, pd.z, q.x, q.y, q.z, lx, ly, ilx, ily, rc2, eps,
                                  sig2, acc, flag);
        }
      }
    }
    const int64_t i = order[a];
    if (accumulate) {
      acc.fx += forces[3 * i + 0];
      acc.fy += forces[3 * i + 1];
      acc.fz += forces[3 * i + 2];
    }
    forces[3 * i + 0] = acc.fx;
    forces[3 * i + 1] = acc.fy;
    forces[3 * i + 2] = acc.fz;
    e_sum += acc.e;
  }
  if (flag) atomicOr(status, SLAB_STATUS_COINCIDENT_DEV);
  red[threadIdx.x] = e_sum;
  __syncthreads();
  for (int w = kSRThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[blockIdx.x] = red[0];
}

// all pairs (ncx < 3 or ncy < 3): grid (i tiles, j splits)
template <int KIND>
__global__ void __launch_bounds__(128) brute_pair_kernel(
    const double* __restrict__ pos, const double* __restrict__ q, int64_t n, int64_t i_begin,
    int64_t i_end, int jsplit, double lx, double ly, double alpha, double rc2, double eps,
    double sig2, double* __restrict__ fbuf, double* __restrict__ eblk, int* __restrict__ status) {
  __shared__ double etab[KIND == 0 ? kErfcxTabSize : 1];
  if constexpr (KIND == 0) load_erfcx_table(etab);
  __syncthreads();
  const int64_t i = i_begin + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int js = blockIdx.y;
  const int64_t per = (n + jsplit - 1) / jsplit;
  const int64_t j0 = js * per, j1 = j0 + per < n ? j0 + per : n;
  const double c = kTwoOverSqrtPi * alpha;
  const double ilx = 1.0 / lx, ily = 1.0 / ly;
  PairAcc acc{0.0, 0.0, 0.0, 0.0};
  int flag = 0;
  if (i < i_end) {
    const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2];
    const double qi = KIND == 0 ? q[i] : 0.0;
    for (int64_t j = j0; j < j1; ++j) {
      if (j == i) continue;
      if constexpr (KIND == 0)
        pair_accumulate(xi, yi, zi, qi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], q[j], lx, ly,
                        ilx, ily, alpha, rc2, c, etab, acc, flag);
      else
        wca_accumulate<false>(xi, yi, zi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], lx, ly, ilx,
                              ily, rc2, eps, sig2, acc, flag);
    }
    double* f = fbuf + ((size_t)js * n + i) * 3;
    f[0] = acc.fx;
    f[1] = acc.fy;
    f[2] = acc.fz;
  }
  if (flag) atomicOr(status, SLAB_STATUS_COINCIDENT_DEV);
  __shared__ double red[128];
  red[threadIdx.x] = acc.e;
  __syncthreads();
  for (int s = 64; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[(size_t)js * gridDim.x + blockIdx.x] = red[0];
}

__global__ void brute_force_reduce_kernel(const double* __restrict__ fbuf, int jsplit, int64_t n3,
                                          double* __restrict__ forces, int accumulate) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n3) return;
  double v = 0.0;
  for (int s = 0; s < jsplit; ++s) v += fbuf[(size_t)s * n3 + e];
  forces[e] = accumulate ? forces[e] + v : v;
}

// u_s = 1/2 * sum of the per-block full-shell partials, fixed order
__global__ void __launch_bounds__(1024) half_sum_kernel(const double* __restrict__ eblk,
                                                        int64_t m, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += 1024) s += eblk[k];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = 0.5 * red[0];
}

// pair_list_kernel grid: one resident wave (kPairCtas CTAs per SM), grid-striding
static int64_t pair_grid(int64_t blocks) {
  return blocks < 148 * kPairCtas ? blocks : 148 * kPairCtas;
}
// lanes per home: fill one resident wave (148 SMs x kPairCtas CTAs x 128 threads)
// when there are fewer homes than that (cfg2, N = 1e4: 8 lanes per home)
static int pair_split(int64_t nh) {
  int s = 1;
  while (s < 8 && nh * s < (int64_t)148 * kPairCtas * kSRThreads) s *= 2;
  return s;
}

template <int KIND>
static void launch_pair_split(int split, unsigned grid, cudaStream_t st, const double4* cp,
                              const int32_t* order, const int32_t* nbr, const int32_t* nn,
                              int64_t h0, int64_t h1, int kcap, double lx, double ly,
                              double alpha, double rc2, double eps, double sig2, double* forces,
                              double* eblk, int* status, int accumulate) {
#define SLAB_PAIR_LAUNCH(S)                                                                 \
  pair_list_kernel<KIND, S><<<grid, kSRThreads, 0, st>>>(cp, order, nbr, nn, h0, h1, kcap, lx, \
                                                         ly, alpha, rc2, eps, sig2, forces,   \
                                                         eblk, status, accumulate)
  if (split >= 8) SLAB_PAIR_LAUNCH(8);
  else if (split == 4) SLAB_PAIR_LAUNCH(4);
  else if (split == 2) SLAB_PAIR_LAUNCH(2);
  else SLAB_PAIR_LAUNCH(1);
#undef SLAB_PAIR_LAUNCH
}

static void launch_pair_list(int kind, int split, unsigned grid, cudaStream_t st,
                             const double4* cp, const int32_t* order, const int32_t* nbr,
                             const int32_t* nn, int64_t h0, int64_t h1, int kcap, double lx,
                             double ly, double alpha, double rc2, double eps, double sig2,
                             double* forces, double* eblk, int* status, int accumulate) {
  if (kind == 2)
    launch_pair_split<2>(split, grid, st, cp, order, nbr, nn, h0, h1, kcap, lx, ly, alpha, rc2,
                         eps, sig2, forces, eblk, status, accumulate);
  else if (kind == 0)
    launch_pair_split<0>(split, grid, st, cp, order, nbr, nn, h0, h1, kcap, lx, ly, alpha, rc2,
                         eps, sig2, forces, eblk, status, accumulate);
  else
    launch_pair_split<1>(split, grid, st, cp, order, nbr, nn, h0, h1, kcap, lx, ly, alpha, rc2,
                         eps, sig2, forces, eblk, status, accumulate);
}

#ifndef SLAB_SHORT_SPAN_DEFAULT
#define SLAB_SHORT_SPAN_DEFAULT 3  // cfg4: nbr_build 1.12 -> 1.02 ms (pair_list +0.04)
#endif
constexpr int kShortSpan = SLAB_SHORT_SPAN_DEFAULT;

#ifndef SLAB_TILE_MIN_N
#define SLAB_TILE_MIN_N 40000
#endif
constexpr int64_t kTileMinN = SLAB_TILE_MIN_N;
#ifndef SLAB_NBR_TILE
#define SLAB_NBR_TILE 0  // cfg4: warp-window screen 1.46 ms (2.7x the candidates) vs nbr_build 1.10 ms
#endif
constexpr bool kNbrTile = SLAB_NBR_TILE;
#ifndef SLAB_TILE_DEFAULT
#define SLAB_TILE_DEFAULT 0  // cfg4: tile 4.5 ms vs neighbour rows 3.2 ms (DESIGN 4.3)
#endif
constexpr bool kTileDefault = SLAB_TILE_DEFAULT;

ShortPlan short_plan(int64_t n, double lx, double ly, double lz, double rc, int max_span) {
  ShortPlan p{};
  p.n = n;
  int ncx = (int)(lx / rc), ncy = (int)(ly / rc), ncz = (int)(lz / rc);
  ncx = ncx < 1 ? 1 : ncx;
  ncy = ncy < 1 ? 1 : ncy;
  ncz = ncz < 1 ? 1 : ncz;
  p.brute = (ncx < 3 || ncy < 3);
  p.span = 1;
  if (p.brute) {
    ncx = ncy = ncz = 1;
  } else {
    // cells of edge >= r_c / S searched over (2S+1)^2 columns: ncx, ncy >= 3S >=
    // 2S+1 here.  SLAB_SHORT_SPAN (1..3) overrides the default for tuning.
    const char* env = getenv("SLAB_SHORT_SPAN");
    int S = kShortSpan;
    if (env && env[0] >= '1' && env[0] <= '3') S = env[0] - '0';
    S = S < max_span ? S : max_span;
    if (S >= 2) {
      p.span = S;
      ncx = (int)(S * lx / rc);
      ncy = (int)(S * ly / rc);
      ncz = (int)(S * lz / rc);
      ncz = ncz < 1 ? 1 : ncz;
    }
  }
  p.ncx = ncx;
  p.ncy = ncy;
  p.ncz = ncz;
  p.ncell = (int64_t)ncx * ncy * ncz;
  // the fused tile kernel (short_tile.cu) for the erfc Coulomb sum of larger
  // systems: its column window (a warp's ~2 x 2-cell box +- S cells) must fit in
  // the box without aliasing; small systems keep the neighbour-row kernels tuned
  // for them.  SLAB_SHORT_TILE=0/1 overrides (A/B timing).
  p.tile = 0;
  if (kTileDefault && !p.brute && max_span >= 3 && p.span == 3 && ncx >= 2 * p.span + 6 &&
      ncy >= 2 * p.span + 6 && n >= kTileMinN)
    p.tile = 1;
  if (const char* env = getenv("SLAB_SHORT_TILE"))
    p.tile = (env[0] == '1' && !p.brute && max_span >= 3 && p.span >= 2) ? 1 :
             (env[0] == '0' ? 0 : p.tile);
  const int64_t nbx = (n + 127) / 128;
  int js = (int)(592 / (nbx > 0 ? nbx : 1));
  p.jsplit = p.brute ? (js < 1 ? 1 : (js > 64 ? 64 : js)) : 1;
  p.nblk = p.brute ? (int64_t)p.jsplit * (nbx > 0 ? nbx : 1)
                   : (int64_t)148 * 5;  // pair_grid cap: any home count / split
  // neighbour-row capacity: 1.6x the mean-density sphere count + slack, rounded to
  // whole 32-byte sectors; grown by the caller after an overflow report
  const double dens = n / (lx * ly * lz);
  // (rows past capacity are evaluated by overflow_pairs_kernel, so this only
  // trades row memory -- 21 GB at N = 1e7 with 1.6x + 96 -- against fallback work)
  int64_t kc = (int64_t)(1.3 * 4.18879 * rc * rc * rc * dens) + 48;
  if (kc > n + 8) kc = n + 8;
  p.kcap = (int)((kc + 7) / 8 * 8);  // whole 32-byte sectors
  return p;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t short_work_bytes(const ShortPlan& p) {
  const size_t n = (size_t)(p.n > 0 ? p.n : 1);
  size_t b = align256(sizeof(double) * ((p.nblk > 0 ? p.nblk : 1) + kOvfBlocks));  // eblk
  if (p.brute) {
    b += align256(sizeof(double) * 3 * n * p.jsplit);
  } else {
    b += 2 * align256(sizeof(uint32_t) * n) + 2 * align256(sizeof(int32_t) * n);
    b += align256(sizeof(int32_t) * radix_hist_entries(p.n));
    b += align256(sizeof(int32_t) * (p.ncell + 1));
    b += align256(sizeof(double4) * n) + align256(sizeof(float4) * n);
    b += tile_work_bytes(p.n, p.ncx, p.ncy, p.ncz);  // home order (tile kernels)
    if (!p.tile)
      b += align256(sizeof(int32_t) * n * (size_t)p.kcap) + align256(sizeof(int32_t) * n);
    b += align256(sizeof(int));
  }
  return b + 256;
}

cudaError_t short_run(const ShortPlan& p, void* work, const double* pos, const double* charge,
                      double lx, double ly, double lz, double alpha, double rc, double* forces,
                      double* energy_out, int* status, int64_t h0, int64_t h1,
                      int* maxnn_out, cudaStream_t st, int kind, double lj_eps,
                      double lj_sigma, int accumulate, cudaEvent_t pairs_after,
                      cudaEvent_t charge_ready) {
  const int64_t n = p.n;
  const double sig2 = lj_sigma * lj_sigma;
  if (n < 2 || h1 <= h0) {
    cudaMemsetAsync(energy_out, 0, sizeof(double), st);
    if (n > 0 && !accumulate) cudaMemsetAsync(forces, 0, sizeof(double) * 3 * n, st);
    return cudaGetLastError();
  }
  // a shard (multi-GPU) writes only its home particles: clear the rest first
  const bool partial = h0 > 0 || h1 < n;
  if (partial && accumulate) return cudaErrorInvalidValue;
  if (partial) cudaMemsetAsync(forces, 0, sizeof(double) * 3 * n, st);
  const int64_t nh = h1 - h0;
  char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(work) + 255) & ~(uintptr_t)255);
  double* eblk = reinterpret_cast<double*>(w);
  w += align256(sizeof(double) * (p.nblk + kOvfBlocks));
  const double rc2 = rc * rc;
  // the cell search needs positions only: a host-buffer caller's charges may
  // still be landing (they are first read by the gather / brute kernel)
  if (p.brute) {
    if (charge_ready) cudaStreamWaitEvent(st, charge_ready, 0);
    double* fbuf = reinterpret_cast<double*>(w);
    const unsigned nbx = (unsigned)((nh + 127) / 128);
    if (partial) cudaMemsetAsync(fbuf, 0, sizeof(double) * 3 * n * p.jsplit, st);
    if (kind == 0)
      brute_pair_kernel<0><<<dim3(nbx, p.jsplit), 128, 0, st>>>(
          pos, charge, n, h0, h1, p.jsplit, lx, ly, alpha, rc2, 0.0, 0.0, fbuf, eblk, status);
    else
      brute_pair_kernel<1><<<dim3(nbx, p.jsplit), 128, 0, st>>>(
          pos, charge, n, h0, h1, p.jsplit, lx, ly, 0.0, rc2, lj_eps, sig2, fbuf, eblk, status);
    brute_force_reduce_kernel<<<(unsigned)((3 * n + 255) / 256), 256, 0, st>>>(
        fbuf, p.jsplit, 3 * n, forces, accumulate);
    half_sum_kernel<<<1, 1024, 0, st>>>(eblk, (int64_t)nbx * p.jsplit, energy_out);
    return cudaGetLastError();
  } else {
    uint32_t* k0 = reinterpret_cast<uint32_t*>(w);
    w += align256(sizeof(uint32_t) * n);
    uint32_t* k1 = reinterpret_cast<uint32_t*>(w);
    w += align256(sizeof(uint32_t) * n);
    int32_t* v0 = reinterpret_cast<int32_t*>(w);
    w += align256(sizeof(int32_t) * n);
    int32_t* v1 = reinterpret_cast<int32_t*>(w);
    w += align256(sizeof(int32_t) * n);
    int32_t* hist = reinterpret_cast<int32_t*>(w);
    w += align256(sizeof(int32_t) * radix_hist_entries(n));
    int32_t* start = reinterpret_cast<int32_t*>(w);
    w += align256(sizeof(int32_t) * (p.ncell + 1));
    double4* cp = reinterpret_cast<double4*>(w);
    w += align256(sizeof(double4) * n);
    float4* cpf = reinterpret_cast<float4*>(w);
    w += align256(sizeof(float4) * n);
    int* maxnn = maxnn_out;
    cell_index_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pos, n, lx, ly, lz, p.ncx,
                                                                  p.ncy, p.ncz, k0, v0);
    int bits = 8;
    while (bits < 32 && ((int64_t)1 << bits) <= p.ncell) bits += 8;
    uint32_t* skey;
    int32_t* order;
    cudaError_t e = radix_sort_pairs<uint32_t>(k0, v0, k1, v1, hist, n, bits, st, &skey, &order);
    if (e != cudaSuccess) return e;
    cell_start_kernel<<<(unsigned)((p.ncell + 1 + 255) / 256), 256, 0, st>>>(skey, n, p.ncell,
                                                                             start);
    if (charge_ready) cudaStreamWaitEvent(st, charge_ready, 0);
    cell_gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pos, charge, order, n, lx,
                                                                    ly, cp, cpf);
    void* twork = w;  // home-order work (tile_work_bytes)
    w += tile_work_bytes(p.n, p.ncx, p.ncy, p.ncz);
    if (p.tile) {  // fused screen + pair kernel: no neighbour rows
      if (accumulate) return cudaErrorInvalidValue;  // Coulomb callers overwrite
      int32_t* hperm = nullptr;
      e = tile_homes(start, skey, n, p.ncx, p.ncy, p.ncz, twork, &hperm, st);
      if (e != cudaSuccess) return e;
      const int grid = tile_grid(nh) < p.nblk ? tile_grid(nh) : (int)p.nblk;
      e = tile_pairs(cp, cpf, start, hperm, order, h0, h1, p.ncx, p.ncy, p.ncz, lx, ly, lz,
                     alpha, rc, forces, eblk, grid, status, st);
      if (e != cudaSuccess) return e;
      half_sum_kernel<<<1, 1024, 0, st>>>(eblk, grid, energy_out);
      return cudaGetLastError();
    }
    int32_t* nbr = reinterpret_cast<int32_t*>(w);
    w += align256(sizeof(int32_t) * n * (size_t)p.kcap);
    int32_t* nn = reinterpret_cast<int32_t*>(w);
    w += align256(sizeof(int32_t) * n);
    // conservative fp32 screen: positions rounded to fp32 move d2 by < 1e-2 for
    // |r| <= 1e3; the exact fp64 test is applied to every survivor
    const float rc2f = (float)(rc2 * (1.0 + 1e-3) + 1e-2);
    const int64_t nblk = (nh + kSRThreads - 1) / kSRThreads;
    const int64_t cblk = (p.ncell + kSRThreads / 32 - 1) / (kSRThreads / 32);
    const bool cells = nh <= kNbrCellsMaxHomes;
    // the warp-cooperative screen (short_tile.cu) for large full home ranges; its
    // rows follow the cell order like nbr_build's (a shard's home range is a
    // cell-order range, which the brick home order does not tile)
    const bool tile_screen = kNbrTile && !cells && h0 == 0 && h1 == n && p.span >= 2 &&
                             p.ncx >= 2 * p.span + 6 && p.ncy >= 2 * p.span + 6;
    if (tile_screen) {
      int32_t* hperm = nullptr;
      e = tile_homes(start, skey, n, p.ncx, p.ncy, p.ncz, twork, &hperm, st);
      if (e != cudaSuccess) return e;
      e = nbr_tile(cpf, start, hperm, 0, n, p.ncx, p.ncy, p.ncz, lx, ly, lz, rc2f, p.kcap, nbr, nn,
                   maxnn, status, st);
      if (e != cudaSuccess) return e;
    } else if (cells && p.span == 3)
      nbr_cells_kernel<3><<<(unsigned)cblk, kSRThreads, 0, st>>>(
          cpf, start, p.ncell, h0, h1, p.ncx, p.ncy, p.ncz, (float)lx, (float)ly, (float)lz,
          rc2f, p.kcap, nbr, nn, maxnn, status);
    else if (cells && p.span == 2)
      nbr_cells_kernel<2><<<(unsigned)cblk, kSRThreads, 0, st>>>(
          cpf, start, p.ncell, h0, h1, p.ncx, p.ncy, p.ncz, (float)lx, (float)ly, (float)lz,
          rc2f, p.kcap, nbr, nn, maxnn, status);
    else if (p.span == 3)
      nbr_build_kernel<3><<<(unsigned)nblk, kSRThreads, 0, st>>>(
          cpf, skey, start, h0, h1, p.ncx, p.ncy, p.ncz, (float)lx, (float)ly, (float)lz, rc2f, p.kcap, nbr,
          nn, maxnn, status);
    else if (p.span == 2)
      nbr_build_kernel<2><<<(unsigned)nblk, kSRThreads, 0, st>>>(
          cpf, skey, start, h0, h1, p.ncx, p.ncy, p.ncz, (float)lx, (float)ly, (float)lz, rc2f, p.kcap, nbr,
          nn, maxnn, status);
    else
      nbr_build_kernel<1><<<(unsigned)nblk, kSRThreads, 0, st>>>(
          cpf, skey, start, h0, h1, p.ncx, p.ncy, p.ncz, (float)lx, (float)ly, (float)lz, rc2f, p.kcap, nbr,
          nn, maxnn, status);
    if (pairs_after) cudaStreamWaitEvent(st, pairs_after, 0);
    const int split = pair_split(nh);
    const int64_t pgrid = pair_grid((nh * split + kSRThreads - 1) / kSRThreads);
    // every pair has alpha d <= alpha r_c: below the table end -> branch-free form
    const bool tab_only = alpha * sqrt(rc2) < 0.999 * SLAB_ERFCX_NINT / SLAB_ERFCX_INV_W &&
                          (!SLAB_PAIR_RAT || alpha * sqrt(rc2) <= 0.999 * kErfcxRatMax);
    const int kk = kind == 0 ? (tab_only ? 2 : 0) : 1;
    launch_pair_list(kk, split, (unsigned)pgrid, st, cp, order, nbr, nn, h0, h1, p.kcap, lx, ly,
                     kind == 0 ? alpha : 0.0, rc2, kind == 0 ? 0.0 : lj_eps,
                     kind == 0 ? 0.0 : sig2, forces, eblk, status, accumulate);
    // homes whose row overflowed (nn = -1), evaluated directly; in-stream, so
    // no pair is dropped and no host rerun is needed
#define SLAB_OVF_LAUNCH(S_, K_)                                                              \
  overflow_pairs_kernel<S_, K_><<<kOvfBlocks, kSRThreads, 0, st>>>(                          \
      cp, cpf, skey, start, order, nn, h0, h1, p.ncx, p.ncy, p.ncz, (float)lx, (float)ly,    \
      (float)lz, rc2f, lx, ly, kind == 0 ? alpha : 0.0, rc2, kind == 0 ? 0.0 : lj_eps,        \
      kind == 0 ? 0.0 : sig2, forces, eblk + pgrid, status, accumulate)
    if (kind == 1) {
      if (p.span == 3) SLAB_OVF_LAUNCH(3, 1);
      else if (p.span == 2) SLAB_OVF_LAUNCH(2, 1);
      else SLAB_OVF_LAUNCH(1, 1);
    } else {
      if (p.span == 3) SLAB_OVF_LAUNCH(3, 0);
      else if (p.span == 2) SLAB_OVF_LAUNCH(2, 0);
      else SLAB_OVF_LAUNCH(1, 0);
    }
#undef SLAB_OVF_LAUNCH
    half_sum_kernel<<<1, 1024, 0, st>>>(eblk, pgrid + kOvfBlocks, energy_out);
  }
  return cudaGetLastError();
}

}  // namespace slab
