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
// each cell) -> cell-sorted SoA + cell_start by binary search.  One CTA per home
// cell; each thread owns home particles and sums over the full 27-cell shell
// (both orders of every pair) so each force is accumulated by exactly one
// thread: deterministic, no atomics.  u_s = 1/2 of the full-shell sum.
#include "common.cuh"
#include "kernels.cuh"

namespace slab {

struct PairAcc {
  double fx, fy, fz, e;
};

__device__ __forceinline__ void pair_accumulate(double xi, double yi, double zi, double qi,
                                                double xj, double yj, double zj, double qj,
                                                double lx, double ly, double alpha, double rc2,
                                                double c, PairAcc& acc, int& flag) {
  // rounding exactly as the numba reference (no FMA contraction in the geometry)
  double dx = __dsub_rn(xi, xj), dy = __dsub_rn(yi, yj);
  const double dz = __dsub_rn(zi, zj);
  dx = __dsub_rn(dx, __dmul_rn(lx, rint(__ddiv_rn(dx, lx))));
  dy = __dsub_rn(dy, __dmul_rn(ly, rint(__ddiv_rn(dy, ly))));
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  if (d2 > rc2) return;
  if (d2 < 1e-24) {
    flag = 1;
    return;
  }
  const double d = sqrt(d2);
  const double qq = qi * qj;
  const double e = erfc(alpha * d);
  acc.e += qq * e / d;
  const double fmag = qq * (e / (d2 * d) + c * exp(-alpha * alpha * d2) / d2);
  acc.fx = fma(fmag, dx, acc.fx);
  acc.fy = fma(fmag, dy, acc.fy);
  acc.fz = fma(fmag, dz, acc.fz);
}

// ewald2d.py:126-138
__global__ void cell_index_kernel(const double* __restrict__ pos, int64_t n, double lx, double ly,
                                  double lz, int ncx, int ncy, int ncz, uint32_t* __restrict__ key,
                                  int32_t* __restrict__ val) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  long long cx = (long long)(pos[3 * i + 0] / lx * ncx);
  long long cy = (long long)(pos[3 * i + 1] / ly * ncy);
  long long cz = (long long)(pos[3 * i + 2] / lz * ncz);
  cx = ((cx % ncx) + ncx) % ncx;
  cy = ((cy % ncy) + ncy) % ncy;
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

__global__ void cell_gather_kernel(const double* __restrict__ pos, const double* __restrict__ q,
                                   const int32_t* __restrict__ order, int64_t n,
                                   double4* __restrict__ cp) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  int64_t i = order[a];
  cp[a] = make_double4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], q[i]);
}

constexpr int kCellThreads = 64;

__global__ void __launch_bounds__(kCellThreads) cell_pair_kernel(
    const double4* __restrict__ cp, const int32_t* __restrict__ order,
    const int32_t* __restrict__ start, int ncx, int ncy, int ncz, double lx, double ly,
    double alpha, double rc2, double* __restrict__ forces, double* __restrict__ eblk,
    int* __restrict__ status) {
  const int cid = blockIdx.x;
  const int cz = cid % ncz, cy = (cid / ncz) % ncy, cx = cid / (ncz * ncy);
  const int h0 = start[cid], h1 = start[cid + 1];
  const double c = kTwoOverSqrtPi * alpha;
  double esum = 0.0;
  int flag = 0;
  for (int ii = h0 + threadIdx.x; ii < h1; ii += kCellThreads) {
    const double4 pi = cp[ii];
    PairAcc acc{0.0, 0.0, 0.0, 0.0};
    for (int off = 0; off < 27; ++off) {
      const int dxc = off / 9 - 1, dyc = (off / 3) % 3 - 1, dzc = off % 3 - 1;
      const int nz = cz + dzc;
      if (nz < 0 || nz >= ncz) continue;
      const int nx = (cx + dxc + ncx) % ncx, ny = (cy + dyc + ncy) % ncy;
      const int nid = (nx * ncy + ny) * ncz + nz;
      const int b0 = start[nid], b1 = start[nid + 1];
      for (int jj = b0; jj < b1; ++jj) {
        if (jj == ii) continue;
        const double4 pj = cp[jj];
        pair_accumulate(pi.x, pi.y, pi.z, pi.w, pj.x, pj.y, pj.z, pj.w, lx, ly, alpha, rc2, c,
                        acc, flag);
      }
    }
    const int64_t i = order[ii];
    forces[3 * i + 0] = acc.fx;
    forces[3 * i + 1] = acc.fy;
    forces[3 * i + 2] = acc.fz;
    esum += acc.e;
  }
  if (flag) atomicOr(status, SLAB_STATUS_COINCIDENT_DEV);
  // fixed-order block reduction
  __shared__ double red[kCellThreads];
  red[threadIdx.x] = esum;
  __syncthreads();
  for (int s = kCellThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[cid] = red[0];
}

// all pairs (ncx < 3 or ncy < 3): grid (i tiles, j splits)
__global__ void __launch_bounds__(128) brute_pair_kernel(
    const double* __restrict__ pos, const double* __restrict__ q, int64_t n, int jsplit,
    double lx, double ly, double alpha, double rc2, double* __restrict__ fbuf,
    double* __restrict__ eblk, int* __restrict__ status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int js = blockIdx.y;
  const int64_t per = (n + jsplit - 1) / jsplit;
  const int64_t j0 = js * per, j1 = j0 + per < n ? j0 + per : n;
  const double c = kTwoOverSqrtPi * alpha;
  PairAcc acc{0.0, 0.0, 0.0, 0.0};
  int flag = 0;
  if (i < n) {
    const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2], qi = q[i];
    for (int64_t j = j0; j < j1; ++j) {
      if (j == i) continue;
      pair_accumulate(xi, yi, zi, qi, pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], q[j], lx, ly,
                      alpha, rc2, c, acc, flag);
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
                                          double* __restrict__ forces) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= n3) return;
  double v = 0.0;
  for (int s = 0; s < jsplit; ++s) v += fbuf[(size_t)s * n3 + e];
  forces[e] = v;
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

ShortPlan short_plan(int64_t n, double lx, double ly, double lz, double rc) {
  ShortPlan p{};
  p.n = n;
  int ncx = (int)(lx / rc), ncy = (int)(ly / rc), ncz = (int)(lz / rc);
  ncx = ncx < 1 ? 1 : ncx;
  ncy = ncy < 1 ? 1 : ncy;
  ncz = ncz < 1 ? 1 : ncz;
  p.brute = (ncx < 3 || ncy < 3);
  if (p.brute) ncx = ncy = ncz = 1;
  p.ncx = ncx;
  p.ncy = ncy;
  p.ncz = ncz;
  p.ncell = (int64_t)ncx * ncy * ncz;
  const int64_t nbx = (n + 127) / 128;
  int js = (int)(592 / (nbx > 0 ? nbx : 1));
  p.jsplit = p.brute ? (js < 1 ? 1 : (js > 64 ? 64 : js)) : 1;
  p.nblk = p.brute ? (int64_t)p.jsplit * (nbx > 0 ? nbx : 1) : p.ncell;
  return p;
}

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t short_work_bytes(const ShortPlan& p) {
  const size_t n = (size_t)(p.n > 0 ? p.n : 1);
  size_t b = 0;
  b += align256(sizeof(double) * p.nblk);  // eblk
  if (p.brute) {
    b += align256(sizeof(double) * 3 * n * p.jsplit);
  } else {
    b += 2 * align256(sizeof(uint32_t) * n) + 2 * align256(sizeof(int32_t) * n);
    b += align256(sizeof(int32_t) * radix_hist_entries(p.n));
    b += align256(sizeof(int32_t) * (p.ncell + 1));
    b += align256(sizeof(double4) * n);
  }
  return b + 256;
}

cudaError_t short_run(const ShortPlan& p, void* work, const double* pos, const double* charge,
                      double lx, double ly, double lz, double alpha, double rc, double* forces,
                      double* energy_out, int* status, cudaStream_t st) {
  const int64_t n = p.n;
  if (n < 2) {
    cudaMemsetAsync(energy_out, 0, sizeof(double), st);
    if (n > 0) cudaMemsetAsync(forces, 0, sizeof(double) * 3 * n, st);
    return cudaGetLastError();
  }
  char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(work) + 255) & ~(uintptr_t)255);
  double* eblk = reinterpret_cast<double*>(w);
  w += align256(sizeof(double) * p.nblk);
  const double rc2 = rc * rc;
  if (p.brute) {
    double* fbuf = reinterpret_cast<double*>(w);
    const unsigned nbx = (unsigned)((n + 127) / 128);
    brute_pair_kernel<<<dim3(nbx, p.jsplit), 128, 0, st>>>(pos, charge, n, p.jsplit, lx, ly, alpha,
                                                           rc2, fbuf, eblk, status);
    brute_force_reduce_kernel<<<(unsigned)((3 * n + 255) / 256), 256, 0, st>>>(fbuf, p.jsplit,
                                                                               3 * n, forces);
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
    cell_gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pos, charge, order, n, cp);
    cell_pair_kernel<<<(unsigned)p.ncell, kCellThreads, 0, st>>>(
        cp, order, start, p.ncx, p.ncy, p.ncz, lx, ly, alpha, rc2, forces, eblk, status);
  }
  half_sum_kernel<<<1, 1024, 0, st>>>(eblk, p.nblk, energy_out);
  return cudaGetLastError();
}

}  // namespace slab
