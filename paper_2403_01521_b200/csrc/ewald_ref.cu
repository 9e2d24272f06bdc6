// ewald_ref.cu -- the O(N^2 K) Ewald2D reference solver on device
// (the accuracy oracle behind the error scans).
//
// Replaces reference ewald2d.py:331-442 (_fourier_ref_kernel, ring-factored
// pairwise Fourier sweep, "stable" and "naive" xi kernels) and 477-501
// (_zero_mode_kernel, G(z) = z erf(a z) + exp(-a^2 z^2) / (a sqrt(pi))).
//
// One thread per particle i over every j != i (full shell): the force on i is
// owned by one thread (deterministic, no atomics); each pair's energy is
// counted from both sides and halved in the block-partial sum.  Per pair the
// xi kernels are evaluated once per ring of equal |k| (ewald2d.py:310-328) and
// the angular factors come from cos/sin recurrences in the integer mode
// indices, as in the reference.
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace slab {

constexpr int kRefThreads = 128;
constexpr int kRefMaxRing = 256;  // rings of equal |k| per call (host splits larger sets)
constexpr int kRefMaxM = 64;      // |mx|, |my| bound for the recurrence tables

// erfcx for x >= 0 in the form of ewald2d.py:96-107 (direct product below 25,
// continued fraction beyond); libdevice erfcx is the accurate version of both
__device__ __forceinline__ double erfcx_pos(double x) { return erfcx(x); }

__global__ void __launch_bounds__(kRefThreads) ewald_ref_fourier_kernel(
    const double* __restrict__ pos, const double* __restrict__ charge, int64_t n, double lx,
    double ly, double alpha, const int* __restrict__ mxy, const int* __restrict__ ring_id,
    int nmode, const double* __restrict__ kappa, int nring, int mxmax, int mymax, int naive,
    double* __restrict__ forces, double* __restrict__ eblk) {
  __shared__ double sk[kRefMaxRing];    // kappa
  __shared__ double shalf[kRefMaxRing];  // kappa / 2a
  __shared__ double sdamp[kRefMaxRing];  // exp(-(kappa/2a)^2)
  __shared__ double red[kRefThreads];
  for (int r = threadIdx.x; r < nring; r += blockDim.x) {
    sk[r] = kappa[r];
    shalf[r] = kappa[r] / (2.0 * alpha);
    sdamp[r] = exp(-shalf[r] * shalf[r]);
  }
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double pref = kPi / (lx * ly), fx = 2.0 * kPi / lx, fy = 2.0 * kPi / ly;
  double fxi_t = 0.0, fyi_t = 0.0, fzi_t = 0.0, e_t = 0.0;
  if (i < n) {
    const double xi = pos[3 * i], yi = pos[3 * i + 1], zi = pos[3 * i + 2], qi = charge[i];
    double xs[kRefMaxRing], xd[kRefMaxRing];
    double ca[kRefMaxM + 1], sa[kRefMaxM + 1], cb[kRefMaxM + 1], sb[kRefMaxM + 1];
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double qq = qi * charge[j];
      const double dx = xi - pos[3 * j], dy = yi - pos[3 * j + 1];
      double z = zi - pos[3 * j + 2];
      double sgn = 0.0;
      if (z > 0.0) {
        sgn = 1.0;
      } else if (z < 0.0) {
        sgn = -1.0;
        z = -z;
      }
      const double gz = exp(-alpha * alpha * z * z);
      for (int r = 0; r < nring; ++r) {
        const double kap = sk[r], h = shalf[r];
        double xp, xm;
        if (naive) {
          xp = exp(kap * z) * erfc(h + alpha * z);
          xm = exp(-kap * z) * erfc(h - alpha * z);
        } else {
          const double damp = sdamp[r] * gz;
          xp = erfcx_pos(h + alpha * z) * damp;
          xm = alpha * z > h ? 2.0 * exp(-kap * z) - erfcx_pos(alpha * z - h) * damp
                             : erfcx_pos(h - alpha * z) * damp;
        }
        xs[r] = (xp + xm) / kap;
        xd[r] = xp - xm;
      }
      double su, cu, sv, cv;
      sincos(fx * dx, &su, &cu);
      sincos(fy * dy, &sv, &cv);
      ca[0] = 1.0;
      sa[0] = 0.0;
      for (int t = 1; t <= mxmax; ++t) {
        ca[t] = ca[t - 1] * cu - sa[t - 1] * su;
        sa[t] = sa[t - 1] * cu + ca[t - 1] * su;
      }
      cb[0] = 1.0;
      sb[0] = 0.0;
      for (int t = 1; t <= mymax; ++t) {
        cb[t] = cb[t - 1] * cv - sb[t - 1] * sv;
        sb[t] = sb[t - 1] * cv + cb[t - 1] * sv;
      }
      double fxs = 0.0, fys = 0.0, fzs = 0.0, esum = 0.0;
      for (int t = 0; t < nmode; ++t) {
        const int ax = mxy[2 * t], by = mxy[2 * t + 1];
        const int aax = ax < 0 ? -ax : ax, aby = by < 0 ? -by : by;
        const double cxv = ca[aax], sxv = ax >= 0 ? sa[aax] : -sa[aax];
        const double cyv = cb[aby], syv = by >= 0 ? sb[aby] : -sb[aby];
        const double cosw = cxv * cyv - sxv * syv;
        const double sinw = sxv * cyv + cxv * syv;
        const int r = ring_id[t];
        esum += cosw * xs[r];
        fxs += sinw * xs[r] * ax;
        fys += sinw * xs[r] * by;
        fzs += cosw * xd[r];
      }
      const double cc = pref * qq;
      e_t += cc * esum;
      fxi_t += cc * fxs * fx;
      fyi_t += cc * fys * fy;
      fzi_t -= cc * fzs * sgn;
    }
    forces[3 * i + 0] = fxi_t;
    forces[3 * i + 1] = fyi_t;
    forces[3 * i + 2] = fzi_t;
  }
  red[threadIdx.x] = 0.5 * e_t;  // each pair counted from both sides
  __syncthreads();
  for (int w = kRefThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[blockIdx.x] = red[0];
}

// ewald2d.py:477-501: u_pair = sum_{i<j} q_i q_j G(|z_ij|), fz_i = sum_j q_i q_j erf(a |z_ij|) sgn
__global__ void __launch_bounds__(kRefThreads) ewald_ref_zero_kernel(
    const double* __restrict__ pos, const double* __restrict__ charge, int64_t n, double alpha,
    double* __restrict__ fz, double* __restrict__ eblk) {
  __shared__ double red[kRefThreads];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double inv = 1.0 / (alpha * kSqrtPi);
  double e_t = 0.0, f_t = 0.0;
  if (i < n) {
    const double zi = pos[3 * i + 2], qi = charge[i];
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double dz = zi - pos[3 * j + 2];
      double sgn = 1.0;
      if (dz < 0.0) {
        sgn = -1.0;
        dz = -dz;
      }
      const double qq = qi * charge[j];
      const double e = erf(alpha * dz);
      e_t += qq * (dz * e + exp(-alpha * alpha * dz * dz) * inv);
      f_t += qq * e * sgn;
    }
    fz[i] = f_t;
  }
  red[threadIdx.x] = 0.5 * e_t;
  __syncthreads();
  for (int w = kRefThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(1024) ewald_ref_sum_kernel(const double* __restrict__ part,
                                                             int64_t m, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += 1024) s += part[k];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

int64_t ewald_ref_partials(int64_t n) { return (n + kRefThreads - 1) / kRefThreads; }
int ewald_ref_max_ring() { return kRefMaxRing; }
int ewald_ref_max_m() { return kRefMaxM; }

cudaError_t ewald_ref_fourier(const double* pos, const double* charge, int64_t n, double lx,
                              double ly, double alpha, const int* mxy, const int* ring_id,
                              int nmode, const double* kappa, int nring, int mxmax, int mymax,
                              int naive, double* forces, double* energy, double* part,
                              cudaStream_t st) {
  const int64_t nb = ewald_ref_partials(n);
  if (n > 0) {
    ewald_ref_fourier_kernel<<<(unsigned)nb, kRefThreads, 0, st>>>(
        pos, charge, n, lx, ly, alpha, mxy, ring_id, nmode, kappa, nring, mxmax, mymax, naive,
        forces, part);
    ewald_ref_sum_kernel<<<1, 1024, 0, st>>>(part, nb, energy);
  }
  return cudaGetLastError();
}

cudaError_t ewald_ref_zero(const double* pos, const double* charge, int64_t n, double alpha,
                           double* fz, double* energy, double* part, cudaStream_t st) {
  const int64_t nb = ewald_ref_partials(n);
  if (n > 0) {
    ewald_ref_zero_kernel<<<(unsigned)nb, kRefThreads, 0, st>>>(pos, charge, n, alpha, fz, part);
    ewald_ref_sum_kernel<<<1, 1024, 0, st>>>(part, nb, energy);
  }
  return cudaGetLastError();
}

}  // namespace slab
