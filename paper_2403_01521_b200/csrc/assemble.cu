// assemble.cu -- EnergyBreakdown and the scatter of forces back to input order.
//
// Replaces the numpy assembly of rbse2d.py:289-317 / soewald2d.py:401-438 and
// the O(N) terms self_energy (ewald2d.py:527-529) and slab_energy_forces
// (ewald2d.py:532-545):
//   forces_sorted[:,2] += (2 pi / A) q fz            (soewald2d.py:433)
//   out[perm] = forces_sorted; total = f_s + out + f_ps
//   u_self = alpha/sqrt(pi) sum q^2, u_ps = sum q phi(z),
//   phi(z) = -2 pi [sigma_top (lz - z) + sigma_bot z], F_ps,z = -2 pi q (st - sb)
//   u_l_0 = -sqrt(pi) Q /(alpha A) - (2 pi / A) u_pair  (soewald2d.py:415,430-432)
#include "common.cuh"
#include "kernels.cuh"

namespace slab {

__global__ void assemble_forces_kernel(int64_t n, const int32_t* __restrict__ perm,
                                       const double* __restrict__ qs,
                                       const double* __restrict__ fsorted,
                                       const double* __restrict__ fzf,
                                       const double* __restrict__ fzb, double zpref,
                                       const double* __restrict__ fshort,
                                       const double* __restrict__ charge, double plane,
                                       double* __restrict__ forces) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const int64_t i = perm[a];
  double fx = fsorted[3 * a], fy = fsorted[3 * a + 1], fz = fsorted[3 * a + 2];
  if (fzf) fz += zpref * qs[a] * (fzf[a] - fzb[a]);
  double sx = 0.0, sy = 0.0, sz = 0.0;
  if (fshort) {
    sx = fshort[3 * i];
    sy = fshort[3 * i + 1];
    sz = fshort[3 * i + 2];
  }
  forces[3 * i] = sx + fx;
  forces[3 * i + 1] = sy + fy;
  forces[3 * i + 2] = sz + fz + (-2.0 * kPi * charge[i]) * plane;
}

constexpr int kEBlocks = 296;  // partial sums for Q = sum q^2 and u_ps

__global__ void __launch_bounds__(256) energy_partials_kernel(
    int64_t n, const double* __restrict__ charge, const double* __restrict__ pos, double lz,
    double sigma_top, double sigma_bot, double* __restrict__ part) {
  __shared__ double r0[256], r1[256];
  double q2 = 0.0, ups = 0.0;
  for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += (int64_t)kEBlocks * 256) {
    const double q = charge[i], z = pos[3 * i + 2];
    q2 = fma(q, q, q2);
    ups += q * (-2.0 * kPi * (sigma_top * (lz - z) + sigma_bot * z));
  }
  r0[threadIdx.x] = q2;
  r1[threadIdx.x] = ups;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      r0[threadIdx.x] += r0[threadIdx.x + s];
      r1[threadIdx.x] += r1[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = r0[0];
    part[kEBlocks + blockIdx.x] = r1[0];
  }
}

__global__ void __launch_bounds__(512) assemble_energy_kernel(
    int64_t n, const double* __restrict__ part, double alpha, double area, double charge_const,
    const double* __restrict__ u_s, const double* __restrict__ u_sweep,
    const double* __restrict__ u_pair, const int* __restrict__ status,
    double* __restrict__ energy, int include_constants) {
  __shared__ double r0[512], r1[512];
  r0[threadIdx.x] = threadIdx.x < kEBlocks ? part[threadIdx.x] : 0.0;
  r1[threadIdx.x] = threadIdx.x < kEBlocks ? part[kEBlocks + threadIdx.x] : 0.0;
  __syncthreads();
  for (int s = 256; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      r0[threadIdx.x] += r0[threadIdx.x + s];
      r1[threadIdx.x] += r1[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double Q = r0[0];
    energy[0] = u_s ? u_s[0] : 0.0;
    energy[1] = charge_const + (u_sweep ? u_sweep[0] : 0.0);
    double u0 = (n && include_constants) ? -kSqrtPi * Q / (alpha * area) : 0.0;
    if (u_pair) u0 += -2.0 * kPi / area * u_pair[0];
    energy[2] = u0;
    energy[3] = include_constants ? alpha / kSqrtPi * Q : 0.0;
    energy[4] = include_constants ? r1[0] : 0.0;
    const int st = status ? status[0] : 0;
    energy[5] = (double)st;
    energy[6] = include_constants ? Q : 0.0;
    // status again, one 8-bit counter per bit (bit k -> 256^k): the multi-GPU
    // all-reduce SUMS the packed energies, which keeps "any rank set bit k"
    // recoverable for up to 255 ranks (slot 5 is the single-rank form)
    double spread = 0.0, w = 1.0;
    for (int k = 0; k < 6; ++k, w *= 256.0)
      if (st & (1 << k)) spread += w;
    energy[7] = spread;
  }
}

cudaError_t assemble_forces(int64_t n, const int32_t* perm, const double* qs,
                            const double* fsorted, const double* fzf, const double* fzb,
                            double zpref, const double* fshort, const double* charge,
                            double fz_plane, double* forces, cudaStream_t st) {
  if (n > 0)
    assemble_forces_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        n, perm, qs, fsorted, fzf, fzb, zpref, fshort, charge, fz_plane, forces);
  return cudaGetLastError();
}

cudaError_t assemble_energy(int64_t n, const double* charge, const double* pos, double lz,
                            double sigma_top, double sigma_bot, double alpha, double area,
                            double charge_const, const double* u_s, const double* u_sweep,
                            const double* u_pair, const int* status, double* energy,
                            double* energy_scratch, int include_constants, cudaStream_t st) {
  // the 2*kEBlocks partials live in energy[8..] (callers pass >= 8 + 2*kEBlocks doubles
  // of scratch through `energy_scratch`)
  energy_partials_kernel<<<kEBlocks, 256, 0, st>>>(n, charge, pos, lz, sigma_top, sigma_bot,
                                                    energy_scratch);
  assemble_energy_kernel<<<1, 512, 0, st>>>(n, energy_scratch, alpha, area, charge_const, u_s,
                                            u_sweep, u_pair, status, energy, include_constants);
  return cudaGetLastError();
}

}  // namespace slab

namespace slab {

__global__ void fz_accumulate_kernel(int64_t n, const double* __restrict__ fzf,
                                     const double* __restrict__ fzb, double* __restrict__ fz) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) fz[a] += fzf[a] - fzb[a];
}

cudaError_t fz_accumulate(int64_t n, const double* fzf, const double* fzb, double* fz,
                          cudaStream_t st) {
  if (n > 0) fz_accumulate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, fzf, fzb, fz);
  return cudaGetLastError();
}

// soewald2d.py:42-64 recursive_pair_sum: one forward recursion for a single
// complex beta (a test / API utility, not on the evaluation path):
// out[a] = sum_{j<a} q_j exp(-i theta_j - beta (z_a - z_j)).  Chunked like the
// sweep: per-chunk aggregates, carry over chunks, exact recursion per chunk.
__global__ void rps_aggregate_kernel(const double* __restrict__ q, const double* __restrict__ th,
                                     const double* __restrict__ z, int64_t n, int R, double br,
                                     double bi, double2* __restrict__ agg) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  int64_t a0 = (int64_t)c * R;
  if (a0 >= n) return;
  int64_t a1 = a0 + R < n ? a0 + R : n;
  const double zend = z[a1 - 1];
  C2 acc{0.0, 0.0};
  for (int64_t j = a0; j < a1; ++j) {
    double s, co;
    sincos_fast(th[j], &s, &co);
    const double dz = zend - z[j];
    C2 e = cexp_neg(br * dz, bi * dz);
    C2 u{q[j] * co, -q[j] * s};
    C2 t = cmul(u, e);
    acc.re += t.re;
    acc.im += t.im;
  }
  agg[c] = make_double2(acc.re, acc.im);
}

__global__ void rps_final_kernel(const double* __restrict__ q, const double* __restrict__ th,
                                 const double* __restrict__ z, int64_t n, int R, int nch,
                                 double br, double bi, const double2* __restrict__ agg,
                                 double* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nch) return;
  // carry-in: inclusive state at the end of chunk c-1, rebuilt from the aggregates
  C2 T{0.0, 0.0};
  for (int k = 0; k < c; ++k) {
    const int64_t e0 = (int64_t)k * R;
    const int64_t e1 = e0 + R < n ? e0 + R : n;
    if (k > 0) {
      const double dz = z[e1 - 1] - z[e0 - 1];
      T = cmul(T, cexp_neg(br * dz, bi * dz));
    }
    T.re += agg[k].x;
    T.im += agg[k].y;
  }
  const int64_t a0 = (int64_t)c * R, a1 = a0 + R < n ? a0 + R : n;
  for (int64_t a = a0; a < a1; ++a) {
    if (a > 0) {
      const double dz = z[a] - z[a - 1];
      T = cmul(T, cexp_neg(br * dz, bi * dz));
    } else {
      T = C2{0.0, 0.0};
    }
    out[2 * a] = T.re;
    out[2 * a + 1] = T.im;
    double s, co;
    sincos_fast(th[a], &s, &co);
    T.re += q[a] * co;
    T.im -= q[a] * s;
  }
}

cudaError_t recursive_pair_sum(const double* q, const double* theta, const double* z, int64_t n,
                               double beta_re, double beta_im, double* out, double2* agg,
                               cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int R = 64;
  const int nch = (int)((n + R - 1) / R);
  rps_aggregate_kernel<<<(nch + 63) / 64, 64, 0, st>>>(q, theta, z, n, R, beta_re, beta_im, agg);
  rps_final_kernel<<<(nch + 63) / 64, 64, 0, st>>>(q, theta, z, n, R, nch, beta_re, beta_im, agg,
                                                   out);
  return cudaGetLastError();
}

}  // namespace slab

// ---------------------------------------------------------------------------
// FP64 roofline denominator: a DFMA throughput microbenchmark (8 independent
// chains per thread, 2 CTAs of 1024 threads per SM).  MEASURED_PEAKS.json has
// no fp64 figure, so bench.py measures it live on the box it runs on.
// ---------------------------------------------------------------------------
namespace slab {
__global__ void __launch_bounds__(1024) dfma_peak_kernel(double* out, int iters, double a,
                                                         double b) {
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

cudaError_t fp64_peak(double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaError_t e = cudaMalloc(&out, sizeof(double));
  if (e != cudaSuccess) return e;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 2 * sms, threads = 1024, iters = 20000;
  dfma_peak_kernel<<<blocks, threads>>>(out, 200, 1.0000001, 1e-7);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dfma_peak_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  *tflops = 2.0 * 8.0 * iters * (double)blocks * threads / (best * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError();
}
}  // namespace slab
