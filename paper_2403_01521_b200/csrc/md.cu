// md.cu -- device-resident MD step around the evaluator.
//
// Replaces the O(N) numpy parts of reference md.py: wall_forces (59-77),
// langevin_step (180-193) with its Gaussian noise, the plain velocity-Verlet
// kick / drift (300-305), the Nose-Hoover velocity scaling (196-224), the xy
// wrap with accumulated image shifts (run_simulation 245-250) and
// kinetic_energy (176-177).  The WCA pair core (lj_forces 34-56) runs through
// the short-range pair machinery (short.cu, KIND 1).
//
// Thermostat noise: counter-based Philox4x32-10 (seed = key, (step, particle)
// = counter, a domain word separate from the mode sampler) + Box-Muller in
// fp64, instead of numpy's Generator: reproducible per seed, not
// numpy-identical (the same policy as the mode sampler).  The step counter
// lives in device memory and is advanced by the kernel that consumes it, so a
// whole MD step can be captured in a CUDA graph.
#include "common.cuh"
#include "kernels.cuh"
#include "philox.cuh"

namespace slab {

constexpr uint32_t kNoiseDomain = 0x4D44u;  // 'MD'
constexpr int kMdThreads = 256;

__device__ __forceinline__ void wrap_xy(double* __restrict__ p, double* __restrict__ shift,
                                        int64_t i, double lx, double ly) {
  // run_simulation.wrap (md.py:245-250): moved = floor(p / L); shift += moved L; p -= moved L
  const double mx = floor(p[3 * i] / lx), my = floor(p[3 * i + 1] / ly);
  if (shift) {
    shift[2 * i] += mx * lx;
    shift[2 * i + 1] += my * ly;
  }
  p[3 * i] -= mx * lx;
  p[3 * i + 1] -= my * ly;
}

// v += 0.5 dt F / m ; x += 0.5 dt v ; v = c v + sqrt((1 - c^2) T / m) xi ; x += 0.5 dt v ;
// wrap.  counter[0] = this step's noise counter (read; advanced by md_counter_kernel).
__global__ void langevin_kernel(double* __restrict__ pos, double* __restrict__ vel,
                                const double* __restrict__ forces, const double* __restrict__ mass,
                                int64_t n, double dt, double c, double temperature, uint64_t seed,
                                const int64_t* __restrict__ counter, double* __restrict__ shift,
                                double lx, double ly) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t ctr = ((uint64_t)counter[0] * (uint64_t)n + (uint64_t)i) * 2;
  const uint4 r0 = Philox::gen(seed, ctr, kNoiseDomain);
  const uint4 r1 = Philox::gen(seed, ctr + 1, kNoiseDomain);
  double xi[4];
  {
    const double u1 = u01_open(r0.x, r0.y), u2 = u01_open(r0.z, r0.w);
    const double rad = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    xi[0] = rad * cs;
    xi[1] = rad * sn;
    const double u3 = u01_open(r1.x, r1.y), u4 = u01_open(r1.z, r1.w);
    const double rad2 = sqrt(-2.0 * log(u3));
    sincospi(2.0 * u4, &sn, &cs);
    xi[2] = rad2 * cs;
    xi[3] = rad2 * sn;
  }
  const double m = mass[i], inv_m = 1.0 / m;
  const double amp = sqrt((1.0 - c * c) * temperature / m);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double v = vel[3 * i + d] + 0.5 * dt * forces[3 * i + d] * inv_m;
    double x = pos[3 * i + d] + 0.5 * dt * v;
    v = c * v + amp * xi[d];
    x = x + 0.5 * dt * v;
    vel[3 * i + d] = v;
    pos[3 * i + d] = x;
  }
  wrap_xy(pos, shift, i, lx, ly);
}

__global__ void md_counter_kernel(int64_t* counter) {
  if (threadIdx.x == 0 && blockIdx.x == 0) counter[0] += 1;
}

// v += h F / m
__global__ void kick_kernel(double* __restrict__ vel, const double* __restrict__ forces,
                            const double* __restrict__ mass, int64_t n, double h) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= 3 * n) return;
  vel[e] += h * forces[e] / mass[e / 3];
}

// x += dt v ; wrap
__global__ void drift_kernel(double* __restrict__ pos, const double* __restrict__ vel, int64_t n,
                             double dt, double* __restrict__ shift, double lx, double ly) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int d = 0; d < 3; ++d) pos[3 * i + d] += dt * vel[3 * i + d];
  wrap_xy(pos, shift, i, lx, ly);
}

__global__ void scale_kernel(double* __restrict__ vel, int64_t n3, double s) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < n3) vel[e] *= s;
}

// md.py:59-77: repulsive WCA form on the distances to z = 0 and z = lz.
// F_z += sign 24 eps (2 s6^2 - s6) / d; energy partials per block (fixed order).
__global__ void __launch_bounds__(kMdThreads) walls_kernel(
    const double* __restrict__ pos, int64_t n, double lz, double eps, double sigma,
    double* __restrict__ forces, double* __restrict__ part, int* __restrict__ status) {
  __shared__ double red[kMdThreads];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double cut = 1.122462048309373 * sigma;  // 2^(1/6) sigma
  double u = 0.0;
  if (i < n) {
    const double z = pos[3 * i + 2];
    double fz = 0.0;
    int bad = 0;
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      const double d = w == 0 ? z : lz - z;
      const double sign = w == 0 ? 1.0 : -1.0;
      if (d < cut) {
        if (d <= 0.0) {
          bad = 1;
        } else {
          const double sd = sigma / d;
          const double s2 = sd * sd, s6 = s2 * s2 * s2;
          u += 4.0 * eps * (s6 * s6 - s6) + eps;
          fz += sign * 24.0 * eps * (2.0 * s6 * s6 - s6) / d;
        }
      }
    }
    if (bad) atomicOr(status, SLAB_STATUS_WALL_DEV);
    forces[3 * i + 2] += fz;
  }
  red[threadIdx.x] = u;
  __syncthreads();
  for (int w = kMdThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// 0.5 sum m v^2 (md.py:176-177): block partials
__global__ void __launch_bounds__(kMdThreads) kinetic_kernel(const double* __restrict__ vel,
                                                             const double* __restrict__ mass,
                                                             int64_t n, double* __restrict__ part) {
  __shared__ double red[kMdThreads];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double k = 0.0;
  if (i < n) {
    const double vx = vel[3 * i], vy = vel[3 * i + 1], vz = vel[3 * i + 2];
    k = 0.5 * mass[i] * (vx * vx + vy * vy + vz * vz);
  }
  red[threadIdx.x] = k;
  __syncthreads();
  for (int w = kMdThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// fixed-order sum of block partials: out[0] = scale * sum (+ out[0] if accumulate)
__global__ void __launch_bounds__(1024) partial_sum_kernel(const double* __restrict__ part,
                                                           int64_t m, double* __restrict__ out,
                                                           int accumulate) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t k = threadIdx.x; k < m; k += 1024) s += part[k];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = accumulate ? out[0] + red[0] : red[0];
}

static unsigned blocks_for(int64_t n) { return (unsigned)((n + kMdThreads - 1) / kMdThreads); }
int64_t md_partials(int64_t n) { return (n + kMdThreads - 1) / kMdThreads; }

cudaError_t md_langevin(double* pos, double* vel, const double* forces, const double* mass,
                        int64_t n, double dt, double gamma, double temperature, uint64_t seed,
                        int64_t* counter, double* shift, double lx, double ly, cudaStream_t st) {
  if (n > 0)
    langevin_kernel<<<blocks_for(n), kMdThreads, 0, st>>>(pos, vel, forces, mass, n, dt,
                                                          exp(-gamma * dt), temperature, seed,
                                                          counter, shift, lx, ly);
  md_counter_kernel<<<1, 32, 0, st>>>(counter);
  return cudaGetLastError();
}

cudaError_t md_kick(double* vel, const double* forces, const double* mass, int64_t n, double h,
                    cudaStream_t st) {
  if (n > 0) kick_kernel<<<blocks_for(3 * n), kMdThreads, 0, st>>>(vel, forces, mass, n, h);
  return cudaGetLastError();
}

cudaError_t md_drift(double* pos, const double* vel, int64_t n, double dt, double* shift, double lx,
                     double ly, cudaStream_t st) {
  if (n > 0) drift_kernel<<<blocks_for(n), kMdThreads, 0, st>>>(pos, vel, n, dt, shift, lx, ly);
  return cudaGetLastError();
}

cudaError_t md_scale(double* vel, int64_t n, double s, cudaStream_t st) {
  if (n > 0) scale_kernel<<<blocks_for(3 * n), kMdThreads, 0, st>>>(vel, 3 * n, s);
  return cudaGetLastError();
}

cudaError_t md_walls(const double* pos, int64_t n, double lz, double eps, double sigma,
                     double* forces, double* energy, int* status, double* part, int accumulate,
                     cudaStream_t st) {
  if (n > 0) {
    walls_kernel<<<blocks_for(n), kMdThreads, 0, st>>>(pos, n, lz, eps, sigma, forces, part,
                                                       status);
    partial_sum_kernel<<<1, 1024, 0, st>>>(part, md_partials(n), energy, accumulate);
  } else if (!accumulate) {
    cudaMemsetAsync(energy, 0, sizeof(double), st);
  }
  return cudaGetLastError();
}

cudaError_t md_kinetic(const double* vel, const double* mass, int64_t n, double* out,
                       double* part, cudaStream_t st) {
  if (n > 0) {
    kinetic_kernel<<<blocks_for(n), kMdThreads, 0, st>>>(vel, mass, n, part);
    partial_sum_kernel<<<1, 1024, 0, st>>>(part, md_partials(n), out, 0);
  } else {
    cudaMemsetAsync(out, 0, sizeof(double), st);
  }
  return cudaGetLastError();
}

}  // namespace slab
