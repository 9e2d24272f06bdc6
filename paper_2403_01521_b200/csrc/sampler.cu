// sampler.cu -- Metropolis importance sampling of the P Fourier modes on device.
//
// Replaces reference rbse2d.py:96-214 (_axis_logq, _chain_kernel, ModeSampler).
// Same chain: independence proposals m* = rint(N(0,1) sigma) per axis with
// sigma = 1/(a sqrt 2), a = pi/(alpha L); target log weight -((a_x mx)^2 +
// (a_y my)^2); proposal log mass of the rounded normal (erf differences); the
// (0,0) proposal counts as a step and is rejected; every thin-th step is
// recorded (repeats kept); burn-in in chunks of 4*burn_in steps until
// >= burn_in acceptances.  The random stream is a counter-based
// Philox4x32-10 (seed = key, step = counter) instead of numpy's Philox
// Generator, so draws are reproducible per seed but not numpy-identical.
//
// Parallel form: proposals and their log weights r = logt - logq are computed
// one thread per step; the accept chain (accept iff log U_i < r_i - r_cur) runs
// one warp per 32 steps with a ballot fixed-point (exact: the dependency is
// triangular, lane k is final after k rounds; high acceptance converges fast).
#include "common.cuh"
#include "kernels.cuh"
#include "philox.cuh"

namespace slab {

// rbse2d.py:96-102, tail-stable form (erfc differences) for |m| >= 1
__device__ __forceinline__ double axis_logq(long long m, double ax) {
  const long long am = m < 0 ? -m : m;
  if (am == 0) return log(erf(0.5 * ax));
  return log(0.5 * (erfc((am - 0.5) * ax) - erfc((am + 0.5) * ax)));
}

__global__ void proposal_kernel(uint64_t seed, const int64_t* __restrict__ state, int64_t nsteps,
                                double axx, double axy, double* __restrict__ pxy,
                                double* __restrict__ rr, double* __restrict__ logu) {
  int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nsteps) return;
  const uint64_t ctr0 = (uint64_t)state[3];
  const uint4 a = Philox::gen(seed, ctr0 + 2 * (uint64_t)s);
  const uint4 b = Philox::gen(seed, ctr0 + 2 * (uint64_t)s + 1);
  const double u1 = u01_open(a.x, a.y), u2 = u01_open(a.z, a.w), u3 = u01_open(b.x, b.y);
  const double rad = sqrt(-2.0 * log(u1));
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  const double sigx = 1.0 / (axx * 1.4142135623730951), sigy = 1.0 / (axy * 1.4142135623730951);
  const double px = rint(rad * cs * sigx), py = rint(rad * sn * sigy);
  pxy[2 * s] = px;
  pxy[2 * s + 1] = py;
  const long long ix = (long long)px, iy = (long long)py;
  const bool zero = (ix == 0 && iy == 0);
  const double logt = -((axx * px) * (axx * px) + (axy * py) * (axy * py));
  rr[s] = zero ? -INFINITY : logt - (axis_logq(ix, axx) + axis_logq(iy, axy));
  logu[s] = log(u3);
}

// state: {mx, my, since, counter, accepted, steps}
// mode 0: batch (record P), mode 1: burn-in chunk (no record)
__global__ void __launch_bounds__(32) chain_kernel(int64_t* __restrict__ state, int64_t nsteps,
                                                   const double* __restrict__ pxy,
                                                   const double* __restrict__ rr,
                                                   const double* __restrict__ logu, int thin,
                                                   int64_t P, double axx, double axy, double lx,
                                                   double ly, double* __restrict__ modes,
                                                   int64_t* __restrict__ idx,
                                                   int64_t* __restrict__ acc_out) {
  const int lane = threadIdx.x;
  __syncwarp();
  long long mx = state[0], my = state[1], since = state[2];
  double rcur = -((axx * (double)mx) * (axx * (double)mx) + (axy * (double)my) * (axy * (double)my)) -
                (axis_logq(mx, axx) + axis_logq(my, axy));
  int64_t nrec = 0, nacc = 0, used = 0;
  bool done = false;
  for (int64_t base = 0; base < nsteps && !done; base += 32) {
    const int64_t s = base + lane;
    const bool in = s < nsteps;
    const double r = in ? rr[s] : -INFINITY;
    const double lu = in ? logu[s] : 0.0;
    unsigned acc = 0;
    for (int it = 0; it < 33; ++it) {
      const unsigned below = acc & ((1u << lane) - 1u);
      const int src = below ? 31 - __clz(below) : -1;
      const double rp = __shfl_sync(0xffffffffu, r, src < 0 ? 0 : src);
      const double rprev = src < 0 ? rcur : rp;
      const bool a = in && (lu < r - rprev);
      const unsigned nacc_mask = __ballot_sync(0xffffffffu, a);
      if (nacc_mask == acc) break;
      acc = nacc_mask;
    }
    // state after each lane's step
    const unsigned upto = acc & (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u));
    const int last = upto ? 31 - __clz(upto) : -1;
    const double lpx = __shfl_sync(0xffffffffu, in ? pxy[2 * s] : 0.0, last < 0 ? 0 : last);
    const double lpy = __shfl_sync(0xffffffffu, in ? pxy[2 * s + 1] : 0.0, last < 0 ? 0 : last);
    const long long smx = last < 0 ? mx : (long long)lpx;
    const long long smy = last < 0 ? my : (long long)lpy;
    // recording: step s records when (since + (s - base) + 1) hits thin (since resets)
    const long long sn = since + lane + 1;
    const bool rec = in && P > 0 && (sn % thin) == 0;
    const unsigned recmask = __ballot_sync(0xffffffffu, rec);
    // the chain stops right after the P-th record (rbse2d.py:125-126)
    int stop_lane = 31;
    const int64_t need = P - nrec;
    if (P > 0 && __popc(recmask) >= need) {
      unsigned m = recmask;
      for (int k = 1; k < need; ++k) m &= m - 1;  // drop the lowest need-1 records
      stop_lane = __ffs(m) - 1;
      done = true;
    }
    const int64_t nin = nsteps - base < 32 ? nsteps - base : 32;
    const int last_lane = done ? stop_lane : (int)nin - 1;
    if (rec && lane <= last_lane) {
      const int64_t k = nrec + __popc(recmask & ((1u << lane) - 1u));
      const double kx = 2.0 * kPi * (double)smx / lx, ky = 2.0 * kPi * (double)smy / ly;
      modes[3 * k] = kx;
      modes[3 * k + 1] = ky;
      modes[3 * k + 2] = hypot(kx, ky);
      if (idx) {
        idx[2 * k] = smx;
        idx[2 * k + 1] = smy;
      }
    }
    const unsigned valid_upto = last_lane == 31 ? 0xffffffffu : ((2u << last_lane) - 1u);
    nrec += __popc(recmask & valid_upto);
    nacc += __popc(acc & valid_upto);
    used += last_lane + 1;
    // carry the chain state from last_lane
    mx = __shfl_sync(0xffffffffu, smx, last_lane);
    my = __shfl_sync(0xffffffffu, smy, last_lane);
    const unsigned upto_last = acc & valid_upto;
    const int la = upto_last ? 31 - __clz(upto_last) : -1;
    if (la >= 0) rcur = __shfl_sync(0xffffffffu, r, la);
    const long long sl = __shfl_sync(0xffffffffu, sn, last_lane);
    since = (P > 0) ? sl % thin : sl;
  }
  if (lane == 0) {
    state[0] = mx;
    state[1] = my;
    state[2] = since;
    if (P > 0) {
      state[4] += nacc;
      state[5] += used;
    }
    if (acc_out) *acc_out = nacc;
    state[3] += 2 * nsteps;  // Philox blocks consumed by proposal_kernel
  }
}

// initial state: first proposal that is not (0,0) (rbse2d.py:168-171)
__global__ void chain_init_kernel(int64_t* __restrict__ state, const double* __restrict__ pxy,
                                  int64_t nsteps) {
  if (threadIdx.x || blockIdx.x) return;
  state[3] += 2 * nsteps;
  for (int64_t s = 0; s < nsteps; ++s) {
    const long long px = (long long)pxy[2 * s], py = (long long)pxy[2 * s + 1];
    if (px != 0 || py != 0) {
      state[0] = px;
      state[1] = py;
      state[2] = 0;
      return;
    }
  }
  state[0] = 1;  // (unreachable in practice)
  state[1] = 0;
  state[2] = 0;
}

int64_t sampler_scratch_doubles(int64_t P, int thin, int burn_in) {
  int64_t steps = P * thin + thin;
  int64_t b = 4 * (int64_t)(burn_in > 0 ? burn_in : 1);
  if (b > steps) steps = b;
  if (steps < 64) steps = 64;
  return 4 * steps + 8;
}

cudaError_t sample_modes(int64_t* state, uint64_t seed, double alpha, double lx, double ly,
                         int thin, int burn_in, int64_t P, double* modes, int64_t* idx,
                         double* scratch, int64_t scratch_doubles, cudaStream_t st) {
  const double axx = kPi / (alpha * lx), axy = kPi / (alpha * ly);
  const int64_t cap = (scratch_doubles - 8) / 4;
  double* pxy = scratch;
  double* rr = scratch + 2 * cap;
  double* lu = scratch + 3 * cap;
  int64_t* accbuf = reinterpret_cast<int64_t*>(scratch + 4 * cap);
  cudaError_t e;
  if (burn_in > 0) {  // ModeSampler.__init__ (rbse2d.py:163-181): host-driven, once per chain
    const int64_t ninit = 64;
    proposal_kernel<<<1, 64, 0, st>>>(seed, state, ninit, axx, axy, pxy, rr, lu);
    chain_init_kernel<<<1, 1, 0, st>>>(state, pxy, ninit);
    int64_t got = 0;
    const int64_t chunk = 4 * (int64_t)burn_in;
    if (chunk > cap) return cudaErrorInvalidValue;
    while (got < burn_in) {
      proposal_kernel<<<(unsigned)((chunk + 255) / 256), 256, 0, st>>>(seed, state, chunk, axx,
                                                                       axy, pxy, rr, lu);
      chain_kernel<<<1, 32, 0, st>>>(state, chunk, pxy, rr, lu, thin, 0, axx, axy, lx, ly,
                                     nullptr, nullptr, accbuf);
      int64_t na = 0;
      e = cudaMemcpyAsync(&na, accbuf, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
      if (e != cudaSuccess) return e;
      e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) return e;
      got += na;
    }
    cudaMemsetAsync(state + 2, 0, sizeof(int64_t), st);  // since = 0
  }
  if (P > 0) {  // batch_indices (rbse2d.py:187-200): no host sync, graph-capturable
    const int64_t need = P * thin + thin;  // >= P*thin - since + thin for any since
    if (need > cap) return cudaErrorInvalidValue;
    proposal_kernel<<<(unsigned)((need + 255) / 256), 256, 0, st>>>(seed, state, need, axx, axy,
                                                                    pxy, rr, lu);
    chain_kernel<<<1, 32, 0, st>>>(state, need, pxy, rr, lu, thin, P, axx, axy, lx, ly, modes, idx,
                                   nullptr);
  }
  return cudaGetLastError();
}

}  // namespace slab
