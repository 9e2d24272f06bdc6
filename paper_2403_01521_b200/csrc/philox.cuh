// philox.cuh -- counter-based Philox4x32-10 stream shared by the mode sampler and
// the Langevin integrator: draw (seed = key, counter) is a pure function, so
// every thread draws its own numbers independently and results do not depend
// on launch geometry.
#pragma once
#include <stdint.h>

namespace slab {

struct Philox {
  __device__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  // `domain` separates independent streams under one seed (sampler / thermostat)
  __device__ static uint4 gen(uint64_t seed, uint64_t ctr, uint32_t domain = 0x5AB5u) {
    uint4 c = make_uint4((uint32_t)ctr, (uint32_t)(ctr >> 32), domain, 0x2403u);
    uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

__device__ __forceinline__ double u01_open(uint32_t a, uint32_t b) {
  // 53-bit uniform in (0, 1]
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6) + 1.0) * (1.0 / 9007199254740992.0);
}

}  // namespace slab
