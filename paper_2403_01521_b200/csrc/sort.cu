// sort.cu -- stable LSD radix sort of particles by z (and of cell ids), plus the
// gather into the z-sorted SoA the recurrence kernels stream.
//
// Replaces reference core.py:166-208 (_bucket_sort_perm / sort_by_z).  The
// reference result equals np.argsort(z, kind="stable") (tests/test_core.py:206);
// an LSD radix sort over an order-preserving uint64 image of z, with each pass a
// stable scatter, gives the same permutation bit for bit.  -0.0 is folded onto
// +0.0 (the reference compares with '>' so they tie and keep input order).
//
// All passes' digit counts in one read, then one Onesweep kernel per pass
// (decoupled look-back for the tile offsets, stable scatter with warp
// match_any ranks, 16 rounds of 256 keys per 4096-key tile).  8 passes for
// 64-bit keys, ceil(bits/8) for the 32-bit cell-id keys of the cell list.
#include "common.cuh"
#include "kernels.cuh"

namespace slab {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;  // 4096 keys per tile
// small inputs: 4 keys per thread (1024 per tile): 4x the tiles and a quarter of
// the per-tile rounds, for the latency-bound passes of a few-tile sort
constexpr int kSortItemsSmall = 4;
#ifndef SLAB_SORT_SMALL_LOG2
#define SLAB_SORT_SMALL_LOG2 18
#endif
constexpr int64_t kSortSmallN = (int64_t)1 << SLAB_SORT_SMALL_LOG2;
static int sort_items(int64_t n) { return n < kSortSmallN ? kSortItemsSmall : kSortItems; }

__global__ void zkey_init_kernel(const double* __restrict__ z, int64_t stride, int64_t n,
                                 uint64_t* __restrict__ keys, int32_t* __restrict__ idx,
                                 int* __restrict__ status) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const double zi = z[i * stride];
    keys[i] = z_key(zi);
    idx[i] = (int32_t)i;
    // core.py:206-207 rejects non-finite z; reported through the status word
    if (status && !isfinite(zi)) atomicOr(status, SLAB_STATUS_NONFINITE_DEV);
  }
}

// ---------------------------------------------------------------------------
// Onesweep-style LSD radix sort: one kernel per digit pass.
//   radix_digit_counts: all passes' global digit counts in one read of the keys
//                       (digit totals do not depend on the key order);
//   radix_digit_bases:  exclusive scans -> global base of every digit, per pass;
//   radix_onesweep:     per 4096-key tile (tiles taken in launch order from an
//                       atomic counter, so waiting only ever targets a running
//                       tile): count the tile's digits, publish them, look back
//                       over earlier tiles' published counts (decoupled
//                       look-back) for the tile's exclusive offsets, then the
//                       stable scatter (warp match_any ranks, 16 rounds).
// ---------------------------------------------------------------------------
constexpr uint32_t kLbAgg = 1u << 30;   // look-back word: tile aggregate published
constexpr uint32_t kLbInc = 2u << 30;   // inclusive prefix published
constexpr uint32_t kLbVal = (1u << 30) - 1u;
constexpr int kMaxPasses = 8;

template <typename K>
__global__ void __launch_bounds__(kSortThreads) radix_digit_counts_kernel(
    const K* __restrict__ keys, int64_t n, int passes, uint32_t* __restrict__ counts) {
  __shared__ uint32_t cnt[kMaxPasses][256];
  for (int e = threadIdx.x; e < kMaxPasses * 256; e += blockDim.x) (&cnt[0][0])[e] = 0;
  __syncthreads();
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const K k = keys[p];
    for (int ps = 0; ps < passes; ++ps) atomicAdd(&cnt[ps][(unsigned)(k >> (8 * ps)) & 255u], 1u);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < passes * 256; e += blockDim.x) {
    const uint32_t v = (&cnt[0][0])[e];
    if (v) atomicAdd(&counts[e], v);
  }
}

// one block per pass: bases[ps][d] = sum_{d' < d} counts[ps][d']
__global__ void __launch_bounds__(256) radix_digit_bases_kernel(const uint32_t* __restrict__ counts,
                                                                uint32_t* __restrict__ bases) {
  __shared__ uint32_t s[256];
  const int ps = blockIdx.x, d = threadIdx.x;
  s[d] = counts[ps * 256 + d];
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const uint32_t y = d >= o ? s[d - o] : 0u;
    __syncthreads();
    s[d] += y;
    __syncthreads();
  }
  bases[ps * 256 + d] = s[d] - counts[ps * 256 + d];
}

template <typename K, int ITEMS>
__global__ void __launch_bounds__(kSortThreads) radix_onesweep_kernel(
    const K* __restrict__ kin, const int32_t* __restrict__ vin, K* __restrict__ kout,
    int32_t* __restrict__ vout, int64_t n, int shift, const uint32_t* __restrict__ bases,
    uint32_t* __restrict__ look, int* __restrict__ tile_ctr) {
  __shared__ int32_t base[256];
  __shared__ int32_t wcnt[kSortThreads / 32][256];
  __shared__ uint32_t tcnt[256];
  __shared__ int tile_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) tile_s = atomicAdd(tile_ctr, 1);
  tcnt[tid] = 0u;
  __syncthreads();
  const int tile = tile_s;
  const int64_t tile0 = (int64_t)tile * (kSortThreads * ITEMS);
  K keys[ITEMS];
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
    const int64_t p = tile0 + r * kSortThreads + tid;
    keys[r] = p < n ? kin[p] : K(0);
    if (p < n) atomicAdd(&tcnt[(unsigned)(keys[r] >> shift) & 255u], 1u);
  }
  __syncthreads();
  // decoupled look-back for digit `tid`
  {
    const uint32_t own = tcnt[tid];
    volatile uint32_t* lk = look;
    uint32_t excl = 0;
    if (tile == 0) {
      lk[tid] = kLbInc | own;
    } else {
      lk[(size_t)tile * 256 + tid] = kLbAgg | own;
      for (int t = tile - 1; t >= 0; --t) {
        uint32_t v;
        do {
          v = lk[(size_t)t * 256 + tid];
        } while ((v & ~kLbVal) == 0u);
        excl += v & kLbVal;
        if (v & kLbInc) break;
      }
      lk[(size_t)tile * 256 + tid] = kLbInc | (excl + own);
    }
    base[tid] = (int32_t)(bases[tid] + excl);
  }
  const unsigned lt_mask = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < ITEMS; ++r) {
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][tid] = 0;
    __syncthreads();
    const int64_t p = tile0 + r * kSortThreads + tid;
    const bool valid = p < n;
    const K key = keys[r];
    const unsigned digit = valid ? (unsigned)(key >> shift) & 255u : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, digit);
    const int rank = __popc(peers & lt_mask);
    if (valid && rank == 0) wcnt[warp][digit] = __popc(peers);
    __syncthreads();
    {  // digit tid: exclusive prefix over warps, advance the tile-running base
      int32_t run = base[tid];
#pragma unroll
      for (int w = 0; w < kSortThreads / 32; ++w) {
        const int32_t c = wcnt[w][tid];
        wcnt[w][tid] = run;
        run += c;
      }
      base[tid] = run;
    }
    __syncthreads();
    if (valid) {
      const int32_t dst = wcnt[warp][digit] + rank;
      SLAB_BOUND(dst, n);
      kout[dst] = key;
      vout[dst] = vin[p];
    }
    __syncthreads();  // wcnt is reset by the next round
  }
}

__global__ void gather_sorted_kernel(const double* __restrict__ pos,
                                     const double* __restrict__ charge,
                                     const int32_t* __restrict__ perm, int64_t n,
                                     double* __restrict__ xs, double* __restrict__ ys,
                                     double* __restrict__ zs, double* __restrict__ qs,
                                     int64_t* __restrict__ perm64) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) {
    int64_t i = perm[a];
    xs[a] = pos[3 * i + 0];
    ys[a] = pos[3 * i + 1];
    zs[a] = pos[3 * i + 2];
    qs[a] = charge[i];
    if (perm64) perm64[a] = i;
  }
}

__global__ void perm_to_int64_kernel(const int32_t* __restrict__ p, int64_t n,
                                     int64_t* __restrict__ out) {
  int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a < n) out[a] = p[a];
}

template <typename K>
cudaError_t radix_sort_pairs(K* keys, int32_t* vals, K* keys_alt, int32_t* vals_alt,
                             int32_t* hist, int64_t n, int key_bits, cudaStream_t st,
                             K** keys_out, int32_t** vals_out) {
  const int items = sort_items(n);
  const int tile_keys = kSortThreads * items;
  const int ntiles = (int)((n + tile_keys - 1) / tile_keys);
  const int passes = (key_bits + 7) / 8;
  K *ki = keys, *ko = keys_alt;
  int32_t *vi = vals, *vo = vals_alt;
  if (n > 0) {
    // workspace: counts [passes][256] | bases [passes][256] | tile counters [passes]
    //            | look-back words [passes][ntiles][256]
    uint32_t* counts = reinterpret_cast<uint32_t*>(hist);
    uint32_t* bases = counts + kMaxPasses * 256;
    int* tctr = reinterpret_cast<int*>(bases + kMaxPasses * 256);
    uint32_t* look = reinterpret_cast<uint32_t*>(tctr + 64);
    const size_t clear = sizeof(uint32_t) * ((size_t)kMaxPasses * 256 * 2 + 64 +
                                            (size_t)passes * ntiles * 256);
    cudaMemsetAsync(hist, 0, clear, st);
    int grid = (int)((n + kSortThreads - 1) / kSortThreads);
    grid = grid < 4 * 148 ? grid : 4 * 148;
    radix_digit_counts_kernel<K><<<grid, kSortThreads, 0, st>>>(ki, n, passes, counts);
    radix_digit_bases_kernel<<<passes, 256, 0, st>>>(counts, bases);
    for (int ps = 0; ps < passes; ++ps) {
      if (items == kSortItems)
        radix_onesweep_kernel<K, kSortItems><<<ntiles, kSortThreads, 0, st>>>(
            ki, vi, ko, vo, n, 8 * ps, bases + ps * 256, look + (size_t)ps * ntiles * 256,
            tctr + ps);
      else
        radix_onesweep_kernel<K, kSortItemsSmall><<<ntiles, kSortThreads, 0, st>>>(
            ki, vi, ko, vo, n, 8 * ps, bases + ps * 256, look + (size_t)ps * ntiles * 256,
            tctr + ps);
      K* tk = ki; ki = ko; ko = tk;
      int32_t* tv = vi; vi = vo; vo = tv;
    }
  }
  *keys_out = ki;
  *vals_out = vi;
  return cudaGetLastError();
}

int64_t radix_hist_entries(int64_t n) {
  const int64_t tile_keys = (int64_t)kSortThreads * sort_items(n);
  const int64_t ntiles = (n + tile_keys - 1) / tile_keys;
  return (int64_t)kMaxPasses * 256 * 2 + 64 + (int64_t)kMaxPasses * (ntiles > 0 ? ntiles : 1) * 256;
}

cudaError_t sort_by_z_device(const double* z, int64_t stride, int64_t n, SortWork& w,
                             cudaStream_t st, int32_t** perm_out, int* status) {
  if (n > 0)
    zkey_init_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(z, stride, n, w.k0, w.v0,
                                                                  status);
  uint64_t* kout;
  return radix_sort_pairs<uint64_t>(w.k0, w.v0, w.k1, w.v1, w.hist, n, 64, st, &kout, perm_out);
}

cudaError_t gather_sorted(const double* pos, const double* charge, const int32_t* perm, int64_t n,
                          double* xs, double* ys, double* zs, double* qs, int64_t* perm64,
                          cudaStream_t st) {
  if (n > 0)
    gather_sorted_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pos, charge, perm, n, xs, ys,
                                                                      zs, qs, perm64);
  return cudaGetLastError();
}

cudaError_t perm_to_int64(const int32_t* p, int64_t n, int64_t* out, cudaStream_t st) {
  if (n > 0) perm_to_int64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(p, n, out);
  return cudaGetLastError();
}

template cudaError_t radix_sort_pairs<uint32_t>(uint32_t*, int32_t*, uint32_t*, int32_t*,
                                                int32_t*, int64_t, int, cudaStream_t,
                                                uint32_t**, int32_t**);

}  // namespace slab
