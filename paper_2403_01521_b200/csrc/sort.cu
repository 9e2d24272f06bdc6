// sort.cu -- stable LSD radix sort of particles by z (and of cell ids), plus the
// gather into the z-sorted SoA the recurrence kernels stream.
//
// Replaces reference core.py:166-208 (_bucket_sort_perm / sort_by_z).  The
// reference result equals np.argsort(z, kind="stable") (tests/test_core.py:206);
// an LSD radix sort over an order-preserving uint64 image of z, with each pass a
// stable scatter, gives the same permutation bit for bit.  -0.0 is folded onto
// +0.0 (the reference compares with '>' so they tie and keep input order).
//
// Per pass: histogram (per tile, smem atomics) -> one-block exclusive scan over
// [digit][tile] -> stable scatter (warp match_any ranks + per-warp digit
// prefix, 16 rounds of 256 keys per 4096-key tile).  8 passes for 64-bit keys,
// ceil(bits/8) for the 32-bit cell-id keys of the short-range cell list.
#include "common.cuh"
#include "kernels.cuh"

namespace slab {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 16;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys per tile

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

template <typename K>
__global__ void __launch_bounds__(kSortThreads) radix_hist_kernel(const K* __restrict__ keys,
                                                                  int64_t n, int shift,
                                                                  int32_t* __restrict__ hist,
                                                                  int ntiles) {
  __shared__ int32_t cnt[256];
  cnt[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
  for (int r = 0; r < kSortItems; ++r) {
    int64_t p = base + r * kSortThreads + threadIdx.x;
    if (p < n) atomicAdd(&cnt[(unsigned)(keys[p] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[threadIdx.x * (int64_t)ntiles + blockIdx.x] = cnt[threadIdx.x];
}

// Row-wise exclusive scan of hist[256][ntiles] (one block per digit row); the
// row total lands in rowtot[digit].
__global__ void __launch_bounds__(1024) scan_rows_kernel(int32_t* __restrict__ hist, int ntiles,
                                                         int32_t* __restrict__ rowtot) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t carry;
  int32_t* row = hist + (int64_t)blockIdx.x * ntiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < ntiles; base += 1024) {
    int i = base + threadIdx.x;
    int32_t v = i < ntiles ? row[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t s = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    if (i < ntiles) row[i] = carry + (warp ? wsum[warp - 1] : 0) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) rowtot[blockIdx.x] = carry;
}

// offsets[d][t] += sum_{d' < d} rowtot[d']
__global__ void __launch_bounds__(256) add_digit_base_kernel(int32_t* __restrict__ hist, int ntiles,
                                                             const int32_t* __restrict__ rowtot) {
  __shared__ int32_t pre[256];
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int d = 0; d < 256; ++d) { pre[d] = run; run += rowtot[d]; }
  }
  __syncthreads();
  int64_t total = (int64_t)256 * ntiles;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    hist[i] += pre[i / ntiles];
}

template <typename K>
__global__ void __launch_bounds__(kSortThreads) radix_scatter_kernel(
    const K* __restrict__ kin, const int32_t* __restrict__ vin, K* __restrict__ kout,
    int32_t* __restrict__ vout, int64_t n, int shift, const int32_t* __restrict__ offsets,
    int ntiles) {
  __shared__ int32_t base[256];
  __shared__ int32_t wcnt[kSortThreads / 32][256];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  base[tid] = offsets[tid * (int64_t)ntiles + blockIdx.x];
  const unsigned lt_mask = (1u << lane) - 1u;
  int64_t tile0 = (int64_t)blockIdx.x * kSortTile;
  for (int r = 0; r < kSortItems; ++r) {
#pragma unroll
    for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][tid] = 0;
    __syncthreads();
    int64_t p = tile0 + r * kSortThreads + tid;
    bool valid = p < n;
    K key = valid ? kin[p] : K(0);
    unsigned digit = valid ? (unsigned)(key >> shift) & 255u : 256u;
    unsigned peers = __match_any_sync(0xffffffffu, digit);
    int rank = __popc(peers & lt_mask);
    if (valid && rank == 0) wcnt[warp][digit] = __popc(peers);
    __syncthreads();
    {  // digit tid: exclusive prefix over warps, advance the tile-running base
      int32_t run = base[tid];
#pragma unroll
      for (int w = 0; w < kSortThreads / 32; ++w) {
        int32_t c = wcnt[w][tid];
        wcnt[w][tid] = run;
        run += c;
      }
      base[tid] = run;
    }
    __syncthreads();
    if (valid) {
      int32_t dst = wcnt[warp][digit] + rank;
      kout[dst] = key;
      vout[dst] = vin[p];
    }
    __syncthreads();
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
  const int ntiles = (int)((n + kSortTile - 1) / kSortTile);
  K *ki = keys, *ko = keys_alt;
  int32_t *vi = vals, *vo = vals_alt;
  if (n > 0) {
    for (int shift = 0; shift < key_bits; shift += 8) {
      radix_hist_kernel<K><<<ntiles, kSortThreads, 0, st>>>(ki, n, shift, hist, ntiles);
      scan_rows_kernel<<<256, 1024, 0, st>>>(hist, ntiles, hist + (int64_t)256 * ntiles);
      add_digit_base_kernel<<<(unsigned)((256 * (int64_t)ntiles + 255) / 256 < 1184 ? (256 * (int64_t)ntiles + 255) / 256 : 1184), 256, 0, st>>>(
          hist, ntiles, hist + (int64_t)256 * ntiles);
      radix_scatter_kernel<K><<<ntiles, kSortThreads, 0, st>>>(ki, vi, ko, vo, n, shift, hist,
                                                               ntiles);
      K* tk = ki; ki = ko; ko = tk;
      int32_t* tv = vi; vi = vo; vo = tv;
    }
  }
  *keys_out = ki;
  *vals_out = vi;
  return cudaGetLastError();
}

int64_t radix_hist_entries(int64_t n) {
  int64_t ntiles = (n + kSortTile - 1) / kSortTile;
  return 256 * (ntiles > 0 ? ntiles : 1) + 256;  // + row totals
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
