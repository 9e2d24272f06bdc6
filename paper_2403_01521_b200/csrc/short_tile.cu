// short_tile.cu -- the erfc(alpha r)/r short range as ONE fused kernel: the
// candidate screen and the exact fp64 pair term run from shared-memory tiles,
// with no neighbour rows in HBM (reference ewald2d.py:160-231, the same pair set
// and pair term as short.cu).
//
// Layout.  Particles are cell-sorted as in short.cu (cells of edge >= r_c / S,
// column-major, z fastest: a column's z range is one contiguous index range).
// HOMES are visited in a second order: bricks of 2 x 2 x 4 cells in serpentine
// order (consecutive bricks are neighbours), z level then the 2 x 2 cells inside
// a brick.  A warp takes 32 consecutive homes of that order -- a compact ~2 x 2 x
// 3.4-cell box -- and screens the candidates of every column within r_c of the
// box's bounding box (z range trimmed per column to the r_c-swept box):
//
//   stage   32 candidates at a time into shared memory (coalesced loads of the
//           fp32 screen image and the fp64 record, periodic image shift applied)
//   screen  lane = home: 32 broadcast reads, fp32 distance test -> hit bitmask
//   queue   the hits in home-major order (warp prefix sum of the popcounts)
//   pairs   lane = queue entry: the exact fp64 term of 32 pairs at a time (full
//           warps whatever the per-home hit counts), forces combined per home by a
//           segmented shuffle scan (entries are home-sorted) and added by the
//           segment's last lane into the home's shared accumulator
//
// Every pair is evaluated from both ends (full shell, u_s = 1/2 sum) and each
// home's force is summed in a fixed order: deterministic, no atomics, and no
// capacity to overflow.  The host uses this path when the box holds enough cells
// that a warp's column window cannot alias across the periodic boundary.
#include <stdio.h>

#include "common.cuh"
#include "kernels.cuh"

namespace slab {

constexpr int kTileWarps = 4;
constexpr int kTileThreads = 32 * kTileWarps;

// home-order slot of cell (cx, cy, cz): bricks of 2 x 2 x 4 cells; brick columns
// serpentine in y (per x brick) and bricks serpentine in z (per brick column);
// inside a brick z level (reversed in descending bricks) then the 2 x 2 cells
__host__ __device__ __forceinline__ int64_t home_slot(int cx, int cy, int cz, int nby, int nbz) {
  const int bx = cx >> 1, by = cy >> 1, bz = cz >> 2;
  const int bys = (bx & 1) ? nby - 1 - by : by;
  const int64_t col = (int64_t)bx * nby + bys;
  const bool down = (col & 1) != 0;
  const int bzs = down ? nbz - 1 - bz : bz;
  const int lz = down ? 3 - (cz & 3) : (cz & 3);
  return ((col * nbz + bzs) << 4) + (lz << 2) + ((cx & 1) << 1) + (cy & 1);
}

// cnt[slot] = particles of the cell at that slot (slots of absent cells stay 0)
__global__ void home_count_kernel(const int32_t* __restrict__ start, int ncx, int ncy, int ncz,
                                  int nby, int nbz, int32_t* __restrict__ cnt) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= (int64_t)ncx * ncy * ncz) return;
  const int cz = (int)(c % ncz), cy = (int)((c / ncz) % ncy), cx = (int)(c / ((int64_t)ncz * ncy));
  cnt[home_slot(cx, cy, cz, nby, nbz)] = start[c + 1] - start[c];
}

// hperm[off[slot(cell of a)] + rank of a in its cell] = a (cell-sorted index)
__global__ void home_scatter_kernel(const uint32_t* __restrict__ skey,
                                    const int32_t* __restrict__ start,
                                    const int32_t* __restrict__ off, int64_t n, int ncy, int ncz,
                                    int nby, int nbz, int32_t* __restrict__ hperm) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= n) return;
  const uint32_t c = skey[a];
  const int cz = (int)(c % ncz), cy = (int)((c / ncz) % ncy), cx = (int)(c / ((uint32_t)ncz * ncy));
  hperm[off[home_slot(cx, cy, cz, nby, nbz)] + (a - start[c])] = (int32_t)a;
}

// exclusive prefix sum of int32 (three passes: per-block sums, their scan, block scans)
constexpr int kScanThreads = 256, kScanItems = 4, kScanTile = kScanThreads * kScanItems;
__global__ void __launch_bounds__(kScanThreads) scan_block_sums_kernel(
    const int32_t* __restrict__ in, int64_t n, int32_t* __restrict__ bsum) {
  __shared__ int32_t red[kScanThreads];
  const int64_t base = blockIdx.x * (int64_t)kScanTile;
  int32_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k * kScanThreads + threadIdx.x;
    s += i < n ? in[i] : 0;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = kScanThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = red[0];
}

// one block: exclusive scan of nb block sums in place (nb <= 64K)
__global__ void __launch_bounds__(1024) scan_sums_kernel(int32_t* __restrict__ bsum, int nb) {
  __shared__ int32_t part[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(nb, b0 + per);
  int32_t s = 0;
  for (int b = b0; b < b1; ++b) s += bsum[b];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = part[threadIdx.x] - s;  // exclusive
  for (int b = b0; b < b1; ++b) {
    const int32_t v = bsum[b];
    bsum[b] = run;
    run += v;
  }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(
    const int32_t* __restrict__ in, int64_t n, const int32_t* __restrict__ bsum,
    int32_t* __restrict__ out) {
  __shared__ int32_t wsum[kScanThreads / 32];
  const int64_t base = blockIdx.x * (int64_t)kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t v[kScanItems], s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    s += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int32_t wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += wsum[w];
  int32_t run = bsum[blockIdx.x] + wbase + incl - s;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
}

static cudaError_t exclusive_scan(const int32_t* in, int64_t n, int32_t* bsum, int32_t* out,
                                  cudaStream_t st) {
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb > 65536) return cudaErrorInvalidValue;
  scan_block_sums_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, bsum);
  scan_sums_kernel<<<1, 1024, 0, st>>>(bsum, (int)nb);
  scan_apply_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, bsum, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// the fused kernel
// ---------------------------------------------------------------------------
constexpr int kTileQueue = 32 * 32;  // at most 32 hits per home per staged batch

// the exact fp64 pair term (ewald2d.py:199-230), masked: a dead entry or an
// out-of-range / coincident pair contributes exact zeros
template <bool kTabOnly>
__device__ __forceinline__ void tile_pair(double xi, double yi, double zi, double qi, double xj,
                                          double yj, double zj, double qj, bool live, double lx,
                                          double ly, double ilx, double ily, double alpha,
                                          double rc2, double c, const double* __restrict__ etab,
                                          double& e, double& fx, double& fy, double& fz,
                                          int& flag) {
  double dx = xi - xj, dy = yi - yj;
  const double dz = zi - zj;
  // minimum image as the reference, dx - lx rint(dx / lx); lx * rint(.) is exact
  // for the shifts -1, 0, 1 of a box of >= 3 r_c, so the fused form rounds alike
  dx = fma(-lx, rint(dx * ilx), dx);
  dy = fma(-ly, rint(dy * ily), dy);
  // the reference's rounding order, so the cutoff test d2 <= r_c^2 decides alike
  const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  const bool in = live && d2 <= rc2;
  const bool coincident = d2 < 1e-24;
  flag |= (in && coincident) ? 1 : 0;
  const bool use = in && !coincident;
  const double d2u = use ? d2 : rc2;
  const double inv_d = rsqrt(d2u);
  const double d = d2u * inv_d;
  const double qq = use ? qi * qj : 0.0;
  double er, g;
#if SLAB_TILE_TABLE
  erfc_gauss<kTabOnly>(alpha * d, etab, &er, &g);  // the 48-interval erfcx table (short.cu's)
#else
  erfc_gauss_rat<kTabOnly>(alpha * d, &er, &g);
#endif
  const double qe = qq * er;
  e = qe * inv_d;
  const double fmag = fma(qq * c, g, qe * inv_d) * (inv_d * inv_d);
  fx = fmag * dx;
  fy = fmag * dy;
  fz = fmag * dz;
}

#ifndef SLAB_TILE_TABLE
#define SLAB_TILE_TABLE 0
#endif
struct TileShared {
#if SLAB_TILE_TABLE
  double etab[kErfcxTabSize];
#endif
  float nfx[kTileWarps][32], nfy[kTileWarps][32];  // staged candidates: -(fp32 screen image)
  float nfz[kTileWarps][32];                       //   (SoA: float2 pairs for the f32x2 screen)
  int32_t cj[kTileWarps][32];                      // staged candidates: cell-sorted index
  int32_t ha[kTileWarps][32];                      // homes: cell-sorted index
  double cx[kTileWarps][32], cy[kTileWarps][32];  // staged candidates: raw fp64 record (SoA:
  double cz[kTileWarps][32], cq[kTileWarps][32];  //   lanes read distinct words, <= 2-way banks)
  double hx[kTileWarps][32], hy[kTileWarps][32];  // homes
  double hz[kTileWarps][32], hq[kTileWarps][32];
  double f[kTileWarps][3][32];                    // home force accumulators
  uint16_t q[kTileWarps][kTileQueue];             // (home << 5 | candidate), home-major
  double red[kTileThreads];
};

template <bool kTabOnly>
__global__ void __launch_bounds__(kTileThreads) short_tile_kernel(
    const double4* __restrict__ cp, const float4* __restrict__ cpf,
    const int32_t* __restrict__ start, const int32_t* __restrict__ hperm,
    const int32_t* __restrict__ order, int64_t h0, int64_t h1, int ncx, int ncy, int ncz,
    double lx, double ly, float lxf, float lyf, float lzf, double alpha, double rc2,
    float rc2f, float rcf, double* __restrict__ forces, double* __restrict__ eblk,
    int* __restrict__ status) {
  __shared__ TileShared sh;
#if SLAB_TILE_TABLE
  load_erfcx_table(sh.etab);
  __syncthreads();
  const double* etab = sh.etab;
#else
  const double* etab = nullptr;
#endif
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const double c = kTwoOverSqrtPi * alpha, ilx = 1.0 / lx, ily = 1.0 / ly;
  const float ex = lxf / ncx, ey = lyf / ncy, izc = ncz / lzf;
  const float ilxf = 1.0f / lxf, ilyf = 1.0f / lyf;
  double E = 0.0;
  int flag = 0;
  uint16_t* q_w = sh.q[warp];
  double* f0 = sh.f[warp][0];
  double* f1 = sh.f[warp][1];
  double* f2 = sh.f[warp][2];
  const int64_t ngroups = (h1 - h0 + 31) / 32;
  for (int64_t grp = blockIdx.x * (int64_t)kTileWarps + warp; grp < ngroups;
       grp += (int64_t)gridDim.x * kTileWarps) {
    const int64_t hidx = h0 + grp * 32 + lane;
    const bool hact = hidx < h1;
    const int a = hact ? hperm[hidx] : -1;
    const float4 pf = hact ? cpf[a] : make_float4(0.f, 0.f, 0.f, 0.f);
    sh.ha[warp][lane] = a;
    {
      const double4 pd = hact ? cp[a] : make_double4(0.0, 0.0, 0.0, 0.0);
      sh.hx[warp][lane] = pd.x;
      sh.hy[warp][lane] = pd.y;
      sh.hz[warp][lane] = pd.z;
      sh.hq[warp][lane] = pd.w;
    }
    f0[lane] = f1[lane] = f2[lane] = 0.0;
    // bounding box of the active homes (fp32 screen image)
    float x0 = hact ? pf.x : 3e30f, x1 = hact ? pf.x : -3e30f;
    float y0 = hact ? pf.y : 3e30f, y1 = hact ? pf.y : -3e30f;
    float z0 = hact ? pf.z : 3e30f, z1 = hact ? pf.z : -3e30f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x0 = fminf(x0, __shfl_xor_sync(full, x0, o));
      x1 = fmaxf(x1, __shfl_xor_sync(full, x1, o));
      y0 = fminf(y0, __shfl_xor_sync(full, y0, o));
      y1 = fmaxf(y1, __shfl_xor_sync(full, y1, o));
      z0 = fminf(z0, __shfl_xor_sync(full, z0, o));
      z1 = fmaxf(z1, __shfl_xor_sync(full, z1, o));
    }
    // candidate columns (unwrapped indices) whose xy rectangle is within r_c of the box
    const int ix0 = (int)floorf((x0 - rcf) / ex), ix1 = (int)floorf((x1 + rcf) / ex);
    const int iy0 = (int)floorf((y0 - rcf) / ey), iy1 = (int)floorf((y1 + rcf) / ey);
    // A window wider than the box (a very sparse warp, a small box) would visit a
    // column twice: clamp it to every column once and screen with the per-pair
    // minimum image instead of the column's image shift (warp-uniform mode).
    const bool wrap_x = ix1 - ix0 + 1 > ncx, wrap_y = iy1 - iy0 + 1 > ncy;
    const bool minimg = wrap_x || wrap_y;
    const int nX = wrap_x ? ncx : ix1 - ix0 + 1;
    const int nY = wrap_y ? ncy : iy1 - iy0 + 1;
    const int ncol = nX * nY;
#pragma unroll 1
    for (int q0 = 0; q0 < ncol; q0 += 32) {
      const int qc = q0 + lane;
      int j0 = 0, len = 0;
      float shx = 0.f, shy = 0.f;
      if (qc < ncol) {
        const int ux = ix0 + qc / nY, uy = iy0 + qc % nY;
        const int mx = ux >= 0 ? ux / ncx : -((-ux + ncx - 1) / ncx);  // floor division
        const int my = uy >= 0 ? uy / ncy : -((-uy + ncy - 1) / ncy);
        const int wx = ux - mx * ncx, wy = uy - my * ncy;
        shx = (float)mx * lxf;
        shy = (float)my * lyf;
        const float dxr = wrap_x ? 0.0f : fmaxf(0.0f, fmaxf(ux * ex - x1, x0 - (ux + 1) * ex));
        const float dyr = wrap_y ? 0.0f : fmaxf(0.0f, fmaxf(uy * ey - y1, y0 - (uy + 1) * ey));
        const float dxy2 = fmaf(dxr, dxr, dyr * dyr);
        if (dxy2 <= rc2f) {
          const float h = sqrtf(rc2f - dxy2);
          int zlo = (int)floorf((z0 - h) * izc - 1e-3f);
          int zhi = (int)floorf((z1 + h) * izc + 1e-3f);
          zlo = zlo < 0 ? 0 : (zlo >= ncz ? ncz - 1 : zlo);
          zhi = zhi < 0 ? 0 : (zhi >= ncz ? ncz - 1 : zhi);
          const int64_t col = ((int64_t)wx * ncy + wy) * ncz;
          j0 = start[col + zlo];
          len = start[col + zhi + 1] - j0;
        }
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(full, incl, 31);
      const int excl = incl - len;
#pragma unroll 1
      for (int fb = 0; fb < total; fb += 32) {
        // ---- stage 32 candidates: owner column by binary search on the prefix
        const int f = fb + lane;
        int k = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int v = __shfl_sync(full, incl, k + step - 1);
          if (v <= f) k += step;
        }
        const int jk = __shfl_sync(full, j0, k & 31);
        const int ek = __shfl_sync(full, excl, k & 31);
        const float sx = __shfl_sync(full, shx, k & 31);
        const float sy = __shfl_sync(full, shy, k & 31);
        const bool valid = f < total;
        const int j = jk + (f - ek);
        const float4 cfj = valid ? cpf[j] : make_float4(3e30f, 3e30f, 3e30f, 0.f);
        const double4 cdj = valid ? cp[j] : make_double4(0.0, 0.0, 0.0, 0.0);
        sh.nfx[warp][lane] = -(cfj.x + sx);
        sh.nfy[warp][lane] = -(cfj.y + sy);
        sh.nfz[warp][lane] = -cfj.z;
        sh.cj[warp][lane] = valid ? j : -2;
        sh.cx[warp][lane] = cdj.x;
        sh.cy[warp][lane] = cdj.y;
        sh.cz[warp][lane] = cdj.z;
        sh.cq[warp][lane] = cdj.w;
        __syncwarp();
        // ---- screen: lane = home, the 32 staged candidates broadcast two at a
        // time to paired fp32 (f32x2) arithmetic; the sign bit of d^2 - r_c^2 is
        // the hit, funnel-shifted into the row mask (invalid slots sit far away,
        // so the trip count is constant and fully unrolled).  The home itself is
        // screened in and masked out of the pair terms.
        unsigned row = 0u;
        if (!minimg) {
          const float2 px = make_float2(pf.x, pf.x), py = make_float2(pf.y, pf.y);
          const float2 pz = make_float2(pf.z, pf.z), nrc = make_float2(-rc2f, -rc2f);
          const float* nx = sh.nfx[warp];
          const float* ny = sh.nfy[warp];
          const float* nz = sh.nfz[warp];
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            const float2 dx = __fadd2_rn(px, *reinterpret_cast<const float2*>(nx + t));
            const float2 dy = __fadd2_rn(py, *reinterpret_cast<const float2*>(ny + t));
            const float2 dz = __fadd2_rn(pz, *reinterpret_cast<const float2*>(nz + t));
            float2 d = __ffma2_rn(dz, dz, nrc);
            d = __ffma2_rn(dy, dy, d);
            d = __ffma2_rn(dx, dx, d);
            row = __funnelshift_l(__float_as_uint(d.x), row, 1);
            row = __funnelshift_l(__float_as_uint(d.y), row, 1);
          }
          row = __brev(row);  // bit t = candidate t
        } else {
#pragma unroll 4
          for (int t = 0; t < 32; ++t) {
            float dx = pf.x + sh.nfx[warp][t], dy = pf.y + sh.nfy[warp][t];
            const float dz = pf.z + sh.nfz[warp][t];
            dx = fmaf(-lxf, rintf(dx * ilxf), dx);
            dy = fmaf(-lyf, rintf(dy * ilyf), dy);
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (d2 <= rc2f && sh.cj[warp][t] >= 0) row |= 1u << t;
          }
        }
        if (!hact) row = 0u;
        // ---- queue the hits home-major
        const int cnt = __popc(row);
        int ofs = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(full, ofs, o);
          if (lane >= o) ofs += v;
        }
        const int T = __shfl_sync(full, ofs, 31);
        {
          int p = ofs - cnt;
          unsigned r = row;
          while (r) {
            const int t = __ffs(r) - 1;
            r &= r - 1u;
            SLAB_BOUND(p, kTileQueue);
            q_w[p++] = (uint16_t)((lane << 5) | t);
          }
        }
        __syncwarp();
        if (T == 0) continue;
        // ---- exact pair terms: lane l takes the R consecutive queue entries
        // [l R, l R + R) over R rounds (full warps whatever the per-home hit
        // counts).  Its entries are home-sorted: forces accumulate in registers
        // while the home stays the same; a segment that starts AND ends inside
        // the lane is exclusive to it and goes straight to the home's shared
        // accumulator; the lane's first and last pieces may be shared with its
        // neighbours and are combined below in a fixed order.
        const int R = (T + 31) >> 5;
        const int e_lo = lane * R;
        const int e_hi = e_lo + R < T ? e_lo + R : T;
        int cur = -1, head = -1;
        double ax = 0.0, ay = 0.0, az = 0.0, bx = 0.0, by = 0.0, bz = 0.0;
        // home-run bookkeeping of one evaluated entry
        auto take = [&](bool live, int hh, double fx, double fy, double fz) {
          if (live && hh != cur) {  // a new segment starts in this lane
            if (cur >= 0) {
              if (head < 0) {  // closing the lane's first piece: hold it
                head = cur;
                bx = ax;
                by = ay;
                bz = az;
              } else {  // an interior segment: exclusive to this lane
                SLAB_BOUND(cur, 32);
                f0[cur] += ax;
                f1[cur] += ay;
                f2[cur] += az;
              }
            }
            cur = hh;
            ax = ay = az = 0.0;
          }
          ax += fx;
          ay += fy;
          az += fz;
        };
        // two independent pair terms per iteration: the uniform constants of the
        // transcendentals are materialised once per two pairs
#pragma unroll 1
        for (int r = 0; r < R; r += 2) {
          const int e1 = e_lo + r, e2 = e1 + 1;
          const int qe1 = q_w[e1 < e_hi ? e1 : 0], qe2 = q_w[e2 < e_hi ? e2 : 0];
          const int h1_ = qe1 >> 5, k1 = qe1 & 31, h2_ = qe2 >> 5, k2 = qe2 & 31;
          const bool l1 = e1 < e_hi && sh.cj[warp][k1] != sh.ha[warp][h1_];
          const bool l2 = e2 < e_hi && sh.cj[warp][k2] != sh.ha[warp][h2_];
          double pe1, fx1, fy1, fz1, pe2, fx2, fy2, fz2;
          tile_pair<kTabOnly>(sh.hx[warp][h1_], sh.hy[warp][h1_], sh.hz[warp][h1_],
                              sh.hq[warp][h1_], sh.cx[warp][k1], sh.cy[warp][k1], sh.cz[warp][k1],
                              sh.cq[warp][k1], l1, lx, ly, ilx, ily, alpha, rc2, c, etab, pe1, fx1, fy1,
                              fz1, flag);
          tile_pair<kTabOnly>(sh.hx[warp][h2_], sh.hy[warp][h2_], sh.hz[warp][h2_],
                              sh.hq[warp][h2_], sh.cx[warp][k2], sh.cy[warp][k2], sh.cz[warp][k2],
                              sh.cq[warp][k2], l2, lx, ly, ilx, ily, alpha, rc2, c, etab, pe2, fx2, fy2,
                              fz2, flag);
          E += pe1;
          E += pe2;
          take(e1 < e_hi, h1_, fx1, fy1, fz1);
          take(e2 < e_hi, h2_, fx2, fy2, fz2);
        }
        // last piece: when the first piece was closed, the open one started here
        // and is the only piece of its home that starts in this lane -> no two
        // lanes write the same home in this step
        if (head >= 0) {
          f0[cur] += ax;
          f1[cur] += ay;
          f2[cur] += az;
        } else {  // one piece: it is the head
          head = cur;
          bx = ax;
          by = ay;
          bz = az;
        }
        __syncwarp();
        // heads: runs of equal home over consecutive lanes, segmented scan by
        // home (keys ascend over the lanes; empty lanes get distinct keys)
        const int key = head >= 0 ? head : 64 + lane;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double ux = __shfl_up_sync(full, bx, o);
          const double uy = __shfl_up_sync(full, by, o);
          const double uz = __shfl_up_sync(full, bz, o);
          const int kp = __shfl_up_sync(full, key, o);
          if (lane >= o && kp == key) {
            bx += ux;
            by += uy;
            bz += uz;
          }
        }
        const int kn = __shfl_down_sync(full, key, 1);
        if (head >= 0 && (lane == 31 || kn != key)) {
          f0[head] += bx;
          f1[head] += by;
          f2[head] += bz;
        }
        __syncwarp();
      }
    }
    __syncwarp();
    if (hact) {
      const int64_t i = order[a];
      forces[3 * i + 0] = f0[lane];
      forces[3 * i + 1] = f1[lane];
      forces[3 * i + 2] = f2[lane];
    }
    __syncwarp();
  }
  if (flag) atomicOr(status, SLAB_STATUS_COINCIDENT_DEV);
  sh.red[threadIdx.x] = E;
  __syncthreads();
  for (int w = kTileThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh.red[threadIdx.x] += sh.red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) eblk[blockIdx.x] = sh.red[0];
}

// ---------------------------------------------------------------------------
// the same warp-cooperative screen, writing neighbour rows for pair_list_kernel
// ---------------------------------------------------------------------------
// Replaces nbr_build_kernel's per-lane candidate streams (each lane loading its
// own candidates: L1-throughput bound, lanes idling on uneven column lengths)
// with the tile kernel's screen: a warp's 32 homes (a compact brick of the home
// order) test every candidate of their r_c window, staged 32 at a time in shared
// memory and compared two at a time in paired fp32; each lane appends its hits to
// its home's row (cell-sorted index a -> row a, as nbr_build writes them).  A row
// that would exceed kcap is marked nn = -1 (overflow_pairs_kernel evaluates it).
constexpr int kNbrTileWarps = 4;
__global__ void __launch_bounds__(32 * kNbrTileWarps) nbr_tile_kernel(
    const float4* __restrict__ cpf, const int32_t* __restrict__ start,
    const int32_t* __restrict__ hperm, int64_t h0, int64_t h1, int ncx, int ncy, int ncz,
    float lxf, float lyf, float lzf, float rc2f, float rcf, int kcap,
    int32_t* __restrict__ nbr, int32_t* __restrict__ nn, int* __restrict__ maxnn,
    int* __restrict__ status) {
  __shared__ float s_nx[kNbrTileWarps][32], s_ny[kNbrTileWarps][32], s_nz[kNbrTileWarps][32];
  __shared__ int32_t s_j[kNbrTileWarps][32];
  // per-lane ring of pending row entries (slot-major: conflict-free), written to
  // the row as whole 32-byte sectors, as nbr_build does
  constexpr int kTRing = 16;
  __shared__ int32_t s_ring[kNbrTileWarps][kTRing][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const float ex = lxf / ncx, ey = lyf / ncy, izc = ncz / lzf;
  const float ilxf = 1.0f / lxf, ilyf = 1.0f / lyf;
  float* snx = s_nx[warp];
  float* sny = s_ny[warp];
  float* snz = s_nz[warp];
  int32_t* sj = s_j[warp];
  const int64_t ngroups = (h1 - h0 + 31) / 32;
  for (int64_t grp = blockIdx.x * (int64_t)kNbrTileWarps + warp; grp < ngroups;
       grp += (int64_t)gridDim.x * kNbrTileWarps) {
    const int64_t hidx = h0 + grp * 32 + lane;
    const bool hact = hidx < h1;
    const int a = hact ? hperm[hidx] : -1;
    const float4 pf = hact ? cpf[a] : make_float4(0.f, 0.f, 0.f, 0.f);
    int32_t* row = nbr + (hact ? (int64_t)a : 0) * kcap;  // rows indexed by cell order
    int cnt = 0, done = 0;  // hits found / hits already written to the row
    int32_t* ring = &s_ring[warp][0][lane];
    auto flush8 = [&]() {
      if (done + 8 <= kcap) {
        const int s0 = done & (kTRing - 1);
        const int4 v0 = make_int4(ring[(s0 + 0) * 32], ring[(s0 + 1) * 32], ring[(s0 + 2) * 32],
                                  ring[(s0 + 3) * 32]);
        const int4 v1 = make_int4(ring[(s0 + 4) * 32], ring[(s0 + 5) * 32], ring[(s0 + 6) * 32],
                                  ring[(s0 + 7) * 32]);
        int4* dst = reinterpret_cast<int4*>(row + done);
        dst[0] = v0;
        dst[1] = v1;
      }
      done += 8;
    };
    float x0 = hact ? pf.x : 3e30f, x1 = hact ? pf.x : -3e30f;
    float y0 = hact ? pf.y : 3e30f, y1 = hact ? pf.y : -3e30f;
    float z0 = hact ? pf.z : 3e30f, z1 = hact ? pf.z : -3e30f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      x0 = fminf(x0, __shfl_xor_sync(full, x0, o));
      x1 = fmaxf(x1, __shfl_xor_sync(full, x1, o));
      y0 = fminf(y0, __shfl_xor_sync(full, y0, o));
      y1 = fmaxf(y1, __shfl_xor_sync(full, y1, o));
      z0 = fminf(z0, __shfl_xor_sync(full, z0, o));
      z1 = fmaxf(z1, __shfl_xor_sync(full, z1, o));
    }
    const int ix0 = (int)floorf((x0 - rcf) / ex), ix1 = (int)floorf((x1 + rcf) / ex);
    const int iy0 = (int)floorf((y0 - rcf) / ey), iy1 = (int)floorf((y1 + rcf) / ey);
    const bool wrap_x = ix1 - ix0 + 1 > ncx, wrap_y = iy1 - iy0 + 1 > ncy;
    const bool minimg = wrap_x || wrap_y;
    const int nX = wrap_x ? ncx : ix1 - ix0 + 1;
    const int nY = wrap_y ? ncy : iy1 - iy0 + 1;
    const int ncol = nX * nY;
#pragma unroll 1
    for (int q0 = 0; q0 < ncol; q0 += 32) {
      const int qc = q0 + lane;
      int j0 = 0, len = 0;
      float shx = 0.f, shy = 0.f;
      if (qc < ncol) {
        const int ux = ix0 + qc / nY, uy = iy0 + qc % nY;
        const int mx = ux >= 0 ? ux / ncx : -((-ux + ncx - 1) / ncx);
        const int my = uy >= 0 ? uy / ncy : -((-uy + ncy - 1) / ncy);
        const int wx = ux - mx * ncx, wy = uy - my * ncy;
        shx = (float)mx * lxf;
        shy = (float)my * lyf;
        const float dxr = wrap_x ? 0.0f : fmaxf(0.0f, fmaxf(ux * ex - x1, x0 - (ux + 1) * ex));
        const float dyr = wrap_y ? 0.0f : fmaxf(0.0f, fmaxf(uy * ey - y1, y0 - (uy + 1) * ey));
        const float dxy2 = fmaf(dxr, dxr, dyr * dyr);
        if (dxy2 <= rc2f) {
          const float h = sqrtf(rc2f - dxy2);
          int zlo = (int)floorf((z0 - h) * izc - 1e-3f);
          int zhi = (int)floorf((z1 + h) * izc + 1e-3f);
          zlo = zlo < 0 ? 0 : (zlo >= ncz ? ncz - 1 : zlo);
          zhi = zhi < 0 ? 0 : (zhi >= ncz ? ncz - 1 : zhi);
          const int64_t col = ((int64_t)wx * ncy + wy) * ncz;
          j0 = start[col + zlo];
          len = start[col + zhi + 1] - j0;
        }
      }
      int incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(full, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(full, incl, 31);
      const int excl = incl - len;
#pragma unroll 1
      for (int fb = 0; fb < total; fb += 32) {
        const int f = fb + lane;
        int k = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
          const int v = __shfl_sync(full, incl, k + step - 1);
          if (v <= f) k += step;
        }
        const int jk = __shfl_sync(full, j0, k & 31);
        const int ek = __shfl_sync(full, excl, k & 31);
        const float sx = __shfl_sync(full, shx, k & 31);
        const float sy = __shfl_sync(full, shy, k & 31);
        const bool valid = f < total;
        const int j = jk + (f - ek);
        const float4 cfj = valid ? cpf[j] : make_float4(3e30f, 3e30f, 3e30f, 0.f);
        snx[lane] = -(cfj.x + sx);
        sny[lane] = -(cfj.y + sy);
        snz[lane] = -cfj.z;
        sj[lane] = valid ? j : -2;
        __syncwarp();
        unsigned hits = 0u;
        if (!minimg) {
          const float2 px = make_float2(pf.x, pf.x), py = make_float2(pf.y, pf.y);
          const float2 pz = make_float2(pf.z, pf.z), nrc = make_float2(-rc2f, -rc2f);
#pragma unroll
          for (int t = 0; t < 32; t += 2) {
            const float2 dx = __fadd2_rn(px, *reinterpret_cast<const float2*>(snx + t));
            const float2 dy = __fadd2_rn(py, *reinterpret_cast<const float2*>(sny + t));
            const float2 dz = __fadd2_rn(pz, *reinterpret_cast<const float2*>(snz + t));
            float2 d = __ffma2_rn(dz, dz, nrc);
            d = __ffma2_rn(dy, dy, d);
            d = __ffma2_rn(dx, dx, d);
            hits = __funnelshift_l(__float_as_uint(d.x), hits, 1);
            hits = __funnelshift_l(__float_as_uint(d.y), hits, 1);
          }
          hits = __brev(hits);
        } else {
#pragma unroll 4
          for (int t = 0; t < 32; ++t) {
            float dx = pf.x + snx[t], dy = pf.y + sny[t];
            const float dz = pf.z + snz[t];
            dx = fmaf(-lxf, rintf(dx * ilxf), dx);
            dy = fmaf(-lyf, rintf(dy * ilyf), dy);
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            if (d2 <= rc2f && sj[t] >= 0) hits |= 1u << t;
          }
        }
        if (!hact) hits = 0u;
        // append the hits (the home itself is screened in: skip it by index)
        while (hits) {
          const int t = __ffs(hits) - 1;
          hits &= hits - 1u;
          const int jj = sj[t];
          if (jj != a) {
            ring[(cnt & (kTRing - 1)) * 32] = jj;
            ++cnt;
            if (cnt - done >= 8) flush8();
          }
        }
        __syncwarp();
      }
    }
    if (hact && cnt <= kcap)
      for (int e = done; e < cnt; ++e) row[e] = ring[(e & (kTRing - 1)) * 32];
    if (hact) {
      nn[a] = cnt <= kcap ? cnt : -1;  // -1: overflowed, evaluated by overflow_pairs_kernel
      if (cnt > kcap) {
        atomicOr(status, SLAB_STATUS_NBR_OVERFLOW_DEV);
        atomicMax(maxnn, cnt);
      }
    }
  }
}

cudaError_t nbr_tile(const float4* cpf, const int32_t* start, const int32_t* hperm, int64_t h0,
                     int64_t h1, int ncx, int ncy, int ncz, double lx, double ly, double lz,
                     float rc2f, int kcap, int32_t* nbr, int32_t* nn, int* maxnn, int* status,
                     cudaStream_t st) {
  const int64_t groups = (h1 - h0 + 31) / 32;
  int64_t ctas = (groups + kNbrTileWarps - 1) / kNbrTileWarps;
  const int64_t cap = 148 * 12;
  ctas = ctas < cap ? (ctas > 0 ? ctas : 1) : cap;
  nbr_tile_kernel<<<(unsigned)ctas, 32 * kNbrTileWarps, 0, st>>>(
      cpf, start, hperm, h0, h1, ncx, ncy, ncz, (float)lx, (float)ly, (float)lz, rc2f,
      sqrtf(rc2f), kcap, nbr, nn, maxnn, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
int64_t tile_home_slots(int ncx, int ncy, int ncz) {
  const int64_t nbx = (ncx + 1) / 2, nby = (ncy + 1) / 2, nbz = (ncz + 3) / 4;
  return nbx * nby * nbz * 16;
}

size_t tile_work_bytes(int64_t n, int ncx, int ncy, int ncz) {
  const int64_t slots = tile_home_slots(ncx, ncy, ncz);
  const int64_t nb = (slots + kScanTile - 1) / kScanTile;
  auto a256 = [](size_t b) { return (b + 255) & ~(size_t)255; };
  return 2 * a256(sizeof(int32_t) * (size_t)slots) + a256(sizeof(int32_t) * (size_t)(nb + 1)) +
         a256(sizeof(int32_t) * (size_t)(n > 0 ? n : 1)) + 1024;
}

int tile_grid(int64_t nhomes) {
  const int64_t groups = (nhomes + 31) / 32;
  const int64_t ctas = (groups + kTileWarps - 1) / kTileWarps;
  const int64_t cap = 148 * 8;  // resident CTAs (~26 KB shared, <= 96 registers)
  return (int)(ctas < cap ? (ctas > 0 ? ctas : 1) : cap);
}

cudaError_t tile_homes(const int32_t* start, const uint32_t* skey, int64_t n, int ncx, int ncy,
                       int ncz, void* work, int32_t** hperm_out, cudaStream_t st) {
  const int nby = (ncy + 1) / 2, nbz = (ncz + 3) / 4;
  const int64_t slots = tile_home_slots(ncx, ncy, ncz);
  const int64_t nb = (slots + kScanTile - 1) / kScanTile;
  auto a256 = [](size_t b) { return (b + 255) & ~(size_t)255; };
  char* w = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(work) + 255) & ~(uintptr_t)255);
  int32_t* cnt = reinterpret_cast<int32_t*>(w);
  w += a256(sizeof(int32_t) * (size_t)slots);
  int32_t* off = reinterpret_cast<int32_t*>(w);
  w += a256(sizeof(int32_t) * (size_t)slots);
  int32_t* bsum = reinterpret_cast<int32_t*>(w);
  w += a256(sizeof(int32_t) * (size_t)(nb + 1));
  int32_t* hperm = reinterpret_cast<int32_t*>(w);
  cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)slots, st);
  const int64_t ncell = (int64_t)ncx * ncy * ncz;
  home_count_kernel<<<(unsigned)((ncell + 255) / 256), 256, 0, st>>>(start, ncx, ncy, ncz, nby,
                                                                       nbz, cnt);
  cudaError_t e = exclusive_scan(cnt, slots, bsum, off, st);
  if (e != cudaSuccess) return e;
  home_scatter_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(skey, start, off, n, ncy, ncz,
                                                                   nby, nbz, hperm);
  *hperm_out = hperm;
  return cudaGetLastError();
}

cudaError_t tile_pairs(const double4* cp, const float4* cpf, const int32_t* start,
                       const int32_t* hperm, const int32_t* order, int64_t h0, int64_t h1,
                       int ncx, int ncy, int ncz, double lx, double ly, double lz, double alpha,
                       double rc, double* forces, double* eblk, int grid, int* status,
                       cudaStream_t st) {
  const double rc2 = rc * rc;
  const float rc2f = (float)(rc2 * (1.0 + 1e-3) + 1e-2);  // conservative, as short.cu
  const float rcf = sqrtf(rc2f);
  const bool tab_only = alpha * rc <= 0.999 * kErfcxRatMax;
  if (tab_only)
    short_tile_kernel<true><<<grid, kTileThreads, 0, st>>>(
        cp, cpf, start, hperm, order, h0, h1, ncx, ncy, ncz, lx, ly, (float)lx, (float)ly,
        (float)lz, alpha, rc2, rc2f, rcf, forces, eblk, status);
  else
    short_tile_kernel<false><<<grid, kTileThreads, 0, st>>>(
        cp, cpf, start, hperm, order, h0, h1, ncx, ncy, ncz, lx, ly, (float)lx, (float)ly,
        (float)lz, alpha, rc2, rc2f, rcf, forces, eblk, status);
  return cudaGetLastError();
}

}  // namespace slab
