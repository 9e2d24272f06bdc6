// kernels.cuh -- internal host-side launch API shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace slab {

// ---------------------------------------------------------------- sort.cu
struct SortWork {
  uint64_t* k0;
  uint64_t* k1;
  int32_t* v0;
  int32_t* v1;
  int32_t* hist;
};
int64_t radix_hist_entries(int64_t n);
cudaError_t sort_by_z_device(const double* z, int64_t stride, int64_t n, SortWork& w,
                             cudaStream_t st, int32_t** perm_out, int* status = nullptr);
template <typename K>
cudaError_t radix_sort_pairs(K* keys, int32_t* vals, K* keys_alt, int32_t* vals_alt,
                             int32_t* hist, int64_t n, int key_bits, cudaStream_t st,
                             K** keys_out, int32_t** vals_out);
cudaError_t gather_sorted(const double* pos, const double* charge, const int32_t* perm, int64_t n,
                          double* xs, double* ys, double* zs, double* qs, int64_t* perm64,
                          cudaStream_t st);
cudaError_t perm_to_int64(const int32_t* p, int64_t n, int64_t* out, cudaStream_t st);

// ---------------------------------------------------------------- SOE constants
struct BVec {  // b_l = alpha * s_l for the pair representatives l < mh
  double re[12];
  double im[12];
};
struct WVec {
  double re[12];
  double im[12];
};
struct ZCoef {  // zero-mode pair coefficients (all doubled for the conj partner)
  double ws2[24];   // 2 w/s      (re,im interleaved)
  double w2[24];    // 2 w
  double f2[24];    // 2 (w/s + w s / 2)
  double aw2[24];   // 2 alpha w
};

// ---------------------------------------------------------------- fourier.cu
struct FourierPlan {
  int64_t n;
  int P;          // modes
  int mh;         // SOE pairs
  int R;          // particles per chunk
  int nch;        // chunks
  int ngroups;    // item groups per chunk
  int upg;        // units per group: modes (paired) or items
  int warps;      // warps per CTA
  int nbuf;       // partial force buffers (2 per group x warp, + 2 for the remainder)
  int items;      // active (mode, direction) items: 2P, or P for energy-only (forward)
  int c0, c1;     // chunk range this plan scans (z-split multi-GPU rank), default [0, nch)
  size_t smem_sweep;
  int swap;       // 1: real inputs swapped (u_r, u_i) -> (u_i, -u_r), i.e. the pass's result
                  // times -i (lone complex SOE terms, capi.cu prepare_soe)
  int paired;     // 1: a warp = 16 modes x 2 directions (force plans); 0: 32 forward items
  int units_main; // modes (paired) / items of the main sweep (whole warps when rem > 0)
  int items_main; // items of the main sweep
  int rem;        // leftover items per chunk run by the remainder sweep (0: none)
  int rem_g;      // chunks per remainder warp (32 / (rem_spl rem))
  int rem_spl;    // lanes per remainder item (2: its pairs split over two lanes)
  int rem_buf;    // the remainder's partial force buffer
};
FourierPlan fourier_plan(int64_t n, int P, int mh, int dirs = 2, int ranks = 1);
// bytes of device workspace the plan needs (carry, chunk decays, mode table, partials)
struct FourierWork {
  double* modetab;   // P * mode_stride
  double2* carry;    // nch * (2mh+1) * 2P
  double2* dchunk;   // 2 * nch * mh   (Df, Db)
  double* zbound;    // 2 * nch        (z_end, z_start)
  double* epart;     // nch * P
  double* fpart;     // nbuf * n * 3
  double* segmap;    // carry-scan segment maps (4 doubles each)
  double* tin;       // z-split: state entering the chunk range, per (comp, item) (double2)
};
size_t fourier_work_doubles(const FourierPlan& p);
void fourier_work_carve(const FourierPlan& p, double* base, FourierWork& w);
// rows [a_lo, a_hi] of the (n + 1)-row table (default: all; a z-split rank
// without the k = 0 mode needs only its chunk range's rows)
cudaError_t decay_table(const double* zs, int64_t n, int mh, const BVec& b, double2* dtab,
                        cudaStream_t st, int64_t a_lo = 0, int64_t a_hi = -1);
cudaError_t fourier_run(const FourierPlan& p, const FourierWork& w, const double* xs,
                        const double* ys, const double* zs, const double* qs,
                        const double2* dtab, const double* modes, const double* commonv,
                        double commonv_scalar, double area, const BVec& b, const WVec& wv,
                        int want_forces, double* energy_out, int* status, double* forces_sorted,
                        cudaStream_t st, int seg_len = 0);  // seg_len > 0: energy per segment
cudaError_t add_into(double* dst, const double* src, int count, cudaStream_t st);
// the same as two phases around a z-split exchange: phase 1 builds the chunk
// range's aggregates (and, with `totals`, its total map per (comp, item):
// 4 doubles each, the all-gather payload); fourier_zsplit_tin composes the
// gathered totals of the other ranks into `tin`; phase 2 finishes from `tin`
cudaError_t fourier_phase1(const FourierPlan& p, const FourierWork& w, const double* xs,
                           const double* ys, const double* zs, const double* qs,
                           const double* modes, const double* commonv, double commonv_scalar,
                           double area, const BVec& b, const WVec& wv, int* status,
                           double* totals, cudaStream_t st);
cudaError_t fourier_zsplit_tin(const FourierPlan& p, const double* totals, int W, int r,
                               double* tin, cudaStream_t st);
cudaError_t fourier_phase2(const FourierPlan& p, const FourierWork& w, const double* xs,
                           const double* ys, const double* zs, const double* qs,
                           const double2* dtab, const BVec& b, int want_forces,
                           double* energy_out, double* forces_sorted, const double* tin,
                           cudaStream_t st, int seg_len = 0);

// ---------------------------------------------------------------- zero.cu
struct ZeroPlan {
  int64_t n;
  int mh;
  int R;
  int nch;
};
ZeroPlan zero_plan(int64_t n, int mh);
size_t zero_work_doubles(const ZeroPlan& p);
cudaError_t zero_run_b(const ZeroPlan& p, double* work, const double* zs, const double* qs,
                       const double2* dtab, const ZCoef& zc, const BVec& b, double alpha,
                       int want_forces, double* fzf, double* fzb, double* upair,
                       cudaStream_t st);

// ---------------------------------------------------------------- short.cu
struct ShortPlan {
  int64_t n;
  int ncx, ncy, ncz;
  int brute;
  int64_t ncell;
  int jsplit;     // brute path: j-range splits
  int64_t nblk;   // energy partial count
  int kcap;       // neighbour-row capacity (multiple of 8)
  int span;       // cell search span S: cells of edge >= r_c / S, (2S+1)^2 columns
  int tile;       // 1: fused screen + pair kernel (short_tile.cu), no neighbour rows
};
// short_tile.cu: homes in brick order, fused screen + exact pair terms
int64_t tile_home_slots(int ncx, int ncy, int ncz);
size_t tile_work_bytes(int64_t n, int ncx, int ncy, int ncz);
int tile_grid(int64_t nhomes);
cudaError_t tile_homes(const int32_t* start, const uint32_t* skey, int64_t n, int ncx, int ncy,
                       int ncz, void* work, int32_t** hperm_out, cudaStream_t st);
cudaError_t nbr_tile(const float4* cpf, const int32_t* start, const int32_t* hperm, int64_t h0,
                     int64_t h1, int ncx, int ncy, int ncz, double lx, double ly, double lz,
                     float rc2f, int kcap, int32_t* nbr, int32_t* nn, int* maxnn, int* status,
                     cudaStream_t st);
cudaError_t tile_pairs(const double4* cp, const float4* cpf, const int32_t* start,
                       const int32_t* hperm, const int32_t* order, int64_t h0, int64_t h1,
                       int ncx, int ncy, int ncz, double lx, double ly, double lz, double alpha,
                       double rc, double* forces, double* eblk, int grid, int* status,
                       cudaStream_t st);
// max_span 1: cells of edge >= rc (fewer cells: the short WCA cutoff of a big box
// would otherwise need ~6e7 half-edge cells at N = 1e6)
ShortPlan short_plan(int64_t n, double lx, double ly, double lz, double rc, int max_span = 3);
size_t short_work_bytes(const ShortPlan& p);
cudaError_t short_run(const ShortPlan& p, void* work, const double* pos, const double* charge,
                      double lx, double ly, double lz, double alpha, double rc, double* forces,
                      double* energy_out, int* status, int64_t home_begin, int64_t home_end,
                      int* maxnn_out, cudaStream_t st, int kind = 0, double lj_eps = 0.0,
                      double lj_sigma = 0.0,  // kind 1: WCA core instead of erfc Coulomb
                      int accumulate = 0,     // 1: forces += (full home range only)
                      cudaEvent_t pairs_after = nullptr,   // pair kernel waits on it
                      cudaEvent_t charge_ready = nullptr);  // charges read from here on

// ---------------------------------------------------------------- md.cu
int64_t md_partials(int64_t n);
cudaError_t md_langevin(double* pos, double* vel, const double* forces, const double* mass,
                        int64_t n, double dt, double gamma, double temperature, uint64_t seed,
                        int64_t* counter, double* shift, double lx, double ly, cudaStream_t st);
cudaError_t md_kick(double* vel, const double* forces, const double* mass, int64_t n, double h,
                    cudaStream_t st);
cudaError_t md_drift(double* pos, const double* vel, int64_t n, double dt, double* shift, double lx,
                     double ly, cudaStream_t st);
cudaError_t md_scale(double* vel, int64_t n, double s, cudaStream_t st);
cudaError_t md_walls(const double* pos, int64_t n, double lz, double eps, double sigma,
                     double* forces, double* energy, int* status, double* part, int accumulate,
                     cudaStream_t st);
cudaError_t md_kinetic(const double* vel, const double* mass, int64_t n, double* out,
                       double* part, cudaStream_t st);

// ---------------------------------------------------------------- assemble.cu
cudaError_t assemble_forces(int64_t n, const int32_t* perm, const double* qs,
                            const double* fsorted, const double* fzf, const double* fzb,
                            double zpref, const double* fshort, const double* charge,
                            double fz_plane, double* forces, cudaStream_t st);
cudaError_t assemble_energy(int64_t n, const double* charge, const double* pos, double lz,
                            double sigma_top, double sigma_bot, double alpha, double area,
                            double charge_const, const double* u_s, const double* u_sweep,
                            const double* u_pair, const int* status, double* energy,
                            double* energy_scratch, int include_constants, cudaStream_t st);

// ---------------------------------------------------------------- sampler.cu
cudaError_t sample_modes(int64_t* state, uint64_t seed, double alpha, double lx, double ly,
                         int thin, int burn_in, int64_t P, double* modes, int64_t* idx,
                         double* scratch, int64_t scratch_doubles, cudaStream_t st);
int64_t sampler_scratch_doubles(int64_t P, int thin, int burn_in);

// ---------------------------------------------------------------- misc
cudaError_t recursive_pair_sum(const double* q, const double* theta, const double* z, int64_t n,
                               double beta_re, double beta_im, double* out, double2* agg,
                               cudaStream_t st);
cudaError_t fz_accumulate(int64_t n, const double* fzf, const double* fzb, double* fz,
                          cudaStream_t st);

}  // namespace slab

namespace slab {
cudaError_t fp64_peak(double* tflops);
// ---------------------------------------------------------------- ewald_ref.cu
int64_t ewald_ref_partials(int64_t n);
int ewald_ref_max_ring();
int ewald_ref_max_m();
cudaError_t ewald_ref_fourier(const double* pos, const double* charge, int64_t n, double lx,
                              double ly, double alpha, const int* mxy, const int* ring_id,
                              int nmode, const double* kappa, int nring, int mxmax, int mymax,
                              int naive, double* forces, double* energy, double* part,
                              cudaStream_t st);
cudaError_t ewald_ref_zero(const double* pos, const double* charge, int64_t n, double alpha,
                           double* fz, double* energy, double* part, cudaStream_t st);

}  // namespace slab
