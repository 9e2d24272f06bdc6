/*
 * slabewald_b200.h -- C ABI of the B200-native RBSE2D / SOEwald2D energy-force path.
 *
 * The reference (arXiv 2403.01521 artifact, package `slabewald`) has no FFI; its
 * operator boundary is the Python function layer above its numba kernels
 * (SURVEY.md 8(b)).  Each entry point below replaces one of those kernels or
 * the evaluation that strings them together, with plain pointers and sizes:
 *
 *   slab_sort_by_z          <- core.py:166-208  _bucket_sort_perm / sort_by_z
 *   slab_fourier_sweep      <- soewald2d.py:85-208  _fourier_soe_sweep
 *                              (+ _decay_table soewald2d.py:76-82, fused on device)
 *   slab_zero_mode_sweep    <- soewald2d.py:211-296 _zero_mode_soe_sweep
 *   slab_short_range        <- ewald2d.py:280-303  short_range_energy_forces
 *                              (build_cell_list 141-157, _pair_kernel_cells 160-231,
 *                               _pair_kernel_brute 234-277)
 *   slab_sample_modes       <- rbse2d.py:105-207  _chain_kernel / ModeSampler.batch
 *   slab_evaluate           <- rbse2d.py:274-317 rb_energy_forces and
 *                              soewald2d.py:398-438 soe_energy_forces
 *
 * Conventions
 *   - Every array pointer is DEVICE memory unless the name starts with h_.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Positions are (n,3) float64 row-major AoS exactly like ParticleSystem.pos;
 *     per-particle scalars are float64 (n,).  Modes are (P,3) float64 rows
 *     (kx, ky, |k|) as EwaldParams.kmodes / ModeSampler.batch.
 *   - SOE coefficients are passed as host arrays of the M complex terms (re/im
 *     split); M must be even and conjugate-paired (term M-1-l == conj(term l)),
 *     which every contour from build_soe_contour satisfies (soe.py:77-84).
 *   - Outputs are written (not accumulated) unless stated.
 *   - Calls are stream-ordered and asynchronous; status that depends on device
 *     data (coincident particles) is reported through device status words the
 *     caller reads after synchronising.
 *   - Return value: SLAB_OK or an error code; slab_last_error() gives text.
 */
#ifndef SLABEWALD_B200_H
#define SLABEWALD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SLAB_OK = 0,
  SLAB_ERR_ARG = 1,          /* bad argument (sizes, M odd / unpaired, ...) */
  SLAB_ERR_CUDA = 2,         /* CUDA runtime error */
  SLAB_ERR_UNSUPPORTED = 3,  /* e.g. unpaired SOE table */
  SLAB_ERR_NOMEM = 4
};

/* device status word bits (written by kernels, read by the host after sync) */
enum {
  SLAB_STATUS_COINCIDENT = 1, /* d2 < 1e-24 pair: ewald2d.py:207-209,301-302 */
  SLAB_STATUS_SINGULAR = 2,   /* reserved: singular terms (|b_l - k| < 2e-6 k) are now
                               * evaluated (soewald2d.py:116-124), this bit is never set */
  SLAB_STATUS_NBR_OVERFLOW = 4, /* a short-range neighbour row exceeded its capacity; those
                                   homes were evaluated in-stream by the overflow kernel, so the
                                   results are COMPLETE -- raising the capacity
                                   (slab_ctx_neighbor_capacity) only makes later runs faster */
  SLAB_STATUS_NONFINITE = 8,    /* a z coordinate is not finite (core.py:206-207): results invalid */
  SLAB_STATUS_WALL = 16         /* a particle at or beyond a wall (md.py:72) */
};

typedef struct SlabBox {
  double lx, ly, lz, sigma_top, sigma_bot; /* core.py:25-51 BoxGeometry */
} SlabBox;

typedef struct SlabSOE {
  int m;                 /* number of complex terms (even) */
  const double* h_w_re;  /* host, length m */
  const double* h_w_im;
  const double* h_s_re;
  const double* h_s_im;
} SlabSOE;

/* One full energy + force evaluation.  rb_energy_forces when commonv_scalar is
 * used ((H/P)(2 alpha/sqrt(pi)), rbse2d.py:301); soe_energy_forces when
 * d_commonv carries (2 alpha/sqrt(pi)) exp(-k^2/4alpha^2) per mode
 * (soewald2d.py:421-422). */
typedef struct SlabEvalArgs {
  int64_t n;
  const double* d_pos;      /* (n,3) input order */
  const double* d_charge;   /* (n,) */
  SlabBox box;
  double alpha;
  double r_c;
  SlabSOE soe;
  const double* d_modes;    /* (P,3) kx,ky,|k| */
  int64_t nmode;
  const double* d_commonv;  /* (P,) or NULL -> commonv_scalar for every mode */
  double commonv_scalar;
  double charge_const;      /* C_Q (rbse2d.py:77-89) or u_q (soewald2d.py:408-413) */
  int want_forces;          /* 0: energies only (forces untouched) */
  int skip_short_range;     /* 1: u_s = 0, no short-range forces (sub-path calls) */
  double* d_forces;         /* (n,3) out, input order */
  double* d_energy;         /* (8,) out: u_s, u_l_k, u_l_0, u_self, u_ps, status bits,
                               Q = sum q^2 (lead rank), status as sum_k bit_k 256^k (a
                               SUM all-reduce over ranks keeps every bit recoverable) */
  int64_t* d_perm;          /* optional (n,) out: the z-sort permutation, or NULL */
  /* Multi-GPU (one process per GPU, particles replicated): this
   * rank evaluates only its share and the caller sums d_forces and d_energy[0..4]
   * over ranks with ONE allreduce.  The caller passes this rank's slice of the
   * sampled modes (d_modes/nmode) with commonv for the GLOBAL batch size; the
   * library takes home particles [rank*n/count, (rank+1)*n/count) of the
   * short-range cell order, and rank 0 alone adds the k = 0 mode, the constants
   * (charge_const, self, slab) and the plane forces.  shard_count <= 1: all. */
  int shard_rank;
  int shard_count;
  /* optional cudaEvent_t (as void*) recorded on `stream` around the SOE scan
   * kernels (Fourier 3-phase scan + k = 0 mode) for roofline timing */
  void* ev_scan_begin;
  void* ev_scan_end;
  /* multi-GPU decomposition (shard_count > 1):
   *   SLAB_SHARD_MODES  (0): rank r evaluates its slice of d_modes (one call);
   *   SLAB_SHARD_ZSPLIT (1): rank r scans ALL modes over its contiguous range of
   *     the z-sorted particles (chunks nch*r/W .. nch*(r+1)/W), in two calls
   *     around an all-gather (SURVEY 8(e) alternative):
   *       phase 1 writes this rank's chunk-range total maps to d_xchg
   *         (slab_zsplit_exchange_doubles() doubles);
   *       the caller all-gathers them into d_xchg[W][...] (rank order);
   *       phase 2 (same arguments, d_xchg = gathered) finishes the evaluation.
   *   phase 0 = the whole evaluation in one call (shard_mode MODES, or W = 1). */
  int shard_mode;
  int phase;
  double* d_xchg;
  /* cudaEvent_t or NULL: d_modes is complete once this event has fired (e.g. a
   * device sampler on another stream).  The evaluation waits on it only before
   * its first use of the k-set, so the sampler overlaps the z sort. */
  void* ev_modes_ready;
} SlabEvalArgs;

enum { SLAB_SHARD_MODES = 0, SLAB_SHARD_ZSPLIT = 1 };

typedef struct SlabCtx SlabCtx;

int slab_ctx_create(SlabCtx** out);
int slab_ctx_destroy(SlabCtx* ctx);
const char* slab_last_error(void);
const char* slab_version(void);

/* Short-range neighbour rows: grow-only minimum capacity, and the longest row
 * seen by the last short-range run (synchronous read) for SLAB_STATUS_NBR_OVERFLOW. */
int slab_ctx_neighbor_capacity(SlabCtx* ctx, int capacity);
int slab_ctx_last_max_neighbors(SlabCtx* ctx, int* out);

/* core.py:203-208: stable ascending-z permutation; z read as d_z[i*stride]. */
int slab_sort_by_z(SlabCtx* ctx, const double* d_z, int64_t stride, int64_t n, int64_t* d_perm,
                   void* stream);

/* soewald2d.py:85-208 on ALREADY z-sorted SoA (x,y,z,q).  Writes the Kahan-
 * combined mode energy to d_energy[0] (without any charge constant) and, when
 * want_forces, ADDS the Fourier forces into d_forces_sorted (n,3) like the
 * reference (which accumulates).  b_l = alpha * s_l. */
int slab_fourier_sweep(SlabCtx* ctx, const double* d_x, const double* d_y, const double* d_z,
                       const double* d_q, int64_t n, const double* d_modes,
                       const double* d_commonv, double commonv_scalar, int64_t nmode,
                       SlabSOE soe, double alpha, double area, int want_forces,
                       double* d_forces_sorted, double* d_energy, int* d_status, void* stream);

/* soewald2d.py:211-296 on sorted z,q: d_energy[0] = u_pair; when want_forces,
 * ADDS fz (the bracket, before the 2 pi/A q factor) into d_fz. */
int slab_zero_mode_sweep(SlabCtx* ctx, const double* d_z, const double* d_q, int64_t n,
                         SlabSOE soe, double alpha, int want_forces, double* d_fz,
                         double* d_energy, void* stream);

/* ewald2d.py:280-303 (no r_c > L/2 check here; the host layer raises).  Writes
 * d_energy[0] = u_s, d_forces (n,3) input order, ORs status bits. */
int slab_short_range(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                     SlabBox box, double alpha, double r_c, double* d_forces, double* d_energy,
                     int* d_status, void* stream);

/* rbse2d.py:151-207 Metropolis independence chain over integer (mx,my) != 0 with
 * a counter-based Philox4x32-10 stream.  d_state = {mx, my, since, counter,
 * accepted, steps} (int64) persists across calls.  Writes P rows (kx,ky,|k|) to
 * d_modes and the integer indices to d_idx (P,2) if not NULL.  burn_in > 0
 * initialises the chain first (ModeSampler.__init__). */
int slab_sample_modes(SlabCtx* ctx, int64_t* d_state, uint64_t seed, double alpha, double lx,
                      double ly, int thin, int burn_in, int64_t P, double* d_modes,
                      int64_t* d_idx, void* stream);

/* Full evaluation (sort, gather, short range, Fourier sweep, zero mode, self,
 * slab, assembly, scatter to input order). */
int slab_evaluate(SlabCtx* ctx, const SlabEvalArgs* args, void* stream);

/* slab_evaluate on HOST buffers -- the call behind rb_energy_forces /
 * soe_energy_forces (rbse2d.py:274-317, soewald2d.py:398-438), whose inputs and
 * outputs are numpy arrays.  h_pos (n x 3, AoS) and h_charge (n) are read,
 * h_forces (n x 3, input order; may be NULL when want_forces = 0) and
 * h_energy (8, the d_energy layout) are written; args->d_pos / d_charge /
 * d_forces / d_energy are ignored (the context keeps device copies) while
 * d_modes / d_commonv stay DEVICE pointers (the device sampler's output).
 * Uploads run on a context-owned stream, the charges overlapping the z sort;
 * page-locked host memory copies at DMA speed.  Synchronises `stream` before
 * returning.  Unsharded (shard_mode 0, phase 0) evaluations only. */
int slab_evaluate_host(SlabCtx* ctx, const SlabEvalArgs* args, const double* h_pos,
                       const double* h_charge, double* h_forces, double* h_energy,
                       void* stream);

/* Size of one rank's z-split exchange payload (doubles): 4 (M + 1) 2P with
 * forces, 4 (M + 1) P energy-only; M = SOE terms, P = modes. */
int64_t slab_zsplit_exchange_doubles(int64_t nmode, int soe_terms, int want_forces);

/* rbse2d.py:320-330 _rb_batch_energy_kernel (the body of run_many_batches):
 * for b < nbatch, d_out[b] = Kahan-combined forward-sweep energy of modes
 * d_modes[b*P .. (b+1)*P) (rows kx, ky, |k|), commonv = commonv_scalar for every
 * mode, no charge constant.  Particles in input order (pos AoS, charge): sorted
 * once, decay table once, modes swept in groups on device.  ORs status bits
  * (NONFINITE) into d_status. */
int slab_batch_energies(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                        SlabSOE soe, double alpha, double area, const double* d_modes,
                        int64_t nbatch, int64_t P, double commonv_scalar, double* d_out,
                        int* d_status, void* stream);

/* ---- device-resident MD step (md.py) ---------------------
 * WCA core of md.py:34-56 (lj_forces: 4 eps[(s/r)^12 - (s/r)^6] + eps below
 * 2^(1/6) s, minimum image in x, y): ADDS into d_forces (n,3, input order),
 * d_energy[0] = energy; coincident pairs set SLAB_STATUS_COINCIDENT. */
int slab_wca(SlabCtx* ctx, const double* d_pos, int64_t n, SlabBox box, double eps, double sigma,
             double* d_forces, double* d_energy, int* d_status, void* stream);
/* md.py:59-77 wall_forces: ADDS the wall z-forces, d_energy[0] = energy,
 * SLAB_STATUS_WALL for a particle at or beyond a wall. */
int slab_walls(SlabCtx* ctx, const double* d_pos, int64_t n, double lz, double eps, double sigma,
               double* d_forces, double* d_energy, int* d_status, void* stream);
/* md.py:180-193 langevin_step (kick, drift, exact OU with Philox4x32-10 noise
 * keyed by (seed, *d_counter, particle), drift) followed by the xy wrap of
 * run_simulation (md.py:245-250) accumulating image offsets into d_shift (n,2)
 * if not NULL; advances *d_counter on device (graph-capturable). */
int slab_md_langevin(double* d_pos, double* d_vel, const double* d_forces, const double* d_mass,
                     int64_t n, double dt, double gamma, double temperature, uint64_t seed,
                     int64_t* d_counter, double* d_shift, double lx, double ly, void* stream);
/* v += h F / m */
int slab_md_kick(double* d_vel, const double* d_forces, const double* d_mass, int64_t n,
                 double h, void* stream);
/* x += dt v, then the xy wrap (d_shift as above) */
int slab_md_drift(double* d_pos, const double* d_vel, int64_t n, double dt, double* d_shift,
                  double lx, double ly, void* stream);
/* v *= s (Nose-Hoover, md.py:205-217) */
int slab_md_scale(double* d_vel, int64_t n, double s, void* stream);
/* d_out[0] = 0.5 sum m v^2 (md.py:176-177), fixed-order reduction */
int slab_md_kinetic(SlabCtx* ctx, const double* d_vel, const double* d_mass, int64_t n,
                    double* d_out, void* stream);

/* ---- O(N^2 K) Ewald2D reference solver -------------------
 * ewald2d.py:331-442 _fourier_ref_kernel: pairwise Fourier sum over the modes
 * (integer indices d_mxy (nmode,2), ring of equal |k| d_ring, ring norms
 * d_kappa), "stable" (naive = 0) or "naive" xi kernels.  d_energy[0] = the pair
 * sum (without the charge term u_q), d_forces (n,3) written.  At most 256 rings
 * and |mx|, |my| <= 64 (SLAB_ERR_UNSUPPORTED otherwise). */
int slab_ewald_ref_fourier(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                           double lx, double ly, double alpha, const int* d_mxy,
                           const int* d_ring, int nmode, const double* d_kappa, int nring,
                           int mxmax, int mymax, int naive, double* d_forces, double* d_energy,
                           void* stream);
/* ewald2d.py:477-501 _zero_mode_kernel: d_energy[0] = sum_{i<j} q_i q_j G(|z_ij|),
 * d_fz[i] = sum_j q_i q_j erf(a |z_ij|) sign(z_ij) (before the 2 pi / A factor). */
int slab_ewald_ref_zero(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                        double alpha, double* d_fz, double* d_energy, void* stream);

/* Recursion of soewald2d.py:42-64 recursive_pair_sum on sorted z:
 * out[a] = sum_{j<a} q_j exp(-i theta_j - beta (z_a - z_j)), complex interleaved. */
int slab_recursive_pair_sum(SlabCtx* ctx, const double* d_q, const double* d_theta,
                            const double* d_z, int64_t n, double beta_re, double beta_im,
                            double* d_out, void* stream);

/* The position-only constants of an evaluation, by the same device reduction
 * slab_evaluate's assembly uses (ewald2d.py:527-545 self_energy and
 * slab_energy_forces): d_energy[3] = u_self = alpha/sqrt(pi) sum q^2,
 * d_energy[4] = u_ps = sum q phi(z); other slots as slab_evaluate with no
 * short-range, Fourier or k = 0 terms.  (Lets the O(N^2 K) reference solver
 * report bitwise the same u_self / u_ps as the SOE paths, as the reference's
 * total_breakdown test requires.)  d_energy: >= 8 doubles. */
int slab_constant_terms(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                        SlabBox box, double alpha, double* d_energy, void* stream);

/* FP64 roofline denominator: DFMA throughput microbenchmark on the current
 * device (TFLOP/s, 2 flops per DFMA).  Synchronous. */
int slab_fp64_peak(double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* SLABEWALD_B200_H */
