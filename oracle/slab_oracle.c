/*
 * slab_oracle.c -- CPU restatement of the reference RBSE2D / SOEwald2D hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; it is never linked into, loaded by, or
 * called from the product path (paper_2403_01521_b200/*), which fails loudly
 * without its CUDA library.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may use it.
 *
 * Each function restates, loop for loop, the numba kernel it cites in the
 * reference package /root/reference/pkg/src/slabewald (scalar, same loop order,
 * no FMA contraction: build with -ffp-contract=off, as numba without fastmath).
 * Complex arithmetic is written out in re/im form the way LLVM lowers numba's
 * complex128 ops (mul: ar*br - ai*bi, ar*bi + ai*br).
 *
 * Parity pin: tests/test_oracle.py checks these functions against fixtures
 * produced by the real reference (tests/golden/make_golden.py).
 *
 * The *_mt variants parallelise over modes / cells with OpenMP for the
 * "--impl reference" arm (all host threads); per-thread force buffers are
 * reduced in fixed thread order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SINGULAR_TOL 2e-6
static const double SQRT_PI = 1.7724538509055159;   /* np.sqrt(np.pi) */

typedef struct { double re, im; } cplx;
static inline cplx cx(double r, double i) { cplx c = {r, i}; return c; }
static inline cplx cadd(cplx a, cplx b) { return cx(a.re + b.re, a.im + b.im); }
static inline cplx cmul(cplx a, cplx b) {
  return cx(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
static inline cplx cscale(double s, cplx a) { return cx(s * a.re, s * a.im); }
/* complex / complex, Smith-free textbook form as used for c_l = w/(b^2-k^2) */
static inline cplx cdiv(cplx a, cplx b) {
  /* numba lowers complex division through a scaled algorithm; the tiny
   * differences are far below the 1e-10 parity tolerance. */
  double d = b.re * b.re + b.im * b.im;
  return cx((a.re * b.re + a.im * b.im) / d, (a.im * b.re - a.re * b.im) / d);
}
static inline double cabs_(cplx a) { return hypot(a.re, a.im); }
static inline cplx cexp_(cplx a) {
  double e = exp(a.re);
  return cx(e * cos(a.im), e * sin(a.im));
}

/* ---------------------------------------------------------------------------
 * core.py:166-200  _bucket_sort_perm -- stable z ordering
 * ------------------------------------------------------------------------- */
void oracle_sort_perm(const double* z, int64_t n, double lz, int64_t* perm) {
  int64_t nb = n > 0 ? n : 1;
  int64_t* counts = (int64_t*)calloc((size_t)nb + 1, sizeof(int64_t));
  int64_t* ids = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    int64_t b = (int64_t)(z[i] / lz * (double)nb);
    if (b < 0) b = 0;
    else if (b >= nb) b = nb - 1;
    ids[i] = b;
    counts[b + 1] += 1;
  }
  for (int64_t b = 0; b < nb; ++b) counts[b + 1] += counts[b];
  int64_t* fill = (int64_t*)malloc((size_t)nb * sizeof(int64_t));
  memcpy(fill, counts, (size_t)nb * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) perm[fill[ids[i]]++] = i;
  for (int64_t b = 0; b < nb; ++b) {
    int64_t lo = counts[b], hi = counts[b + 1];
    for (int64_t i = lo + 1; i < hi; ++i) {
      int64_t pi = perm[i];
      double zi = z[pi];
      int64_t j = i - 1;
      while (j >= lo && z[perm[j]] > zi) { perm[j + 1] = perm[j]; --j; }
      perm[j + 1] = pi;
    }
  }
  free(counts); free(ids); free(fill);
}

/* soewald2d.py:76-82  _decay_table: d[a*m + l] = exp(-b_l (z_a - z_{a-1})), row 0 = 1 */
void oracle_decay_table(const double* z, int64_t n, const double* b_re, const double* b_im,
                        int m, double* d_re, double* d_im) {
  for (int64_t a = 0; a < n; ++a)
    for (int l = 0; l < m; ++l) {
      if (a == 0) { d_re[l] = 1.0; d_im[l] = 0.0; continue; }
      double dz = z[a] - z[a - 1];
      cplx e = cexp_(cx(-(dz * b_re[l]), -(dz * b_im[l])));
      d_re[a * m + l] = e.re;
      d_im[a * m + l] = e.im;
    }
}

/* ---------------------------------------------------------------------------
 * soewald2d.py:85-208  _fourier_soe_sweep (modes [t0, t1)); forces (n,3) row-major,
 * accumulated (+=) exactly as the reference.  Returns the Kahan-summed energy.
 * ------------------------------------------------------------------------- */
static double fourier_range(const double* x, const double* y, const double* z, const double* q,
                            int64_t n, const double* kxv, const double* kyv, const double* kv,
                            const double* commonv, int64_t t0, int64_t t1, const double* w_re,
                            const double* w_im, const double* b_re, const double* b_im, int m,
                            double area, const double* d_re, const double* d_im,
                            int want_forces, double* forces) {
  const double pref = M_PI / area;
  cplx* Gl = (cplx*)malloc(sizeof(cplx) * (size_t)m);
  cplx* c = (cplx*)malloc(sizeof(cplx) * (size_t)m);
  double* cost = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double* sint = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double* decay_k = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  double u_total = 0.0, comp = 0.0, k_prev = -1.0;
  for (int64_t t = t0; t < t1; ++t) {
    const double k = kv[t];
    int any_flag = 0;
    cplx wsing = cx(0, 0), kappa_c = cx(0, 0);
    for (int l = 0; l < m; ++l) {
      cplx bl = cx(b_re[l], b_im[l]);
      if (cabs_(cx(bl.re - k, bl.im)) < SINGULAR_TOL * k) {
        c[l] = cx(0, 0);
        wsing = cadd(wsing, cx(w_re[l], w_im[l]));
        any_flag = 1;
      } else {
        cplx den = cx(bl.re * bl.re - bl.im * bl.im - k * k, bl.re * bl.im + bl.im * bl.re);
        c[l] = cdiv(cx(w_re[l], w_im[l]), den);
        kappa_c = cadd(kappa_c, cmul(cscale(2.0, c[l]), bl));
      }
    }
    const double ck = pref * commonv[t] / k;
    const double cz = pref * commonv[t];
    if (k != k_prev) {
      decay_k[0] = 1.0;
      for (int64_t a = 1; a < n; ++a) decay_k[a] = exp(-k * (z[a] - z[a - 1]));
      k_prev = k;
    }
    for (int64_t a = 0; a < n; ++a) {
      double th = kxv[t] * x[a] + kyv[t] * y[a];
      cost[a] = cos(th);
      sint[a] = sin(th);
    }
    /* forward sweep */
    for (int l = 0; l < m; ++l) Gl[l] = cx(0, 0);
    cplx gk = cx(0, 0), bk = cx(0, 0);
    double u_mode = 0.0;
    for (int64_t a = 0; a < n; ++a) {
      if (a > 0) {
        cplx push = cx(q[a - 1] * cost[a - 1], q[a - 1] * -sint[a - 1]);
        cplx tmp = cadd(gk, push);
        gk = cscale(decay_k[a], tmp);
        if (any_flag) bk = cscale(decay_k[a], cadd(bk, cscale(z[a] - z[a - 1], tmp)));
        for (int l = 0; l < m; ++l)
          Gl[l] = cmul(cadd(Gl[l], push), cx(d_re[a * m + l], d_im[a * m + l]));
      }
      cplx sg = cx(0, 0), sgb = cx(0, 0);
      for (int l = 0; l < m; ++l) {
        sg = cadd(sg, cmul(c[l], Gl[l]));
        sgb = cadd(sgb, cmul(cmul(c[l], cx(b_re[l], b_im[l])), Gl[l]));
      }
      cplx p = cadd(cmul(kappa_c, gk), cscale(-2.0 * k, sg));
      if (any_flag) p = cadd(p, cmul(wsing, cadd(cscale(1.0 / k, gk), bk)));
      cplx ph = cx(cost[a], sint[a]);
      cplx epa = cmul(ph, p);
      u_mode += q[a] * epa.re;
      if (want_forces == 1) {
        forces[a * 3 + 0] += ck * q[a] * kxv[t] * epa.im;
        forces[a * 3 + 1] += ck * q[a] * kyv[t] * epa.im;
        cplx zt = cadd(cscale(2.0, sgb), cscale(-1.0, cmul(kappa_c, gk)));
        if (any_flag) zt = cadd(zt, cscale(-1.0, cmul(wsing, bk)));
        forces[a * 3 + 2] -= cz * q[a] * cmul(ph, zt).re;
      }
    }
    if (want_forces == 1) {
      for (int l = 0; l < m; ++l) Gl[l] = cx(0, 0);
      gk = cx(0, 0);
      bk = cx(0, 0);
      for (int64_t a = n - 1; a >= 0; --a) {
        if (a < n - 1) {
          cplx push = cx(q[a + 1] * cost[a + 1], q[a + 1] * sint[a + 1]);
          cplx tmp = cadd(gk, push);
          gk = cscale(decay_k[a + 1], tmp);
          if (any_flag) bk = cscale(decay_k[a + 1], cadd(bk, cscale(z[a + 1] - z[a], tmp)));
          for (int l = 0; l < m; ++l)
            Gl[l] = cmul(cadd(Gl[l], push), cx(d_re[(a + 1) * m + l], d_im[(a + 1) * m + l]));
        }
        cplx sg = cx(0, 0), sgb = cx(0, 0);
        for (int l = 0; l < m; ++l) {
          sg = cadd(sg, cmul(c[l], Gl[l]));
          sgb = cadd(sgb, cmul(cmul(c[l], cx(b_re[l], b_im[l])), Gl[l]));
        }
        cplx p = cadd(cmul(kappa_c, gk), cscale(-2.0 * k, sg));
        if (any_flag) p = cadd(p, cmul(wsing, cadd(cscale(1.0 / k, gk), bk)));
        cplx ph = cx(cost[a], -sint[a]);
        cplx epa = cmul(ph, p);
        forces[a * 3 + 0] -= ck * q[a] * kxv[t] * epa.im;
        forces[a * 3 + 1] -= ck * q[a] * kyv[t] * epa.im;
        cplx zt = cadd(cscale(2.0, sgb), cscale(-1.0, cmul(kappa_c, gk)));
        if (any_flag) zt = cadd(zt, cscale(-1.0, cmul(wsing, bk)));
        forces[a * 3 + 2] += cz * q[a] * cmul(ph, zt).re;
      }
    }
    double y_k = ck * u_mode - comp;
    double t_k = u_total + y_k;
    comp = (t_k - u_total) - y_k;
    u_total = t_k;
  }
  free(Gl); free(c); free(cost); free(sint); free(decay_k);
  return u_total;
}

double oracle_fourier_sweep(const double* x, const double* y, const double* z, const double* q,
                            int64_t n, const double* kxv, const double* kyv, const double* kv,
                            const double* commonv, int64_t nmode, const double* w_re,
                            const double* w_im, const double* b_re, const double* b_im, int m,
                            double area, const double* d_re, const double* d_im,
                            int want_forces, double* forces) {
  return fourier_range(x, y, z, q, n, kxv, kyv, kv, commonv, 0, nmode, w_re, w_im, b_re, b_im, m,
                       area, d_re, d_im, want_forces, forces);
}

/* Same sweep split over modes across OpenMP threads (CPU baseline only).  Per-mode
 * energies are still combined in mode order with the Kahan recurrence. */
double oracle_fourier_sweep_mt(const double* x, const double* y, const double* z, const double* q,
                               int64_t n, const double* kxv, const double* kyv, const double* kv,
                               const double* commonv, int64_t nmode, const double* w_re,
                               const double* w_im, const double* b_re, const double* b_im, int m,
                               double area, const double* d_re, const double* d_im,
                               int want_forces, double* forces, int nthreads) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
  nthreads = 1;
#endif
  if (nthreads > nmode) nthreads = (int)(nmode > 0 ? nmode : 1);
  double* e = (double*)calloc((size_t)(nmode ? nmode : 1), sizeof(double));
  double** fbuf = (double**)calloc((size_t)nthreads, sizeof(double*));
#pragma omp parallel num_threads(nthreads)
  {
#ifdef _OPENMP
    int tid = omp_get_thread_num();
#else
    int tid = 0;
#endif
    fbuf[tid] = (double*)calloc((size_t)(3 * n + 1), sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t t = 0; t < nmode; ++t) {
      /* one mode at a time; energy of a single mode needs no Kahan state */
      e[t] = fourier_range(x, y, z, q, n, kxv, kyv, kv, commonv, t, t + 1, w_re, w_im, b_re,
                           b_im, m, area, d_re, d_im, want_forces, fbuf[tid]);
    }
  }
  if (want_forces == 1)
    for (int th = 0; th < nthreads; ++th)
      for (int64_t i = 0; i < 3 * n; ++i) forces[i] += fbuf[th][i];
  double u_total = 0.0, comp = 0.0;
  for (int64_t t = 0; t < nmode; ++t) {
    double y_k = e[t] - comp;
    double t_k = u_total + y_k;
    comp = (t_k - u_total) - y_k;
    u_total = t_k;
  }
  for (int th = 0; th < nthreads; ++th) free(fbuf[th]);
  free(fbuf); free(e);
  return u_total;
}

/* ---------------------------------------------------------------------------
 * soewald2d.py:211-296  _zero_mode_soe_sweep.  fz accumulated (+=).  Returns u_pair.
 * ------------------------------------------------------------------------- */
double oracle_zero_mode_sweep(const double* z, const double* q, int64_t n, const double* w_re,
                              const double* w_im, const double* s_re, const double* s_im,
                              const double* b_re, const double* b_im, int m, double alpha,
                              double area, const double* d_re, const double* d_im,
                              int want_forces, double* fz) {
  (void)area;
  const double TWO_OVER_SQRT_PI = 2.0 / SQRT_PI;
  cplx* Al = (cplx*)calloc((size_t)m, sizeof(cplx));
  cplx* Bl = (cplx*)calloc((size_t)m, sizeof(cplx));
  cplx* wos = (cplx*)malloc(sizeof(cplx) * (size_t)m);   /* w_l / s_l */
  cplx* fcoef = (cplx*)malloc(sizeof(cplx) * (size_t)m); /* w/s + 0.5 w s */
  for (int l = 0; l < m; ++l) {
    cplx w = cx(w_re[l], w_im[l]), s = cx(s_re[l], s_im[l]);
    wos[l] = cdiv(w, s);
    fcoef[l] = cadd(wos[l], cmul(cscale(0.5, w), s));
  }
  double csum = 0.0, szsum = 0.0, t0 = 0.0, t1 = 0.0, t2 = 0.0, comp0 = 0.0;
  for (int64_t a = 0; a < n; ++a) {
    if (a > 0) {
      double dz = z[a] - z[a - 1];
      double push = q[a - 1];
      csum += push;
      szsum += push * z[a - 1];
      for (int l = 0; l < m; ++l) {
        cplx d = cx(d_re[a * m + l], d_im[a * m + l]);
        cplx tmp = cx(Al[l].re + push, Al[l].im);
        Bl[l] = cmul(cadd(Bl[l], cscale(dz, tmp)), d);
        Al[l] = cmul(tmp, d);
      }
    }
    double term0 = q[a] * (z[a] * csum - szsum);
    double yv = term0 - comp0;
    double tt = t0 + yv;
    comp0 = (tt - t0) - yv;
    t0 = tt;
    cplx sw_b = cx(0, 0), sw_a = cx(0, 0);
    for (int l = 0; l < m; ++l) {
      sw_b = cadd(sw_b, cmul(wos[l], Bl[l]));
      sw_a = cadd(sw_a, cmul(cx(w_re[l], w_im[l]), Al[l]));
    }
    t1 += q[a] * sw_b.re;
    t2 += q[a] * sw_a.re;
  }
  double u_pair = t0 - TWO_OVER_SQRT_PI * t1 + t2 / (alpha * SQRT_PI);
  if (want_forces == 1) {
    for (int l = 0; l < m; ++l) { Al[l] = cx(0, 0); Bl[l] = cx(0, 0); }
    csum = 0.0;
    for (int64_t a = 0; a < n; ++a) {
      if (a > 0) {
        double dz = z[a] - z[a - 1];
        double push = q[a - 1];
        csum += push;
        for (int l = 0; l < m; ++l) {
          cplx d = cx(d_re[a * m + l], d_im[a * m + l]);
          cplx tmp = cx(Al[l].re + push, Al[l].im);
          Bl[l] = cmul(cadd(Bl[l], cscale(dz, tmp)), d);
          Al[l] = cmul(tmp, d);
        }
      }
      cplx sw = cx(0, 0);
      for (int l = 0; l < m; ++l)
        sw = cadd(sw, cadd(cmul(fcoef[l], Al[l]),
                           cscale(-1.0, cmul(cscale(alpha, cx(w_re[l], w_im[l])), Bl[l]))));
      fz[a] += csum - TWO_OVER_SQRT_PI * sw.re;
    }
    for (int l = 0; l < m; ++l) { Al[l] = cx(0, 0); Bl[l] = cx(0, 0); }
    csum = 0.0;
    for (int64_t a = n - 1; a >= 0; --a) {
      if (a < n - 1) {
        double dz = z[a + 1] - z[a];
        double push = q[a + 1];
        csum += push;
        for (int l = 0; l < m; ++l) {
          cplx d = cx(d_re[(a + 1) * m + l], d_im[(a + 1) * m + l]);
          cplx tmp = cx(Al[l].re + push, Al[l].im);
          Bl[l] = cmul(cadd(Bl[l], cscale(dz, tmp)), d);
          Al[l] = cmul(tmp, d);
        }
      }
      cplx sw = cx(0, 0);
      for (int l = 0; l < m; ++l)
        sw = cadd(sw, cadd(cmul(fcoef[l], Al[l]),
                           cscale(-1.0, cmul(cscale(alpha, cx(w_re[l], w_im[l])), Bl[l]))));
      fz[a] -= csum - TWO_OVER_SQRT_PI * sw.re;
    }
  }
  free(Al); free(Bl); free(wos); free(fcoef);
  return u_pair;
}

/* ---------------------------------------------------------------------------
 * ewald2d.py:126-303  short-range erfc sum: cell list (half shell, 13+1 cells)
 * or all pairs when ncx<3 or ncy<3.  Returns energy; *flag = 1 on a coincident
 * pair (d2 < 1e-24).  forces (n,3) accumulated.
 * ------------------------------------------------------------------------- */
static inline void pair_term(const double* pos, const double* charge, int64_t i, int64_t j,
                             double lx, double ly, double alpha, double rc2, double c,
                             double* energy, double* comp, int* flag, double* forces) {
  double dx = pos[i * 3 + 0] - pos[j * 3 + 0];
  double dy = pos[i * 3 + 1] - pos[j * 3 + 1];
  double dz = pos[i * 3 + 2] - pos[j * 3 + 2];
  dx -= lx * nearbyint(dx / lx);
  dy -= ly * nearbyint(dy / ly);
  double d2 = dx * dx + dy * dy + dz * dz;
  if (d2 > rc2) return;
  if (d2 < 1e-24) { *flag = 1; return; }
  double d = sqrt(d2);
  double qq = charge[i] * charge[j];
  double e = erfc(alpha * d);
  double term = qq * e / d;
  double fmag = qq * (e / (d2 * d) + c * exp(-alpha * alpha * d2) / d2);
  double yv = term - *comp;
  double t2 = *energy + yv;
  *comp = (t2 - *energy) - yv;
  *energy = t2;
  forces[i * 3 + 0] += fmag * dx;
  forces[i * 3 + 1] += fmag * dy;
  forces[i * 3 + 2] += fmag * dz;
  forces[j * 3 + 0] -= fmag * dx;
  forces[j * 3 + 1] -= fmag * dy;
  forces[j * 3 + 2] -= fmag * dz;
}

static int64_t build_cells(const double* pos, int64_t n, double lx, double ly, double lz,
                           double rc, int64_t* ncxyz, int64_t** cell_start_out,
                           int64_t** order_out) {
  int64_t ncx = (int64_t)(lx / rc), ncy = (int64_t)(ly / rc), ncz = (int64_t)(lz / rc);
  if (ncx < 1) ncx = 1;
  if (ncy < 1) ncy = 1;
  if (ncz < 1) ncz = 1;
  if (ncx < 3 || ncy < 3) ncx = ncy = ncz = 1;
  int64_t ncell = ncx * ncy * ncz;
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t* start = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    /* ewald2d.py:126-138: int() truncation then python modulo (non-negative) */
    int64_t cxi = (int64_t)(pos[i * 3 + 0] / lx * (double)ncx);
    int64_t cyi = (int64_t)(pos[i * 3 + 1] / ly * (double)ncy);
    cxi = ((cxi % ncx) + ncx) % ncx;
    cyi = ((cyi % ncy) + ncy) % ncy;
    int64_t czi = (int64_t)(pos[i * 3 + 2] / lz * (double)ncz);
    if (czi < 0) czi = 0;
    else if (czi >= ncz) czi = ncz - 1;
    idx[i] = (cxi * ncy + cyi) * ncz + czi;
    start[idx[i] + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)ncell);
  memcpy(fill, start, sizeof(int64_t) * (size_t)ncell);
  for (int64_t i = 0; i < n; ++i) order[fill[idx[i]]++] = i; /* stable argsort of idx */
  free(fill); free(idx);
  ncxyz[0] = ncx; ncxyz[1] = ncy; ncxyz[2] = ncz;
  *cell_start_out = start;
  *order_out = order;
  return ncell;
}

static double cells_range(const double* pos, const double* charge, double lx, double ly,
                          double alpha, double rc, const int64_t* nc, const int64_t* start,
                          const int64_t* order, int64_t cx0, int64_t cx1, int* flag,
                          double* forces) {
  const double rc2 = rc * rc, c = 2.0 / SQRT_PI * alpha;
  double energy = 0.0, comp = 0.0;
  int64_t ncx = nc[0], ncy = nc[1], ncz = nc[2];
  for (int64_t cxi = cx0; cxi < cx1; ++cxi)
    for (int64_t cyi = 0; cyi < ncy; ++cyi)
      for (int64_t czi = 0; czi < ncz; ++czi) {
        int64_t cid = (cxi * ncy + cyi) * ncz + czi;
        int64_t a0 = start[cid], a1 = start[cid + 1];
        for (int off = 0; off < 27; ++off) {
          int dxc = off / 9 - 1, dyc = (off / 3) % 3 - 1, dzc = off % 3 - 1;
          if (dxc < 0 || (dxc == 0 && (dyc < 0 || (dyc == 0 && dzc < 0)))) continue;
          int64_t nz = czi + dzc;
          if (nz < 0 || nz >= ncz) continue;
          int64_t nx = ((cxi + dxc) % ncx + ncx) % ncx;
          int64_t ny = ((cyi + dyc) % ncy + ncy) % ncy;
          int64_t nid = (nx * ncy + ny) * ncz + nz;
          int64_t b0 = start[nid], b1 = start[nid + 1];
          int same = nid == cid;
          for (int64_t ii = a0; ii < a1; ++ii) {
            int64_t i = order[ii];
            for (int64_t jj = same ? ii + 1 : b0; jj < b1; ++jj)
              pair_term(pos, charge, i, order[jj], lx, ly, alpha, rc2, c, &energy, &comp, flag,
                        forces);
          }
        }
      }
  return energy;
}

double oracle_short_range(const double* pos, const double* charge, int64_t n, double lx,
                          double ly, double lz, double alpha, double rc, double* forces,
                          int* flag, int nthreads) {
  *flag = 0;
  if (n < 2) return 0.0;
  int64_t nc[3];
  int64_t *start, *order;
  build_cells(pos, n, lx, ly, lz, rc, nc, &start, &order);
  double energy = 0.0;
  if (nc[0] == 1) {
    /* ewald2d.py:234-277 all pairs */
    const double rc2 = rc * rc, c = 2.0 / SQRT_PI * alpha;
    double comp = 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = i + 1; j < n; ++j)
        pair_term(pos, charge, i, j, lx, ly, alpha, rc2, c, &energy, &comp, flag, forces);
  } else if (nthreads == 1) {
    energy = cells_range(pos, charge, lx, ly, alpha, rc, nc, start, order, 0, nc[0], flag,
                         forces);
  } else {
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#else
    nthreads = 1;
#endif
    /* slabs of x-cells, fixed assignment, reduced in slab order */
    int64_t nslab = nc[0];
    double* e = (double*)calloc((size_t)nslab, sizeof(double));
    int* fl = (int*)calloc((size_t)nslab, sizeof(int));
    double** fb = (double**)calloc((size_t)nthreads, sizeof(double*));
#pragma omp parallel num_threads(nthreads)
    {
#ifdef _OPENMP
      int tid = omp_get_thread_num();
#else
      int tid = 0;
#endif
      fb[tid] = (double*)calloc((size_t)(3 * n), sizeof(double));
#pragma omp for schedule(dynamic, 1)
      for (int64_t s = 0; s < nslab; ++s)
        e[s] = cells_range(pos, charge, lx, ly, alpha, rc, nc, start, order, s, s + 1, &fl[s],
                           fb[tid]);
    }
    for (int th = 0; th < nthreads; ++th) {
      for (int64_t i = 0; i < 3 * n; ++i) forces[i] += fb[th][i];
      free(fb[th]);
    }
    for (int64_t s = 0; s < nslab; ++s) { energy += e[s]; *flag |= fl[s]; }
    free(fb); free(e); free(fl);
  }
  free(start); free(order);
  return energy;
}

/* ---------------------------------------------------------------------------
 * rbse2d.py:274-317 / soewald2d.py:398-438 assembly (sorted view, sweeps,
 * scatter to input order).  The caller supplies the k-set, commonv (per mode),
 * the deterministic charge constant (c_q or u_q) and the SOE.  out_e[5] =
 * {u_s, u_l_k, u_l_0, u_self, u_ps}; forces (n,3) zero-initialised by caller.
 * Returns 0, or 1 on coincident particles.
 * ------------------------------------------------------------------------- */
int oracle_energy_forces(const double* pos, const double* charge, int64_t n, double lx,
                         double ly, double lz, double sigma_top, double sigma_bot, double alpha,
                         double rc, const double* kx, const double* ky, const double* kv,
                         const double* commonv, int64_t nmode, double charge_const,
                         const double* w_re, const double* w_im, const double* s_re,
                         const double* s_im, int m, int nthreads, double* out_e,
                         double* forces) {
  if (n < 0) return 2;
  const double area = lx * ly;
  int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  double* zin = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) zin[i] = pos[i * 3 + 2];
  oracle_sort_perm(zin, n, lz, perm);
  double* xs = (double*)malloc(sizeof(double) * (size_t)(4 * (n ? n : 1)));
  double *ys = xs + n, *zs = xs + 2 * n, *qs = xs + 3 * n;
  for (int64_t a = 0; a < n; ++a) {
    int64_t i = perm[a];
    xs[a] = pos[i * 3 + 0]; ys[a] = pos[i * 3 + 1]; zs[a] = pos[i * 3 + 2]; qs[a] = charge[i];
  }
  int flag = 0;
  double* fs = (double*)calloc((size_t)(3 * n + 1), sizeof(double));
  double u_s = oracle_short_range(pos, charge, n, lx, ly, lz, alpha, rc, fs, &flag, nthreads);
  double u_ps = 0.0, Q = 0.0, qsum2 = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double phi = -2.0 * M_PI * (sigma_top * (lz - pos[i * 3 + 2]) + sigma_bot * pos[i * 3 + 2]);
    u_ps += charge[i] * phi;
    qsum2 += charge[i] * charge[i];
  }
  for (int64_t a = 0; a < n; ++a) Q += qs[a] * qs[a];
  double u_self = alpha / SQRT_PI * qsum2;
  double u_0 = n ? -SQRT_PI * Q / (alpha * area) : 0.0;
  double u_k = charge_const;
  double* fsorted = (double*)calloc((size_t)(3 * n + 1), sizeof(double));
  if (n >= 2) {
    double* b_re = (double*)malloc(sizeof(double) * (size_t)m);
    double* b_im = (double*)malloc(sizeof(double) * (size_t)m);
    for (int l = 0; l < m; ++l) { b_re[l] = alpha * s_re[l]; b_im[l] = alpha * s_im[l]; }
    double* d_re = (double*)malloc(sizeof(double) * (size_t)(n * m));
    double* d_im = (double*)malloc(sizeof(double) * (size_t)(n * m));
    oracle_decay_table(zs, n, b_re, b_im, m, d_re, d_im);
    if (nmode > 0)
      u_k += (nthreads == 1)
                 ? oracle_fourier_sweep(xs, ys, zs, qs, n, kx, ky, kv, commonv, nmode, w_re,
                                        w_im, b_re, b_im, m, area, d_re, d_im, 1, fsorted)
                 : oracle_fourier_sweep_mt(xs, ys, zs, qs, n, kx, ky, kv, commonv, nmode, w_re,
                                           w_im, b_re, b_im, m, area, d_re, d_im, 1, fsorted,
                                           nthreads);
    double* fz = (double*)calloc((size_t)n, sizeof(double));
    u_0 += -2.0 * M_PI / area *
           oracle_zero_mode_sweep(zs, qs, n, w_re, w_im, s_re, s_im, b_re, b_im, m, alpha, area,
                                  d_re, d_im, 1, fz);
    for (int64_t a = 0; a < n; ++a) fsorted[a * 3 + 2] += 2.0 * M_PI / area * qs[a] * fz[a];
    free(fz); free(d_re); free(d_im); free(b_re); free(b_im);
  }
  for (int64_t a = 0; a < n; ++a) {
    int64_t i = perm[a];
    forces[i * 3 + 0] = fs[i * 3 + 0] + fsorted[a * 3 + 0];
    forces[i * 3 + 1] = fs[i * 3 + 1] + fsorted[a * 3 + 1];
    forces[i * 3 + 2] = fs[i * 3 + 2] + fsorted[a * 3 + 2] + (-2.0 * M_PI * charge[i]) * (sigma_top - sigma_bot);
  }
  out_e[0] = u_s; out_e[1] = u_k; out_e[2] = u_0; out_e[3] = u_self; out_e[4] = u_ps;
  free(perm); free(zin); free(xs); free(fs); free(fsorted);
  return flag;
}

/* ---------------------------------------------------------------------------
 * Multi-GPU shard check (tests only): the short-range share of one rank as the
 * device path computes it -- full-shell forces and half the pair energy for the
 * home particles [h0, h1) of the stable cell order (ewald2d.py:141-157 cells).
 * Summing over ranks reproduces oracle_short_range.
 * ------------------------------------------------------------------------- */
double oracle_short_range_home(const double* pos, const double* charge, int64_t n, double lx,
                               double ly, double lz, double alpha, double rc, int64_t h0,
                               int64_t h1, double* forces, int* flag) {
  *flag = 0;
  if (n < 2) return 0.0;
  int64_t nc[3];
  int64_t *start, *order;
  build_cells(pos, n, lx, ly, lz, rc, nc, &start, &order);
  const double rc2 = rc * rc, c = 2.0 / SQRT_PI * alpha;
  double energy = 0.0, comp = 0.0;
  double* tmp = (double*)calloc((size_t)(3 * n), sizeof(double));
  for (int64_t hh = h0; hh < h1; ++hh) {
    /* the brute path (one cell) uses input order for the home split */
    int64_t i = nc[0] == 1 ? hh : order[hh];
    double e_i = 0.0, c_i = 0.0;
    double fi[3] = {0, 0, 0};
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      double ej = 0.0, cj = 0.0;
      memset(tmp + 3 * i, 0, 3 * sizeof(double));
      memset(tmp + 3 * j, 0, 3 * sizeof(double));
      pair_term(pos, charge, i, j, lx, ly, alpha, rc2, c, &ej, &cj, flag, tmp);
      e_i += ej;
      fi[0] += tmp[3 * i]; fi[1] += tmp[3 * i + 1]; fi[2] += tmp[3 * i + 2];
    }
    forces[3 * i] += fi[0]; forces[3 * i + 1] += fi[1]; forces[3 * i + 2] += fi[2];
    double yv = 0.5 * e_i - comp;
    double t2 = energy + yv;
    comp = (t2 - energy) - yv;
    energy = t2;
    (void)c_i;
  }
  free(tmp); free(start); free(order);
  return energy;
}
