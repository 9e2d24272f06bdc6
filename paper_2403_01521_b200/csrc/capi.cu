// capi.cu -- extern "C" boundary (include/slabewald_b200.h): context, workspace
// arena, argument checks, and the evaluation pipeline that strings the kernels
// together in the order of rbse2d.py:283-317 / soewald2d.py:401-438.
#include <complex>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/slabewald_b200.h"
#include "common.cuh"
#include "kernels.cuh"

using cd = std::complex<double>;

static thread_local std::string g_err;

int slab_record_cuda(cudaError_t e) {
  g_err = std::string("CUDA error: ") + cudaGetErrorString(e);
  return SLAB_ERR_CUDA;
}
static int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}
#define CK(expr)                                   \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return slab_record_cuda(_e); \
  } while (0)

struct SlabCtx {
  void* arena = nullptr;
  size_t arena_bytes = 0;
  double* small = nullptr;  // scalars: [0]=u_s [1]=u_sweep [2]=u_pair ...
  int* status = nullptr;
  double* sampler_scratch = nullptr;
  int64_t sampler_cap = 0;
  int kcap_min = 0;        // learned short-range neighbour-row capacity (grow-only)
  int* d_maxnn = nullptr;  // longest neighbour row of the last short-range run
  double* md_part = nullptr;  // block partials of the O(N) MD reductions
  int64_t md_part_cap = 0;
  int32_t* zs_perm = nullptr;  // z-split: the sort permutation between phase 1 and phase 2
  // slab_evaluate_host: device copies of the host buffers, an upload stream and
  // its events (created on first use)
  double* h_dpos = nullptr;
  double* h_dq = nullptr;
  double* h_dforces = nullptr;
  double* h_denergy = nullptr;
  int64_t h_cap = -1;
  cudaStream_t up_stream = nullptr;
  cudaEvent_t ev_pos = nullptr, ev_q = nullptr;
  // evaluation fork: the Fourier / k = 0 chain on a high-priority stream, the
  // short range on a low-priority one (its CTAs fill the SMs the scan's small
  // and tail kernels leave idle); joined back into the caller's stream
  cudaStream_t hi = nullptr, lo = nullptr, aux = nullptr;  // aux: the k = 0 chain
  cudaEvent_t ev_fork = nullptr, ev_short = nullptr, ev_long = nullptr, ev_x = nullptr;
  cudaEvent_t ev_dtab = nullptr, ev_zero = nullptr;
};

namespace {

struct Carver {
  char* p;
  template <typename T>
  T* take(size_t count) {
    uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 255) & ~(uintptr_t)255;
    T* r = reinterpret_cast<T*>(a);
    p = reinterpret_cast<char*>(a + sizeof(T) * (count ? count : 1));
    return r;
  }
};

size_t pad(size_t b) { return ((b ? b : 1) + 255) & ~(size_t)255; }

int ensure_arena(SlabCtx* c, size_t bytes) {
  if (c->small == nullptr) {
    CK(cudaMalloc(&c->small, 1024 * sizeof(double)));
    CK(cudaMalloc(&c->status, 16 * sizeof(int)));
    CK(cudaMalloc(&c->d_maxnn, sizeof(int)));
    CK(cudaMemset(c->d_maxnn, 0, sizeof(int)));
  }
  if (bytes <= c->arena_bytes) return SLAB_OK;
  if (c->arena) {
    CK(cudaDeviceSynchronize());
    CK(cudaFree(c->arena));
    c->arena = nullptr;
    c->arena_bytes = 0;
  }
  size_t want = bytes + bytes / 8;
  if (cudaMalloc(&c->arena, want) != cudaSuccess) {
    cudaGetLastError();
    return fail(SLAB_ERR_NOMEM, "device workspace allocation failed");
  }
  c->arena_bytes = want;
  return SLAB_OK;
}

struct SOEHost {
  int m = 0, mh = 0;
  int real_terms = 0;  // self-conjugate terms carried as pairs (mh = (m + real_terms) / 2)
  slab::BVec b{};
  slab::WVec w{};
  slab::ZCoef z{};
  // lone complex terms (no conjugate partner): the swapped second pass, pairs
  // (s_l, i w_l / 2) evaluated with inputs (u_i, -u_r) -- see prepare_soe
  int mh2 = 0;
  slab::BVec b2{};
  slab::WVec w2{};
};

// The kernels run over conjugate PAIRS (s, w), (conj s, conj w): per pair two
// complex recurrences with real inputs carry both terms.  A table is accepted
// when every term is either real (s and w real: carried as the pair
// (s, w/2), (s, w/2) -- halving is exact, so c G + c G = (w / (b^2 - k^2)) G)
// or has its conjugate elsewhere in the table (bitwise).  Built contours are
// conjugate-symmetric in mirrored order; m = 1 real-exponent tables are what
// soe.py's removable-singularity tests use.
int prepare_soe(const SlabSOE& soe, double alpha, SOEHost& out) {
  if (soe.m < 1 || soe.m > 24) return fail(SLAB_ERR_ARG, "SOE term count must be in [1, 24]");
  if (!soe.h_w_re || !soe.h_w_im || !soe.h_s_re || !soe.h_s_im)
    return fail(SLAB_ERR_ARG, "SOE arrays must be given");
  const int m = soe.m;
  for (int l = 0; l < m; ++l)
    if (!(soe.h_s_re[l] > 0)) return fail(SLAB_ERR_ARG, "every exponent must have positive real part");
  bool used[24] = {false};
  cd ps[24], pw[24];
  int mh = 0;
  out.real_terms = 0;
  out.mh2 = 0;
  for (int l = 0; l < m; ++l) {
    if (used[l]) continue;
    used[l] = true;
    if (soe.h_s_im[l] == 0.0 && soe.h_w_im[l] == 0.0) {  // self-conjugate: half weight twice
      ps[mh] = cd(soe.h_s_re[l], 0.0);
      pw[mh] = cd(0.5 * soe.h_w_re[l], 0.0);
      ++mh;
      ++out.real_terms;
      continue;
    }
    int r = -1;
    for (int j = m - 1; j > l; --j)  // mirrored order first (built contours)
      if (!used[j] && soe.h_s_re[j] == soe.h_s_re[l] && soe.h_s_im[j] == -soe.h_s_im[l] &&
          soe.h_w_re[j] == soe.h_w_re[l] && soe.h_w_im[j] == -soe.h_w_im[l]) {
        r = j;
        break;
      }
    if (r < 0) {
      // A lone complex term F(s, w) (soewald2d.py:85-208 accepts any table).  With
      // G(s, w) = F(s, w) + F(conj s, conj w) -- one pair of the main pass --
      // F(s, w) = 1/2 G(s, w) - (i/2) G(s, i w): the pair (s, w/2) joins the main
      // pass, and the pair (s, i w/2) a second pass whose real inputs are swapped
      // (u_r, u_i) -> (u_i, -u_r), which multiplies that pass's p, zeta and g chain
      // by -i (FourierPlan::swap).  The k = 0 mode has real inputs, so there the
      // lone term is exactly the half-weight pair.
      const cd s_l(soe.h_s_re[l], soe.h_s_im[l]), w_l(soe.h_w_re[l], soe.h_w_im[l]);
      if (std::abs(s_l.imag()) < 1e-5 * s_l.real())
        return fail(SLAB_ERR_UNSUPPORTED,
                    "a lone complex SOE term with a near-real exponent is not supported");
      if (out.mh2 >= 12) return fail(SLAB_ERR_UNSUPPORTED, "more than 12 lone complex SOE terms");
      ps[mh] = s_l;
      pw[mh] = 0.5 * w_l;
      ++mh;
      const cd w2 = cd(0.0, 0.5) * w_l;
      out.b2.re[out.mh2] = alpha * s_l.real();
      out.b2.im[out.mh2] = alpha * s_l.imag();
      out.w2.re[out.mh2] = w2.real();
      out.w2.im[out.mh2] = w2.imag();
      ++out.mh2;
      continue;
    }
    used[r] = true;
    ps[mh] = cd(soe.h_s_re[l], soe.h_s_im[l]);
    pw[mh] = cd(soe.h_w_re[l], soe.h_w_im[l]);
    ++mh;
  }
  if (mh > 12) return fail(SLAB_ERR_UNSUPPORTED, "more than 12 SOE pairs");
  out.m = m;
  out.mh = mh;
  for (int l = 0; l < mh; ++l) {
    const cd s = ps[l], w = pw[l];
    out.b.re[l] = alpha * s.real();
    out.b.im[l] = alpha * s.imag();
    out.w.re[l] = w.real();
    out.w.im[l] = w.imag();
    const cd ws = w / s;
    const cd ws2 = 2.0 * ws, w2 = 2.0 * w, f2 = 2.0 * (ws + 0.5 * w * s), aw2 = 2.0 * alpha * w;
    out.z.ws2[2 * l] = ws2.real();
    out.z.ws2[2 * l + 1] = ws2.imag();
    out.z.w2[2 * l] = w2.real();
    out.z.w2[2 * l + 1] = w2.imag();
    out.z.f2[2 * l] = f2.real();
    out.z.f2[2 * l + 1] = f2.imag();
    out.z.aw2[2 * l] = aw2.real();
    out.z.aw2[2 * l + 1] = aw2.imag();
  }
  return SLAB_OK;
}

// plan of the lone-term pass (prepare_soe): same modes, mh2 swapped pairs
slab::FourierPlan lone_plan(const SOEHost& sh, int64_t n, int nmode, int dirs) {
  auto p = slab::fourier_plan(n, nmode, sh.mh2 > 0 ? sh.mh2 : 1, dirs);
  p.swap = 1;
  return p;
}

// workspace for the z-sorted part of an evaluation
struct SortedWork {
  slab::SortWork sw;
  double *xs, *ys, *zs, *qs;
  double2* dtab;
  double2* dtab2;  // decay table of the lone-term pass (mh2 columns)
  double* elone;   // energies of the lone-term pass (one per batch / one)
  double* fwork;
  double* zwork;
  double *fsorted, *fzf, *fzb;
};

size_t sorted_bytes(int64_t n, int mh, const slab::FourierPlan& fp, const slab::ZeroPlan& zp,
                    bool with_sort, int mh2 = 0, const slab::FourierPlan* fp2 = nullptr) {
  const size_t N = (size_t)(n > 0 ? n : 1);
  size_t b = 0;
  if (with_sort) {
    b += 2 * pad(8 * N) + 2 * pad(4 * N) + pad(4 * (size_t)slab::radix_hist_entries(n));
    b += 4 * pad(8 * N);
  }
  b += pad(sizeof(double2) * (N + 1) * mh);
  b += pad(sizeof(double2) * (N + 1) * (size_t)mh2) + pad(8 * 4096);
  size_t fw = slab::fourier_work_doubles(fp);
  if (fp2 && slab::fourier_work_doubles(*fp2) > fw) fw = slab::fourier_work_doubles(*fp2);
  b += pad(8 * fw);
  b += pad(8 * slab::zero_work_doubles(zp));
  b += pad(24 * N) + 2 * pad(8 * N);
  return b;
}

void carve_sorted(Carver& cv, int64_t n, int mh, const slab::FourierPlan& fp,
                  const slab::ZeroPlan& zp, bool with_sort, SortedWork& w, int mh2 = 0,
                  const slab::FourierPlan* fp2 = nullptr) {
  const size_t N = (size_t)(n > 0 ? n : 1);
  if (with_sort) {
    w.sw.k0 = cv.take<uint64_t>(N);
    w.sw.k1 = cv.take<uint64_t>(N);
    w.sw.v0 = cv.take<int32_t>(N);
    w.sw.v1 = cv.take<int32_t>(N);
    w.sw.hist = cv.take<int32_t>(slab::radix_hist_entries(n));
    w.xs = cv.take<double>(N);
    w.ys = cv.take<double>(N);
    w.zs = cv.take<double>(N);
    w.qs = cv.take<double>(N);
  }
  w.dtab = cv.take<double2>((N + 1) * mh);
  w.dtab2 = cv.take<double2>((N + 1) * (size_t)mh2);
  w.elone = cv.take<double>(4096);
  size_t fwd = slab::fourier_work_doubles(fp);
  if (fp2 && slab::fourier_work_doubles(*fp2) > fwd) fwd = slab::fourier_work_doubles(*fp2);
  w.fwork = cv.take<double>(fwd);
  w.zwork = cv.take<double>(slab::zero_work_doubles(zp));
  w.fsorted = cv.take<double>(3 * N);
  w.fzf = cv.take<double>(N);
  w.fzb = cv.take<double>(N);
}

}  // namespace

extern "C" {

const char* slab_last_error(void) { return g_err.c_str(); }
const char* slab_version(void) { return "slabewald_b200 0.1 (sm_100a)"; }

int slab_ctx_create(SlabCtx** out) {
  if (!out) return fail(SLAB_ERR_ARG, "null output pointer");
  *out = new SlabCtx();
  return SLAB_OK;
}

int slab_ctx_destroy(SlabCtx* ctx) {
  if (!ctx) return SLAB_OK;
  cudaDeviceSynchronize();
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->small) cudaFree(ctx->small);
  if (ctx->status) cudaFree(ctx->status);
  if (ctx->sampler_scratch) cudaFree(ctx->sampler_scratch);
  if (ctx->d_maxnn) cudaFree(ctx->d_maxnn);
  if (ctx->md_part) cudaFree(ctx->md_part);
  if (ctx->h_dpos) cudaFree(ctx->h_dpos);
  if (ctx->h_dq) cudaFree(ctx->h_dq);
  if (ctx->h_dforces) cudaFree(ctx->h_dforces);
  if (ctx->h_denergy) cudaFree(ctx->h_denergy);
  if (ctx->up_stream) cudaStreamDestroy(ctx->up_stream);
  if (ctx->hi) cudaStreamDestroy(ctx->hi);
  if (ctx->lo) cudaStreamDestroy(ctx->lo);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_short, ctx->ev_long, ctx->ev_x, ctx->ev_dtab,
                        ctx->ev_zero})
    if (e) cudaEventDestroy(e);
  if (ctx->ev_pos) cudaEventDestroy(ctx->ev_pos);
  if (ctx->ev_q) cudaEventDestroy(ctx->ev_q);
  delete ctx;
  return SLAB_OK;
}

int slab_ctx_neighbor_capacity(SlabCtx* ctx, int capacity) {
  if (!ctx || capacity < 0) return fail(SLAB_ERR_ARG, "bad capacity");
  if (capacity > ctx->kcap_min) ctx->kcap_min = (capacity + 7) / 8 * 8;
  return SLAB_OK;
}

int slab_ctx_last_max_neighbors(SlabCtx* ctx, int* out) {
  if (!ctx || !out) return fail(SLAB_ERR_ARG, "bad arguments");
  *out = 0;
  if (ctx->d_maxnn) CK(cudaMemcpy(out, ctx->d_maxnn, sizeof(int), cudaMemcpyDeviceToHost));
  return SLAB_OK;
}

int slab_sort_by_z(SlabCtx* ctx, const double* d_z, int64_t stride, int64_t n, int64_t* d_perm,
                   void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!d_z || !d_perm)) || stride < 1)
    return fail(SLAB_ERR_ARG, "bad sort arguments");
  if (n > INT32_MAX) return fail(SLAB_ERR_ARG, "n exceeds int32 indexing");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t N = (size_t)(n > 0 ? n : 1);
  const size_t bytes = 2 * pad(8 * N) + 2 * pad(4 * N) + pad(4 * (size_t)slab::radix_hist_entries(n)) + 1024;
  int rc = ensure_arena(ctx, bytes);
  if (rc) return rc;
  Carver cv{(char*)ctx->arena};
  slab::SortWork sw;
  sw.k0 = cv.take<uint64_t>(N);
  sw.k1 = cv.take<uint64_t>(N);
  sw.v0 = cv.take<int32_t>(N);
  sw.v1 = cv.take<int32_t>(N);
  sw.hist = cv.take<int32_t>(slab::radix_hist_entries(n));
  int32_t* perm;
  CK(slab::sort_by_z_device(d_z, stride, n, sw, st, &perm));
  CK(slab::perm_to_int64(perm, n, d_perm, st));
  return SLAB_OK;
}

int slab_fourier_sweep(SlabCtx* ctx, const double* d_x, const double* d_y, const double* d_z,
                       const double* d_q, int64_t n, const double* d_modes,
                       const double* d_commonv, double commonv_scalar, int64_t nmode,
                       SlabSOE soe, double alpha, double area, int want_forces,
                       double* d_forces_sorted, double* d_energy, int* d_status, void* stream) {
  if (!ctx || n < 0 || nmode < 0 || !d_energy) return fail(SLAB_ERR_ARG, "bad sweep arguments");
  if (nmode > 100000) return fail(SLAB_ERR_ARG, "too many modes for one sweep");
  SOEHost sh;
  int rc = prepare_soe(soe, alpha, sh);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int dirs = (want_forces && d_forces_sorted) ? 2 : 1;
  auto fp = slab::fourier_plan(n, (int)nmode, sh.mh, dirs);
  auto fp2 = lone_plan(sh, n, (int)nmode, dirs);
  auto zp = slab::zero_plan(n, sh.mh);
  rc = ensure_arena(ctx, sorted_bytes(n, sh.mh, fp, zp, false, sh.mh2, &fp2) + 4096);
  if (rc) return rc;
  Carver cv{(char*)ctx->arena};
  SortedWork w{};
  carve_sorted(cv, n, sh.mh, fp, zp, false, w, sh.mh2, &fp2);
  slab::FourierWork fw;
  slab::fourier_work_carve(fp, w.fwork, fw);
  CK(cudaMemsetAsync(d_energy, 0, sizeof(double), st));
  if (n < 2 || nmode == 0) return SLAB_OK;
  CK(slab::decay_table(d_z, n, sh.mh, sh.b, w.dtab, st));
  int* status = d_status ? d_status : ctx->status;
  if (!d_status) CK(cudaMemsetAsync(ctx->status, 0, sizeof(int), st));
  CK(slab::fourier_run(fp, fw, d_x, d_y, d_z, d_q, w.dtab, d_modes, d_commonv, commonv_scalar,
                       area, sh.b, sh.w, want_forces && d_forces_sorted, d_energy, status,
                       d_forces_sorted, st));
  if (sh.mh2) {  // lone complex terms: the swapped pass, added in
    CK(slab::decay_table(d_z, n, sh.mh2, sh.b2, w.dtab2, st));
    slab::fourier_work_carve(fp2, w.fwork, fw);
    CK(slab::fourier_run(fp2, fw, d_x, d_y, d_z, d_q, w.dtab2, d_modes, d_commonv,
                         commonv_scalar, area, sh.b2, sh.w2, want_forces && d_forces_sorted,
                         w.elone, status, d_forces_sorted, st));
    CK(slab::add_into(d_energy, w.elone, 1, st));
  }
  return SLAB_OK;
}

int slab_zero_mode_sweep(SlabCtx* ctx, const double* d_z, const double* d_q, int64_t n,
                         SlabSOE soe, double alpha, int want_forces, double* d_fz,
                         double* d_energy, void* stream) {
  if (!ctx || n < 0 || !d_energy) return fail(SLAB_ERR_ARG, "bad zero-mode arguments");
  SOEHost sh;
  int rc = prepare_soe(soe, alpha, sh);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  auto fp = slab::fourier_plan(n, 0, sh.mh);
  auto zp = slab::zero_plan(n, sh.mh);
  rc = ensure_arena(ctx, sorted_bytes(n, sh.mh, fp, zp, false) + 4096);
  if (rc) return rc;
  Carver cv{(char*)ctx->arena};
  SortedWork w{};
  carve_sorted(cv, n, sh.mh, fp, zp, false, w);
  if (n < 2) return cudaMemsetAsync(d_energy, 0, sizeof(double), st) == cudaSuccess ? SLAB_OK : SLAB_ERR_CUDA;
  CK(slab::decay_table(d_z, n, sh.mh, sh.b, w.dtab, st));
  CK(slab::zero_run_b(zp, w.zwork, d_z, d_q, w.dtab, sh.z, sh.b, alpha, want_forces && d_fz,
                      w.fzf, w.fzb, d_energy, st));
  if (want_forces && d_fz) CK(slab::fz_accumulate(n, w.fzf, w.fzb, d_fz, st));
  return SLAB_OK;
}

int slab_short_range(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                     SlabBox box, double alpha, double r_c, double* d_forces, double* d_energy,
                     int* d_status, void* stream) {
  if (!ctx || n < 0 || !d_energy || !d_status || (n > 0 && (!d_pos || !d_charge || !d_forces)))
    return fail(SLAB_ERR_ARG, "bad short-range arguments");
  if (!(alpha > 0) || !(r_c > 0)) return fail(SLAB_ERR_ARG, "alpha and r_c must be positive");
  cudaStream_t st = (cudaStream_t)stream;
  auto sp = slab::short_plan(n, box.lx, box.ly, box.lz, r_c);
  if (sp.kcap < ctx->kcap_min) sp.kcap = ctx->kcap_min;
  int rc = ensure_arena(ctx, slab::short_work_bytes(sp) + 1024);
  if (rc) return rc;
  CK(cudaMemsetAsync(ctx->d_maxnn, 0, sizeof(int), st));
  CK(slab::short_run(sp, ctx->arena, d_pos, d_charge, box.lx, box.ly, box.lz, alpha, r_c,
                     d_forces, d_energy, d_status, 0, n, ctx->d_maxnn, st));
  return SLAB_OK;
}

int slab_sample_modes(SlabCtx* ctx, int64_t* d_state, uint64_t seed, double alpha, double lx,
                      double ly, int thin, int burn_in, int64_t P, double* d_modes,
                      int64_t* d_idx, void* stream) {
  if (!ctx || !d_state || thin < 1 || P < 0 || burn_in < 0 || (P > 0 && !d_modes))
    return fail(SLAB_ERR_ARG, "bad sampler arguments");
  if (!(alpha > 0) || !(lx > 0) || !(ly > 0)) return fail(SLAB_ERR_ARG, "alpha and box must be positive");
  const int64_t need = slab::sampler_scratch_doubles(P, thin, burn_in);
  if (need > ctx->sampler_cap) {
    if (ctx->sampler_scratch) {
      CK(cudaDeviceSynchronize());
      CK(cudaFree(ctx->sampler_scratch));
    }
    CK(cudaMalloc(&ctx->sampler_scratch, sizeof(double) * need));
    ctx->sampler_cap = need;
  }
  CK(slab::sample_modes(d_state, seed, alpha, lx, ly, thin, burn_in, P, d_modes, d_idx,
                        ctx->sampler_scratch, ctx->sampler_cap, (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_batch_energies(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                        SlabSOE soe, double alpha, double area, const double* d_modes,
                        int64_t nbatch, int64_t P, double commonv_scalar, double* d_out,
                        int* d_status, void* stream) {
  if (!ctx || n < 0 || nbatch < 0 || P < 1 || !d_out || !d_status ||
      (n > 0 && (!d_pos || !d_charge)) || (nbatch > 0 && !d_modes))
    return fail(SLAB_ERR_ARG, "bad batch-energy arguments");
  if (n > INT32_MAX) return fail(SLAB_ERR_ARG, "n exceeds int32 indexing");
  if (!(alpha > 0)) return fail(SLAB_ERR_ARG, "alpha must be positive");
  SOEHost sh;
  int rc = prepare_soe(soe, alpha, sh);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (nbatch == 0) return SLAB_OK;
  if (n < 2) {
    CK(cudaMemsetAsync(d_out, 0, sizeof(double) * nbatch, st));
    return SLAB_OK;
  }
  // batches per launch: ~4096 modes keeps the carries modest and the grid full
  int64_t per = 4096 / P;
  per = per < 1 ? 1 : (per > nbatch ? nbatch : per);
  // the full passes and the (shorter) tail pass have their own plans (chunk
  // length, chunk count, buffer counts): the arena is carved for the larger of
  // the two work areas and each pass re-carves it with its own plan
  auto fp = slab::fourier_plan(n, (int)(per * P), sh.mh, 1);
  auto fp2 = lone_plan(sh, n, (int)(per * P), 1);
  const int64_t tail = nbatch % per;
  if (tail) {
    auto ft = slab::fourier_plan(n, (int)(tail * P), sh.mh, 1);
    if (slab::fourier_work_doubles(ft) > slab::fourier_work_doubles(fp)) fp = ft;
    auto ft2 = lone_plan(sh, n, (int)(tail * P), 1);
    if (slab::fourier_work_doubles(ft2) > slab::fourier_work_doubles(fp2)) fp2 = ft2;
  }
  auto zp = slab::zero_plan(n, sh.mh);
  rc = ensure_arena(ctx, sorted_bytes(n, sh.mh, fp, zp, true, sh.mh2, &fp2) + 8192);
  if (rc) return rc;
  Carver cv{(char*)ctx->arena};
  SortedWork w{};
  carve_sorted(cv, n, sh.mh, fp, zp, true, w, sh.mh2, &fp2);
  int32_t* perm = nullptr;
  CK(slab::sort_by_z_device(d_pos + 2, 3, n, w.sw, st, &perm, d_status));
  CK(slab::gather_sorted(d_pos, d_charge, perm, n, w.xs, w.ys, w.zs, w.qs, nullptr, st));
  CK(slab::decay_table(w.zs, n, sh.mh, sh.b, w.dtab, st));
  if (sh.mh2) CK(slab::decay_table(w.zs, n, sh.mh2, sh.b2, w.dtab2, st));
  for (int64_t b0 = 0; b0 < nbatch; b0 += per) {
    const int64_t nb = nbatch - b0 < per ? nbatch - b0 : per;
    auto fpb = slab::fourier_plan(n, (int)(nb * P), sh.mh, 1);
    slab::FourierWork fw;
    slab::fourier_work_carve(fpb, w.fwork, fw);
    CK(slab::fourier_run(fpb, fw, w.xs, w.ys, w.zs, w.qs, w.dtab, d_modes + 3 * b0 * P, nullptr,
                         commonv_scalar, area, sh.b, sh.w, 0, d_out + b0, d_status, nullptr, st,
                         (int)P));
    if (sh.mh2) {  // lone complex terms: the swapped pass, per batch, added in
      auto fpb2 = lone_plan(sh, n, (int)(nb * P), 1);
      slab::fourier_work_carve(fpb2, w.fwork, fw);
      CK(slab::fourier_run(fpb2, fw, w.xs, w.ys, w.zs, w.qs, w.dtab2, d_modes + 3 * b0 * P,
                           nullptr, commonv_scalar, area, sh.b2, sh.w2, 0, w.elone, d_status,
                           nullptr, st, (int)P));
      CK(slab::add_into(d_out + b0, w.elone, (int)nb, st));
    }
  }
  return SLAB_OK;
}

// ---------------------------------------------------------------- MD step (md.cu)
static int ensure_md_part(SlabCtx* ctx, int64_t n) {
  const int64_t need = slab::md_partials(n) + 1;
  if (need <= ctx->md_part_cap) return SLAB_OK;
  if (ctx->md_part) {
    CK(cudaDeviceSynchronize());
    CK(cudaFree(ctx->md_part));
  }
  CK(cudaMalloc(&ctx->md_part, sizeof(double) * need));
  ctx->md_part_cap = need;
  return SLAB_OK;
}

int slab_wca(SlabCtx* ctx, const double* d_pos, int64_t n, SlabBox box, double eps, double sigma,
             double* d_forces, double* d_energy, int* d_status, void* stream) {
  if (!ctx || n < 0 || !d_energy || !d_status || (n > 0 && (!d_pos || !d_forces)))
    return fail(SLAB_ERR_ARG, "bad WCA arguments");
  if (!(sigma > 0) || eps < 0) return fail(SLAB_ERR_ARG, "WCA needs sigma > 0, eps >= 0");
  if (n > INT32_MAX) return fail(SLAB_ERR_ARG, "n exceeds int32 indexing");
  cudaStream_t st = (cudaStream_t)stream;
  const double cut = 1.122462048309373 * sigma;  // WCA_CUT = 2^(1/6), md.py:31
  auto sp = slab::short_plan(n, box.lx, box.ly, box.lz, cut, 1);
  if (sp.kcap < ctx->kcap_min) sp.kcap = ctx->kcap_min;
  int rc = ensure_arena(ctx, slab::short_work_bytes(sp) + 1024);
  if (rc) return rc;
  CK(cudaMemsetAsync(ctx->d_maxnn, 0, sizeof(int), st));
  CK(slab::short_run(sp, ctx->arena, d_pos, d_pos /* charges unused */, box.lx, box.ly, box.lz,
                     0.0, cut, d_forces, d_energy, d_status, 0, n, ctx->d_maxnn, st, 1, eps,
                     sigma, 1));
  return SLAB_OK;
}

int slab_walls(SlabCtx* ctx, const double* d_pos, int64_t n, double lz, double eps, double sigma,
               double* d_forces, double* d_energy, int* d_status, void* stream) {
  if (!ctx || n < 0 || !d_energy || !d_status || (n > 0 && (!d_pos || !d_forces)))
    return fail(SLAB_ERR_ARG, "bad wall arguments");
  int rc = ensure_md_part(ctx, n);
  if (rc) return rc;
  CK(slab::md_walls(d_pos, n, lz, eps, sigma, d_forces, d_energy, d_status, ctx->md_part, 0,
                    (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_md_langevin(double* d_pos, double* d_vel, const double* d_forces, const double* d_mass,
                     int64_t n, double dt, double gamma, double temperature, uint64_t seed,
                     int64_t* d_counter, double* d_shift, double lx, double ly, void* stream) {
  if (n < 0 || !d_counter || (n > 0 && (!d_pos || !d_vel || !d_forces || !d_mass)))
    return fail(SLAB_ERR_ARG, "bad Langevin arguments");
  CK(slab::md_langevin(d_pos, d_vel, d_forces, d_mass, n, dt, gamma, temperature, seed, d_counter,
                       d_shift, lx, ly, (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_md_kick(double* d_vel, const double* d_forces, const double* d_mass, int64_t n,
                 double h, void* stream) {
  if (n < 0 || (n > 0 && (!d_vel || !d_forces || !d_mass)))
    return fail(SLAB_ERR_ARG, "bad kick arguments");
  CK(slab::md_kick(d_vel, d_forces, d_mass, n, h, (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_md_drift(double* d_pos, const double* d_vel, int64_t n, double dt, double* d_shift,
                  double lx, double ly, void* stream) {
  if (n < 0 || (n > 0 && (!d_pos || !d_vel))) return fail(SLAB_ERR_ARG, "bad drift arguments");
  CK(slab::md_drift(d_pos, d_vel, n, dt, d_shift, lx, ly, (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_md_scale(double* d_vel, int64_t n, double s, void* stream) {
  if (n < 0 || (n > 0 && !d_vel)) return fail(SLAB_ERR_ARG, "bad scale arguments");
  CK(slab::md_scale(d_vel, n, s, (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_md_kinetic(SlabCtx* ctx, const double* d_vel, const double* d_mass, int64_t n,
                    double* d_out, void* stream) {
  if (!ctx || n < 0 || !d_out || (n > 0 && (!d_vel || !d_mass)))
    return fail(SLAB_ERR_ARG, "bad kinetic-energy arguments");
  int rc = ensure_md_part(ctx, n);
  if (rc) return rc;
  CK(slab::md_kinetic(d_vel, d_mass, n, d_out, ctx->md_part, (cudaStream_t)stream));
  return SLAB_OK;
}

// ---------------------------------------------------------------- Ewald2D reference (ewald_ref.cu)
int slab_ewald_ref_fourier(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                           double lx, double ly, double alpha, const int* d_mxy,
                           const int* d_ring, int nmode, const double* d_kappa, int nring,
                           int mxmax, int mymax, int naive, double* d_forces, double* d_energy,
                           void* stream) {
  if (!ctx || n < 0 || nmode < 0 || nring < 0 || !d_energy ||
      (n > 0 && (!d_pos || !d_charge || !d_forces)) ||
      (nmode > 0 && (!d_mxy || !d_ring || !d_kappa)))
    return fail(SLAB_ERR_ARG, "bad Ewald2D reference arguments");
  if (nring > slab::ewald_ref_max_ring() || mxmax > slab::ewald_ref_max_m() ||
      mymax > slab::ewald_ref_max_m() || mxmax < 0 || mymax < 0)
    return fail(SLAB_ERR_UNSUPPORTED, "mode set too large for the device Ewald2D reference");
  int rc = ensure_md_part(ctx, 2 * n);  // 128-thread block partials (MD uses 256)
  if (rc) return rc;
  CK(slab::ewald_ref_fourier(d_pos, d_charge, n, lx, ly, alpha, d_mxy, d_ring, nmode, d_kappa,
                             nring, mxmax, mymax, naive, d_forces, d_energy, ctx->md_part,
                             (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_ewald_ref_zero(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                        double alpha, double* d_fz, double* d_energy, void* stream) {
  if (!ctx || n < 0 || !d_energy || (n > 0 && (!d_pos || !d_charge || !d_fz)))
    return fail(SLAB_ERR_ARG, "bad k = 0 reference arguments");
  int rc = ensure_md_part(ctx, 2 * n);
  if (rc) return rc;
  CK(slab::ewald_ref_zero(d_pos, d_charge, n, alpha, d_fz, d_energy, ctx->md_part,
                          (cudaStream_t)stream));
  return SLAB_OK;
}

int slab_recursive_pair_sum(SlabCtx* ctx, const double* d_q, const double* d_theta,
                            const double* d_z, int64_t n, double beta_re, double beta_im,
                            double* d_out, void* stream) {
  if (!ctx || n < 0 || (n > 0 && (!d_q || !d_theta || !d_z || !d_out)))
    return fail(SLAB_ERR_ARG, "bad recursive_pair_sum arguments");
  int rc = ensure_arena(ctx, pad(sizeof(double2) * (size_t)(n / 64 + 2)) + 512);
  if (rc) return rc;
  CK(slab::recursive_pair_sum(d_q, d_theta, d_z, n, beta_re, beta_im, d_out,
                              reinterpret_cast<double2*>(ctx->arena), (cudaStream_t)stream));
  return SLAB_OK;
}

// short-range home-particle boundary of rank r of W (sharding.py home_range): the
// lead rank (which also runs the k = 0 mode) takes LEAD_HOME_TENTHS[W] tenths of a
// regular share
static int64_t home_bound(int64_t n, int r, int W) {
  static const int kLeadTenths[9] = {10, 10, 8, 8, 7, 5, 4, 2, 1};
  if (W <= 1 || r >= W) return r <= 0 ? 0 : n;
  if (r <= 0) return 0;
  const int64_t lead = W < 9 ? kLeadTenths[W] : 0;
  return n * (lead + 10 * (int64_t)(r - 1)) / (lead + 10 * (int64_t)(W - 1));
}

static int evaluate_impl(SlabCtx* ctx, const SlabEvalArgs* a, cudaStream_t st,
                         cudaEvent_t pos_ready, cudaEvent_t charge_ready, bool host_entry);

// Concurrent short range up to this many particles (cfg3, N = 1e5: 3.30 ->
// 3.07 ms).  Beyond it both halves fill the GPU on their own: at N = 1e6 the
// overlap bought 1.6% while stretching the scan kernels' measured span (its
// roofline figure) by 45% as the short range's CTAs shared their SMs.
#ifndef SLAB_FORK_MAX_N
#define SLAB_FORK_MAX_N 400000
#endif
constexpr int64_t kForkMaxN = SLAB_FORK_MAX_N;
// Host-buffer entry: fork everything regardless of N.  Off since round 2: with
// the faster scan the cfg4 call measured 9.85 ms forked against 9.58 ms with
// the device-buffer rule (z sort beside the short range, scan after it).
#ifndef SLAB_FORK_HOST
#define SLAB_FORK_HOST 0
#endif
constexpr bool kForkHost = SLAB_FORK_HOST;
#ifndef SLAB_FORK_SORT
#define SLAB_FORK_SORT 1
#endif
constexpr bool kForkSort = SLAB_FORK_SORT;
#ifndef SLAB_SPLIT_SHORT
#define SLAB_SPLIT_SHORT 0
#endif
constexpr bool kSplitShort = SLAB_SPLIT_SHORT;
#ifndef SLAB_PAR_ZERO
#define SLAB_PAR_ZERO 1
#endif
constexpr bool kParZero = SLAB_PAR_ZERO;

// A caller's timing event: inside a stream capture it must be an EXTERNAL
// record node (a plain record there only orders captured work), so that a
// replayed graph stamps it -- the scan span is then timed inside the same
// graph the bench replays.
static cudaError_t record_timing_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(s, &cs);
  if (e != cudaSuccess) return e;
  if (cs == cudaStreamCaptureStatusActive)
    return cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  return cudaEventRecord(ev, s);
}

static int ensure_fork(SlabCtx* ctx) {
  if (ctx->hi) return SLAB_OK;
  int least = 0, greatest = 0;
  CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
  // (the scan chain one notch below the greatest priority, so that the remainder
  // sweep and the k = 0 chain take SM slots as soon as sweep CTAs retire rather
  // than after its last wave, stretched the main sweep by more than the tail it
  // saved: cfg4 8.49 -> 8.60 ms; the k = 0 chain and decay table enqueued before
  // the scan's wait for the short range, to run beside the pair kernel, delayed
  // the pair kernel instead: 8.48 -> 8.74 ms; the k = 0 chain alone above the
  // scan's priority ran inside the aggregate and stretched it: 8.48 -> 8.63 ms)
  CK(cudaStreamCreateWithPriority(&ctx->hi, cudaStreamNonBlocking, greatest));
#ifndef SLAB_SHORT_HI
#define SLAB_SHORT_HI 0
#endif
  CK(cudaStreamCreateWithPriority(&ctx->lo, cudaStreamNonBlocking, SLAB_SHORT_HI ? greatest : least));
  CK(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, greatest));
  for (cudaEvent_t* e : {&ctx->ev_fork, &ctx->ev_short, &ctx->ev_long, &ctx->ev_x,
                         &ctx->ev_dtab, &ctx->ev_zero})
    CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return SLAB_OK;
}

int slab_evaluate(SlabCtx* ctx, const SlabEvalArgs* a, void* stream) {
  if (!ctx || !a) return fail(SLAB_ERR_ARG, "null context or arguments");
  return evaluate_impl(ctx, a, (cudaStream_t)stream, nullptr, nullptr, false);
}

int slab_evaluate_host(SlabCtx* ctx, const SlabEvalArgs* args, const double* h_pos,
                       const double* h_charge, double* h_forces, double* h_energy,
                       void* stream) {
  if (!ctx || !args || !h_energy) return fail(SLAB_ERR_ARG, "null context or arguments");
  const int64_t n = args->n;
  if (n < 0) return fail(SLAB_ERR_ARG, "bad evaluation arguments");
  if (n > 0 && (!h_pos || !h_charge)) return fail(SLAB_ERR_ARG, "host inputs missing");
  if (args->want_forces && n > 0 && !h_forces) return fail(SLAB_ERR_ARG, "forces output missing");
  if (args->shard_mode != SLAB_SHARD_MODES || args->phase != 0)
    return fail(SLAB_ERR_ARG, "the host-buffer form runs unsharded-mode evaluations only");
  cudaStream_t st = (cudaStream_t)stream;
  if (!ctx->up_stream) {
    CK(cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_pos, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_q, cudaEventDisableTiming));
    CK(cudaMalloc(&ctx->h_denergy, 8 * sizeof(double)));
  }
  if (n > ctx->h_cap) {
    CK(cudaStreamSynchronize(st));
    if (ctx->h_dpos) CK(cudaFree(ctx->h_dpos));
    if (ctx->h_dq) CK(cudaFree(ctx->h_dq));
    if (ctx->h_dforces) CK(cudaFree(ctx->h_dforces));
    const size_t cap = (size_t)(n > 0 ? n : 1);
    CK(cudaMalloc(&ctx->h_dpos, 3 * sizeof(double) * cap));
    CK(cudaMalloc(&ctx->h_dq, sizeof(double) * cap));
    CK(cudaMalloc(&ctx->h_dforces, 3 * sizeof(double) * cap));
    ctx->h_cap = n;
  }
  // uploads on the side stream, concurrent with work already queued on `stream`
  // (e.g. the device sampler's chain for this batch): positions first (the z
  // sort needs only them), then charges, which land while the sort runs.  The
  // buffers are private to this entry point, which leaves both streams idle
  // on return (success or failure), so no earlier work can still read them.
  if (n > 0) {
    CK(cudaMemcpyAsync(ctx->h_dpos, h_pos, 3 * sizeof(double) * n, cudaMemcpyHostToDevice,
                       ctx->up_stream));
    CK(cudaEventRecord(ctx->ev_pos, ctx->up_stream));
    CK(cudaMemcpyAsync(ctx->h_dq, h_charge, sizeof(double) * n, cudaMemcpyHostToDevice,
                       ctx->up_stream));
  } else {
    CK(cudaEventRecord(ctx->ev_pos, ctx->up_stream));
  }
  CK(cudaEventRecord(ctx->ev_q, ctx->up_stream));
  SlabEvalArgs a = *args;
  a.d_pos = ctx->h_dpos;
  a.d_charge = ctx->h_dq;
  a.d_forces = args->want_forces ? ctx->h_dforces : nullptr;
  a.d_energy = ctx->h_denergy;
  const int rc = evaluate_impl(ctx, &a, st, ctx->ev_pos, ctx->ev_q, true);
  if (rc) {
    cudaStreamSynchronize(ctx->up_stream);
    cudaStreamSynchronize(st);
    return rc;
  }
  if (args->want_forces && n > 0)
    CK(cudaMemcpyAsync(h_forces, ctx->h_dforces, 3 * sizeof(double) * n,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_energy, ctx->h_denergy, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return SLAB_OK;
}

static int evaluate_impl(SlabCtx* ctx, const SlabEvalArgs* a, cudaStream_t st,
                         cudaEvent_t pos_ready, cudaEvent_t charge_ready, bool host_entry) {
  const int64_t n = a->n;
  if (n < 0 || a->nmode < 0 || !a->d_energy || (n > 0 && (!a->d_pos || !a->d_charge)))
    return fail(SLAB_ERR_ARG, "bad evaluation arguments");
  if (a->want_forces && n > 0 && !a->d_forces) return fail(SLAB_ERR_ARG, "forces output missing");
  if (n > INT32_MAX) return fail(SLAB_ERR_ARG, "n exceeds int32 indexing");
  if (a->nmode > 0 && !a->d_modes) return fail(SLAB_ERR_ARG, "modes missing");
  if (!(a->alpha > 0)) return fail(SLAB_ERR_ARG, "alpha must be positive");
  SOEHost sh;
  int rc = prepare_soe(a->soe, a->alpha, sh);
  if (rc) return rc;
  const SlabBox& box = a->box;
  const double area = box.lx * box.ly;
  const int scount = a->shard_count > 1 ? a->shard_count : 1;
  const int srank = scount > 1 ? a->shard_rank : 0;
  if (srank < 0 || srank >= scount) return fail(SLAB_ERR_ARG, "shard_rank out of range");
  const bool zsplit = a->shard_mode == SLAB_SHARD_ZSPLIT;
  if (a->shard_mode != SLAB_SHARD_MODES && !zsplit) return fail(SLAB_ERR_ARG, "bad shard_mode");
  if (a->phase < 0 || a->phase > 2) return fail(SLAB_ERR_ARG, "phase must be 0, 1 or 2");
  if (a->phase != 0 && !zsplit) return fail(SLAB_ERR_ARG, "phases belong to the z-split mode");
  if (zsplit && a->phase == 0) return fail(SLAB_ERR_ARG, "z-split runs as phase 1 + phase 2");
  if (zsplit && a->nmode > 0 && !a->d_xchg) return fail(SLAB_ERR_ARG, "z-split needs d_xchg");
  if (zsplit && (sh.real_terms || sh.mh2))  // the exchange is sized for m = 2 mh
    return fail(SLAB_ERR_UNSUPPORTED,
                "z-split needs a table of conjugate pairs (no real or lone complex terms)");
  const bool forces = a->want_forces && n > 0;
  auto fp = slab::fourier_plan(n, (int)a->nmode, sh.mh, forces ? 2 : 1, zsplit ? scount : 1);
  if (zsplit) {  // this rank's contiguous chunk range of the z-sorted particles
    fp.c0 = (int)((int64_t)fp.nch * srank / scount);
    fp.c1 = (int)((int64_t)fp.nch * (srank + 1) / scount);
  }
  auto zp = slab::zero_plan(n, sh.mh);
  auto fp2 = lone_plan(sh, n, (int)a->nmode, forces ? 2 : 1);
  auto sp = slab::short_plan(n, box.lx, box.ly, box.lz, a->r_c);
  if (sp.kcap < ctx->kcap_min) sp.kcap = ctx->kcap_min;
  const size_t N = (size_t)(n > 0 ? n : 1);
  size_t bytes = sorted_bytes(n, sh.mh, fp, zp, true, sh.mh2, &fp2) + pad(24 * N) +
                 (a->skip_short_range ? 0 : pad(slab::short_work_bytes(sp))) + 8192;
  if (a->phase == 2 && bytes > ctx->arena_bytes)
    return fail(SLAB_ERR_ARG, "phase 2 without a matching phase 1 on this context");
  rc = ensure_arena(ctx, bytes);
  if (rc) return rc;
  Carver cv{(char*)ctx->arena};
  SortedWork w{};
  carve_sorted(cv, n, sh.mh, fp, zp, true, w, sh.mh2, &fp2);
  double* fshort = cv.take<double>(3 * N);
  void* swork = a->skip_short_range ? nullptr : cv.take<char>(slab::short_work_bytes(sp));
  slab::FourierWork fw;
  slab::fourier_work_carve(fp, w.fwork, fw);
  double* u_s = ctx->small;
  double* u_sweep = ctx->small + 1;
  double* u_pair = ctx->small + 2;
  const bool lead = srank == 0;  // the rank that owns the k = 0 mode and the constants
  int32_t* perm = nullptr;

  // Fork: the short range runs on ctx->lo (lowest priority) concurrently with
  // the sort / Fourier / k = 0 chain on ctx->hi (highest priority); both join
  // back into `st` before the assembly.  (A z-split phase 1 joins its short
  // range before returning: each phase is capturable as its own graph.)
  const bool fork_all = !a->skip_short_range && n > 0 && (n <= kForkMaxN || (host_entry && kForkHost));
  // Large systems on device buffers: only the z sort + gather run beside the
  // short range (latency-bound passes that barely compete with it); the scan
  // waits for the short range, so its kernels keep the GPU to themselves.
  // (Also in z-split phase 1; round 1 ran a z-split rank's sort after its
  // short range, 0.26 ms of a 1.8 ms rank step at W = 8.)
  const bool fork_sort = kForkSort && !fork_all && !a->skip_short_range && n > 0;
  const bool fork = fork_all || fork_sort;
  // ... and with SLAB_SPLIT_SHORT the neighbour screen (no fp64 work) also runs
  // beside the scan's first phase while the pair kernel waits for the scan's end
  const bool split_short = kSplitShort && fork_sort;
  // the k = 0 chain (aggregate, carry, sweep: low-occupancy kernels) runs on
  // ctx->aux beside the Fourier chain once the decay table exists
  const bool par_zero = kParZero && a->phase == 0 && n >= 2 && lead;
  if (fork || par_zero) {
    rc = ensure_fork(ctx);
    if (rc) return rc;
  }
  cudaStream_t sl = fork ? ctx->hi : st;  // the long (scan) chain's stream
  if (a->phase != 2) {  // ---- sort, short range, aggregates
    CK(cudaMemsetAsync(ctx->status, 0, sizeof(int), st));
    CK(cudaMemsetAsync(ctx->small, 0, 8 * sizeof(double), st));
    CK(cudaMemsetAsync(ctx->d_maxnn, 0, sizeof(int), st));
    if (fork) {
      CK(cudaEventRecord(ctx->ev_fork, st));
      CK(cudaStreamWaitEvent(ctx->hi, ctx->ev_fork, 0));
      CK(cudaStreamWaitEvent(ctx->lo, ctx->ev_fork, 0));
    }
    if (!a->skip_short_range && !split_short) {
      cudaStream_t ss = fork ? ctx->lo : st;
      if (pos_ready) CK(cudaStreamWaitEvent(ss, pos_ready, 0));
      // (charges: waited for inside, before the first kernel that reads them)
      const int64_t h0 = home_bound(n, srank, scount), h1 = home_bound(n, srank + 1, scount);
      CK(slab::short_run(sp, swork, a->d_pos, a->d_charge, box.lx, box.ly, box.lz, a->alpha,
                         a->r_c, fshort, u_s, ctx->status, h0, h1, ctx->d_maxnn, ss, 0, 0.0, 0.0,
                         0, nullptr, charge_ready));
      if (fork) CK(cudaEventRecord(ctx->ev_short, ctx->lo));
    }
    if (pos_ready) CK(cudaStreamWaitEvent(sl, pos_ready, 0));
    if (n > 0) {
      CK(slab::sort_by_z_device(a->d_pos + 2, 3, n, w.sw, sl, &perm, ctx->status));
      if (charge_ready) CK(cudaStreamWaitEvent(sl, charge_ready, 0));
      CK(slab::gather_sorted(a->d_pos, a->d_charge, perm, n, w.xs, w.ys, w.zs, w.qs, a->d_perm,
                             sl));
    }
    ctx->zs_perm = perm;
    if (fork_sort && !split_short)  // scan after the short range
      CK(cudaStreamWaitEvent(sl, ctx->ev_short, 0));
    if (a->ev_scan_begin) CK(record_timing_event((cudaEvent_t)a->ev_scan_begin, sl));
    if (n >= 2) {
      if (zsplit && !lead)  // rows of this rank's chunk range only (no k = 0 mode here)
        CK(slab::decay_table(w.zs, n, sh.mh, sh.b, w.dtab, sl, (int64_t)fp.c0 * fp.R,
                             std::min<int64_t>(n, (int64_t)fp.c1 * fp.R)));
      else
        CK(slab::decay_table(w.zs, n, sh.mh, sh.b, w.dtab, sl));
      if (par_zero) {
        CK(cudaEventRecord(ctx->ev_dtab, sl));
        CK(cudaStreamWaitEvent(ctx->aux, ctx->ev_dtab, 0));
        CK(slab::zero_run_b(zp, w.zwork, w.zs, w.qs, w.dtab, sh.z, sh.b, a->alpha,
                            forces ? 1 : 0, w.fzf, w.fzb, u_pair, ctx->aux));
        CK(cudaEventRecord(ctx->ev_zero, ctx->aux));
      }
      if (forces) CK(cudaMemsetAsync(w.fsorted, 0, sizeof(double) * 3 * n, sl));
      if (a->nmode > 0 && a->ev_modes_ready)
        CK(cudaStreamWaitEvent(sl, (cudaEvent_t)a->ev_modes_ready, 0));
      if (a->nmode > 0)
        CK(slab::fourier_phase1(fp, fw, w.xs, w.ys, w.zs, w.qs, a->d_modes, a->d_commonv,
                                a->commonv_scalar, area, sh.b, sh.w, ctx->status,
                                a->phase == 1 ? a->d_xchg : nullptr, sl));
    } else if (forces) {
      CK(cudaMemsetAsync(w.fsorted, 0, sizeof(double) * 3 * N, sl));
    }
    if (a->phase == 1) {  // the exchange payload is read on `st` by the caller
      if (fork) {
        CK(cudaEventRecord(ctx->ev_long, sl));
        CK(cudaStreamWaitEvent(st, ctx->ev_long, 0));
        // the short range is joined here too, so that each phase is
        // self-contained (a rank captures the two phases as separate CUDA
        // graphs around the exchange; with the sort fork the scan waited for
        // it already)
        if (!a->skip_short_range && !split_short) CK(cudaStreamWaitEvent(st, ctx->ev_short, 0));
      }
      return SLAB_OK;
    }
  } else {
    perm = ctx->zs_perm;
    if (fork) {  // the gathered exchange was written on `st`
      CK(cudaEventRecord(ctx->ev_x, st));
      CK(cudaStreamWaitEvent(sl, ctx->ev_x, 0));
    }
  }

  // ---- carried-in states, sweep, k = 0 mode, assembly
  if (n >= 2) {
    if (a->nmode > 0) {
      const double* tin = nullptr;
      if (a->phase == 2) {
        CK(slab::fourier_zsplit_tin(fp, a->d_xchg, scount, srank, fw.tin, sl));
        tin = fw.tin;
      }
      CK(slab::fourier_phase2(fp, fw, w.xs, w.ys, w.zs, w.qs, w.dtab, sh.b, forces ? 1 : 0,
                              u_sweep, w.fsorted, tin, sl));
      if (sh.mh2) {  // lone complex terms: the swapped pass (phase 0 only, see above)
        CK(slab::decay_table(w.zs, n, sh.mh2, sh.b2, w.dtab2, sl));
        slab::FourierWork fw2;
        slab::fourier_work_carve(fp2, w.fwork, fw2);
        CK(slab::fourier_run(fp2, fw2, w.xs, w.ys, w.zs, w.qs, w.dtab2, a->d_modes,
                             a->d_commonv, a->commonv_scalar, area, sh.b2, sh.w2,
                             forces ? 1 : 0, w.elone, ctx->status, w.fsorted, sl));
        CK(slab::add_into(u_sweep, w.elone, 1, sl));
      }
    }
    if (lead && !par_zero)
      CK(slab::zero_run_b(zp, w.zwork, w.zs, w.qs, w.dtab, sh.z, sh.b, a->alpha, forces ? 1 : 0,
                          w.fzf, w.fzb, u_pair, sl));
    if (par_zero) CK(cudaStreamWaitEvent(sl, ctx->ev_zero, 0));
  }
  if (a->ev_scan_end) CK(record_timing_event((cudaEvent_t)a->ev_scan_end, sl));
  if (split_short) {  // enqueued after the scan chain so the pair kernel can wait on its end
    CK(cudaEventRecord(ctx->ev_long, sl));
    if (pos_ready) CK(cudaStreamWaitEvent(ctx->lo, pos_ready, 0));
    const int64_t h0 = home_bound(n, srank, scount), h1 = home_bound(n, srank + 1, scount);
    CK(slab::short_run(sp, swork, a->d_pos, a->d_charge, box.lx, box.ly, box.lz, a->alpha,
                       a->r_c, fshort, u_s, ctx->status, h0, h1, ctx->d_maxnn, ctx->lo, 0, 0.0,
                       0.0, 0, ctx->ev_long, charge_ready));
    CK(cudaEventRecord(ctx->ev_short, ctx->lo));
  }
  if (fork) {  // join (a phase 2 joined its short range at the end of phase 1)
    CK(cudaEventRecord(ctx->ev_long, sl));
    CK(cudaStreamWaitEvent(st, ctx->ev_long, 0));
    if (a->phase != 2 || split_short) CK(cudaStreamWaitEvent(st, ctx->ev_short, 0));
  }
  if (forces) {
    const double plane = lead ? box.sigma_top - box.sigma_bot : 0.0;
    CK(slab::assemble_forces(n, perm, w.qs, w.fsorted, (n >= 2 && lead) ? w.fzf : nullptr, w.fzb,
                             2.0 * slab::kPi / area, a->skip_short_range ? nullptr : fshort,
                             a->d_charge, plane, a->d_forces, st));
  }
  CK(slab::assemble_energy(n, a->d_charge, a->d_pos, box.lz, box.sigma_top, box.sigma_bot,
                           a->alpha, area, lead ? a->charge_const : 0.0, u_s, u_sweep,
                           lead ? u_pair : nullptr, ctx->status, a->d_energy, ctx->small + 64,
                           lead ? 1 : 0, st));
  return SLAB_OK;
}

int slab_constant_terms(SlabCtx* ctx, const double* d_pos, const double* d_charge, int64_t n,
                        SlabBox box, double alpha, double* d_energy, void* stream) {
  if (!ctx || n < 0 || !d_energy || (n > 0 && (!d_pos || !d_charge)))
    return fail(SLAB_ERR_ARG, "bad constant-term arguments");
  if (!(alpha > 0)) return fail(SLAB_ERR_ARG, "alpha must be positive");
  int rc = ensure_arena(ctx, 4096);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(ctx->status, 0, sizeof(int), st));
  CK(slab::assemble_energy(n, d_charge, d_pos, box.lz, box.sigma_top, box.sigma_bot, alpha,
                           box.lx * box.ly, 0.0, nullptr, nullptr, nullptr, ctx->status, d_energy,
                           ctx->small + 64, 1, st));
  return SLAB_OK;
}

int64_t slab_zsplit_exchange_doubles(int64_t nmode, int soe_terms, int want_forces) {
  if (nmode <= 0 || soe_terms <= 0) return 0;
  return 4 * (int64_t)(soe_terms + 1) * (want_forces ? 2 : 1) * nmode;
}

}  // extern "C"

extern "C" int slab_fp64_peak(double* tflops) {
  if (!tflops) return fail(SLAB_ERR_ARG, "null output");
  CK(slab::fp64_peak(tflops));
  return SLAB_OK;
}
