// In-library L-BFGS-B drivers of the two continuous steps of the solver:
// the certificate ascent (refine_eta_max, certificate.py:187-224) and the
// joint slide (local_descent, solvers.py:197-240). The objective is evaluated
// by the device kernels (sfw3d_atom_sums / sfw3d_cost_grad); the optimiser
// (lbfgsb.cuh) runs on the calling host thread, so one C call replaces the
// reference's scipy loop with its Python callback per evaluation.
#include <cmath>
#include <vector>

#include "internal.cuh"
#include "lbfgsb.cuh"

namespace sfw3d {
namespace {

lbfgsb::Options make_options(int maxcor, double ftol, double gtol, int maxiter, int maxfun, int maxls) {
  lbfgsb::Options o;
  o.m = maxcor > 0 ? maxcor : 10;
  o.factr = ftol / lbfgsb::detail::EPS;
  o.pgtol = gtol;
  o.maxiter = maxiter;
  o.maxfun = maxfun > 0 ? maxfun : 15000;
  o.maxls = maxls > 0 ? maxls : 20;
  return o;
}

void fill_info(int32_t* info, const lbfgsb::Result& r) {
  if (!info) return;
  info[0] = r.status;
  info[1] = r.iterations;
  info[2] = r.evaluations;
}

struct RefineUser {
  sfw3d_ctx* ctx;
  int dtype;
  const int* dims;
  const void* back;
  double lam;
  double row[6];
  double sums[6];
  bool first = true;
  double f_first = 0.0;
  std::vector<AtomGeo> atom;
};

// neg_eta (certificate.py:201-209): -<G_theta, back>/lam and its 5-gradient
int refine_objective(void* user, const double* x, double* f, double* g) {
  RefineUser* u = static_cast<RefineUser*>(user);
  u->row[0] = 1.0;
  for (int i = 0; i < 5; ++i) u->row[1 + i] = x[i];
  int rc = build_atoms(u->dims, u->row, 1, u->atom);
  if (rc != SFW3D_OK) return rc;
  rc = refine_sums_impl(u->ctx, u->dtype, u->dims, u->back, u->atom[0], u->sums);
  if (rc != SFW3D_OK) return rc;
  for (int c = 0; c < 6; ++c)
    if (!std::isfinite(u->sums[c])) {
      set_error("non-finite certificate value; atom parameters left the smooth regime");
      return SFW3D_ENONFINITE;
    }
  *f = -(u->sums[0] / u->lam);
  for (int i = 0; i < 5; ++i) g[i] = -(u->sums[1 + i] / u->lam);
  if (u->first) { u->first = false; u->f_first = *f; }
  return 0;
}

struct DescentUser {
  sfw3d_ctx* ctx;
  const sfw3d_psf* psf;
  int dtype;
  const void* y;
  int k;
  double lam;
  std::vector<double> rows;
  bool first = true;
  double f_first = 0.0;
};

// fun of local_descent (solvers.py:218-220): rows from x with w = max(0, w)
int descent_objective(void* user, const double* x, double* f, double* g) {
  DescentUser* u = static_cast<DescentUser*>(user);
  const size_t n = size_t(u->k) * 6;
  for (size_t i = 0; i < n; ++i) {
    if (!std::isfinite(x[i])) {
      set_error("invalid argument: non-finite atom parameters");
      return SFW3D_EINVAL;
    }
    u->rows[i] = x[i];
  }
  for (int i = 0; i < u->k; ++i)
    if (!(u->rows[size_t(i) * 6] > 0.0)) u->rows[size_t(i) * 6] = 0.0;
  const int rc = sfw3d_cost_grad(u->ctx, u->psf, u->dtype, u->y, u->rows.data(), u->k, u->lam, f, g, nullptr);
  if (rc != SFW3D_OK) return rc;
  if (u->first) { u->first = false; u->f_first = *f; }
  return 0;
}

}  // namespace
}  // namespace sfw3d

using namespace sfw3d;

extern "C" int sfw3d_lbfgsb_minimize(int n, double* x, const double* lower, const double* upper,
                                     const int32_t* nbd, int maxcor, double ftol, double gtol,
                                     int maxiter, int maxfun, int maxls, sfw3d_objective_fn fn,
                                     void* user, double* f_out, int32_t info[3]) {
  SFW3D_CHECK_ARG(n > 0 && x && lower && upper && nbd && fn && f_out, "NULL argument");
  SFW3D_CHECK_ARG(ftol >= 0.0 && gtol >= 0.0 && maxiter >= 0, "tolerances");
  for (int i = 0; i < n; ++i) {
    SFW3D_CHECK_ARG(nbd[i] >= 0 && nbd[i] <= 3, "nbd must be 0..3");
    SFW3D_CHECK_ARG(nbd[i] != 2 || lower[i] <= upper[i], "lower bound above upper bound");
  }
  std::vector<int> nb(nbd, nbd + n);
  lbfgsb::Minimizer opt(n, make_options(maxcor, ftol, gtol, maxiter, maxfun, maxls));
  const lbfgsb::Result r = opt.minimize(x, lower, upper, nb.data(), fn, user);
  *f_out = r.f;
  fill_info(info, r);
  if (r.status == lbfgsb::CALLBACK_ERROR) return r.callback_code > 0 && r.callback_code <= SFW3D_ENOMEM
                                                     ? r.callback_code : SFW3D_EINVAL;
  return SFW3D_OK;
}

extern "C" int sfw3d_refine_eta_max(sfw3d_ctx* ctx, int dtype, const int dims[3], const void* back_dev,
                                    double lam, const double start[5], const double lower[5],
                                    const double upper[5], int max_iter, double gtol,
                                    double theta_out[5], double* eta_out, int32_t info[3]) {
  SFW3D_CHECK_ARG(ctx && back_dev && start && lower && upper && theta_out && eta_out, "NULL argument");
  SFW3D_CHECK_ARG(lam > 0.0, "lam must be > 0");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(dims[0] > 0 && dims[1] > 0 && dims[2] > 0, "dims must be positive");
  SFW3D_TRY(begin_call(ctx));
  RefineUser u{ctx, dtype, dims, back_dev, lam};
  double x[5];
  int nb[5];
  for (int i = 0; i < 5; ++i) {
    SFW3D_CHECK_ARG(lower[i] <= upper[i], "lower bound above upper bound");
    x[i] = start[i];
    nb[i] = 2;
  }
  // scipy defaults of the reference call: ftol 2.220446049250313e-09, maxcor 10
  lbfgsb::Minimizer opt(5, make_options(10, 2.220446049250313e-09, gtol, max_iter, 15000, 20));
  const lbfgsb::Result r = opt.minimize(x, lower, upper, nb, refine_objective, &u);
  fill_info(info, r);
  if (r.status == lbfgsb::CALLBACK_ERROR) return r.callback_code;
  if (!std::isfinite(r.f)) {
    set_error("certificate ascent diverged to a non-finite value");
    return SFW3D_ENONFINITE;
  }
  const double start_val = -u.f_first;
  if (-r.f < start_val) {  // keep the seed if the ascent did not improve it
    for (int i = 0; i < 5; ++i) theta_out[i] = std::min(std::max(start[i], lower[i]), upper[i]);
    *eta_out = start_val;
  } else {
    for (int i = 0; i < 5; ++i) theta_out[i] = x[i];
    *eta_out = -r.f;
  }
  return SFW3D_OK;
}

extern "C" int sfw3d_local_descent(sfw3d_ctx* ctx, const sfw3d_psf* psf, int dtype, const void* y_dev,
                                   double* params_host, int k, double lam, const double lower[5],
                                   const double upper[5], double gtol, double ftol, int max_iter,
                                   double* cost_out, int32_t info[3]) {
  SFW3D_CHECK_ARG(ctx && psf && y_dev && params_host && lower && upper && cost_out, "NULL argument");
  SFW3D_CHECK_ARG(k > 0, "k must be positive");
  SFW3D_CHECK_ARG(lam > 0.0, "lam must be > 0");
  const int n = 6 * k;
  std::vector<double> x(params_host, params_host + n), lo(n), hi(n);
  std::vector<int> nb(n);
  for (int i = 0; i < k; ++i) {
    lo[6 * i] = 0.0;  // w >= 0, no upper bound
    hi[6 * i] = 0.0;
    nb[6 * i] = 1;
    for (int c = 0; c < 5; ++c) {
      SFW3D_CHECK_ARG(lower[c] <= upper[c], "lower bound above upper bound");
      lo[6 * i + 1 + c] = lower[c];
      hi[6 * i + 1 + c] = upper[c];
      nb[6 * i + 1 + c] = 2;
    }
  }
  DescentUser u{ctx, psf, dtype, y_dev, k, lam, std::vector<double>(size_t(n))};
  lbfgsb::Minimizer opt(n, make_options(10, ftol, gtol, max_iter, 15000, 20));
  const lbfgsb::Result r = opt.minimize(x.data(), lo.data(), hi.data(), nb.data(), descent_objective, &u);
  fill_info(info, r);
  if (r.status == lbfgsb::CALLBACK_ERROR) return r.callback_code;
  if (!std::isfinite(r.f) || r.f > u.f_first) {  // keep the start (solvers.py:236-237)
    *cost_out = u.f_first;
    if (info) info[0] |= 0x100;
    return SFW3D_OK;
  }
  for (int i = 0; i < n; ++i) params_host[i] = x[i];
  *cost_out = r.f;
  return SFW3D_OK;
}
