// The solver's outer loop (solvers.py:286-395: SFW / boosted SFW) as ONE
// library call: certificate (grid argmax + ascent), new atom's phi, cached
// Gram rows, non-negative LASSO, residual + criterion, prune, duplicate
// guard, the slide(s) and the final re-check run from a C++ controller on
// the calling thread over the device kernels — no Python between the steps.
// The atoms' blurred volumes phi_i live in a caller-owned device arena; the
// host keeps only k x 6 parameters, the k x k Gram matrix and the trace.
#include <chrono>
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace sfw3d {
namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// numpy's float64 sum (pairwise with an 8-way unrolled base case): the
// reference's weights.sum() in the criterion (solvers.py:266)
double np_sum(const double* a, size_t n) {
  if (n < 8) {
    double r = 0.0;
    for (size_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    size_t i = 8;
    for (; i + 8 <= n; i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  size_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_sum(a, n2) + np_sum(a + n2, n - n2);
}

struct Atom {
  double theta[5];
  double w;
  void* phi;   // device volume H * G(theta)
  int gslot;   // row / column in the Gram cache, -1 = not yet computed
  int xlo, xhi;  // x planes outside which phi is exactly zero (xlo > xhi: wrapped)
};

struct Loop {
  sfw3d_ctx* ctx;
  const sfw3d_psf* psf;
  const sfw3d_table* table;
  int dtype;
  const void* y;
  const sfw3d_solve_options* o;
  int dims[3];
  int64_t n;
  size_t vol_bytes;
  // phi arena slots
  std::vector<void*> free_slots;
  void* rvol = nullptr;      // residual volume
  void* scratch = nullptr;   // render target / back-projection
  bool rvol_valid = false;   // rvol = y - sum w phi of the current state
  // Gram cache over live slots
  std::vector<double> G;     // gcap x gcap row-major
  std::vector<double> b;
  std::vector<void*> gphi;   // phi per Gram slot
  int gcap = 0;

  int render_phi(Atom& a) {
    const double row[6] = {1.0, a.theta[0], a.theta[1], a.theta[2], a.theta[3], a.theta[4]};
    SFW3D_TRY(sfw3d_render(ctx, dtype, dims, row, 1, scratch));
    SFW3D_TRY(sfw3d_psf_apply(ctx, psf, dtype, scratch, a.phi, 0));
    // support along x: the render box (the geometry the render kernel uses)
    // dilated by the PSF's x extent; the separable passes produce exact
    // zeros outside it (a cuFFT PSF does not: full range)
    a.xlo = 0;
    a.xhi = dims[0] - 1;
    std::vector<AtomGeo> geo;
    SFW3D_TRY(build_atoms(dims, row, 1, geo));
    if (psf->separable && !geo[0].full[0]) {
      const long long lo = (long long)geo[0].start[0] + psf->lo[0];
      const long long hi = (long long)geo[0].start[0] + geo[0].len[0] - 1 + psf->hi[0];
      if (hi - lo + 1 < dims[0]) {
        a.xlo = int(((lo % dims[0]) + dims[0]) % dims[0]);
        a.xhi = int(((hi % dims[0]) + dims[0]) % dims[0]);
      }
    }
    return SFW3D_OK;
  }

  // <vecs[q], v> over the x planes [xlo, xhi] of v's support (v is exactly
  // zero elsewhere): one sfw3d_dots per contiguous plane segment
  int dots_on(const std::vector<void*>& vecs, const void* v, int xlo, int xhi, double* out) {
    const int k = int(vecs.size());
    const long long plane = (long long)dims[1] * dims[2];
    const size_t es = dtype_size(dtype);
    int seg[2][2] = {{xlo, xhi}, {0, -1}};
    if (xlo > xhi) { seg[0][1] = dims[0] - 1; seg[1][0] = 0; seg[1][1] = xhi; }
    std::vector<double> part(k);
    std::vector<const void*> ptr(k);
    for (int q = 0; q < k; ++q) out[q] = 0.0;
    for (auto& sg : seg) {
      if (sg[1] < sg[0]) continue;
      const size_t off = size_t(sg[0]) * size_t(plane) * es;
      for (int q = 0; q < k; ++q) ptr[q] = static_cast<const char*>(vecs[q]) + off;
      SFW3D_TRY(sfw3d_dots(ctx, dtype, (long long)(sg[1] - sg[0] + 1) * plane, ptr.data(), k,
                           static_cast<const char*>(v) + off, part.data()));
      for (int q = 0; q < k; ++q) out[q] += part[q];
    }
    return SFW3D_OK;
  }

  // <phi_i, phi_j> and <phi_i, y> for the listed atoms, new rows only
  int gram_system(std::vector<Atom>& atoms, std::vector<double>& g, std::vector<double>& bb) {
    // drop the slots of phis that left the state, compact
    std::vector<int> live(gphi.size(), 0);
    for (const Atom& a : atoms)
      if (a.gslot >= 0) live[a.gslot] = 1;
    bool dead = false;
    for (int v : live) dead = dead || !v;
    if (dead) {
      std::vector<int> map(gphi.size(), -1);
      int m = 0;
      for (size_t s = 0; s < gphi.size(); ++s)
        if (live[s]) map[s] = m++;
      std::vector<double> G2(size_t(m) * m), b2(m);
      std::vector<void*> p2(m);
      for (size_t s = 0; s < gphi.size(); ++s) {
        if (map[s] < 0) continue;
        p2[map[s]] = gphi[s];
        b2[map[s]] = b[s];
        for (size_t t = 0; t < gphi.size(); ++t)
          if (map[t] >= 0) G2[size_t(map[s]) * m + map[t]] = G[s * gcap + t];
      }
      G.swap(G2); b.swap(b2); gphi.swap(p2);
      gcap = m;
      for (Atom& a : atoms)
        if (a.gslot >= 0) a.gslot = map[a.gslot];
    }
    for (Atom& a : atoms) {
      if (a.gslot >= 0) continue;
      const int s = int(gphi.size());
      // grow the matrix by one row / column
      std::vector<double> G2(size_t(s + 1) * (s + 1), 0.0);
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < s; ++j) G2[size_t(i) * (s + 1) + j] = G[size_t(i) * gcap + j];
      G.swap(G2);
      gcap = s + 1;
      b.push_back(0.0);
      gphi.push_back(a.phi);
      a.gslot = s;
      std::vector<double> row(s + 1);
      SFW3D_TRY(dots_on(gphi, a.phi, a.xlo, a.xhi, row.data()));
      for (int q = 0; q <= s; ++q) {
        G[size_t(s) * gcap + q] = row[q];
        G[size_t(q) * gcap + s] = row[q];
      }
      // <phi, y>: y streamed against phi on phi's planes
      const std::vector<void*> yy = {const_cast<void*>(y)};
      SFW3D_TRY(dots_on(yy, a.phi, a.xlo, a.xhi, &b[s]));
    }
    const int k = int(atoms.size());
    g.assign(size_t(k) * k, 0.0);
    bb.assign(k, 0.0);
    for (int i = 0; i < k; ++i) {
      bb[i] = b[atoms[i].gslot];
      for (int j = 0; j < k; ++j) g[size_t(i) * k + j] = G[size_t(atoms[i].gslot) * gcap + atoms[j].gslot];
    }
    return SFW3D_OK;
  }

  // _lasso_on (solvers.py:145-180): fp32 storage takes the exact active-set
  // optimum when it applies, fp64 the reference's coordinate descent
  int lasso(std::vector<Atom>& atoms) {
    std::vector<double> g, bb;
    SFW3D_TRY(gram_system(atoms, g, bb));
    const int k = int(atoms.size());
    std::vector<double> w(k), w0(k);
    for (int i = 0; i < k; ++i) w0[i] = atoms[i].w;
    int32_t info[2] = {0, 0};
    double kkt = 0.0;
    bool done = false;
    if (dtype == SFW3D_F32 && k > 0) {
      w = w0;
      SFW3D_TRY(sfw3d_nnlasso_qp(ctx, k, g.data(), bb.data(), o->lam, o->lasso_tol, o->lasso_max_iter,
                                 w.data(), info, &kkt));
      done = info[1] != 3;
    }
    if (!done) {
      w = w0;
      SFW3D_TRY(sfw3d_nnlasso_cd(ctx, k, g.data(), bb.data(), o->lam, o->lasso_tol, o->lasso_max_iter,
                                 w.data(), info, &kkt));
    }
    for (int i = 0; i < k; ++i) atoms[i].w = w[i];
    return SFW3D_OK;
  }

  // residual volume of the state into rvol, returns 1/2 ||r||^2 + lam sum w
  int criterion(const std::vector<Atom>& atoms, double* c) {
    const int k = int(atoms.size());
    std::vector<const void*> ph(std::max(k, 1));
    std::vector<double> w(std::max(k, 1));
    std::vector<int32_t> xr(2 * std::max(k, 1));
    for (int i = 0; i < k; ++i) {
      ph[i] = atoms[i].phi;
      w[i] = atoms[i].w;
      xr[2 * i] = atoms[i].xlo;
      xr[2 * i + 1] = atoms[i].xhi;
    }
    double ss = 0.0;
    SFW3D_TRY(sfw3d_residual_ranged(ctx, dtype, dims, y, k ? ph.data() : nullptr, k ? w.data() : nullptr,
                                    xr.data(), k, rvol, &ss));
    rvol_valid = true;
    *c = 0.5 * ss + o->lam * np_sum(w.data(), size_t(k));
    return SFW3D_OK;
  }

  int ensure_residual(const std::vector<Atom>& atoms) {
    if (rvol_valid) return SFW3D_OK;
    double c;
    return criterion(atoms, &c);
  }

  // certificate_max (certificate.py:227-236): grid argmax, then the ascent
  int certificate(const std::vector<Atom>& atoms, double theta[5], double* eta) {
    SFW3D_TRY(ensure_residual(atoms));
    sfw3d_argmax best;
    SFW3D_TRY(sfw3d_eta_argmax(ctx, table, dtype, rvol, o->lam, o->window, &best, nullptr, nullptr));
    const int i = best.cand / o->n_shape, j = best.cand % o->n_shape;
    const double start[5] = {double(best.pos[0]), double(best.pos[1]), double(best.pos[2]),
                             o->sigma_grid[i], o->shape_grid[j]};
    SFW3D_TRY(sfw3d_psf_apply(ctx, psf, dtype, rvol, scratch, 1));
    int32_t info[3];
    return sfw3d_refine_eta_max(ctx, dtype, dims, scratch, o->lam, start, o->lower, o->upper, 200, 1e-8,
                                theta, eta, info);
  }

  // prune (solvers.py:269-278): weights <= rel * max weight leave the state
  void prune(std::vector<Atom>& atoms) {
    if (atoms.empty()) return;
    double mx = atoms[0].w;
    for (const Atom& a : atoms) mx = std::max(mx, a.w);
    const double tol = o->prune_rel_tol * mx;
    std::vector<Atom> keep;
    for (const Atom& a : atoms) {
      if (a.w > tol) keep.push_back(a);
      else free_slots.push_back(a.phi);
    }
    if (keep.size() != atoms.size()) {
      atoms.swap(keep);
      rvol_valid = false;
    }
  }

  // local_descent (solvers.py:197-240) + re-rendered phis of the result
  int descend(std::vector<Atom>& atoms, double* c_desc) {
    const int k = int(atoms.size());
    std::vector<double> rows(size_t(k) * 6);
    for (int i = 0; i < k; ++i) {
      rows[6 * i] = atoms[i].w;
      for (int c = 0; c < 5; ++c)
        rows[6 * i + 1 + c] = std::min(std::max(atoms[i].theta[c], o->lower[c]), o->upper[c]);
    }
    int32_t info[3];
    SFW3D_TRY(sfw3d_local_descent(ctx, psf, dtype, y, rows.data(), k, o->lam, o->lower, o->upper,
                                  o->descent_gtol, o->descent_ftol, o->descent_max_iter, c_desc, info));
    for (int i = 0; i < k; ++i) {
      atoms[i].w = rows[6 * i];
      for (int c = 0; c < 5; ++c) atoms[i].theta[c] = rows[6 * i + 1 + c];
      SFW3D_TRY(render_phi(atoms[i]));  // in place: the old phi is dead
      atoms[i].gslot = -1;
    }
    // every cached Gram row referred to the old volumes
    G.clear(); b.clear(); gphi.clear(); gcap = 0;
    rvol_valid = false;
    return SFW3D_OK;
  }
};

}  // namespace
}  // namespace sfw3d

using namespace sfw3d;

extern "C" int sfw3d_solve(sfw3d_ctx* ctx, const sfw3d_psf* psf, const sfw3d_table* table, int dtype,
                           const void* y_dev, const sfw3d_solve_options* opts, void* arena_dev,
                           int arena_volumes, double* rows_out, int* n_atoms, double* criterion_out,
                           int* termination, sfw3d_solve_record* records, int* n_records) {
  SFW3D_CHECK_ARG(ctx && psf && table && y_dev && opts && arena_dev && rows_out && n_atoms &&
                      criterion_out && termination && records && n_records, "NULL argument");
  SFW3D_CHECK_ARG(dtype == SFW3D_F32 || dtype == SFW3D_F64, "dtype");
  SFW3D_CHECK_ARG(opts->lam > 0.0, "lam must be > 0");
  SFW3D_CHECK_ARG(opts->max_outer_iterations >= 1, "max_outer_iterations must be >= 1");
  SFW3D_CHECK_ARG(arena_volumes >= 3, "arena too small");  // (SFW3D_ENOMEM when atoms outgrow it)
  SFW3D_CHECK_ARG(opts->sigma_grid && opts->shape_grid && opts->n_sigma > 0 && opts->n_shape > 0, "grids");
  Loop L{ctx, psf, table, dtype, y_dev, opts};
  for (int a = 0; a < 3; ++a) L.dims[a] = psf->dims[a];
  L.n = vol_count(L.dims);
  L.vol_bytes = size_t(L.n) * dtype_size(dtype);
  char* base = static_cast<char*>(arena_dev);
  L.rvol = base;
  L.scratch = base + L.vol_bytes;
  for (int s = arena_volumes - 1; s >= 2; --s) L.free_slots.push_back(base + size_t(s) * L.vol_bytes);

  std::vector<Atom> state;
  double crit = 0.0;
  SFW3D_TRY(L.criterion(state, &crit));  // 1/2 ||y||^2; rvol = y
  const double stop_at = opts->eta_threshold + opts->eta_slack;
  int term = SFW3D_TERM_ITERATION_CAP, dup_streak = 0, nrec = 0;
  const double nan = std::nan("");

  for (int k = 1; k <= opts->max_outer_iterations; ++k) {
    const double c_before = crit;
    sfw3d_solve_record& rec = records[nrec];
    rec = {k, 0.0, c_before, nan, nan, 0, 0.0, 0.0, 0.0};
    double t0 = now_s();
    double theta[5], eta = 0.0;
    SFW3D_TRY(L.certificate(state, theta, &eta));
    rec.eta_max = eta;
    rec.t_certificate = now_s() - t0;

    if (eta <= stop_at) {
      term = SFW3D_TERM_CERTIFICATE;
      if (opts->boosted && !state.empty()) {
        t0 = now_s();
        // final slide and re-check; the slid state replaces the current one
        // only if it lowers the criterion and keeps the certificate
        std::vector<Atom> slid = state;
        double c_desc = 0.0;
        SFW3D_TRY(L.descend(slid, &c_desc));
        L.prune(slid);
        double th2[5], eta_slid = 0.0;
        SFW3D_TRY(L.certificate(slid, th2, &eta_slid));
        if (c_desc <= crit && eta_slid <= stop_at) {
          state.swap(slid);
          crit = c_desc;
        }
        rec.t_descent = now_s() - t0;
      }
      if (opts->boosted) rec.criterion_after_descent = crit;
      rec.atom_count = int(state.size());
      ++nrec;
      break;
    }

    bool duplicate = false;
    for (const Atom& a : state) {
      double mx = 0.0;
      for (int c = 0; c < 5; ++c) mx = std::max(mx, std::fabs(theta[c] - a.theta[c]));
      if (mx <= opts->duplicate_tol) { duplicate = true; break; }
    }

    t0 = now_s();
    if (L.free_slots.empty()) {
      set_error("internal: phi arena exhausted");
      return SFW3D_ENOMEM;
    }
    Atom a{};
    for (int c = 0; c < 5; ++c) a.theta[c] = theta[c];
    a.w = 0.0;
    a.phi = L.free_slots.back();
    a.gslot = -1;
    L.free_slots.pop_back();
    SFW3D_TRY(L.render_phi(a));
    state.push_back(a);
    SFW3D_TRY(L.lasso(state));
    SFW3D_TRY(L.criterion(state, &crit));
    rec.criterion_after_lasso = crit;
    rec.t_lasso = now_s() - t0;

    if (!opts->boosted) {
      t0 = now_s();
      double c_desc = 0.0;
      SFW3D_TRY(L.descend(state, &c_desc));
      crit = c_desc;
      rec.criterion_after_descent = c_desc;
      rec.t_descent = now_s() - t0;
    }
    L.prune(state);
    rec.atom_count = int(state.size());
    ++nrec;

    if (duplicate && crit >= c_before * (1.0 - 1e-12)) {
      if (++dup_streak >= 2) { term = SFW3D_TERM_STALLED; break; }
    } else {
      dup_streak = 0;
    }
  }
  *n_atoms = int(state.size());
  for (size_t i = 0; i < state.size(); ++i) {
    rows_out[6 * i] = state[i].w;
    for (int c = 0; c < 5; ++c) rows_out[6 * i + 1 + c] = state[i].theta[c];
  }
  *criterion_out = crit;
  *termination = term;
  *n_records = nrec;
  return SFW3D_OK;
}
