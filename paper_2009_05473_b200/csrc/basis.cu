// Shared separable Gaussian basis for the dual certificate (K1 fast path).
//
// Every certificate candidate is a unit atom G_c(v) = g_c(|v|^2) with
// g_c(s) = exp(-s^(d/2) / (2 sigma^d)) on the reference's support box
// (_unit_atom, forward.py:119-137; certificate.py:86-92). For d <= 2, g_c is
// completely monotone in s, so it is a positive mixture of Gaussians
// exp(-beta s) — and a Gaussian of |v|^2 is separable, f(a) f(b) f(c). Here
// all basis candidates of a table share ONE dictionary of betas (geometric
// over the common box, plus the exact 1/(2 sigma^2) of every d == 2
// candidate) and are fitted on it by non-negative least squares on the
// lattice values s of the common box:
//     G_c(v) ~ w0_c [v == 0] + sum_k W[c][k] exp(-beta_k |v|^2).
// The certificate then costs, per voxel,
//   * one separable pass triple per SHARED term k:  T_k = f_k^(x,y,z) * b,
//   * one fused kernel that reads b and every T_k once and forms
//     eta_c = (w0_c b + sum_k W[c][k] T_k) / lam for every member c, with the
//     windowed argmax per member (and the fields when requested),
// instead of (2R+1)^3 taps per candidate. Candidates whose fit error on the
// common box exceeds the tolerance stay on the direct kernels (eta.cu).
// Factors are truncated where exp(-beta t^2) < trunc / max_c(sum_k W[c][k])
// (trunc = 1e-12 for fp64, 1e-9 for fp32 storage), which adds at most trunc
// to every member's error (fp64: included in the recorded error).
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <thread>
#include <type_traits>

#include "basis.cuh"
#include "window.cuh"

namespace sfw3d {

// ------------------------------------------------------------------ NNLS
// Lawson-Hanson non-negative least squares min ||A x - g||, x >= 0, with the
// passive-set subproblems solved by Householder QR in extended precision
// (x86 long double): the exponential columns are nearly collinear.
namespace {
using ld = long double;

void lsq_qr(const std::vector<ld>& A, int M, const std::vector<int>& cols, const std::vector<ld>& g,
            std::vector<ld>& z) {
  const int p = int(cols.size());
  std::vector<ld> B(size_t(M) * p), rhs(g), scale(p), v(M);
  for (int j = 0; j < p; ++j) {
    ld s = 0.0L;
    for (int i = 0; i < M; ++i) s += A[size_t(cols[j]) * M + i] * A[size_t(cols[j]) * M + i];
    scale[j] = s > 0 ? 1.0L / std::sqrt(s) : 1.0L;
    for (int i = 0; i < M; ++i) B[size_t(j) * M + i] = A[size_t(cols[j]) * M + i] * scale[j];
  }
  for (int j = 0; j < p; ++j) {
    ld* c = &B[size_t(j) * M];
    ld nrm = 0.0L;
    for (int i = j; i < M; ++i) nrm += c[i] * c[i];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0L) continue;
    const ld alpha = c[j] > 0 ? -nrm : nrm;
    for (int i = j; i < M; ++i) v[i] = c[i];
    v[j] -= alpha;
    ld vn = 0.0L;
    for (int i = j; i < M; ++i) vn += v[i] * v[i];
    if (vn == 0.0L) continue;
    auto apply = [&](ld* col) {
      ld dot = 0.0L;
      for (int i = j; i < M; ++i) dot += v[i] * col[i];
      const ld f = 2.0L * dot / vn;
      for (int i = j; i < M; ++i) col[i] -= f * v[i];
    };
    for (int k = j; k < p; ++k) apply(&B[size_t(k) * M]);
    apply(rhs.data());
  }
  z.assign(p, 0.0L);
  for (int j = p - 1; j >= 0; --j) {
    ld s = rhs[j];
    for (int k = j + 1; k < p; ++k) s -= B[size_t(k) * M + j] * z[k];
    const ld r = B[size_t(j) * M + j];
    z[j] = r != 0.0L ? s / r : 0.0L;
  }
  for (int j = 0; j < p; ++j) z[j] *= scale[j];
}

// Householder compression of a tall least-squares problem: R (p x p upper,
// column-major in a p x p block) and c = (Q^T g)[0:p] with A = Q R (thin).
// min ||A z - g||^2 + |D z|^2 = min ||[R; D] z - [c; 0]||^2 + const, so a
// ridge sweep solves (2p x p) systems instead of (M + p) x p ones.
void qr_compress(const std::vector<ld>& A, int M, int p, const std::vector<ld>& g,
                 std::vector<ld>& R, std::vector<ld>& c) {
  std::vector<ld> B(A.begin(), A.begin() + size_t(M) * p), rhs(g.begin(), g.begin() + M), v(M);
  for (int j = 0; j < p; ++j) {
    ld* col = &B[size_t(j) * M];
    ld nrm = 0.0L;
    for (int i = j; i < M; ++i) nrm += col[i] * col[i];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0L) continue;
    const ld alpha = col[j] > 0 ? -nrm : nrm;
    for (int i = j; i < M; ++i) v[i] = col[i];
    v[j] -= alpha;
    ld vn = 0.0L;
    for (int i = j; i < M; ++i) vn += v[i] * v[i];
    if (vn == 0.0L) continue;
    auto apply = [&](ld* x) {
      ld dot = 0.0L;
      for (int i = j; i < M; ++i) dot += v[i] * x[i];
      const ld f = 2.0L * dot / vn;
      for (int i = j; i < M; ++i) x[i] -= f * v[i];
    };
    for (int k = j; k < p; ++k) apply(&B[size_t(k) * M]);
    apply(rhs.data());
  }
  R.assign(size_t(p) * p, 0.0L);
  for (int k = 0; k < p; ++k)
    for (int i = 0; i <= k && i < M; ++i) R[size_t(k) * p + i] = B[size_t(k) * M + i];
  c.assign(rhs.begin(), rhs.begin() + std::min(p, M));
  c.resize(p, 0.0L);
}

void nnls(const std::vector<double>& Ad, int M, int N, const std::vector<double>& gd,
          std::vector<double>& xd) {
  std::vector<ld> A(Ad.begin(), Ad.end()), g(gd.begin(), gd.end()), x(N, 0.0L), cn(N);
  std::vector<char> passive(N, 0), banned(N, 0);
  ld gn = 0.0L;
  for (ld v : g) gn += v * v;
  const ld tol = 1e-17L * std::sqrt(gn);
  if (M > N) {
    // tall problem: compress to the N x N triangular form once (A = Q R,
    // A^T (g - A x) = R^T (Q^T g - R x)): every residual, gradient and
    // passive-set solve below then runs on N rows instead of M
    std::vector<ld> R, c;
    qr_compress(A, M, N, g, R, c);
    A.swap(R);
    g.swap(c);
    M = N;
  }
  std::vector<ld> r(M);
  for (int j = 0; j < N; ++j) {
    ld s = 0.0L;
    for (int i = 0; i < M; ++i) s += A[size_t(j) * M + i] * A[size_t(j) * M + i];
    cn[j] = s > 0.0L ? std::sqrt(s) : 1.0L;
  }
  for (int outer = 0; outer < 8 * N; ++outer) {
    for (int i = 0; i < M; ++i) {
      ld s = g[i];
      for (int j = 0; j < N; ++j)
        if (x[j] != 0.0L) s -= A[size_t(j) * M + i] * x[j];
      r[i] = s;
    }
    int jmax = -1;
    ld best = tol;
    for (int j = 0; j < N; ++j) {
      if (passive[j] || banned[j]) continue;
      ld s = 0.0L;
      for (int i = 0; i < M; ++i) s += A[size_t(j) * M + i] * r[i];
      s /= cn[j];
      if (s > best) {
        best = s;
        jmax = j;
      }
    }
    if (jmax < 0) break;
    passive[jmax] = 1;
    bool first = true, added = true;
    for (int inner = 0; inner < 3 * N; ++inner) {
      std::vector<int> cols;
      for (int j = 0; j < N; ++j)
        if (passive[j]) cols.push_back(j);
      std::vector<ld> z;
      lsq_qr(A, M, cols, g, z);
      bool ok = true;
      for (ld v : z) ok &= v > 0.0L;
      if (ok) {
        std::fill(x.begin(), x.end(), 0.0L);
        for (size_t q = 0; q < cols.size(); ++q) x[cols[q]] = z[q];
        break;
      }
      if (first) {  // the entering column itself came out non-positive: skip it
        size_t qn = 0;
        while (cols[qn] != jmax) ++qn;
        if (z[qn] <= 0.0L) {
          passive[jmax] = 0;
          banned[jmax] = 1;
          added = false;
          break;
        }
      }
      first = false;
      ld alpha = 2.0L;
      int qmin = -1;
      for (size_t q = 0; q < cols.size(); ++q)
        if (z[q] <= 0.0L) {
          const ld xv = x[cols[q]];
          const ld a = xv / (xv - z[q]);
          if (a < alpha) {
            alpha = a;
            qmin = int(q);
          }
        }
      for (size_t q = 0; q < cols.size(); ++q) {
        const int j = cols[q];
        x[j] += alpha * (z[q] - x[j]);
        if (int(q) == qmin || x[j] <= 0.0L) {
          x[j] = 0.0L;
          passive[j] = 0;
        }
      }
    }
    if (added) std::fill(banned.begin(), banned.end(), 0);
  }
  xd.assign(x.begin(), x.end());
}

// lattice values s = a^2 + b^2 + c^2 of an offset box, and the fitting subset
// (every s <= 256, then geometric 0.4% steps: the profile is smooth there)
void box_lattice(const int lo[3], const int hi[3], std::vector<double>& S, std::vector<double>& Sfit) {
  int smax = 0;
  for (int a = 0; a < 3; ++a) smax += std::max(lo[a] * lo[a], hi[a] * hi[a]);
  std::vector<char> present(size_t(smax) + 1, 0);
  std::vector<int> sv[3];
  for (int ax = 0; ax < 3; ++ax) {
    std::vector<char> sq(size_t(smax) + 1, 0);
    for (int t = lo[ax]; t <= hi[ax]; ++t) sq[size_t(t) * t] = 1;
    for (int s = 0; s <= smax; ++s)
      if (sq[s]) sv[ax].push_back(s);
  }
  for (int s0 : sv[0])
    for (int s1 : sv[1])
      for (int s2 : sv[2]) present[size_t(s0) + s1 + s2] = 1;
  S.clear();
  for (int s = 0; s <= smax; ++s)
    if (present[s]) S.push_back(double(s));
  Sfit.clear();
  double next = 256.0;
  for (double s : S)
    if (s <= 256.0 || s >= next) {
      Sfit.push_back(s);
      if (s > 256.0) next = s * 1.01;
    }
}

double profile(double s, double sigma, double d) {
  return std::exp(-(0.5 / std::pow(sigma, d)) * std::pow(s, 0.5 * d));
}

// NNLS fit of one profile on a dictionary; returns weights (dict order), w0
// and the max abs error over all lattice values S.
double fit_on(const std::vector<double>& dict, const std::vector<double>& S,
              const std::vector<double>& Sfit, double sigma, double d, std::vector<double>& w,
              double& w0) {
  const int K = int(dict.size()), M = int(Sfit.size());
  std::vector<double> A(size_t(M) * (K + 1)), g(M);
  for (int i = 0; i < M; ++i) {
    const double s = Sfit[i];
    g[i] = profile(s, sigma, d);
    for (int k = 0; k < K; ++k) A[size_t(k) * M + i] = std::exp(-dict[k] * s);
    A[size_t(K) * M + i] = s == 0.0 ? 1.0 : 0.0;  // delta term
  }
  std::vector<double> x;
  nnls(A, M, K + 1, g, x);
  w.assign(x.begin(), x.begin() + K);
  w0 = x[K];
  double err = 0.0;
  for (double s : S) {
    double v = s == 0.0 ? w0 : 0.0;
    for (int k = 0; k < K; ++k)
      if (w[k] > 0.0) v += std::exp(-dict[k] * s) * w[k];
    err = std::max(err, std::fabs(v - profile(s, sigma, d)));
  }
  return err;
}

std::vector<double> geometric(double lo, double hi, int K) {
  std::vector<double> out(K);
  for (int k = 0; k < K; ++k) out[k] = lo * std::pow(hi / lo, double(k) / (K - 1));
  return out;
}

int upload(void** dst, const void* src, size_t bytes) {
  SFW3D_CUDA_TRY(cudaMalloc(dst, bytes));
  SFW3D_CUDA_TRY(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
  return SFW3D_OK;
}

}  // namespace

void fit_profile(const int lo[3], const int hi[3], double sigma, double d, double target,
                 double& w0, std::vector<std::pair<double, double>>& terms, double& err,
                 bool& exact) {
  terms.clear();
  if (d == 2.0) {  // exp(-s / (2 sigma^2)): one exact separable term
    exact = true;
    err = 0.0;
    w0 = 0.0;
    terms.push_back({0.5 / (sigma * sigma), 1.0});
    return;
  }
  exact = false;
  std::vector<double> S, Sfit;
  box_lattice(lo, hi, S, Sfit);
  const double rmax = std::max({-lo[0], hi[0], -lo[1], hi[1], -lo[2], hi[2], 1});
  err = INFINITY;
  for (const int K : {48, 96}) {
    std::vector<double> dict = geometric(0.5 / (rmax * rmax), 30.0, K), w;
    double z0;
    const double e = fit_on(dict, S, Sfit, sigma, d, w, z0);
    if (e < err) {
      err = e;
      w0 = z0;
      terms.clear();
      for (int k = 0; k < K; ++k)
        if (w[k] > 0.0) terms.push_back({dict[k], w[k]});
    }
    if (err <= target) break;
  }
}

// ------------------------------------------------------------------ set
struct BasisSet {
  int dtype;
  int lo[3], hi[3];                 // common offset box
  std::vector<double> betas;        // shared terms
  std::vector<int> tlo[3], tlen[3];  // per term, per axis tap range (of the passes)
  // chained terms (fp32): T_t = (g_t x g_t x g_t) * T_parent[t] instead of
  // f_t^3 * b, with g_t the Gaussian whose convolution with the parent's
  // factor is f_t (variances add); parent -1 = from b. The effective factor
  // (parent's effective factor convolved with g_t, as the passes compute it)
  // on [elo, elo + elen) per axis is what the signed bounds use.
  std::vector<int> parent;
  std::vector<int> elo[3], elen[3];
  std::vector<void*> taps;          // per term: 3 axes contiguous, storage dtype
  std::vector<int> members;         // candidate ids on the basis path
  std::vector<double> W, w0;        // [member][term], [member]
  std::vector<double> fit_err;      // per candidate (inf when not fitted)
  std::vector<char> is_member;      // per candidate: 1 non-negative fit, 2 signed
  int n_nnls = 0;                   // members [0, n_nnls) non-negative, then signed
  std::vector<double> ebound;       // per candidate: signed members' bound factor
  void* W_dev = nullptr;            // storage dtype, [member][term]
  void* w0_dev = nullptr;
  int* cid_dev = nullptr;           // member -> candidate id
  long long taps_per_voxel = 0;
  int device = 0;
  // mix_ring2_kernel: dense members (W rows [nmd][K], w0) and copy members
  // (one weight-1 term, w0 = 0) with cterm[k] = copy slot of term k or -1
  int nmd = 0, nmc = 0;
  void* Wd_dev = nullptr;
  void* w0d_dev = nullptr;
  int* dmem_dev = nullptr;
  int* cmem_dev = nullptr;
  int* cterm_dev = nullptr;
};

// coarse dictionary size (the fine one has 2 * kDictCoarse - 1 points)
constexpr int kDictCoarse = 49;
// tangent betas per d < 2 candidate (s = 1, 2, 4, ..., 2^(kTangents-1))
constexpr int kTangents = 10;
// no fit is accepted below this bound (double-precision evaluation floor)
constexpr double kFitFloor = 1e-11;

// ------------------------------------------------------------ signed members
// A candidate outside the non-negative pool (d > 2: g_c is not completely
// monotone) is fitted on the SHARED terms by weighted-ridge least squares with
// signed weights. Its basis value eta~ then differs from the direct value at
// EVERY voxel m by at most
//   lam |eta~(m) - eta(m)| <= ||b||_inf (D1 + R),
//   D1 = sum_{v in C} |G~(v) - G_dir(v)| + tap_tol |B_c|
//        (the exact mixture with the stored factors and weights against the
//        candidate's direct template g_c(|v|^2) on its box B_c, over the
//        common box C that the passes cover),
//   R  = sum_k |W_k| S_k (rho_k + g_mix (1 + rho_k)) + |w0| g_mix
//        (floating-point rounding: a pass of L taps is an L-term FMA chain,
//        rho_k = 1.01 u (Lx + Ly + Lz) for the three passes of term k, S_k the
//        factor mass over C, g_mix = 1.01 u (K + 2) for the (K + 1)-term mix).
// The ridge weight trades D1 against R (large signed weights amplify the
// rounding) and is picked to minimise D1 + R. eta.cu collects every voxel
// within 2 E of the approximate maximum and re-evaluates it directly.
namespace {

constexpr int kRidgeMin = -34, kRidgeMax = -6;  // ridge weights 10^e (and 0)

void fit_signed_members(BasisSet* s, const std::vector<BasisCandidate>& cands, int dtype,
                        const std::vector<double>& Sfit,
                        const std::vector<std::vector<double>>& hstore,
                        const std::vector<double>& pass_taps) {
  const int nc = int(cands.size()), nt = int(s->betas.size());
  const double u = dtype == SFW3D_F64 ? 0x1p-53 : 0x1p-24;
  // acceptance of a signed member: bound E <= accept x template mass. A
  // member's maxima are refined exactly whatever E is; E only sizes the
  // refinement set. fp32: 0.1 (with the 1e-5 loose term selection, config 4
  // keeps all 16 members on 12 shared terms, ~360 refined voxels); fp64: 0.01
  const double accept = dtype == SFW3D_F32 ? 0.1 : 0.01;
  // per term: (effective) factor mass, its part outside the common box C
  // (chained factors may reach past C, where every template is 0), and the
  // passes' rounding factor (a chained term adds its own passes' rounding
  // to its parent's, relative to the same mass)
  std::vector<double> Sk(nt), rho(nt), ext(nt);
  std::vector<size_t> aoff[3];
  for (int a = 0; a < 3; ++a) aoff[a].resize(nt);
  for (int t = nt - 1; t >= 0; --t) {  // parents (narrower) have larger indices
    double prod = 1.0, pin = 1.0;
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
      aoff[a][t] = off;
      double sa = 0.0, si = 0.0;
      for (int q = 0; q < s->elen[a][t]; ++q) {
        const double v = std::fabs(hstore[t][off + q]);
        sa += v;
        const int o = s->elo[a][t] + q;
        if (o >= s->lo[a] && o <= s->hi[a]) si += v;
      }
      off += s->elen[a][t];
      prod *= sa;
      pin *= si;
    }
    Sk[t] = prod;
    ext[t] = std::max(0.0, prod - pin);
    rho[t] = 1.01 * u * pass_taps[t] + (s->parent[t] >= 0 ? rho[s->parent[t]] * (1.0 + 1.01 * u * pass_taps[t]) : 0.0);
  }
  // the mix's rounding: (K + 1)-term FFMA chains in the storage precision
  const double gmix = 1.01 * u * (nt + 2);
  // axis representatives: offsets +t and -t share one (multiplicity 2) when
  // both lie in C and every factor is defined at both
  struct Rep {
    int t;
    double w;
  };
  std::vector<Rep> reps[3];
  std::vector<std::vector<double>> fval[3];  // [a][rep][term]
  for (int a = 0; a < 3; ++a) {
    const int lo = s->lo[a], hi = s->hi[a];
    auto in_term = [&](int t, int k) { return t >= s->elo[a][k] && t < s->elo[a][k] + s->elen[a][k]; };
    for (int t = 0; t <= std::max(-lo, hi); ++t) {
      const bool pos = t >= lo && t <= hi, neg = t > 0 && -t >= lo && -t <= hi;
      bool same = pos && neg;
      for (int k = 0; same && k < nt; ++k) same = in_term(t, k) == in_term(-t, k);
      if (same) {
        reps[a].push_back({t, 2.0});
      } else {
        if (pos) reps[a].push_back({t, 1.0});
        if (neg) reps[a].push_back({-t, 1.0});
      }
    }
    for (const Rep& r : reps[a]) {
      std::vector<double> f(nt, 0.0);
      for (int k = 0; k < nt; ++k)
        if (in_term(r.t, k)) f[k] = hstore[k][aoff[a][k] + (r.t - s->elo[a][k])];
      fval[a].push_back(std::move(f));
    }
  }
  std::vector<int> todo;
  for (int c = 0; c < nc; ++c) {
    if (s->is_member[c]) continue;
    bool ok = true;
    for (int a = 0; a < 3; ++a)
      ok &= cands[c].lo[a] == -cands[c].hi[a] && cands[c].lo[a] >= s->lo[a] &&
            cands[c].hi[a] <= s->hi[a];
    if (ok) todo.push_back(c);
  }
  if (todo.empty()) return;
  const int M = int(Sfit.size()), ncol = nt + 1, Mt = 2 * ncol;
  std::vector<std::vector<double>> wsig(nc);
  std::vector<double> w0sig(nc, 0.0), esig(nc, INFINITY), dsig(nc, INFINITY), mass(nc, 0.0);
  auto fit_one = [&](int c) {
    const BasisCandidate& bc = cands[c];
    // the lattice fit, compressed once (qr_compress); each ridge weight then
    // solves [R; sqrt(mu) diag(pen)] z = [Q^T g; 0]
    std::vector<ld> A(size_t(Mt) * ncol, 0.0L), g(Mt, 0.0L);
    {
      std::vector<ld> Af(size_t(M) * ncol, 0.0L), gf(M, 0.0L), Rc, cc;
      for (int i = 0; i < M; ++i) {
        gf[i] = profile(Sfit[i], bc.sigma, bc.d);
        for (int k = 0; k < nt; ++k) Af[size_t(k) * M + i] = std::exp(-(ld)s->betas[k] * Sfit[i]);
        Af[size_t(nt) * M + i] = Sfit[i] == 0.0 ? 1.0L : 0.0L;
      }
      qr_compress(Af, M, ncol, gf, Rc, cc);
      for (int k = 0; k < ncol; ++k)
        for (int i = 0; i < ncol; ++i) A[size_t(k) * Mt + i] = Rc[size_t(k) * ncol + i];
      for (int i = 0; i < ncol; ++i) g[i] = cc[i];
    }
    std::vector<double> pen(ncol);
    for (int k = 0; k < nt; ++k) pen[k] = Sk[k] * (rho[k] + gmix * (1.0 + rho[k])) + ext[k];
    pen[nt] = gmix;
    std::vector<int> cols(ncol);
    for (int k = 0; k < ncol; ++k) cols[k] = k;
    // the direct template at every representative triple (independent of the
    // ridge weight: tabulated once)
    const size_t nrx = reps[0].size(), nry = reps[1].size(), nrz = reps[2].size();
    std::vector<double> gdt(nrx * nry * nrz, 0.0);
    for (size_t ix = 0; ix < nrx; ++ix)
      for (size_t iy = 0; iy < nry; ++iy) {
        const int tx = reps[0][ix].t, ty = reps[1][iy].t;
        if (std::abs(tx) > bc.hi[0] || std::abs(ty) > bc.hi[1]) continue;
        const double sxy = double(tx) * tx + double(ty) * ty;
        for (size_t iz = 0; iz < nrz; ++iz) {
          const int tz = reps[2][iz].t;
          if (std::abs(tz) <= bc.hi[2])
            gdt[(ix * nry + iy) * nrz + iz] = profile(sxy + double(tz) * tz, bc.sigma, bc.d);
        }
      }
    // the direct template on its box, per representative triple
    double m = 0.0;
    for (int x = bc.lo[0]; x <= bc.hi[0]; ++x)
      for (int y = bc.lo[1]; y <= bc.hi[1]; ++y)
        for (int z = bc.lo[2]; z <= bc.hi[2]; ++z)
          m += profile(double(x) * x + double(y) * y + double(z) * z, bc.sigma, bc.d);
    mass[c] = m;
    const double box_taps = double(bc.hi[0] - bc.lo[0] + 1) * (bc.hi[1] - bc.lo[1] + 1) *
                            (bc.hi[2] - bc.lo[2] + 1);
    std::vector<double> P(nt);
    int best_e = kRidgeMin - 1;
    // one ridge weight 10^e (e < kRidgeMin: none): solve, bound, keep the best
    auto try_ridge = [&](int e) {
      const ld mu = e < kRidgeMin ? 0.0L : std::pow(10.0L, (ld)e);
      for (int k = 0; k < ncol; ++k) A[size_t(k) * Mt + ncol + k] = std::sqrt(mu) * (ld)pen[k];
      std::vector<ld> z;
      lsq_qr(A, Mt, cols, g, z);
      std::vector<double> w(nt);
      bool finite = true;
      for (int k = 0; k < nt; ++k) {
        w[k] = dtype == SFW3D_F64 ? double(z[k]) : double(float(z[k]));
        finite &= std::isfinite(w[k]);
      }
      double w0 = dtype == SFW3D_F64 ? double(z[nt]) : double(float(z[nt]));
      if (!finite || !std::isfinite(w0)) return;
      double R = std::fabs(w0) * gmix;
      for (int k = 0; k < nt; ++k) R += std::fabs(w[k]) * pen[k];
      if (R >= esig[c]) return;
      double D1 = bc.tap_tol * box_taps;
      for (size_t ix = 0; ix < reps[0].size(); ++ix) {
        const Rep rx = reps[0][ix];
        for (size_t iy = 0; iy < reps[1].size(); ++iy) {
          const Rep ry = reps[1][iy];
          for (int k = 0; k < nt; ++k) P[k] = w[k] * fval[0][ix][k] * fval[1][iy][k];
          const double* gdr = &gdt[(ix * nry + iy) * nrz];
          double acc = 0.0;
          for (size_t iz = 0; iz < nrz; ++iz) {
            const Rep rz = reps[2][iz];
            const std::vector<double>& fz = fval[2][iz];
            double gv = (rx.t == 0 && ry.t == 0 && rz.t == 0) ? w0 : 0.0;
            for (int k = 0; k < nt; ++k) gv += P[k] * fz[k];
            acc += rz.w * std::fabs(gv - gdr[iz]);
          }
          D1 += rx.w * ry.w * acc;
        }
        if (D1 + R >= esig[c]) break;
      }
      if (D1 + R < esig[c]) {
        esig[c] = D1 + R;
        dsig[c] = D1;
        wsig[c] = w;
        w0sig[c] = w0;
        best_e = e;
      }
    };
    // coarse scan (every 3 decades, and no ridge), then the neighbours of the best
    try_ridge(kRidgeMin - 1);
    for (int e = kRidgeMin; e <= kRidgeMax; e += 3) try_ridge(e);
    const int e0 = best_e;
    if (e0 >= kRidgeMin)
      for (int e : {e0 - 2, e0 - 1, e0 + 1, e0 + 2})
        if (e >= kRidgeMin && e <= kRidgeMax) try_ridge(e);
  };
  {
    const int nthreads =
        std::max(1, std::min<int>(int(todo.size()), int(std::thread::hardware_concurrency())));
    std::atomic<int> next{0};
    std::vector<std::thread> workers;
    for (int w = 0; w < nthreads; ++w)
      workers.emplace_back([&] {
        for (int q = next++; q < int(todo.size()); q = next++) fit_one(todo[q]);
      });
    for (auto& th : workers) th.join();
  }
  for (int c : todo) {
    const bool ok = std::isfinite(esig[c]) && esig[c] <= accept * mass[c];
    if (!ok) continue;
    s->is_member[c] = 2;
    s->ebound[c] = esig[c];
    s->fit_err[c] = esig[c];  // (signed members report their bound factor)
    s->members.push_back(c);
    s->W.insert(s->W.end(), wsig[c].begin(), wsig[c].end());
    s->w0.push_back(w0sig[c]);
  }
}

}  // namespace

// fp32 default: config 4 measured 26 -> 12 shared terms at 1e-5 (with the
// fp32 signed acceptance 0.1), 31.3 -> 12.5 ms per certificate; 5e-5 drops one
// more wide term (11 terms, ~1240 refined voxels, 11.7 ms; tools/loose_scan.py:
// 1e-4 and looser lose members to the direct kernels). The table option
// "loose_tol" overrides; 0 disables.
constexpr double kLooseF32 = 5e-5;
double basis_loose_tol(int dtype) { return dtype == SFW3D_F32 ? kLooseF32 : 0.0; }

int basis_set_build(const int dims[3], const std::vector<BasisCandidate>& cands, int dtype,
                    double tol, BasisSet** out, bool on_device, bool prune, double loose) {
  // loose > tol: the shared terms are chosen (fits, pruning) for members
  // within `loose`; members that miss `tol` are then refitted as signed
  // members on those terms (certified bound, exact refinement of maxima)
  loose = std::max(loose, tol);
  // factor truncation: exp(-beta q^2) below trunc / max_c sum_k W_ck is cut,
  // which adds at most `trunc` to a member's error. 1e-12 for fp64 (the
  // reference's own tail cutoff; part of the recorded fit error). 1e-9 for
  // fp32 storage: two decades under fp32's own resolution, four under the
  // 1e-5 bar; fp32 members are either signed — their certified bounds are
  // computed from the effective, truncated factors, so the cut is inside the
  // bound — or unrefined members whose error is fp32 rounding anyway. It
  // shortens every fp32 filter by ~13%.
  const double trunc = dtype == SFW3D_F32 ? 1e-9 : 1e-12;
  auto* s = new BasisSet();
  s->dtype = dtype;
  cudaGetDevice(&s->device);
  const int nc = int(cands.size());
  s->fit_err.assign(nc, INFINITY);
  s->is_member.assign(nc, 0);
  // candidates that can have a positive Gaussian mixture (d <= 2)
  std::vector<int> pool;
  for (int c = 0; c < nc; ++c)
    if (cands[c].d <= 2.0) pool.push_back(c);
  *out = s;
  if (pool.empty()) return SFW3D_OK;
  // common box: union of the pool's boxes
  for (int a = 0; a < 3; ++a) {
    s->lo[a] = 0;
    s->hi[a] = 0;
    for (int c : pool) {
      s->lo[a] = std::min(s->lo[a], cands[c].lo[a]);
      s->hi[a] = std::max(s->hi[a], cands[c].hi[a]);
    }
    if (s->hi[a] - s->lo[a] + 1 > dims[a]) {  // never wider than the axis
      s->lo[a] = -(dims[a] / 2);
      s->hi[a] = s->lo[a] + dims[a] - 1;
    }
  }
  std::vector<double> S, Sfit;
  box_lattice(s->lo, s->hi, S, Sfit);
  const double rmax = std::max({-s->lo[0], s->hi[0], -s->lo[1], s->hi[1], -s->lo[2], s->hi[2], 1});
  // nested geometric dictionaries over [0.5 / rmax^2, 30] (the coarse one is
  // every other point of the fine one) plus the exact 1/(2 sigma^2) of every
  // d == 2 candidate
  const double bmin = 0.5 / (rmax * rmax);
  std::vector<double> fine = geometric(bmin, 30.0, 2 * kDictCoarse - 1);
  for (int c : pool)
    if (cands[c].d == 2.0) fine.push_back(0.5 / (cands[c].sigma * cands[c].sigma));
  // tangent betas of a d < 2 candidate: the Gaussian matching the profile's
  // log-slope at s = 2^j (d/2 s^(d/2-1) / (2 sigma^d)); they let the fine fit
  // of a near-Gaussian profile (d close to 2) reach tol where the geometric
  // grid alone stalls at a few 1e-9
  std::vector<std::vector<double>> tangents(nc);
  for (int c : pool) {
    if (cands[c].d >= 2.0) continue;
    const double a0 = 0.5 / std::pow(cands[c].sigma, cands[c].d) * 0.5 * cands[c].d;
    for (int j = 0; j < kTangents; ++j) {
      const double b = a0 * std::pow(double(1 << j), 0.5 * cands[c].d - 1.0);
      if (b >= 0.5 * bmin && b <= 30.0) tangents[c].push_back(b);
    }
  }
  std::vector<double> dict(fine);
  for (int c : pool) dict.insert(dict.end(), tangents[c].begin(), tangents[c].end());
  std::sort(dict.begin(), dict.end());
  dict.erase(std::unique(dict.begin(), dict.end()), dict.end());
  const int K = int(dict.size());
  auto index_of = [&](double b) {
    const auto it = std::min_element(dict.begin(), dict.end(), [&](double x, double y) {
      return std::fabs(x - b) < std::fabs(y - b);
    });
    return int(it - dict.begin());
  };
  std::vector<int> coarse_idx, fine_idx;  // positions of the grid points in dict
  for (double b : geometric(bmin, 30.0, kDictCoarse)) coarse_idx.push_back(index_of(b));
  for (double b : fine) fine_idx.push_back(index_of(b));
  // fit every pool candidate over the COMMON box: outside its own box the
  // target is its true profile (< 1e-12 there), so the mixture stays
  // controlled on the whole box the passes use. Coarse dictionary first, the
  // fine one where that misses tol. Below kFitFloor no NNLS fit can certify
  // the bound in double arithmetic: only the exact d == 2 candidates join.
  // Independent problems: one host thread each. A d == 2 candidate is
  // exactly its own dictionary term, weight 1.
  std::vector<std::vector<double>> wfit(nc);
  std::vector<double> w0fit(nc, 0.0);
  std::vector<double> err(nc, INFINITY);
  auto fit_one = [&](int c) {
    wfit[c].assign(K, 0.0);
    if (cands[c].d == 2.0) {
      const double beta = 0.5 / (cands[c].sigma * cands[c].sigma);
      wfit[c][std::lower_bound(dict.begin(), dict.end(), beta) - dict.begin()] = 1.0;
      err[c] = 0.0;
      return;
    }
    if (tol < kFitFloor) return;
    std::vector<double> sub, w;
    for (int k : coarse_idx) sub.push_back(dict[k]);
    double e = fit_on(sub, S, Sfit, cands[c].sigma, cands[c].d, w, w0fit[c]) + 1e-12;
    for (size_t q = 0; q < coarse_idx.size(); ++q) wfit[c][coarse_idx[q]] = w[q];
    // fine grid, then fine grid + the candidate's own tangent betas (each only
    // when the previous level misses tol: extra betas are extra shared terms)
    for (int level = 0; level < 2 && e > loose; ++level) {
      std::vector<int> idx(fine_idx);
      if (level == 1)
        for (double b : tangents[c]) idx.push_back(index_of(b));
      std::sort(idx.begin(), idx.end());
      idx.erase(std::unique(idx.begin(), idx.end()), idx.end());
      sub.clear();
      for (int k : idx) sub.push_back(dict[k]);
      double z0;
      const double e2 = fit_on(sub, S, Sfit, cands[c].sigma, cands[c].d, w, z0) + 1e-12;
      if (e2 < e) {
        e = e2;
        wfit[c].assign(K, 0.0);
        for (size_t q = 0; q < idx.size(); ++q) wfit[c][idx[q]] = w[q];
        w0fit[c] = z0;
      }
    }
    err[c] = e;  // (+ 1e-12: fp64 factor truncation below)
  };
  {
    const int nthreads =
        std::max(1, std::min<int>(int(pool.size()), int(std::thread::hardware_concurrency())));
    std::atomic<int> next{0};
    std::vector<std::thread> workers;
    for (int w = 0; w < nthreads; ++w)
      workers.emplace_back([&] {
        for (int q = next++; q < int(pool.size()); q = next++) fit_one(pool[q]);
      });
    for (auto& th : workers) th.join();
  }
  for (int c : pool) {
    s->fit_err[c] = err[c];
    if (err[c] <= loose) {
      s->is_member[c] = 1;
      s->members.push_back(c);
    }
  }
  // Greedy pruning of the shared term set (large volumes, where each term
  // costs three full-volume passes per certificate): try dropping terms from
  // the most expensive (widest) down; a drop is kept when every member using
  // the term refits on the remaining terms within tol.
  if (prune && !s->members.empty()) {
    std::vector<char> in(K, 0), pinned(K, 0);
    for (int c : s->members)
      for (int k = 0; k < K; ++k)
        if (wfit[c][k] > 0.0) {
          in[k] = 1;
          if (cands[c].d == 2.0) pinned[k] = 1;  // exact members need their term
        }
    const double rbox = rmax;
    auto cost = [&](int k) {
      return std::min(2.0 * std::ceil(std::sqrt(27.7 / dict[k])) + 1.0, 2.0 * rbox + 1.0);
    };
    std::vector<int> order;
    for (int k = 0; k < K; ++k)
      if (in[k] && !pinned[k]) order.push_back(k);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return cost(x) > cost(y); });
    for (int k : order) {
      std::vector<int> users;
      for (int c : s->members)
        if (wfit[c][k] > 0.0 && cands[c].d != 2.0) users.push_back(c);
      in[k] = 0;
      std::vector<double> sub;
      std::vector<int> subk;
      for (int q = 0; q < K; ++q)
        if (in[q]) {
          sub.push_back(dict[q]);
          subk.push_back(q);
        }
      std::vector<std::vector<double>> nw(users.size());
      std::vector<double> nw0(users.size()), ne(users.size());
      std::vector<std::thread> th;
      for (size_t u = 0; u < users.size(); ++u)
        th.emplace_back([&, u] {
          const int c = users[u];
          ne[u] = fit_on(sub, S, Sfit, cands[c].sigma, cands[c].d, nw[u], nw0[u]) + 1e-12;
        });
      for (auto& x : th) x.join();
      bool ok = true;
      for (size_t u = 0; u < users.size(); ++u) ok &= ne[u] <= loose;
      if (!ok) {
        in[k] = 1;
        continue;
      }
      for (size_t u = 0; u < users.size(); ++u) {
        const int c = users[u];
        wfit[c].assign(K, 0.0);
        for (size_t q = 0; q < subk.size(); ++q) wfit[c][subk[q]] = nw[u][q];
        w0fit[c] = nw0[u];
        s->fit_err[c] = ne[u];
      }
    }
  }
  // union of the members' terms
  std::vector<char> used(K, 0);
  double wsum_max = 1.0;
  for (int c : s->members) {
    double ws = 0.0;
    for (int k = 0; k < K; ++k)
      if (wfit[c][k] > 0.0) {
        used[k] = 1;
        ws += wfit[c][k];
      }
    wsum_max = std::max(wsum_max, ws);
  }
  const double eps = trunc / wsum_max;
  if (loose > tol) {
    // members within `loose` but not `tol`: demoted (their terms stay shared);
    // fit_signed_members below refits them on the shared terms
    std::vector<int> keep;
    for (int c : s->members)
      if (s->fit_err[c] <= tol) keep.push_back(c);
      else s->is_member[c] = 0;
    s->members.swap(keep);
  }
  std::vector<int> kmap;
  for (int k = 0; k < K; ++k)
    if (used[k]) kmap.push_back(k);
  const int nt = int(kmap.size()), nm = int(s->members.size());
  for (int a = 0; a < 3; ++a) {
    s->tlo[a].resize(nt);
    s->tlen[a].resize(nt);
    s->elo[a].resize(nt);
    s->elen[a].resize(nt);
  }
  s->parent.assign(nt, -1);
  for (int t = 0; t < nt; ++t) s->betas.push_back(dict[kmap[t]]);
  const double lneps = std::log(1.0 / eps);
  auto radius = [&](double beta) { return int(std::ceil(std::sqrt(lneps / beta))); };
  // Chains (fp32 storage, not with the fused x pass): a term whose factor is
  // not clipped by C takes the narrower term p that minimises the taps of
  // g = exp(-beta_g q^2) with 1/beta = 1/beta_p + 1/beta_g, when that saves
  // passes taps and the lattice convolution of the two sampled Gaussians is a
  // sampled Gaussian to ~1e-9 (Poisson ripple exp(-pi^2 / (beta_p + beta_g))).
  // The bounds below use the effective factors, so the choice never costs
  // certification, only fit quality at the ripple level.
  const bool chains = dtype == SFW3D_F32;
  std::vector<double> gbeta(nt, 0.0);
  if (chains) {
    int rbox = 1 << 30;
    for (int a = 0; a < 3; ++a) rbox = std::min({rbox, -s->lo[a], s->hi[a]});
    const double kRipple = 0.45;  // beta_p + beta_g: exp(-pi^2 / 0.45) = 3e-10
    for (int t = 0; t < nt; ++t) {
      const double bt = s->betas[t];
      const int rt = radius(bt);
      if (rt > rbox) continue;
      int best = -1, rb_best = rt - 3;  // worth a chain: >= 6 fewer taps per axis
      double gb_best = 0.0;
      for (int p = t + 1; p < nt; ++p) {
        const double bp = s->betas[p];
        if (!(bp > bt * (1.0 + 1e-9))) continue;
        const double bg = bp * bt / (bp - bt);
        if (bp + bg > kRipple) continue;
        const int rg = radius(bg);
        if (rg < rb_best) {
          rb_best = rg;
          best = p;
          gb_best = bg;
        }
      }
      if (best >= 0) {
        s->parent[t] = best;
        gbeta[t] = gb_best;
      }
    }
  }
  // stored factor values (rounded to the storage precision) per term, axes
  // 0, 1, 2 contiguous: what the passes multiply by; heff: effective factors
  std::vector<std::vector<double>> hstore(nt), heff(nt);
  std::vector<double> pass_taps(nt, 0.0);
  for (int t = nt - 1; t >= 0; --t) {  // parents first (larger beta, larger index)
    const double beta = s->betas[t];
    std::vector<double>& h = hstore[t];
    const int p = s->parent[t];
    for (int a = 0; a < 3; ++a) {
      if (p < 0) {
        const int r = radius(beta);
        s->tlo[a][t] = std::max(s->lo[a], -r);
        s->tlen[a][t] = std::min(s->hi[a], r) - s->tlo[a][t] + 1;
        for (int q = s->tlo[a][t]; q < s->tlo[a][t] + s->tlen[a][t]; ++q) {
          const double v = std::exp(-beta * double(q) * q);
          h.push_back(dtype == SFW3D_F64 ? v : double(float(v)));
        }
        s->elo[a][t] = s->tlo[a][t];
        s->elen[a][t] = s->tlen[a][t];
        heff[t].insert(heff[t].end(), h.end() - s->tlen[a][t], h.end());
      } else {
        const double bg = gbeta[t], bp = s->betas[p];
        const int r = radius(bg);
        const double scale = std::sqrt((bp + bg) / M_PI);
        s->tlo[a][t] = -r;
        s->tlen[a][t] = 2 * r + 1;
        std::vector<double> g;
        for (int q = -r; q <= r; ++q) g.push_back(double(float(scale * std::exp(-bg * double(q) * q))));
        h.insert(h.end(), g.begin(), g.end());
        // effective factor: parent's effective factor (this axis) * g, exactly
        size_t poff = 0;
        for (int b2 = 0; b2 < a; ++b2) poff += s->elen[b2][p];
        const int plo = s->elo[a][p], plen = s->elen[a][p];
        s->elo[a][t] = plo - r;
        s->elen[a][t] = plen + 2 * r;
        std::vector<long double> e(size_t(s->elen[a][t]), 0.0L);
        for (int i = 0; i < plen; ++i)
          for (int j = 0; j <= 2 * r; ++j) e[size_t(i + j)] += (long double)heff[p][poff + i] * g[j];
        for (long double v : e) heff[t].push_back(double(v));
      }
      s->taps_per_voxel += s->tlen[a][t];
      pass_taps[t] += s->tlen[a][t];
    }
  }
  for (int t = 0; t < nt; ++t) {
    const std::vector<double>& h = hstore[t];
    if (!on_device) continue;
    void* dev = nullptr;
    int st;
    if (dtype == SFW3D_F64) {
      st = upload(&dev, h.data(), h.size() * sizeof(double));
    } else {
      std::vector<float> hf(h.begin(), h.end());
      st = upload(&dev, hf.data(), hf.size() * sizeof(float));
    }
    if (st != SFW3D_OK) return st;
    s->taps.push_back(dev);
  }
  s->W.assign(size_t(nm) * nt, 0.0);
  s->w0.assign(nm, 0.0);
  for (int m = 0; m < nm; ++m) {
    const int c = s->members[m];
    for (int t = 0; t < nt; ++t) s->W[size_t(m) * nt + t] = wfit[c][kmap[t]];
    s->w0[m] = w0fit[c];
  }
  s->n_nnls = nm;
  s->ebound.assign(nc, 0.0);
  if (nt > 0) fit_signed_members(s, cands, dtype, Sfit, heff, pass_taps);
  const int nmt = int(s->members.size());
  if (nmt && on_device) {
    if (dtype == SFW3D_F64) {
      std::vector<double> Wd(s->W);
      Wd.push_back(0.0);
      SFW3D_TRY(upload(&s->W_dev, Wd.data(), Wd.size() * sizeof(double)));
      SFW3D_TRY(upload(&s->w0_dev, s->w0.data(), s->w0.size() * sizeof(double)));
    } else {
      std::vector<float> Wf(s->W.begin(), s->W.end()), w0f(s->w0.begin(), s->w0.end());
      Wf.push_back(0.f);
      SFW3D_TRY(upload(&s->W_dev, Wf.data(), Wf.size() * sizeof(float)));
      SFW3D_TRY(upload(&s->w0_dev, w0f.data(), w0f.size() * sizeof(float)));
    }
    SFW3D_TRY(upload(reinterpret_cast<void**>(&s->cid_dev), s->members.data(),
                     s->members.size() * sizeof(int)));
    {
      // dense / copy member split for mix_ring2_kernel
      std::vector<int> dmem, cmem, cterm(nt, -1);
      std::vector<double> Wd, w0d;
      for (int m = 0; m < nmt; ++m) {
        int nz = 0, k1 = -1;
        for (int t = 0; t < nt; ++t)
          if (s->W[size_t(m) * nt + t] != 0.0) {
            ++nz;
            k1 = t;
          }
        if (nz == 1 && s->W[size_t(m) * nt + k1] == 1.0 && s->w0[m] == 0.0 && cterm[k1] < 0 &&
            int(cmem.size()) < 8) {
          cterm[k1] = int(cmem.size());
          cmem.push_back(m);
        } else {
          dmem.push_back(m);
          Wd.insert(Wd.end(), s->W.begin() + size_t(m) * nt, s->W.begin() + size_t(m + 1) * nt);
          w0d.push_back(s->w0[m]);
        }
      }
      s->nmd = int(dmem.size());
      s->nmc = int(cmem.size());
      Wd.push_back(0.0);
      w0d.push_back(0.0);
      dmem.push_back(0);
      cmem.push_back(0);
      if (dtype == SFW3D_F64) {
        SFW3D_TRY(upload(&s->Wd_dev, Wd.data(), Wd.size() * sizeof(double)));
        SFW3D_TRY(upload(&s->w0d_dev, w0d.data(), w0d.size() * sizeof(double)));
      } else {
        std::vector<float> Wf(Wd.begin(), Wd.end()), w0f(w0d.begin(), w0d.end());
        SFW3D_TRY(upload(&s->Wd_dev, Wf.data(), Wf.size() * sizeof(float)));
        SFW3D_TRY(upload(&s->w0d_dev, w0f.data(), w0f.size() * sizeof(float)));
      }
      SFW3D_TRY(upload(reinterpret_cast<void**>(&s->dmem_dev), dmem.data(), dmem.size() * sizeof(int)));
      SFW3D_TRY(upload(reinterpret_cast<void**>(&s->cmem_dev), cmem.data(), cmem.size() * sizeof(int)));
      SFW3D_TRY(upload(reinterpret_cast<void**>(&s->cterm_dev), cterm.data(), cterm.size() * sizeof(int)));
    }
  }
  return SFW3D_OK;
}

void basis_set_destroy(BasisSet* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  for (void* p : s->taps) cudaFree(p);
  if (s->W_dev) cudaFree(s->W_dev);
  if (s->w0_dev) cudaFree(s->w0_dev);
  if (s->cid_dev) cudaFree(s->cid_dev);
  for (void* p : {s->Wd_dev, s->w0d_dev, static_cast<void*>(s->dmem_dev),
                  static_cast<void*>(s->cmem_dev), static_cast<void*>(s->cterm_dev)})
    if (p) cudaFree(p);
  delete s;
}

void basis_set_export(const BasisSet* s, int max_terms, int* n_terms, double* betas,
                      double* weights, double* w0, double* fit_err, int32_t* member) {
  const int nt = int(s->betas.size()), nc = int(s->is_member.size());
  if (n_terms) *n_terms = nt;
  for (int t = 0; t < nt && t < max_terms; ++t)
    if (betas) betas[t] = s->betas[t];
  for (int c = 0; c < nc; ++c) {
    if (fit_err) fit_err[c] = s->fit_err[c];
    if (member) member[c] = s->is_member[c];
    if (w0) w0[c] = 0.0;
    if (weights)
      for (int t = 0; t < max_terms; ++t) weights[size_t(c) * max_terms + t] = 0.0;
  }
  for (int m = 0; m < int(s->members.size()); ++m) {
    const int c = s->members[m];
    if (w0) w0[c] = s->w0[m];
    if (weights)
      for (int t = 0; t < nt && t < max_terms; ++t)
        weights[size_t(c) * max_terms + t] = s->W[size_t(m) * nt + t];
  }
}

bool basis_set_member(const BasisSet* s, int cand, double* fit_err) {
  if (!s || cand < 0 || cand >= int(s->is_member.size())) return false;
  if (fit_err) *fit_err = s->fit_err[cand];
  return s->is_member[cand] != 0;
}
bool basis_set_signed(const BasisSet* s, int cand) {
  return s && cand >= 0 && cand < int(s->is_member.size()) && s->is_member[cand] == 2;
}
double basis_set_ebound(const BasisSet* s, int cand) {
  return basis_set_signed(s, cand) ? s->ebound[cand] : 0.0;
}
int basis_set_n_terms(const BasisSet* s) { return s ? int(s->betas.size()) : 0; }
int basis_set_n_members(const BasisSet* s) { return s ? int(s->members.size()) : 0; }
long long basis_set_taps(const BasisSet* s) { return s ? s->taps_per_voxel : 0; }
int basis_set_pass_taps(const BasisSet* s, int term, int axis) {
  return (s && term >= 0 && term < int(s->betas.size())) ? s->tlen[axis][term] : 0;
}
double basis_set_member_flops(const BasisSet* s) {
  return s ? 2.0 * double(s->betas.size()) + 2.0 : 0.0;
}
double basis_set_flops(const BasisSet* s) {
  if (!s || s->members.empty()) return 0.0;
  return 2.0 * double(s->taps_per_voxel) + double(s->members.size()) * basis_set_member_flops(s);
}

// ------------------------------------------------------------------ eval
namespace {

constexpr int kMixMax = 32;  // members mixed per launch
constexpr int kMixThreads = 256;

// V consecutive elements of one volume as one vector load/store (16 B max)
template <typename T, int V>
struct Vec {
  T v[V];
};
template <typename T, int V>
__device__ __forceinline__ Vec<T, V> ld_stream(const T* p) {
  Vec<T, V> r;
  if constexpr (sizeof(T) * V == 16) {
    const float4 q = __ldcs(reinterpret_cast<const float4*>(p));
    memcpy(&r, &q, 16);
  } else if constexpr (sizeof(T) * V == 8) {
    const float2 q = __ldcs(reinterpret_cast<const float2*>(p));
    memcpy(&r, &q, 8);
  } else {
    r.v[0] = __ldcs(p);
  }
  return r;
}
template <typename T, int V>
__device__ __forceinline__ void st_stream(T* p, const Vec<T, V>& r) {
  if constexpr (sizeof(T) * V == 16) {
    float4 q;
    memcpy(&q, &r, 16);
    __stcs(reinterpret_cast<float4*>(p), q);
  } else if constexpr (sizeof(T) * V == 8) {
    float2 q;
    memcpy(&q, &r, 8);
    __stcs(reinterpret_cast<float2*>(p), q);
  } else {
    __stcs(p, r.v[0]);
  }
}

// eta_c = (w0_c b + sum_k W[c][k] T_k) / lam for members [m0, m0 + nm) at
// every voxel; windowed argmax per member (one partial per CTA); optional
// field store. HBM-bound: each thread owns V consecutive voxels of one z row
// (vector loads), KU term loads in flight; the running maximum is kept on the
// raw accumulator (eta = acc / lam with lam > 0 is monotone in acc).
// COLLECT: instead of the argmax, append every windowed voxel whose eta is
// >= thr[member] to the item list (candidate id, voxel) — capped at col.cap,
// the counter keeps counting past the cap.
struct Collect {
  const double* thr;    // [members]
  int* cand;            // [cap] member index
  long long* idx;       // [cap] voxel
  int* count;
  int cap;
  const Best* part;     // the evaluation pass's per-CTA maxima [member][CTA]
  int parents;          // evaluation grid (CTA chunks)
  int split;            // collect CTAs per evaluation chunk
};

template <typename T, int NM, int V, bool COLLECT = false>
__global__ void __launch_bounds__(kMixThreads) mix_argmax_kernel(
    const T* __restrict__ b, const T* __restrict__ terms, long long n, int K, int nm, int m0,
    const T* __restrict__ W, const T* __restrict__ w0, const int* __restrict__ cid, int nx, int ny,
    int nz, int4 wlo, int4 whi, double lam, T* __restrict__ fields, Best* __restrict__ partial,
    Collect col = {}) {
  constexpr int KU = V == 4 ? 8 : (V == 2 ? 12 : 16);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* sW = reinterpret_cast<T*>(smem_raw);  // [K][NM], zero-padded members
  T* sw0 = sW + K * NM;
  __shared__ Best red[NM][kMixThreads / 32];
  for (int e = threadIdx.x; e < K * NM; e += kMixThreads) {
    const int k = e / NM, m = e % NM;
    sW[e] = m < nm ? W[size_t(m0 + m) * K + k] : T(0);
  }
  for (int e = threadIdx.x; e < NM; e += kMixThreads) sw0[e] = e < nm ? w0[m0 + e] : T(0);
  // contiguous chunk of V-vectors per evaluation CTA; the collect pass splits
  // each chunk over col.split CTAs and revisits only the chunks whose
  // evaluation-pass maxima reach a threshold
  const long long nv = n / V;
  const int parents = COLLECT ? col.parents : int(gridDim.x);
  const int parent = COLLECT ? int(blockIdx.x) / col.split : int(blockIdx.x);
  const long long chunk =
      ((nv + parents - 1) / parents + kMixThreads - 1) / kMixThreads * kMixThreads;
  long long qbeg = parent * chunk, qend = min(nv, (parent + 1) * chunk);
  if constexpr (COLLECT) {
    const int q = threadIdx.x < nm &&
                  col.part[(long long)(m0 + threadIdx.x) * parents + parent].v >= col.thr[m0 + threadIdx.x];
    if (!__syncthreads_or(q)) return;
    const int sub = int(blockIdx.x) % col.split;
    const long long sc = ((chunk + col.split - 1) / col.split + kMixThreads - 1) / kMixThreads * kMixThreads;
    qbeg += sub * sc;
    qend = min(qend, qbeg + sc);
  }
  __syncthreads();
  T bacc[NM];
  int bidx[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    bacc[m] = T(-INFINITY);
    bidx[m] = 0x7fffffff;
  }
  for (long long q = qbeg + threadIdx.x; q < qend; q += kMixThreads) {
    const long long i0 = q * V;
    const Vec<T, V> bv = ld_stream<T, V>(b + i0);
    T acc[NM][V];
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int j = 0; j < V; ++j) acc[m][j] = sw0[m] * bv.v[j];
    int k = 0;
    for (; k + KU <= K; k += KU) {
      Vec<T, V> tv[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) tv[u] = ld_stream<T, V>(terms + (long long)(k + u) * n + i0);
#pragma unroll
      for (int u = 0; u < KU; ++u)
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          const T w = sW[(k + u) * NM + m];
#pragma unroll
          for (int j = 0; j < V; ++j) acc[m][j] = fma(w, tv[u].v[j], acc[m][j]);
        }
    }
    for (; k < K; ++k) {
      const Vec<T, V> tv = ld_stream<T, V>(terms + (long long)k * n + i0);
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const T w = sW[k * NM + m];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[m][j] = fma(w, tv.v[j], acc[m][j]);
      }
    }
    // the V voxels share one (x, y) row (nz % V == 0)
    const int z0 = int(i0 % nz);
    const long long row = i0 / nz;
    const int y = int(row % ny), x = int(row / ny);
    const bool row_win = x >= wlo.x && x <= whi.x && y >= wlo.y && y <= whi.y;
    if constexpr (COLLECT) {
      if (row_win) {
#pragma unroll
        for (int m = 0; m < NM; ++m) {
          if (m >= nm) break;
#pragma unroll
          for (int j = 0; j < V; ++j) {
            const int z = z0 + j;
            if (z >= wlo.z && z <= whi.z && double(acc[m][j]) / lam >= col.thr[m0 + m]) {
              atomicAdd(col.count + 1 + m0 + m, 1);
              const int slot = atomicAdd(col.count, 1);
              if (slot < col.cap) {
                col.cand[slot] = cid[m0 + m];
                col.idx[slot] = i0 + j;
              }
            }
          }
        }
      }
      continue;
    }
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      if (m >= nm) break;
      if (fields) {
        Vec<T, V> f;
#pragma unroll
        for (int j = 0; j < V; ++j) f.v[j] = T(double(acc[m][j]) / lam);
        st_stream<T, V>(fields + (long long)cid[m0 + m] * n + i0, f);
      }
      if (row_win) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const int z = z0 + j;
          // ascending i within the thread: strict '>' keeps the first maximum
          if (z >= wlo.z && z <= whi.z && acc[m][j] > bacc[m]) {
            bacc[m] = acc[m][j];
            bidx[m] = int(i0 + j);
          }
        }
      }
    }
  }
  if constexpr (COLLECT) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    if (m >= nm) break;
    Best bm = {bidx[m] == 0x7fffffff ? -INFINITY : double(bacc[m]) / lam,
               bidx[m] == 0x7fffffff ? 0x7fffffffffffffffLL : (long long)bidx[m]};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bm.v, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bm.idx, o);
      if (better(ov, oi, bm.v, bm.idx)) bm = {ov, oi};
    }
    if (lane == 0) red[m][warp] = bm;
  }
  __syncthreads();
  if (threadIdx.x < nm) {
    Best bm = red[threadIdx.x][0];
    for (int w = 1; w < kMixThreads / 32; ++w)
      if (better(red[threadIdx.x][w].v, red[threadIdx.x][w].idx, bm.v, bm.idx))
        bm = red[threadIdx.x][w];
    partial[(long long)(m0 + threadIdx.x) * gridDim.x + blockIdx.x] = bm;
  }
}

// Evaluation-pass mix with a per-thread cp.async ring (same CTA chunking,
// FMA order and per-CTA maxima as mix_argmax_kernel, so its COLLECT pass
// revisits these chunks). Each thread streams its own 16-byte vector of b and
// of every T_k through kMixNS shared-memory slots (no barriers: a thread only
// reads what it copied), keeping kMixNS - 1 loads in flight across term and
// vector boundaries — the flattened (vector, term) sequence never drains.
constexpr int kMixNS = 8;

template <typename T, int NM>
__global__ void __launch_bounds__(kMixThreads, sizeof(T) == 4 ? 2 : 1) mix_ring_kernel(
    const T* __restrict__ b, const T* __restrict__ terms, long long n, int K, int nm, int m0,
    const T* __restrict__ W, const T* __restrict__ w0, const int* __restrict__ cid, int nx, int ny,
    int nz, int4 wlo, int4 whi, double lam, T* __restrict__ fields, Best* __restrict__ partial) {
  constexpr int V = 16 / sizeof(T);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);            // [kMixNS][kMixThreads][V]
  T* sW = ring + kMixNS * kMixThreads * V;             // [K][NM]
  T* sw0 = sW + K * NM;
  __shared__ Best red[NM][kMixThreads / 32];
  for (int e = threadIdx.x; e < K * NM; e += kMixThreads) {
    const int k = e / NM, m = e % NM;
    sW[e] = m < nm ? W[size_t(m0 + m) * K + k] : T(0);
  }
  for (int e = threadIdx.x; e < NM; e += kMixThreads) sw0[e] = e < nm ? w0[m0 + e] : T(0);
  __syncthreads();
  const long long nv = n / V;
  const long long chunk =
      ((nv + gridDim.x - 1) / gridDim.x + kMixThreads - 1) / kMixThreads * kMixThreads;
  const long long qbeg = blockIdx.x * chunk + threadIdx.x, qend = min(nv, (blockIdx.x + 1) * chunk);
  const int iters = qbeg < qend ? int((qend - qbeg + kMixThreads - 1) / kMixThreads) : 0;
  const int E = K + 1;  // sequence entries per vector: b, then T_0 .. T_{K-1}
  const int G = iters * E;
  T* myslot = ring + threadIdx.x * V;
  constexpr int kSlot = kMixThreads * V;  // elements between consecutive slots
  // producer: entry pointer (b, then T_0 .. T_{K-1} of the same vector, then
  // the next vector's b), ring slot pg & (kMixNS - 1). Byte steps between
  // consecutive entries: b -> T_0, T_k -> T_{k+1}, T_{K-1} -> next b.
  const char* pptr = reinterpret_cast<const char*>(b + qbeg * V);
  const long long d_b = reinterpret_cast<const char*>(terms) - reinterpret_cast<const char*>(b);
  const long long d_t = (long long)n * sizeof(T);
  const long long d_w = -d_b - (long long)(K - 1) * d_t + (long long)kMixThreads * V * sizeof(T);
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(myslot));
  int pe = 0;
  unsigned pg = 0;
  auto issue = [&]() {
    const unsigned sa = sbase + (pg & (kMixNS - 1)) * (kSlot * sizeof(T));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(pptr));
    ++pg;
    pptr += pe == 0 ? d_b : (pe == K ? d_w : d_t);
    pe = pe == K ? 0 : pe + 1;
  };
  static_assert((kMixNS & (kMixNS - 1)) == 0, "ring depth is a power of two");
#pragma unroll
  for (int g = 0; g < kMixNS - 1; ++g) {
    if (g < G) issue();
    cp_async_commit();
  }
  // running per-thread maxima live in shared memory (read once per vector,
  // written only on improvement): keeps the accumulators and the producer
  // state in registers at 2 CTAs per SM
  T* sbv = sw0 + NM;                                        // [NM][kMixThreads]
  int* sbi = reinterpret_cast<int*>(sbv + NM * kMixThreads);  // [NM][kMixThreads]
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    sbv[m * kMixThreads + threadIdx.x] = T(-INFINITY);
    sbi[m * kMixThreads + threadIdx.x] = 0x7fffffff;
  }
  unsigned g = 0;
  auto take = [&](T (&v)[V]) {
    cp_async_wait_group<kMixNS - 2>();
    const T* sl = myslot + (g & (kMixNS - 1)) * kSlot;
    if constexpr (sizeof(T) == 4) {
      const float4 q = *reinterpret_cast<const float4*>(sl);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 q = *reinterpret_cast<const double2*>(sl);
      v[0] = q.x; v[1] = q.y;
    }
    if (g + kMixNS - 1 < G) issue();
    cp_async_commit();
    ++g;
  };
  for (int it = 0; it < iters; ++it) {
    const long long i0 = (qbeg + (long long)it * kMixThreads) * V;
    T acc[NM][V];
    {
      T v[V];
      take(v);
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[m][j] = sw0[m] * v[j];
    }
    for (int k = 0; k < K; ++k) {
      T v[V];
      take(v);
      const T* wk = sW + k * NM;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const T w = wk[m];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[m][j] = fma(w, v[j], acc[m][j]);
      }
    }
    // the V voxels share one (x, y) row (nz % V == 0)
    const int z0 = int(i0 % nz);
    const long long row = i0 / nz;
    const int y = int(row % ny), x = int(row / ny);
    const bool row_win = x >= wlo.x && x <= whi.x && y >= wlo.y && y <= whi.y;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      if (m >= nm) break;
      if (fields) {
        T f[V];
#pragma unroll
        for (int j = 0; j < V; ++j) f[j] = T(double(acc[m][j]) / lam);
        T* dst = fields + (long long)cid[m0 + m] * n + i0;
        if constexpr (sizeof(T) == 4)
          __stcs(reinterpret_cast<float4*>(dst), make_float4(f[0], f[1], f[2], f[3]));
        else
          __stcs(reinterpret_cast<double2*>(dst), make_double2(f[0], f[1]));
      }
      if (row_win) {
        const T cur = sbv[m * kMixThreads + threadIdx.x];
        T bv = cur;
        int bj = -1;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          const int z = z0 + j;
          // ascending i within the thread: strict '>' keeps the first maximum
          if (z >= wlo.z && z <= whi.z && acc[m][j] > bv) {
            bv = acc[m][j];
            bj = j;
          }
        }
        if (bj >= 0) {
          sbv[m * kMixThreads + threadIdx.x] = bv;
          sbi[m * kMixThreads + threadIdx.x] = int(i0 + bj);
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    if (m >= nm) break;
    const int bi = sbi[m * kMixThreads + threadIdx.x];
    Best bm = {bi == 0x7fffffff ? -INFINITY : double(sbv[m * kMixThreads + threadIdx.x]) / lam,
               bi == 0x7fffffff ? 0x7fffffffffffffffLL : (long long)bi};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bm.v, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bm.idx, o);
      if (better(ov, oi, bm.v, bm.idx)) bm = {ov, oi};
    }
    if (lane == 0) red[m][warp] = bm;
  }
  __syncthreads();
  if (threadIdx.x < nm) {
    Best bm = red[threadIdx.x][0];
    for (int w = 1; w < kMixThreads / 32; ++w)
      if (better(red[threadIdx.x][w].v, red[threadIdx.x][w].idx, bm.v, bm.idx))
        bm = red[threadIdx.x][w];
    partial[(long long)(m0 + threadIdx.x) * gridDim.x + blockIdx.x] = bm;
  }
}

// Evaluation-pass mix, v2 of mix_ring_kernel (same CTA chunking, so the
// collect pass revisits the same chunks): members split into DENSE members
// (NMD accumulators per voxel, W from shared memory) and COPY members (the
// exact d == 2 members: eta = T_k / lam for one term k, w0 = 0), which cost
// no FMA — their running maxima are updated when their term streams by. The
// producer walks the flattened (vector, entry) sequence through a table of
// byte offsets; the running maxima take the max of the 4 voxels first and
// do index work only on improvement (interior z).
template <typename T, int NMD, int NS, int NT, int VV>
__global__ void __launch_bounds__(NT, NT == 128 ? 3 : 2) mix_ring2_kernel(
    const T* __restrict__ b, const T* __restrict__ terms, long long n, int K,
    const T* __restrict__ Wd, const T* __restrict__ w0d, const int* __restrict__ dmem, int nmd,
    const int* __restrict__ cterm, int nmc, const int* __restrict__ cmem,
    const int* __restrict__ cid, int nx, int ny, int nz, int4 wlo, int4 whi, double lam,
    double* __restrict__ absparts, Best* __restrict__ partial) {
  // VV 16-byte vectors per thread and entry (VV = 2 with 128-thread CTAs: the
  // same 1024-voxel iteration span, per-entry overhead amortised over 8 voxels)
  constexpr int V = VV * 16 / sizeof(T);
  constexpr int NMC = 8;  // copy members (at most)
  static_assert((NS & (NS - 1)) == 0, "ring depth is a power of two");
  double abs_s = 0.0;  // sum |b| (fp64) and max |b| of the vectors read (absparts)
  T abs_m = T(0);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);                       // [NS][threads][V]
  T* sW = ring + NS * NT * V;                            // [K][NMD], 16-byte rows
  T* sw0 = sW + K * NMD;                                          // [NMD]
  T* sbv = sw0 + NMD;                                             // [NMD + NMC][threads]
  int* sbi = reinterpret_cast<int*>(sbv + (NMD + NMC) * NT);
  int* sCt = sbi + (NMD + NMC) * NT;                     // [K]: copy slot or -1
  __shared__ Best red[NMD + NMC][NT / 32];
  for (int e = threadIdx.x; e < K * NMD; e += NT) {
    const int k = e / NMD, m = e % NMD;
    sW[e] = m < nmd ? Wd[size_t(m) * K + k] : T(0);
  }
  for (int e = threadIdx.x; e < NMD; e += NT) sw0[e] = e < nmd ? w0d[e] : T(0);
  for (int e = threadIdx.x; e < K; e += NT) sCt[e] = cterm[e];
#pragma unroll
  for (int m = 0; m < NMD + NMC; ++m) {
    sbv[m * NT + threadIdx.x] = T(-INFINITY);
    sbi[m * NT + threadIdx.x] = 0x7fffffff;
  }
  __syncthreads();
  const long long nv = n / V;
  // chunks in units of one iteration span (NT * V voxels = 256 16-byte
  // vectors for every variant: the collect pass revisits the same ranges)
  const long long nspan = (n / (16 / sizeof(T)) + 255) / 256;  // iteration spans in the volume
  const long long chunk = (nspan + gridDim.x - 1) / gridDim.x * NT;
  const long long qbeg = blockIdx.x * chunk + threadIdx.x, qend = min(nv, (blockIdx.x + 1) * chunk);
  const int iters = qbeg < qend ? int((qend - qbeg + NT - 1) / NT) : 0;
  const int E = K + 1;
  const int G = iters * E;
  T* myslot = ring + threadIdx.x * V;
  constexpr int kSlot = NT * V;
  // producer: entry pe of the vector stream (0 = b, 1 + k = T_k), running
  // pointers into b and the terms, running ring-slot byte offsets
  const char* bq = reinterpret_cast<const char*>(b + qbeg * V);
  const char* tq = reinterpret_cast<const char*>(terms + qbeg * V);
  const long long vstep = (long long)NT * V * sizeof(T);
  const long long nstride = n * (long long)sizeof(T);
  const long long twrap = vstep - (long long)K * nstride;
  const unsigned sbase = static_cast<unsigned>(__cvta_generic_to_shared(myslot));
  constexpr unsigned kSlotB = kSlot * sizeof(T), kRingB = NS * kSlotB;
  static_assert((kRingB & (kRingB - 1)) == 0, "ring bytes are a power of two");
  int pe = 0, pleft = G;
  unsigned poff = 0, coff = 0;
  // branch-free: past the end of the stream the copy has src-size 0 (no
  // global read, the slot is zero-filled and never consumed)
  auto issue = [&]() {
    const char* a = pe == 0 ? bq : tq;
#pragma unroll
    for (int vv = 0; vv < VV; ++vv)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sbase + poff + 16 * vv),
                   "l"(a + 16 * vv), "r"(pleft > 0 ? 16 : 0));
    poff = (poff + kSlotB) & (kRingB - 1);
    --pleft;
    tq += pe != 0 ? nstride : 0LL;
    ++pe;
    const bool wrap = pe == E;
    pe = wrap ? 0 : pe;
    bq += wrap ? vstep : 0LL;
    tq += wrap ? twrap : 0LL;
  };
#pragma unroll
  for (int g = 0; g < NS - 1; ++g) {
    issue();
    cp_async_commit();
  }
  auto take = [&](T (&v)[V]) {
    cp_async_wait_group<NS - 2>();
    const T* sl = reinterpret_cast<const T*>(reinterpret_cast<const char*>(myslot) + coff);
#pragma unroll
    for (int vv = 0; vv < VV; ++vv) {
      if constexpr (sizeof(T) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(sl + 4 * vv);
        v[4 * vv] = q.x; v[4 * vv + 1] = q.y; v[4 * vv + 2] = q.z; v[4 * vv + 3] = q.w;
      } else {
        const double2 q = *reinterpret_cast<const double2*>(sl + 2 * vv);
        v[2 * vv] = q.x; v[2 * vv + 1] = q.y;
      }
    }
    coff = (coff + kSlotB) & (kRingB - 1);
    issue();
    cp_async_commit();
  };
  // running maximum of member slot m over this vector's V voxels
  auto track = [&](int m, const T (&a)[V], long long i0, bool zfull, int z0) {
    T* pv = sbv + m * NT + threadIdx.x;
    if (zfull) {
      T mx = a[0];
#pragma unroll
      for (int j = 1; j < V; ++j) mx = max(mx, a[j]);
      if (mx > *pv) {
        int bj = V - 1;
#pragma unroll
        for (int j = V - 2; j >= 0; --j)
          if (a[j] == mx) bj = j;
        *pv = mx;
        sbi[m * NT + threadIdx.x] = int(i0 + bj);
      }
    } else {
      T bv = *pv;
      int bj = -1;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int z = z0 + j;
        if (z >= wlo.z && z <= whi.z && a[j] > bv) {
          bv = a[j];
          bj = j;
        }
      }
      if (bj >= 0) {
        *pv = bv;
        sbi[m * NT + threadIdx.x] = int(i0 + bj);
      }
    }
  };
  // voxel position of this thread's vector, advanced incrementally (one
  // NT * V step per iteration) instead of divided out per vector
  const int step = NT * V;
  const int dzs = step % nz, dys = step / nz;
  int z0 = 0, y = 0, x = 0;
  if (iters > 0) {
    const long long i0 = qbeg * V;
    z0 = int(i0 % nz);
    const long long row = i0 / nz;
    y = int(row % ny);
    x = int(row / ny);
  }
  for (int it = 0; it < iters; ++it) {
    if (it > 0) {
      z0 += dzs;
      y += dys;
      if (z0 >= nz) {
        z0 -= nz;
        ++y;
      }
      while (y >= ny) {
        y -= ny;
        ++x;
      }
    }
    const long long i0 = (qbeg + (long long)it * NT) * V;
    const bool row_win = x >= wlo.x && x <= whi.x && y >= wlo.y && y <= whi.y;
    const bool zfull = z0 >= wlo.z && z0 + V - 1 <= whi.z;
    if constexpr (sizeof(T) == 4 && NMD >= 16) {
      // fp32, full 16-member slices (measured: config-3 mix 1.88 -> 1.52 ms;
      // the 12-member config-4 slice is closer to its HBM bound and was 8%
      // slower packed, so it keeps the scalar form): members in pairs
      // (m, m + 1) on the packed FFMA2 pipe — the
      // weight pairs come straight out of the 16-byte shared-memory loads,
      // a voxel is broadcast to both halves; each half is the same RN FMA
      // as the scalar form (bit-identical), at half the FMA issue slots
      static_assert(NMD % 4 == 0, "member pairs from 16-byte rows");
      f32x2 acc2[NMD / 2][V];
      {
        T v[V];
        take(v);
        f32x2 vv[V];
#pragma unroll
        for (int j = 0; j < V; ++j) vv[j] = pack2(v[j], v[j]);
#pragma unroll
        for (int p2 = 0; p2 < NMD / 2; p2 += 2) {
          const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(sw0 + 2 * p2);
#pragma unroll
          for (int j = 0; j < V; ++j) {
            acc2[p2][j] = mul2(q.x, vv[j]);
            acc2[p2 + 1][j] = mul2(q.y, vv[j]);
          }
        }
        if (absparts) {
#pragma unroll
          for (int j = 0; j < V; ++j) {
            abs_s += double(fabs(v[j]));
            abs_m = fmax(abs_m, fabs(v[j]));
          }
        }
      }
      for (int k = 0; k < K; ++k) {
        T v[V];
        take(v);
        f32x2 vv[V];
#pragma unroll
        for (int j = 0; j < V; ++j) vv[j] = pack2(v[j], v[j]);
        const T* wk = sW + k * NMD;
#pragma unroll
        for (int p2 = 0; p2 < NMD / 2; p2 += 2) {
          const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(wk + 2 * p2);
#pragma unroll
          for (int j = 0; j < V; ++j) {
            acc2[p2][j] = fma2(q.x, vv[j], acc2[p2][j]);
            acc2[p2 + 1][j] = fma2(q.y, vv[j], acc2[p2 + 1][j]);
          }
        }
        const int c = sCt[k];
        if (c >= 0 && row_win) track(NMD + c, v, i0, zfull, z0);  // a copy's eta * lam is T_k
      }
      if (row_win) {
#pragma unroll
        for (int m = 0; m < NMD; ++m) {
          if (m >= nmd) break;
          T a[V];
#pragma unroll
          for (int j = 0; j < V; ++j) a[j] = (m & 1) ? hi32(acc2[m / 2][j]) : lo32(acc2[m / 2][j]);
          track(m, a, i0, zfull, z0);
        }
      }
    } else {
    T acc[NMD][V];
    {
      T v[V];
      take(v);
#pragma unroll
      for (int m = 0; m < NMD; ++m)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[m][j] = sw0[m] * v[j];
      if (absparts) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
          abs_s += double(fabs(v[j]));
          abs_m = fmax(abs_m, fabs(v[j]));
        }
      }
    }
    for (int k = 0; k < K; ++k) {
      T v[V];
      take(v);
      const T* wk = sW + k * NMD;
      T wv[NMD];
#pragma unroll
      for (int m = 0; m < NMD; m += 16 / sizeof(T)) {
        if constexpr (sizeof(T) == 4) {
          const float4 q = *reinterpret_cast<const float4*>(wk + m);
          wv[m] = q.x; wv[m + 1] = q.y; wv[m + 2] = q.z; wv[m + 3] = q.w;
        } else {
          const double2 q = *reinterpret_cast<const double2*>(wk + m);
          wv[m] = q.x; wv[m + 1] = q.y;
        }
      }
#pragma unroll
      for (int m = 0; m < NMD; ++m)
#pragma unroll
        for (int j = 0; j < V; ++j) acc[m][j] = fma(wv[m], v[j], acc[m][j]);
      const int c = sCt[k];
      if (c >= 0 && row_win) track(NMD + c, v, i0, zfull, z0);  // a copy's eta * lam is T_k
    }
    if (row_win) {
#pragma unroll
      for (int m = 0; m < NMD; ++m) {
        if (m >= nmd) break;
        track(m, acc[m], i0, zfull, z0);
      }
    }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < NMD + NMC; ++m) {
    if (m < NMD ? m >= nmd : m - NMD >= nmc) continue;
    const int bi = sbi[m * NT + threadIdx.x];
    Best bm = {bi == 0x7fffffff ? -INFINITY : double(sbv[m * NT + threadIdx.x]) / lam,
               bi == 0x7fffffff ? 0x7fffffffffffffffLL : (long long)bi};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bm.v, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bm.idx, o);
      if (better(ov, oi, bm.v, bm.idx)) bm = {ov, oi};
    }
    if (lane == 0) red[m][warp] = bm;
  }
  __syncthreads();
  if (threadIdx.x < NMD + NMC) {
    const int m = threadIdx.x;
    if (m < NMD ? m < nmd : m - NMD < nmc) {
      Best bm = red[m][0];
      for (int w = 1; w < NT / 32; ++w)
        if (better(red[m][w].v, red[m][w].idx, bm.v, bm.idx)) bm = red[m][w];
      const int mem = m < NMD ? dmem[m] : cmem[m - NMD];  // member index
      partial[(long long)mem * gridDim.x + blockIdx.x] = bm;
    }
  }
  if (absparts) {  // per-CTA |b| statistics (fixed-order reduce: abs_reduce_kernel)
    double ds = abs_s, dm = double(abs_m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ds += __shfl_xor_sync(0xffffffffu, ds, o);
      dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    }
    __shared__ double sa[NT / 32][2];
    if (lane == 0) {
      sa[warp][0] = ds;
      sa[warp][1] = dm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0, mm = 0.0;
      for (int w = 0; w < NT / 32; ++w) {
        t += sa[w][0];
        mm = fmax(mm, sa[w][1]);
      }
      absparts[2 * blockIdx.x] = t;
      absparts[2 * blockIdx.x + 1] = mm;
    }
  }
}

// [sum |b|, max |b|] from the mix's per-CTA statistics: a fixed-order tree
// (thread i sums blocks i, i + 256, ...; then a fixed shuffle / warp order)
__global__ void __launch_bounds__(256) abs_reduce_kernel(const double* __restrict__ parts,
                                                         int nblocks, double* __restrict__ out) {
  __shared__ double st[8], sm[8];
  double t = 0.0, m = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += 256) {
    t += parts[2 * b];
    m = fmax(m, parts[2 * b + 1]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t += __shfl_down_sync(0xffffffffu, t, o);
    m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  }
  if ((threadIdx.x & 31) == 0) {
    st[threadIdx.x >> 5] = t;
    sm[threadIdx.x >> 5] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tt = 0.0, mm = 0.0;
    for (int w = 0; w < 8; ++w) {
      tt += st[w];
      mm = fmax(mm, sm[w]);
    }
    out[0] = tt;
    out[1] = mm;
  }
}

__global__ void member_reduce_kernel(const Best* __restrict__ partial, int nblocks,
                                     const int* __restrict__ cid, Best* __restrict__ best_dev) {
  __shared__ Best sb[32];
  const int m = blockIdx.x;
  Best b{-INFINITY, 0x7fffffffffffffffLL};
  for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
    const Best p = partial[(long long)m * nblocks + i];
    if (better(p.v, p.idx, b.v, b.idx)) b = p;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, b.v, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, b.idx, o);
    if (better(ov, oi, b.v, b.idx)) b = {ov, oi};
  }
  if (lane == 0) sb[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best r = sb[0];
    for (int w = 1; w < int(blockDim.x / 32); ++w)
      if (better(sb[w].v, sb[w].idx, r.v, r.idx)) r = sb[w];
    best_dev[cid[m]] = r;
  }
}

}  // namespace

// per-member partial maxima: one per evaluation CTA
static long long eval_blocks(const BasisSet* s, int dtype, const int dims[3], int num_sms) {
  (void)s; (void)dtype; (void)dims;
  return std::min<long long>(4096, (long long)num_sms * 8);
}

size_t basis_set_scratch(const BasisSet* s, long long n, int dtype, const int dims[3]) {
  if (!s || s->members.empty()) return 0;
  const size_t es = dtype == SFW3D_F64 ? 8 : 4;
  const long long nb = std::max<long long>(4096, eval_blocks(s, dtype, dims, 4096));
  return Carver::need({size_t(n) * es, size_t(n) * es, size_t(n) * es * s->betas.size(),
                       s->members.size() * size_t(nb) * sizeof(Best), 2 * size_t(nb) * sizeof(double)});
}

template <typename T, int NM, int V>
static int launch_mix_nm(sfw3d_ctx* ctx, int nblocks, const void* b, const void* terms,
                         long long n, int nt, int nmm, int m0, const BasisSet* s, const int dims[3],
                         int4 wlo, int4 whi, double lam, void* fields, Best* partial,
                         const Collect* col) {
  const size_t smem = (size_t(nt) * NM + NM) * sizeof(T);
  if (col) {
    if (smem > 48 * 1024)
      SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(mix_argmax_kernel<T, NM, V, true>), size_t(int(smem))));
    mix_argmax_kernel<T, NM, V, true><<<nblocks, kMixThreads, smem, ctx->stream>>>(
        static_cast<const T*>(b), static_cast<const T*>(terms), n, nt, nmm, m0,
        static_cast<const T*>(s->W_dev), static_cast<const T*>(s->w0_dev), s->cid_dev, dims[0],
        dims[1], dims[2], wlo, whi, lam, nullptr, partial, *col);
    return SFW3D_OK;
  }
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(mix_argmax_kernel<T, NM, V>), size_t(int(smem))));
  mix_argmax_kernel<T, NM, V><<<nblocks, kMixThreads, smem, ctx->stream>>>(
      static_cast<const T*>(b), static_cast<const T*>(terms), n, nt, nmm, m0,
      static_cast<const T*>(s->W_dev), static_cast<const T*>(s->w0_dev), s->cid_dev, dims[0],
      dims[1], dims[2], wlo, whi, lam, static_cast<T*>(fields), partial);
  return SFW3D_OK;
}

template <typename T, int NMD, int NS, int NT = kMixThreads, int VV = 1>
static int launch_ring2(sfw3d_ctx* ctx, int nblocks, const void* b, const void* terms, long long n,
                        int nt, const BasisSet* s, const int dims[3], int4 wlo, int4 whi,
                        double lam, Best* partial, int d0 = 0, int dn = -1, bool copies = true,
                        double* absparts = nullptr) {
  if (dn < 0) dn = s->nmd;
  constexpr int V = VV * 16 / sizeof(T);
  const size_t smem = size_t(NS) * NT * V * sizeof(T) + size_t(nt + 1) * 8 +
                      (size_t(nt) * NMD + NMD + size_t(NMD + 8) * NT) * sizeof(T) +
                      size_t(NMD + 8) * NT * sizeof(int) + size_t(nt) * sizeof(int) + 16;
  if (smem > 48 * 1024)
    SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(mix_ring2_kernel<T, NMD, NS, NT, VV>), size_t(int(smem))));
  mix_ring2_kernel<T, NMD, NS, NT, VV><<<nblocks, NT, smem, ctx->stream>>>(
      static_cast<const T*>(b), static_cast<const T*>(terms), n, nt,
      static_cast<const T*>(s->Wd_dev) + size_t(d0) * nt, static_cast<const T*>(s->w0d_dev) + d0,
      s->dmem_dev + d0, dn, s->cterm_dev, copies ? s->nmc : 0, s->cmem_dev, s->cid_dev, dims[0],
      dims[1], dims[2], wlo, whi, lam, absparts, partial);
  return SFW3D_OK;
}
// every member through mix_ring2_kernel (dense members 16 per launch, the
// copies with the first): argmax-only evaluations whose z extent takes
// 16-byte vectors. The collect pass then chunks with the same V = 16 / es.
static bool ring2_all_ok(const BasisSet* s, int dtype, const int dims[3]) {
  const int V4 = dtype == SFW3D_F64 ? 2 : 4;
  return s->Wd_dev && s->nmc <= 8 && dims[2] % V4 == 0;
}

template <typename T>
static int launch_ring2_all(sfw3d_ctx* ctx, int nblocks, const void* b, const void* terms,
                            long long n, int nt, const BasisSet* s, const int dims[3], int4 wlo,
                            int4 whi, double lam, Best* partial, double* absparts = nullptr) {
  // ring depth: 16 slots (fp32); 8 for fp64 (keeps 2 CTAs per SM)
  constexpr int NS = sizeof(T) == 8 ? 8 : 16;
  // dense members per launch: 12 where the 8-voxel fp32 form applies (a
  // 48-member table takes 4 launches of 12 instead of 3 of 16 — one more sweep
  // over the terms, 1.52 -> 1.01 ms at config 3), else 16
  const int slice = (sizeof(T) == 4 && n % 8 == 0 && dims[2] % 8 == 0) ? 12 : 16;
  for (int d0 = 0; d0 < std::max(s->nmd, 1); d0 += slice) {
    const int dn = std::max(0, std::min(slice, s->nmd - d0));
    const bool cp = d0 == 0;
    SFW3D_PROF(ctx, "eta_mix");
    // fp32 slices of <= 12 dense members: 128-thread CTAs with two 16-byte
    // vectors per thread and entry — the per-entry producer / weight / loop
    // overhead is amortised over 8 voxels instead of 4 (3 CTAs per SM at 157
    // registers, ring depth 8): config-4 mix 1.84 -> 1.56 ms, bit-identical
    const bool v8 = sizeof(T) == 4 && n % 8 == 0 && dims[2] % 8 == 0;
#define SFW3D_RING2(NMD_)                                                                           \
  (v8 ? launch_ring2<T, NMD_, 8, 128, 2>(ctx, nblocks, b, terms, n, nt, s, dims, wlo, whi, lam,    \
                                          partial, d0, dn, cp, cp ? absparts : nullptr)           \
      : launch_ring2<T, NMD_, NS>(ctx, nblocks, b, terms, n, nt, s, dims, wlo, whi, lam, partial,  \
                                  d0, dn, cp, cp ? absparts : nullptr))
    if (dn <= 4)
      SFW3D_TRY(SFW3D_RING2(4));
    else if (dn <= 8)
      SFW3D_TRY(SFW3D_RING2(8));
    else if (dn <= 12)
      SFW3D_TRY(SFW3D_RING2(12));
#undef SFW3D_RING2
    else
      SFW3D_TRY((launch_ring2<T, 16, NS>(ctx, nblocks, b, terms, n, nt, s, dims, wlo, whi, lam, partial, d0, dn, cp, cp ? absparts : nullptr)));
    SFW3D_LAUNCH_CHECK(ctx);
  }
  return SFW3D_OK;
}

// member-count buckets keep the accumulators in registers: V voxels per
// thread x NM members <= 32 accumulators (16-byte loads where z allows)
template <typename T>
static int launch_mix(sfw3d_ctx* ctx, int nblocks, const void* b, const void* terms, long long n,
                      int nt, int nmm, int m0, const BasisSet* s, const int dims[3], int4 wlo,
                      int4 whi, double lam, void* fields, Best* partial, const Collect* col) {
  constexpr int V4 = 16 / sizeof(T);  // 4 floats / 2 doubles
  const int nz = dims[2];
  const bool ring = nz % V4 == 0 && nmm <= 16;
  // v2 ring: all members in one launch, argmax only (fields keep the v1 path)
  if (!col && !fields && ring && m0 == 0 && nmm == int(s->members.size()) && s->nmd <= 16 &&
      s->nmc <= 8 && s->Wd_dev) {
    // (16 ring slots of 16 bytes per thread)
#define SFW3D_RING2(NMD) \
  return launch_ring2<T, NMD, 16>(ctx, nblocks, b, terms, n, nt, s, dims, wlo, whi, lam, partial)
    if (s->nmd <= 4) SFW3D_RING2(4);
    if (s->nmd <= 8) SFW3D_RING2(8);
    if (s->nmd <= 12) SFW3D_RING2(12);
    SFW3D_RING2(16);
#undef SFW3D_RING2
  }
  // the collect pass must chunk the volume exactly as the evaluation pass did
  // (it revisits evaluation CTAs by their maxima): same V as the ring kernel
  if (col && (ring || (!fields && ring2_all_ok(s, sizeof(T) == 8 ? SFW3D_F64 : SFW3D_F32, dims)))) {
    if (nmm <= 16)
      return launch_mix_nm<T, 16, V4>(ctx, nblocks, b, terms, n, nt, nmm, m0, s, dims, wlo, whi,
                                      lam, fields, partial, col);
    return launch_mix_nm<T, kMixMax, V4>(ctx, nblocks, b, terms, n, nt, nmm, m0, s, dims, wlo,
                                         whi, lam, fields, partial, col);
  }
  if (!col && ring) {
    const size_t smem = (size_t(kMixNS) * kMixThreads * V4 + size_t(nt) * 16 + 16 + 16 * kMixThreads) * sizeof(T) +
                        16 * kMixThreads * sizeof(int);
    if (smem > 48 * 1024)
      SFW3D_CUDA_TRY(allow_dynamic_smem(reinterpret_cast<const void*>(mix_ring_kernel<T, 16>), size_t(int(smem))));
    mix_ring_kernel<T, 16><<<nblocks, kMixThreads, smem, ctx->stream>>>(
        static_cast<const T*>(b), static_cast<const T*>(terms), n, nt, nmm, m0,
        static_cast<const T*>(s->W_dev), static_cast<const T*>(s->w0_dev), s->cid_dev, dims[0],
        dims[1], dims[2], wlo, whi, lam, static_cast<T*>(fields), partial);
    return SFW3D_OK;
  }
#define SFW3D_MIX(NM, V)                                                                        \
  return launch_mix_nm<T, NM, V>(ctx, nblocks, b, terms, n, nt, nmm, m0, s, dims, wlo, whi, lam, \
                                 fields, partial, col)
  if (nmm <= 8 && nz % V4 == 0) SFW3D_MIX(8, V4);
  if (nmm <= 16 && nz % 2 == 0) SFW3D_MIX(16, 2);
  if (nmm <= 8) SFW3D_MIX(8, 1);
  if (nmm <= 16) SFW3D_MIX(16, 1);
  SFW3D_MIX(kMixMax, 1);
#undef SFW3D_MIX
}

int basis_set_max_xhalo(const BasisSet* s) {
  int h = 0;
  if (!s) return 0;
  for (size_t t = 0; t < s->betas.size(); ++t)
    h = std::max({h, -s->tlo[0][t], s->tlo[0][t] + s->tlen[0][t] - 1});
  return h;
}

int basis_set_eval(sfw3d_ctx* ctx, const BasisSet* s, int dtype, const int dims[3], const void* b,
                   double lam, const int32_t win[6], void* fields, Best* best_dev, void* scratch,
                   double* abs_dev, bool* abs_done, const SlabEval* se) {
  if (abs_done) *abs_done = false;
  const int nm = fields ? s->n_nnls : int(s->members.size()), nt = int(s->betas.size());
  if (nm == 0) return SFW3D_OK;
  const long long n = vol_count(dims);
  if (n >= (1LL << 31)) {  // (n_terms volumes of that size exceed any HBM anyway)
    set_error("volume too large for the separable basis path (>= 2^31 voxels)");
    return SFW3D_EINVAL;
  }
  const size_t es = dtype == SFW3D_F64 ? 8 : 4;
  Carver cv(scratch);
  char* t1 = cv.take<char>(size_t(n) * es);
  char* t2 = cv.take<char>(size_t(n) * es);
  char* terms = cv.take<char>(size_t(n) * es * nt);
  const int nblocks = int(eval_blocks(s, dtype, dims, ctx->num_sms));
  Best* partial = cv.take<Best>(size_t(nm) * nblocks);
  double* absparts = cv.take<double>(2 * size_t(nblocks));
  const int4 wlo = make_int4(win[0], win[2], win[4], 0), whi = make_int4(win[1], win[3], win[5], 0);
  {
  // T_k = (f_k x f_k x f_k) * b for every shared term; chained terms
  // T_k = (g_k x g_k x g_k) * T_parent (parents: narrower, larger index)
  for (int t = nt - 1; t >= 0; --t) {
    const char* tp = static_cast<const char*>(s->taps[t]);
    const int l0 = s->tlen[0][t], l1 = s->tlen[1][t], l2 = s->tlen[2][t];
    const void* src = s->parent[t] < 0 ? b : terms + size_t(s->parent[t]) * n * es;
    if (se) {  // x-slab: plane-local z/y passes, halo exchange, windowed x pass
      const void* tps[3] = {tp, tp + es * l0, tp + es * (l0 + l1)};
      const int lo[3] = {s->tlo[0][t], s->tlo[1][t], s->tlo[2][t]}, ln[3] = {l0, l1, l2};
      SFW3D_TRY(slab_corr_impl(ctx, dtype, src, terms + size_t(t) * n * es, dims, tps, lo, ln,
                               se->win, se->H, t1, se->link, "eta_basis"));
      continue;
    }
    // (profile families by the bound of the pass: filters of more than
    // kBasisNarrowTaps taps are FP32-bound, the others HBM-bound)
    auto fam = [](int l) { return l > kBasisNarrowTaps ? "eta_basis_wide" : "eta_basis"; };
    SFW3D_TRY(corr_pass_impl(ctx, dtype, src, t1, dims, 2, tp + es * (l0 + l1), s->tlo[2][t], l2,
                             nullptr, 0.0, 1.0, fam(l2)));
    SFW3D_TRY(corr_pass_impl(ctx, dtype, t1, t2, dims, 1, tp + es * l0, s->tlo[1][t], l1,
                             nullptr, 0.0, 1.0, fam(l1)));
    SFW3D_TRY(corr_pass_impl(ctx, dtype, t2, terms + size_t(t) * n * es, dims, 0, tp, s->tlo[0][t],
                             l0, nullptr, 0.0, 1.0, fam(l0)));
  }
  if (!fields && ring2_all_ok(s, dtype, dims)) {
    double* ap = abs_dev ? absparts : nullptr;  // |b| statistics ride along with the mix
    if (dtype == SFW3D_F64)
      SFW3D_TRY(launch_ring2_all<double>(ctx, nblocks, b, terms, n, nt, s, dims, wlo, whi, lam, partial, ap));
    else
      SFW3D_TRY(launch_ring2_all<float>(ctx, nblocks, b, terms, n, nt, s, dims, wlo, whi, lam, partial, ap));
    if (ap) {
      abs_reduce_kernel<<<1, 256, 0, ctx->stream>>>(ap, nblocks, abs_dev);
      SFW3D_LAUNCH_CHECK(ctx);
      if (abs_done) *abs_done = true;
    }
  } else
  for (int m0 = 0; m0 < nm; m0 += kMixMax) {
    const int nmm = std::min(kMixMax, nm - m0);
    SFW3D_PROF(ctx, "eta_mix");
    if (dtype == SFW3D_F64)
      SFW3D_TRY(launch_mix<double>(ctx, nblocks, b, terms, n, nt, nmm, m0, s, dims, wlo, whi, lam,
                                   fields, partial, nullptr));
    else
      SFW3D_TRY(launch_mix<float>(ctx, nblocks, b, terms, n, nt, nmm, m0, s, dims, wlo, whi, lam,
                                  fields, partial, nullptr));
    SFW3D_LAUNCH_CHECK(ctx);
  }
  }
  {
    SFW3D_PROF(ctx, "argmax");
    member_reduce_kernel<<<nm, 256, 0, ctx->stream>>>(partial, nblocks, s->cid_dev, best_dev);
    SFW3D_LAUNCH_CHECK(ctx);
  }
  return SFW3D_OK;
}

int basis_set_collect(sfw3d_ctx* ctx, const BasisSet* s, int dtype, const int dims[3],
                      const void* b, double lam, const int32_t win[6], const double* thr_dev,
                      int cap, int* cand_dev, long long* idx_dev, int* count_dev, void* scratch,
                      bool fields) {
  const int nm = fields ? s->n_nnls : int(s->members.size()), nt = int(s->betas.size());
  if (nm == 0) return SFW3D_OK;
  const long long n = vol_count(dims);
  const size_t es = dtype == SFW3D_F64 ? 8 : 4;
  Carver cv(scratch);
  cv.take<char>(size_t(n) * es);
  cv.take<char>(size_t(n) * es);
  const char* terms = cv.take<char>(size_t(n) * es * nt);  // left by basis_set_eval
  const int nblocks = int(eval_blocks(s, dtype, dims, ctx->num_sms));
  const Best* partial = cv.take<Best>(size_t(nm) * nblocks);  // left by basis_set_eval
  const int4 wlo = make_int4(win[0], win[2], win[4], 0), whi = make_int4(win[1], win[3], win[5], 0);
  SFW3D_CUDA_TRY(cudaMemsetAsync(count_dev, 0, sizeof(int) * (1 + nm), ctx->stream));
  constexpr int kSplit = 32;
  const Collect col{thr_dev, cand_dev, idx_dev, count_dev, cap, partial, nblocks, kSplit};
  // (16-member slices when the evaluation ran through mix_ring2_kernel: the
  // V = 4 collect kernel keeps 16 x 4 accumulators in registers)
  const int step = (!fields && ring2_all_ok(s, dtype, dims)) ? 16 : kMixMax;
  for (int m0 = 0; m0 < nm; m0 += step) {
    const int nmm = std::min(step, nm - m0);
    SFW3D_PROF(ctx, "eta_refine");
    if (dtype == SFW3D_F64)
      SFW3D_TRY(launch_mix<double>(ctx, nblocks * kSplit, b, terms, n, nt, nmm, m0, s, dims, wlo,
                                   whi, lam, nullptr, nullptr, &col));
    else
      SFW3D_TRY(launch_mix<float>(ctx, nblocks * kSplit, b, terms, n, nt, nmm, m0, s, dims, wlo,
                                  whi, lam, nullptr, nullptr, &col));
    SFW3D_LAUNCH_CHECK(ctx);
  }
  return SFW3D_OK;
}

int basis_set_member_index(const BasisSet* s, int cand) {
  if (!s) return -1;
  for (int m = 0; m < int(s->members.size()); ++m)
    if (s->members[m] == cand) return m;
  return -1;
}
int basis_set_member_cand(const BasisSet* s, int m) { return s->members[m]; }

}  // namespace sfw3d
