// Limited-memory BFGS with bounds (L-BFGS-B), host C++.
//
// The reference drives its two continuous steps with scipy's L-BFGS-B
// (refine_eta_max, certificate.py:217-218; local_descent, solvers.py:231-232).
// This is the in-library optimiser that replaces the Python callback loop:
// the published algorithm (Byrd, Lu, Nocedal, Zhu 1995: generalized Cauchy
// point + direct primal subspace minimisation; Morales & Nocedal 2011:
// projected subspace step; More & Thuente 1994 line search), restated with
// the driver conventions scipy.optimize.minimize(method="L-BFGS-B") applies
// (maxcor 10, factr = ftol / eps, pgtol = gtol, maxls 20, maxiter counted on
// accepted iterates, maxfun 15000), so that the iterates follow scipy's to
// rounding.  The objective is a callback: the device kernels evaluate it, the
// (serial, tiny) quasi-Newton algebra runs on the calling host thread.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace sfw3d {
namespace lbfgsb {

enum Status : int {
    CONV_PGTOL = 0,    // ||proj g||_inf <= pgtol
    CONV_FTOL = 1,     // relative reduction of f <= factr * eps
    STOP_MAXITER = 2,  // iteration limit (scipy: warnflag 1)
    STOP_MAXFUN = 3,   // evaluation limit (scipy: warnflag 1)
    ABNORMAL = 4,      // line search gave up (scipy: "ABNORMAL" message, warnflag 2)
    CALLBACK_ERROR = 5 // the objective reported an error
};

struct Options {
    int m = 10;
    double factr = 1e7;   // ftol / eps
    double pgtol = 1e-5;
    int maxiter = 15000;
    int maxfun = 15000;
    int maxls = 20;
};

struct Result {
    int status = ABNORMAL;
    int iterations = 0;
    int evaluations = 0;
    double f = 0.0;
    double pg_norm = 0.0;
    int callback_code = 0;
};

// int fg(user, x, &f, g): 0 = ok; anything else aborts with CALLBACK_ERROR
typedef int (*Objective)(void* user, const double* x, double* f, double* g);

namespace detail {

constexpr double EPS = 2.220446049250313e-16;

inline double dot(int n, const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

// upper Cholesky factor R (R^T R = A) in place on the upper triangle of the
// leading k x k block of a (row-major, leading dimension ld); false if A is
// not positive definite
inline bool cholesky_upper(double* a, int ld, int k) {
    for (int j = 0; j < k; ++j) {
        double s = 0.0;
        for (int i = 0; i < j; ++i) {
            double t = a[i * ld + j];
            for (int p = 0; p < i; ++p) t -= a[p * ld + i] * a[p * ld + j];
            t /= a[i * ld + i];
            a[i * ld + j] = t;
            s += t * t;
        }
        s = a[j * ld + j] - s;
        if (!(s > 0.0)) return false;
        a[j * ld + j] = std::sqrt(s);
    }
    return true;
}
// R x = b (upper), in place
inline bool solve_upper(const double* r, int ld, int k, double* b) {
    for (int i = k - 1; i >= 0; --i) {
        double t = b[i];
        for (int j = i + 1; j < k; ++j) t -= r[i * ld + j] * b[j];
        if (r[i * ld + i] == 0.0) return false;
        b[i] = t / r[i * ld + i];
    }
    return true;
}
// R^T x = b, in place
inline bool solve_upper_t(const double* r, int ld, int k, double* b) {
    for (int i = 0; i < k; ++i) {
        double t = b[i];
        for (int j = 0; j < i; ++j) t -= r[j * ld + i] * b[j];
        if (r[i * ld + i] == 0.0) return false;
        b[i] = t / r[i * ld + i];
    }
    return true;
}

// ---- More-Thuente line search (MINPACK-2 dcsrch / dcstep) ----
struct LineSearch {
    bool brackt = false;
    int stage = 1;
    double ginit = 0, gtest = 0, gx = 0, gy = 0, finit = 0, fx = 0, fy = 0;
    double stx = 0, sty = 0, stmin = 0, stmax = 0, width = 0, width1 = 0;
};
enum LsTask { LS_START, LS_FG, LS_CONV, LS_WARN, LS_ERROR };

inline void dcstep(double& stx, double& fx, double& dx, double& sty, double& fy, double& dy,
                   double& stp, double fp, double dp, bool& brackt, double stpmin, double stpmax) {
    const double sgnd = dp * (dx / std::fabs(dx));
    double stpf, stpc, stpq, theta, s, gamma, p, q, r;
    if (fp > fx) {
        theta = 3.0 * (fx - fp) / (stp - stx) + dx + dp;
        s = std::max({std::fabs(theta), std::fabs(dx), std::fabs(dp)});
        gamma = s * std::sqrt((theta / s) * (theta / s) - (dx / s) * (dp / s));
        if (stp < stx) gamma = -gamma;
        p = (gamma - dx) + theta;
        q = ((gamma - dx) + gamma) + dp;
        r = p / q;
        stpc = stx + r * (stp - stx);
        stpq = stx + ((dx / ((fx - fp) / (stp - stx) + dx)) / 2.0) * (stp - stx);
        if (std::fabs(stpc - stx) < std::fabs(stpq - stx)) stpf = stpc;
        else stpf = stpc + (stpq - stpc) / 2.0;
        brackt = true;
    } else if (sgnd < 0.0) {
        theta = 3.0 * (fx - fp) / (stp - stx) + dx + dp;
        s = std::max({std::fabs(theta), std::fabs(dx), std::fabs(dp)});
        gamma = s * std::sqrt((theta / s) * (theta / s) - (dx / s) * (dp / s));
        if (stp > stx) gamma = -gamma;
        p = (gamma - dp) + theta;
        q = ((gamma - dp) + gamma) + dx;
        r = p / q;
        stpc = stp + r * (stx - stp);
        stpq = stp + (dp / (dp - dx)) * (stx - stp);
        stpf = std::fabs(stpc - stp) > std::fabs(stpq - stp) ? stpc : stpq;
        brackt = true;
    } else if (std::fabs(dp) < std::fabs(dx)) {
        theta = 3.0 * (fx - fp) / (stp - stx) + dx + dp;
        s = std::max({std::fabs(theta), std::fabs(dx), std::fabs(dp)});
        gamma = s * std::sqrt(std::max(0.0, (theta / s) * (theta / s) - (dx / s) * (dp / s)));
        if (stp > stx) gamma = -gamma;
        p = (gamma - dp) + theta;
        q = (gamma + (dx - dp)) + gamma;
        r = p / q;
        if (r < 0.0 && gamma != 0.0) stpc = stp + r * (stx - stp);
        else if (stp > stx) stpc = stpmax;
        else stpc = stpmin;
        stpq = stp + (dp / (dp - dx)) * (stx - stp);
        if (brackt) {
            stpf = std::fabs(stpc - stp) < std::fabs(stpq - stp) ? stpc : stpq;
            if (stp > stx) stpf = std::min(stp + 0.66 * (sty - stp), stpf);
            else stpf = std::max(stp + 0.66 * (sty - stp), stpf);
        } else {
            stpf = std::fabs(stpc - stp) > std::fabs(stpq - stp) ? stpc : stpq;
            stpf = std::min(stpmax, stpf);
            stpf = std::max(stpmin, stpf);
        }
    } else {
        if (brackt) {
            theta = 3.0 * (fp - fy) / (sty - stp) + dy + dp;
            s = std::max({std::fabs(theta), std::fabs(dy), std::fabs(dp)});
            gamma = s * std::sqrt((theta / s) * (theta / s) - (dy / s) * (dp / s));
            if (stp > sty) gamma = -gamma;
            p = (gamma - dp) + theta;
            q = ((gamma - dp) + gamma) + dy;
            r = p / q;
            stpc = stp + r * (sty - stp);
            stpf = stpc;
        } else if (stp > stx) {
            stpf = stpmax;
        } else {
            stpf = stpmin;
        }
    }
    if (fp > fx) {
        sty = stp; fy = fp; dy = dp;
    } else {
        if (sgnd < 0.0) { sty = stx; fy = fx; dy = dx; }
        stx = stp; fx = fp; dx = dp;
    }
    stp = stpf;
}

inline LsTask dcsrch(LineSearch& L, LsTask task, double f, double g, double& stp, double ftol,
                     double gtol, double xtol, double stpmin, double stpmax) {
    if (task == LS_START) {
        if (stp < stpmin || stp > stpmax || g >= 0.0 || stpmax < stpmin) return LS_ERROR;
        L.brackt = false;
        L.stage = 1;
        L.finit = f;
        L.ginit = g;
        L.gtest = ftol * L.ginit;
        L.width = stpmax - stpmin;
        L.width1 = L.width / 0.5;
        L.stx = 0.0; L.fx = L.finit; L.gx = L.ginit;
        L.sty = 0.0; L.fy = L.finit; L.gy = L.ginit;
        L.stmin = 0.0;
        L.stmax = stp + 4.0 * stp;
        return LS_FG;
    }
    const double ftest = L.finit + stp * L.gtest;
    if (L.stage == 1 && f <= ftest && g >= 0.0) L.stage = 2;
    LsTask out = LS_FG;
    if (L.brackt && (stp <= L.stmin || stp >= L.stmax)) out = LS_WARN;
    if (L.brackt && L.stmax - L.stmin <= xtol * L.stmax) out = LS_WARN;
    if (stp == stpmax && f <= ftest && g <= L.gtest) out = LS_WARN;
    if (stp == stpmin && (f > ftest || g >= L.gtest)) out = LS_WARN;
    if (f <= ftest && std::fabs(g) <= gtol * (-L.ginit)) out = LS_CONV;
    if (out != LS_FG) return out;
    if (L.stage == 1 && f <= L.fx && f > ftest) {
        double fm = f - stp * L.gtest, fxm = L.fx - L.stx * L.gtest, fym = L.fy - L.sty * L.gtest;
        double gm = g - L.gtest, gxm = L.gx - L.gtest, gym = L.gy - L.gtest;
        dcstep(L.stx, fxm, gxm, L.sty, fym, gym, stp, fm, gm, L.brackt, L.stmin, L.stmax);
        L.fx = fxm + L.stx * L.gtest;
        L.fy = fym + L.sty * L.gtest;
        L.gx = gxm + L.gtest;
        L.gy = gym + L.gtest;
    } else {
        dcstep(L.stx, L.fx, L.gx, L.sty, L.fy, L.gy, stp, f, g, L.brackt, L.stmin, L.stmax);
    }
    if (L.brackt) {
        if (std::fabs(L.sty - L.stx) >= 0.66 * L.width1) stp = L.stx + 0.5 * (L.sty - L.stx);
        L.width1 = L.width;
        L.width = std::fabs(L.sty - L.stx);
    }
    if (L.brackt) {
        L.stmin = std::min(L.stx, L.sty);
        L.stmax = std::max(L.stx, L.sty);
    } else {
        L.stmin = stp + 1.1 * (stp - L.stx);
        L.stmax = stp + 4.0 * (stp - L.stx);
    }
    stp = std::max(stp, stpmin);
    stp = std::min(stp, stpmax);
    if ((L.brackt && (stp <= L.stmin || stp >= L.stmax)) ||
        (L.brackt && L.stmax - L.stmin <= xtol * L.stmax))
        stp = L.stx;
    return LS_FG;
}

}  // namespace detail

// nbd[i]: 0 unbounded, 1 lower only, 2 both, 3 upper only
class Minimizer {
public:
    Minimizer(int n, const Options& o) : n_(n), m_(o.m), opt_(o) {
        const int m = m_;
        ws_.assign((size_t)n * m, 0.0);
        wy_.assign((size_t)n * m, 0.0);
        sy_.assign((size_t)m * m, 0.0);
        ss_.assign((size_t)m * m, 0.0);
        wt_.assign((size_t)m * m, 0.0);
        wn_.assign((size_t)4 * m * m, 0.0);
        z_.assign(n, 0.0); r_.assign(n, 0.0); d_.assign(n, 0.0); t_.assign(n, 0.0);
        xp_.assign(n, 0.0); g_.assign(n, 0.0);
        p_.assign(2 * m, 0.0); c_.assign(2 * m, 0.0); wbp_.assign(2 * m, 0.0); v_.assign(2 * m, 0.0);
        bt_.assign(n, 0.0);
        iorder_.assign(n, 0); iwhere_.assign(n, 0); index_.assign(n, 0); isfree_.assign(n, 0);
    }

    Result minimize(double* x, const double* l, const double* u, const int* nbd, Objective fg,
                    void* user) {
        using namespace detail;
        const int n = n_;
        Result res;
        l_ = l; u_ = u; nbd_ = nbd;
        col_ = 0; theta_ = 1.0;
        bool updatd = false;
        // project the start into the box, classify the variables
        bool cnstnd = false, boxed = true;
        for (int i = 0; i < n; ++i) {
            if (nbd[i] > 0) {
                if (nbd[i] <= 2 && x[i] <= l[i]) { if (x[i] < l[i]) x[i] = l[i]; }
                else if (nbd[i] >= 2 && x[i] >= u[i]) { if (x[i] > u[i]) x[i] = u[i]; }
            }
        }
        for (int i = 0; i < n; ++i) {
            if (nbd[i] != 2) boxed = false;
            if (nbd[i] == 0) iwhere_[i] = -1;
            else {
                cnstnd = true;
                iwhere_[i] = (nbd[i] == 2 && u[i] - l[i] <= 0.0) ? 3 : 0;
            }
        }
        double f = 0.0;
        double* g = g_.data();
        auto eval = [&](double& fv) -> bool {
            int code = fg(user, x, &fv, g);
            ++res.evaluations;
            if (code != 0) { res.callback_code = code; return false; }
            return true;
        };
        if (!eval(f)) { res.status = CALLBACK_ERROR; res.f = f; return res; }
        double sbgnrm = projgr(x, g);
        if (sbgnrm <= opt_.pgtol) {
            res.status = CONV_PGTOL; res.f = f; res.pg_norm = sbgnrm; return res;
        }
        int iter = 0;
        auto reset_memory = [&]() { col_ = 0; theta_ = 1.0; updatd = false; };
        for (;;) {
            // ---- generalized Cauchy point ----
            int nfree = 0;
            bool have_gcp = true;
            if (!cnstnd && col_ > 0) {
                std::memcpy(z_.data(), x, sizeof(double) * n);
                nfree = n;
                for (int i = 0; i < n; ++i) index_[i] = i;
                have_gcp = false;
            } else {
                if (!cauchy(x, g, sbgnrm)) { reset_memory(); continue; }
                nfree = 0;
                for (int i = 0; i < n; ++i)
                    if (iwhere_[i] <= 0) index_[nfree++] = i;
            }
            // ---- subspace minimisation ----
            if (nfree != 0 && col_ != 0) {
                for (int i = 0; i < n; ++i) isfree_[i] = 0;
                for (int i = 0; i < nfree; ++i) isfree_[index_[i]] = 1;
                if (!formk(nfree)) { reset_memory(); continue; }
                if (!cmprlb(x, g, nfree, cnstnd, have_gcp)) { reset_memory(); continue; }
                if (!subsm(x, g, nfree)) { reset_memory(); continue; }
            }
            // ---- line search along d = z - x ----
            for (int i = 0; i < n; ++i) d_[i] = z_[i] - x[i];
            const double dtd = dot(n, d_.data(), d_.data());
            const double dnorm = std::sqrt(dtd);
            double stpmx = 1e10;
            if (cnstnd) {
                if (iter == 0) stpmx = 1.0;
                else {
                    for (int i = 0; i < n; ++i) {
                        const double a1 = d_[i];
                        if (nbd[i] != 0) {
                            if (a1 < 0.0 && nbd[i] <= 2) {
                                const double a2 = l[i] - x[i];
                                if (a2 >= 0.0) stpmx = 0.0;
                                else if (a1 * stpmx < a2) stpmx = a2 / a1;
                            } else if (a1 > 0.0 && nbd[i] >= 2) {
                                const double a2 = u[i] - x[i];
                                if (a2 <= 0.0) stpmx = 0.0;
                                else if (a1 * stpmx > a2) stpmx = a2 / a1;
                            }
                        }
                    }
                }
            }
            double stp = (iter == 0 && !boxed) ? std::min(1.0 / dnorm, stpmx) : 1.0;
            std::memcpy(t_.data(), x, sizeof(double) * n);
            std::memcpy(r_.data(), g, sizeof(double) * n);
            const double fold = f;
            int ifun = 0, iback = 0;
            double gd = dot(n, g, d_.data());
            const double gdold = gd;
            bool ls_failed = gd >= 0.0;
            LineSearch L;
            LsTask task = LS_START;
            bool cb_error = false;
            if (!ls_failed) {
                for (;;) {
                    task = dcsrch(L, task, f, gd, stp, 1e-3, 0.9, 0.1, 0.0, stpmx);
                    if (task != LS_FG) {
                        if (task == LS_ERROR) ls_failed = true;
                        break;
                    }
                    ++ifun;
                    iback = ifun - 1;
                    if (iback >= opt_.maxls) { ls_failed = true; break; }
                    if (stp == 1.0) std::memcpy(x, z_.data(), sizeof(double) * n);
                    else for (int i = 0; i < n; ++i) x[i] = stp * d_[i] + t_[i];
                    if (!eval(f)) { cb_error = true; break; }
                    gd = dot(n, g, d_.data());
                }
            }
            if (cb_error) { res.status = CALLBACK_ERROR; break; }
            if (ls_failed) {
                std::memcpy(x, t_.data(), sizeof(double) * n);
                std::memcpy(g, r_.data(), sizeof(double) * n);
                f = fold;
                if (col_ == 0) { res.status = ABNORMAL; ++iter; break; }
                reset_memory();
                continue;
            }
            // ---- new iterate ----
            ++iter;
            sbgnrm = projgr(x, g);
            if (iter >= opt_.maxiter) { res.status = STOP_MAXITER; break; }
            if (res.evaluations > opt_.maxfun) { res.status = STOP_MAXFUN; break; }
            if (sbgnrm <= opt_.pgtol) { res.status = CONV_PGTOL; break; }
            const double ddum = std::max({std::fabs(fold), std::fabs(f), 1.0});
            if (fold - f <= EPS * opt_.factr * ddum) { res.status = CONV_FTOL; break; }
            // ---- quasi-Newton update: s = stp d, y = g - g_old ----
            for (int i = 0; i < n; ++i) r_[i] = g[i] - r_[i];
            const double rr = dot(n, r_.data(), r_.data());
            double dr, dd;
            if (stp == 1.0) { dr = gd - gdold; dd = -gdold; }
            else {
                dr = (gd - gdold) * stp;
                for (int i = 0; i < n; ++i) d_[i] *= stp;
                dd = -gdold * stp;
            }
            if (dr <= EPS * dd) { updatd = false; continue; }
            updatd = true;
            matupd(rr, dr, stp, dtd);
            if (!formt()) { reset_memory(); continue; }
        }
        (void)updatd;
        res.iterations = iter;
        res.f = f;
        res.pg_norm = projgr(x, g);
        return res;
    }

    const double* gradient() const { return g_.data(); }

private:
    int n_, m_;
    Options opt_;
    const double *l_ = nullptr, *u_ = nullptr;
    const int* nbd_ = nullptr;
    int col_ = 0;
    double theta_ = 1.0;
    // ws/wy: n x m with the corrections in age order (column 0 oldest)
    std::vector<double> ws_, wy_, sy_, ss_, wt_, wn_;
    std::vector<double> z_, r_, d_, t_, xp_, g_, p_, c_, wbp_, v_, bt_;
    std::vector<int> iorder_, iwhere_, index_, isfree_;

    double projgr(const double* x, const double* g) const {
        double nrm = 0.0;
        for (int i = 0; i < n_; ++i) {
            double gi = g[i];
            if (nbd_[i] != 0) {
                if (gi < 0.0) { if (nbd_[i] >= 2) gi = std::max(x[i] - u_[i], gi); }
                else { if (nbd_[i] <= 2) gi = std::min(x[i] - l_[i], gi); }
            }
            nrm = std::max(nrm, std::fabs(gi));
        }
        return nrm;
    }

    // product of the 2col x 2col middle matrix of the compact form with v
    bool bmv(const double* v, double* p) const {
        using namespace detail;
        const int col = col_, m = m_;
        if (col == 0) return true;
        p[col] = v[col];
        for (int i = 1; i < col; ++i) {
            double sum = 0.0;
            for (int k = 0; k < i; ++k) sum += sy_[i * m + k] * v[k] / sy_[k * m + k];
            p[col + i] = v[col + i] + sum;
        }
        if (!solve_upper_t(wt_.data(), m, col, p + col)) return false;
        for (int i = 0; i < col; ++i) p[i] = v[i] / std::sqrt(sy_[i * m + i]);
        if (!solve_upper(wt_.data(), m, col, p + col)) return false;
        for (int i = 0; i < col; ++i) p[i] = -p[i] / std::sqrt(sy_[i * m + i]);
        for (int i = 0; i < col; ++i) {
            double sum = 0.0;
            for (int k = i + 1; k < col; ++k) sum += sy_[k * m + i] * p[col + k] / sy_[i * m + i];
            p[i] += sum;
        }
        return true;
    }

    // heap of breakpoints (1-based as published): least element moved to t[n]
    static void hpsolb(int n, double* t, int* iorder, int iheap) {
        if (iheap == 0) {
            for (int k = 2; k <= n; ++k) {
                const double ddum = t[k];
                const int indxin = iorder[k];
                int i = k;
                while (i > 1) {
                    const int j = i / 2;
                    if (ddum < t[j]) { t[i] = t[j]; iorder[i] = iorder[j]; i = j; }
                    else break;
                }
                t[i] = ddum; iorder[i] = indxin;
            }
        }
        if (n > 1) {
            int i = 1;
            const double out = t[1];
            const int indxou = iorder[1];
            const double ddum = t[n];
            const int indxin = iorder[n];
            for (;;) {
                int j = i + i;
                if (j <= n - 1) {
                    if (t[j + 1] < t[j]) j = j + 1;
                    if (t[j] < ddum) { t[i] = t[j]; iorder[i] = iorder[j]; i = j; }
                    else break;
                } else break;
            }
            t[i] = ddum; iorder[i] = indxin;
            t[n] = out; iorder[n] = indxou;
        }
    }

    bool cauchy(const double* x, const double* g, double sbgnrm) {
        using namespace detail;
        const int n = n_, m = m_, col = col_, col2 = 2 * col_;
        double* xcp = z_.data();
        if (sbgnrm <= 0.0) { std::memcpy(xcp, x, sizeof(double) * n); return true; }
        bool bnded = true;
        int nfree = n + 1, nbreak = 0, ibkmin = 0;
        double bkmin = 0.0, f1 = 0.0;
        double* p = p_.data();
        double* c = c_.data();
        double* d = d_.data();
        // 1-based scratch for the breakpoint heap
        if ((int)bt_.size() < n + 1) bt_.assign(n + 1, 0.0);
        if ((int)iorder_.size() < n + 2) iorder_.assign(n + 2, 0);
        double* t = bt_.data();
        int* iorder = iorder_.data();
        for (int i = 0; i < col2; ++i) p[i] = 0.0;
        for (int i = 0; i < n; ++i) {
            const double neggi = -g[i];
            double tl = 0.0, tu = 0.0;
            if (iwhere_[i] != 3 && iwhere_[i] != -1) {
                if (nbd_[i] <= 2) tl = x[i] - l_[i];
                if (nbd_[i] >= 2) tu = u_[i] - x[i];
                const bool xlower = nbd_[i] <= 2 && tl <= 0.0;
                const bool xupper = nbd_[i] >= 2 && tu <= 0.0;
                iwhere_[i] = 0;
                if (xlower) { if (neggi <= 0.0) iwhere_[i] = 1; }
                else if (xupper) { if (neggi >= 0.0) iwhere_[i] = 2; }
                else { if (std::fabs(neggi) <= 0.0) iwhere_[i] = -3; }
            }
            if (iwhere_[i] != 0 && iwhere_[i] != -1) {
                d[i] = 0.0;
            } else {
                d[i] = neggi;
                f1 -= neggi * neggi;
                for (int j = 0; j < col; ++j) {
                    p[j] += wy_[(size_t)i * m + j] * neggi;
                    p[col + j] += ws_[(size_t)i * m + j] * neggi;
                }
                if (nbd_[i] <= 2 && nbd_[i] != 0 && neggi < 0.0) {
                    ++nbreak;
                    iorder[nbreak] = i;
                    t[nbreak] = tl / (-neggi);
                    if (nbreak == 1 || t[nbreak] < bkmin) { bkmin = t[nbreak]; ibkmin = nbreak; }
                } else if (nbd_[i] >= 2 && neggi > 0.0) {
                    ++nbreak;
                    iorder[nbreak] = i;
                    t[nbreak] = tu / neggi;
                    if (nbreak == 1 || t[nbreak] < bkmin) { bkmin = t[nbreak]; ibkmin = nbreak; }
                } else {
                    --nfree;
                    iorder[nfree] = i;
                    if (std::fabs(neggi) > 0.0) bnded = false;
                }
            }
        }
        if (theta_ != 1.0)
            for (int j = col; j < col2; ++j) p[j] *= theta_;
        std::memcpy(xcp, x, sizeof(double) * n);
        if (nbreak == 0 && nfree == n + 1) return true;
        for (int j = 0; j < col2; ++j) c[j] = 0.0;
        double f2 = -theta_ * f1;
        const double f2_org = f2;
        if (col > 0) {
            if (!bmv(p, v_.data())) return false;
            f2 -= dot(col2, v_.data(), p);
        }
        double dtm = -f1 / f2;
        double tsum = 0.0;
        bool all_fixed = false;
        if (nbreak > 0) {
            int nleft = nbreak, iter = 1;
            double tj = 0.0;
            for (;;) {
                const double tj0 = tj;
                int ibp;
                if (iter == 1) {
                    tj = bkmin;
                    ibp = iorder[ibkmin];
                } else {
                    if (iter == 2) {
                        if (ibkmin != nbreak) {
                            t[ibkmin] = t[nbreak];
                            iorder[ibkmin] = iorder[nbreak];
                        }
                    }
                    hpsolb(nleft, t, iorder, iter - 2);
                    tj = t[nleft];
                    ibp = iorder[nleft];
                }
                const double dt = tj - tj0;
                if (dtm < dt) break;
                tsum += dt;
                --nleft;
                ++iter;
                const double dibp = d[ibp];
                d[ibp] = 0.0;
                double zibp;
                if (dibp > 0.0) { zibp = u_[ibp] - x[ibp]; xcp[ibp] = u_[ibp]; iwhere_[ibp] = 2; }
                else { zibp = l_[ibp] - x[ibp]; xcp[ibp] = l_[ibp]; iwhere_[ibp] = 1; }
                if (nleft == 0 && nbreak == n) { dtm = dt; all_fixed = true; break; }
                const double dibp2 = dibp * dibp;
                f1 = f1 + dt * f2 + dibp2 - theta_ * dibp * zibp;
                f2 = f2 - theta_ * dibp2;
                if (col > 0) {
                    for (int j = 0; j < col2; ++j) c[j] += dt * p[j];
                    double* wbp = wbp_.data();
                    for (int j = 0; j < col; ++j) {
                        wbp[j] = wy_[(size_t)ibp * m + j];
                        wbp[col + j] = theta_ * ws_[(size_t)ibp * m + j];
                    }
                    if (!bmv(wbp, v_.data())) return false;
                    const double wmc = dot(col2, c, v_.data());
                    const double wmp = dot(col2, p, v_.data());
                    const double wmw = dot(col2, wbp, v_.data());
                    for (int j = 0; j < col2; ++j) p[j] -= dibp * wbp[j];
                    f1 += dibp * wmc;
                    f2 += 2.0 * dibp * wmp - dibp2 * wmw;
                }
                f2 = std::max(EPS * f2_org, f2);
                if (nleft > 0) { dtm = -f1 / f2; continue; }
                if (bnded) { f1 = 0.0; f2 = 0.0; dtm = 0.0; }
                else dtm = -f1 / f2;
                break;
            }
        }
        if (!all_fixed) {
            if (dtm <= 0.0) dtm = 0.0;
            tsum += dtm;
            for (int i = 0; i < n; ++i) xcp[i] += tsum * d[i];
        }
        if (col > 0)
            for (int j = 0; j < col2; ++j) c[j] += dtm * p[j];
        return true;
    }

    // LEL^T factorisation of the indefinite K of the subspace problem
    bool formk(int nfree) {
        using namespace detail;
        const int n = n_, m = m_, col = col_, m2 = 2 * m_;
        (void)nfree;
        double* wn = wn_.data();
        // upper triangle of [ D + Y'ZZ'Y/theta , -L_a' + R_z' ; . , theta S'AA'S ]
        for (int iy = 0; iy < col; ++iy) {
            for (int jy = 0; jy <= iy; ++jy) {
                double yzy = 0.0, sas = 0.0;
                for (int k = 0; k < n; ++k) {
                    if (isfree_[k]) yzy += wy_[(size_t)k * m + iy] * wy_[(size_t)k * m + jy];
                    else sas += ws_[(size_t)k * m + iy] * ws_[(size_t)k * m + jy];
                }
                wn[jy * m2 + iy] = yzy / theta_;
                wn[(col + jy) * m2 + (col + iy)] = sas * theta_;
            }
            wn[iy * m2 + iy] += sy_[iy * m + iy];
        }
        for (int is = 0; is < col; ++is) {
            for (int jy = 0; jy < col; ++jy) {
                // block (2,1) entry (is, jy) of L_a + R_z; stored transposed in the (1,2) block
                double s = 0.0;
                if (is <= jy) {
                    for (int k = 0; k < n; ++k)
                        if (isfree_[k]) s += ws_[(size_t)k * m + is] * wy_[(size_t)k * m + jy];
                    wn[jy * m2 + (col + is)] = s;
                } else {
                    for (int k = 0; k < n; ++k)
                        if (!isfree_[k]) s += ws_[(size_t)k * m + is] * wy_[(size_t)k * m + jy];
                    wn[jy * m2 + (col + is)] = -s;
                }
            }
        }
        if (!cholesky_upper(wn, m2, col)) return false;
        // (1,2) block := L^-1 (-L_a' + R_z'): solve column by column
        std::vector<double>& tmp = v2_;
        tmp.assign(col, 0.0);
        for (int js = col; js < 2 * col; ++js) {
            for (int i = 0; i < col; ++i) tmp[i] = wn[i * m2 + js];
            if (!solve_upper_t(wn, m2, col, tmp.data())) return false;
            for (int i = 0; i < col; ++i) wn[i * m2 + js] = tmp[i];
        }
        for (int is = col; is < 2 * col; ++is)
            for (int js = is; js < 2 * col; ++js) {
                double s = 0.0;
                for (int i = 0; i < col; ++i) s += wn[i * m2 + is] * wn[i * m2 + js];
                wn[is * m2 + js] += s;
            }
        if (!cholesky_upper(wn + (size_t)col * m2 + col, m2, col)) return false;
        // the lower-left block of the 2col x 2col triangular factor is zero
        for (int i = col; i < 2 * col; ++i)
            for (int j = 0; j < col; ++j) wn[i * m2 + j] = 0.0;
        return true;
    }
    std::vector<double> v2_;

    // r = -Z'(B (xcp - x) + g) on the free variables (into r_[0..nfree))
    bool cmprlb(const double* x, const double* g, int nfree, bool cnstnd, bool have_gcp) {
        const int m = m_, col = col_;
        if (!cnstnd && col > 0 && !have_gcp) {
            for (int i = 0; i < n_; ++i) r_[i] = -g[i];
            return true;
        }
        for (int i = 0; i < nfree; ++i) {
            const int k = index_[i];
            r_[i] = -theta_ * (z_[k] - x[k]) - g[k];
        }
        if (!bmv(c_.data(), p_.data())) return false;
        for (int j = 0; j < col; ++j) {
            const double a1 = p_[j], a2 = theta_ * p_[col + j];
            for (int i = 0; i < nfree; ++i) {
                const int k = index_[i];
                r_[i] += wy_[(size_t)k * m + j] * a1 + ws_[(size_t)k * m + j] * a2;
            }
        }
        return true;
    }

    // direct primal subspace minimisation with the projected step
    bool subsm(const double* xx, const double* gg, int nsub) {
        using namespace detail;
        const int n = n_, m = m_, col = col_, m2 = 2 * m_, col2 = 2 * col_;
        if (nsub <= 0) return true;
        double* d = r_.data();   // reduced gradient in, subspace step out
        double* x = z_.data();   // Cauchy point in, subspace minimiser out
        double* wv = v_.data();
        for (int i = 0; i < col; ++i) {
            double t1 = 0.0, t2 = 0.0;
            for (int j = 0; j < nsub; ++j) {
                const int k = index_[j];
                t1 += wy_[(size_t)k * m + i] * d[j];
                t2 += ws_[(size_t)k * m + i] * d[j];
            }
            wv[i] = t1;
            wv[col + i] = theta_ * t2;
        }
        if (!solve_upper_t(wn_.data(), m2, col2, wv)) return false;
        for (int i = 0; i < col; ++i) wv[i] = -wv[i];
        if (!solve_upper(wn_.data(), m2, col2, wv)) return false;
        for (int jy = 0; jy < col; ++jy) {
            const int js = col + jy;
            for (int i = 0; i < nsub; ++i) {
                const int k = index_[i];
                d[i] += wy_[(size_t)k * m + jy] * wv[jy] / theta_ + ws_[(size_t)k * m + jy] * wv[js];
            }
        }
        const double inv = 1.0 / theta_;
        for (int i = 0; i < nsub; ++i) d[i] *= inv;
        // projected Newton point
        int iword = 0;
        std::memcpy(xp_.data(), x, sizeof(double) * n);
        for (int i = 0; i < nsub; ++i) {
            const int k = index_[i];
            const double dk = d[i], xk = x[k];
            if (nbd_[k] != 0) {
                if (nbd_[k] == 1) {
                    x[k] = std::max(l_[k], xk + dk);
                    if (x[k] == l_[k]) iword = 1;
                } else if (nbd_[k] == 2) {
                    const double v = std::max(l_[k], xk + dk);
                    x[k] = std::min(u_[k], v);
                    if (x[k] == l_[k] || x[k] == u_[k]) iword = 1;
                } else {
                    x[k] = std::min(u_[k], xk + dk);
                    if (x[k] == u_[k]) iword = 1;
                }
            } else {
                x[k] = xk + dk;
            }
        }
        if (iword == 0) return true;
        double dd_p = 0.0;
        for (int i = 0; i < n; ++i) dd_p += (x[i] - xx[i]) * gg[i];
        if (dd_p > 0.0) {
            std::memcpy(x, xp_.data(), sizeof(double) * n);
            double alpha = 1.0, temp1 = alpha;
            int ibd = -1;
            for (int i = 0; i < nsub; ++i) {
                const int k = index_[i];
                const double dk = d[i];
                if (nbd_[k] != 0) {
                    if (dk < 0.0 && nbd_[k] <= 2) {
                        const double t2 = l_[k] - x[k];
                        if (t2 >= 0.0) temp1 = 0.0;
                        else if (dk * alpha < t2) temp1 = t2 / dk;
                    } else if (dk > 0.0 && nbd_[k] >= 2) {
                        const double t2 = u_[k] - x[k];
                        if (t2 <= 0.0) temp1 = 0.0;
                        else if (dk * alpha > t2) temp1 = t2 / dk;
                    }
                    if (temp1 < alpha) { alpha = temp1; ibd = i; }
                }
            }
            if (alpha < 1.0 && ibd >= 0) {
                const double dk = d[ibd];
                const int k = index_[ibd];
                if (dk > 0.0) { x[k] = u_[k]; d[ibd] = 0.0; }
                else if (dk < 0.0) { x[k] = l_[k]; d[ibd] = 0.0; }
            }
            for (int i = 0; i < nsub; ++i) x[index_[i]] += alpha * d[i];
        }
        return true;
    }

    // append the correction pair (s = d_, y = r_), oldest dropped when full
    void matupd(double rr, double dr, double stp, double dtd) {
        using namespace detail;
        const int n = n_, m = m_;
        if (col_ == m) {
            for (int i = 0; i < n; ++i) {
                double* a = &ws_[(size_t)i * m];
                double* b = &wy_[(size_t)i * m];
                for (int j = 0; j + 1 < m; ++j) { a[j] = a[j + 1]; b[j] = b[j + 1]; }
            }
            for (int j = 0; j + 1 < m; ++j)
                for (int i = 0; i + 1 < m; ++i) {
                    // upper triangle of SS and lower triangle of SY move up-left
                    if (i <= j) ss_[i * m + j] = ss_[(i + 1) * m + (j + 1)];
                    if (i >= j) sy_[i * m + j] = sy_[(i + 1) * m + (j + 1)];
                }
        } else {
            ++col_;
        }
        const int col = col_, last = col_ - 1;
        for (int i = 0; i < n; ++i) {
            ws_[(size_t)i * m + last] = d_[i];
            wy_[(size_t)i * m + last] = r_[i];
        }
        theta_ = rr / dr;
        for (int j = 0; j < col - 1; ++j) {
            double a = 0.0, b = 0.0;
            for (int i = 0; i < n; ++i) {
                a += d_[i] * wy_[(size_t)i * m + j];
                b += ws_[(size_t)i * m + j] * d_[i];
            }
            sy_[last * m + j] = a;
            ss_[j * m + last] = b;
        }
        ss_[last * m + last] = (stp == 1.0) ? dtd : stp * stp * dtd;
        sy_[last * m + last] = dr;
    }

    // T = theta SS + L D^-1 L', upper Cholesky factor into wt_
    bool formt() {
        using namespace detail;
        const int m = m_, col = col_;
        for (int j = 0; j < col; ++j) wt_[j] = theta_ * ss_[j];
        for (int i = 1; i < col; ++i)
            for (int j = i; j < col; ++j) {
                const int k1 = std::min(i, j);
                double dd = 0.0;
                for (int k = 0; k < k1; ++k) dd += sy_[i * m + k] * sy_[j * m + k] / sy_[k * m + k];
                wt_[i * m + j] = dd + theta_ * ss_[i * m + j];
            }
        return cholesky_upper(wt_.data(), m, col);
    }
};

}  // namespace lbfgsb
}  // namespace sfw3d
