"""Boosted / sliding Frank-Wolfe over x-slabs (BASELINE config 3
"full solve sharded as z-slabs with halo exchange at 1/2/4/8 GPUs").

The outer loop of solvers.py:286-405 runs in lockstep on every rank (one
process per GPU, or ranks as threads in the tests); each rank holds only its
own x-planes of every volume:

* y: the slab window (owned planes + the PSF's x half-extent), static;
* the blurred atoms phi_i: owned planes (rendered on the window from the
  atom pieces that meet it, convolved on the window: sfw3d_render_slab);
* the residual r = y - sum w_i phi_i: owned planes (K5);
* Gram rows <phi_i, phi_j>, b_i = <phi_i, y> and ||r||^2: per-rank partial
  dots, fp64 all-reduced (the weight step then runs identically everywhere);
* the certificate: distributed.SlabCertificate (halo exchange per x pass);
  its L-BFGS-B refine evaluates neg_eta from b = H^T r on a window whose
  halo planes come from the neighbours, the 6 per-atom sums all-reduced per
  callback (sfw3d_atom_sums_slab);
* the descents: distributed.SlabCostGrad, 6k + 1 partials all-reduced on the
  device per callback.

scipy's L-BFGS-B runs on every rank on all-reduced (hence identical) values,
so every rank follows the same trajectory; the result is the single-GPU
solve's up to the summation order of the partial sums.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np
from scipy.optimize import minimize

from . import _native as N
from .certificate import _position_window, build_template_table, make_parameter_grids
from .distributed import SlabCertificate, SlabCostGrad, slab_bounds
from .forward import GRADIENT_COLUMNS, as_psf, code_of, psf_apply_dev
from .optimize import minimize as native_minimize
from .measures import (AtomParams, WeightedMeasure, bounds_box, clamp_to_domain,
                       default_prune_tol, measure_rows, prune_zero_weights)
from .solvers import (BSFW, SFW, TERMINATED_CERTIFICATE, TERMINATED_ITERATION_CAP,
                      TERMINATED_STALLED, IterationRecord, SolveResult, SolveTrace, _is_duplicate,
                      _lasso_on, _rows_from_x, _unpack, residual_dev)


class _Slab:
    """One rank's x-slab of the solve: geometry, y window, collectives."""

    def __init__(self, y, psf, comm, code: int):
        import torch
        self.psf = psf
        self.dims = tuple(psf.dims)
        self.comm = comm.layout(self.dims[0])
        self.x0, self.x1 = slab_bounds(self.dims[0], comm.size, comm.rank)
        self.own = self.x1 - self.x0 + 1
        self.cg = SlabCostGrad(psf, self.dims, self.x0, self.x1)
        self.h = self.cg.halo
        self.code = code
        self.dev = torch.cuda.current_device()
        data = np.asarray(y.data if hasattr(y, "data") else y, dtype=np.float64)
        idx = np.arange(self.x0 - self.h, self.x1 + self.h + 1) % self.dims[0]
        self.y_win = torch.from_numpy(np.ascontiguousarray(data[idx])).to(
            f"cuda:{self.dev}", N.torch_dtype(code))
        self.y_own = self.y_win[self.h:self.h + self.own]

    # -- collectives on host values
    def sum(self, values) -> np.ndarray:
        return self.comm.allreduce(np.asarray(values, dtype=np.float64), "sum")

    # -- volumes on the slab
    def phi(self, theta: AtomParams):
        """Owned planes of H * G(theta) (solvers.py:260-261)."""
        import torch
        row = np.array([[1.0, *theta.m, theta.sigma, theta.d]])
        win = torch.empty(tuple(self.y_win.shape), dtype=self.y_win.dtype, device=self.y_win.device)
        ctx = N.context(self.dev)
        N.check(N.lib().sfw3d_render_slab(ctx.handle, self.code, N.dims_arg(self.dims),
                                          N.f64_ptr(row), 1, self.x0, self.x1, self.h, N.ptr(win)))
        out = psf_apply_dev(self.cg.psf, win, False)
        return out[self.h:self.h + self.own].contiguous()

    def back_window(self, r_own):
        """b = H^T r on a window of the owned planes: the residual's halo planes
        come from the neighbours (one exchange), then the window correlation."""
        import torch
        plane = self.dims[1] * self.dims[2]
        r_win = torch.zeros(tuple(self.y_win.shape), dtype=r_own.dtype, device=r_own.device)
        r_win[self.h:self.h + self.own] = r_own
        self.comm.halo(r_win.view(self.own + 2 * self.h, plane), self.own, self.h, self.h)
        return psf_apply_dev(self.cg.psf, r_win, True)

    def atom_sums(self, b_win, rows) -> np.ndarray:
        """All-reduced raw per-atom sums <P_c(atom), b> (the neg_eta reduction)."""
        rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 6)
        out = np.zeros((rows.shape[0], 6))
        ctx = N.context(self.dev)
        N.check(N.lib().sfw3d_atom_sums_slab(ctx.handle, code_of(b_win), N.dims_arg(self.dims),
                                             N.ptr(b_win), N.f64_ptr(rows), rows.shape[0],
                                             self.x0, self.x1, self.h, N.f64_ptr(out)))
        return self.sum(out.ravel()).reshape(-1, 6)


class _SlabGram:
    """Gram entries and b_i = <phi_i, y>, per pair once, partials all-reduced."""

    def __init__(self, slab: _Slab):
        from .solvers import dots_dev
        self.slab, self.dots = slab, dots_dev
        self.slot, self.keep = {}, []
        self.G, self.b = np.zeros((0, 0)), np.zeros(0)

    def system(self, phis):
        ids = [id(p) for p in phis]
        live = set(ids)
        if any(i not in live for i in self.slot):
            old = [(i, s) for i, s in self.slot.items() if i in live]
            idx = np.array([s for _, s in old], dtype=np.int64)
            self.G, self.b = self.G[np.ix_(idx, idx)], self.b[idx]
            self.keep = [self.keep[s] for s in idx]
            self.slot = {i: n for n, (i, _) in enumerate(old)}
        new = [p for p in phis if id(p) not in self.slot]
        if new:
            m, k0 = len(new), len(self.keep)
            G = np.zeros((k0 + m, k0 + m))
            G[:k0, :k0] = self.G
            b = np.concatenate([self.b, np.zeros(m)])
            for p in new:
                s = len(self.keep)
                self.slot[id(p)] = s
                self.keep.append(p)
                part = np.concatenate([self.dots(self.keep, p), self.dots([p], self.slab.y_own)])
                row = self.slab.sum(part)
                G[s, :s + 1] = row[:-1]
                G[:s + 1, s] = row[:-1]
                b[s] = row[-1]
            self.G, self.b = G, b
        idx = np.array([self.slot[i] for i in ids], dtype=np.int64)
        return self.G[np.ix_(idx, idx)], self.b[idx]


def _minimize(fun, x0, box, max_iter, gtol, ftol=2.220446049250313e-09):
    """The solver's optimiser (N.OPTIMIZER): the in-library L-BFGS-B through its
    callback form, or scipy's; every rank runs it on identical reduced values."""
    if N.OPTIMIZER == "scipy":
        return minimize(fun, x0, jac=True, method="L-BFGS-B", bounds=box,
                        options={"maxiter": max_iter, "gtol": gtol, "ftol": ftol})
    return native_minimize(fun, x0, box, maxiter=max_iter, gtol=gtol, ftol=ftol)


def _refine(slab: _Slab, r_own, lam, start: AtomParams, bounds, max_iter=200, gtol=1e-8):
    """refine_eta_max (certificate.py:187-224) on the slab: neg_eta from the
    all-reduced per-atom sums of the windowed b."""
    start = clamp_to_domain(start, bounds)
    b_win = slab.back_window(r_own)

    def neg_eta(vec):
        s = slab.atom_sums(b_win, np.array([[1.0, *np.asarray(vec, dtype=float)]]))[0]
        val, grad = float(s[0]) / lam, s[1:] / lam
        if not (np.isfinite(val) and np.isfinite(grad).all()):
            raise FloatingPointError(f"non-finite certificate value near {vec}")
        return -val, -grad

    start_val = -neg_eta(start.to_array())[0]
    res = _minimize(neg_eta, start.to_array(), bounds_box(bounds), max_iter, gtol)
    if not np.isfinite(res.fun):
        raise FloatingPointError("certificate ascent diverged to a non-finite value")
    if -res.fun < start_val:
        return start, start_val
    return clamp_to_domain(AtomParams.from_array(res.x), bounds), float(-res.fun)


def _descent(slab: _Slab, measure, lam, bounds, gtol, ftol, max_iter):
    """local_descent (solvers.py:197-240) with the slab-sharded criterion."""
    k = len(measure)
    if k == 0:
        return measure, slab.cg.cost_grad(slab.y_win, np.zeros((0, 6)), lam, slab.comm)[0], False
    start = WeightedMeasure(tuple((clamp_to_domain(th, bounds), w) for th, w in measure.atoms))

    def fun(x):
        value, grad = slab.cg.cost_grad(slab.y_win, _rows_from_x(x, k), lam, slab.comm)
        return value, grad.ravel()

    box = []
    for _ in range(k):
        box.append((0.0, None))
        box.extend(bounds_box(bounds))
    x0 = measure_rows(start).ravel()
    f0 = fun(x0)[0]
    res = _minimize(fun, x0, box, max_iter, gtol, ftol)
    warn = not res.success and "ABNORMAL" in str(res.message).upper()
    if not np.isfinite(res.fun) or res.fun > f0:
        return start, float(f0), warn
    out = WeightedMeasure(tuple((clamp_to_domain(th, bounds), w)
                                for th, w in _unpack(res.x, k).atoms))
    return out, float(res.fun), warn


def sharded_solve(y, psf, opts, bounds, algorithm: str, comm) -> SolveResult:
    """solvers.py:286-395 with every volume sharded as x-slabs over
    `comm.size` ranks (collective: every rank calls it with its comm)."""
    psf = as_psf(psf)
    if tuple(y.dims if hasattr(y, "dims") else np.shape(y)) != tuple(psf.dims):
        raise ValueError("dims mismatch: observation vs kernel")
    if algorithm not in (SFW, BSFW):
        raise ValueError(f"algorithm must be {SFW!r} or {BSFW!r}")
    t_start = time.perf_counter()
    code = N.dtype_code()
    sigma_grid, shape_grid = make_parameter_grids(bounds, opts.n_sigma, opts.n_shape)
    table = build_template_table(psf, sigma_grid, shape_grid, bounds=bounds)
    slab = _Slab(y, psf, comm, code)
    cert = SlabCertificate(table, slab.x0, slab.x1, comm)
    window = _position_window(bounds, slab.dims)
    trace = SolveTrace(algorithm=algorithm, t_table=time.perf_counter() - t_start)
    gram = _SlabGram(slab)
    lam = opts.lam

    def resid(thetas, weights, phis):
        r, ss = residual_dev(slab.y_own, weights, phis)
        return r, float(slab.sum([ss])[0])

    def certificate(thetas, weights, phis):
        r, _ = resid(thetas, weights, phis)
        _, c, pos, _ = cert.argmax(r, lam, window)
        i, j = divmod(c, len(table.shape_grid))
        seed = AtomParams(m=tuple(float(p) for p in pos), sigma=float(table.sigma_grid[i]),
                          d=float(table.shape_grid[j]))
        return _refine(slab, r, lam, seed, bounds)

    def prune(thetas, weights, phis, rel):
        tol = default_prune_tol(WeightedMeasure.from_pairs(thetas, weights), rel)
        keep = [i for i, w in enumerate(weights) if w > tol]
        return ([thetas[i] for i in keep], weights[keep] if len(weights) else weights,
                [phis[i] for i in keep])

    _, yy = resid([], np.zeros(0), [])
    thetas, weights, phis, crit = [], np.zeros(0), [], 0.5 * yy
    termination = TERMINATED_ITERATION_CAP
    stop_at = opts.eta_threshold + opts.eta_slack
    dup_streak = 0
    for k in range(1, opts.max_outer_iterations + 1):
        c_before = crit
        t0 = time.perf_counter()
        theta_star, eta_star = certificate(thetas, weights, phis)
        t_cert = time.perf_counter() - t0
        if eta_star <= stop_at:
            termination = TERMINATED_CERTIFICATE
            t_desc = 0.0
            if algorithm == BSFW and thetas:
                t0 = time.perf_counter()
                slid, c_desc, _ = _descent(slab, WeightedMeasure.from_pairs(thetas, weights), lam,
                                           bounds, opts.descent_gtol, opts.descent_ftol,
                                           opts.descent_max_iter)
                st, sw, sp = prune(list(slid.thetas), slid.weights,
                                   [slab.phi(th) for th in slid.thetas], opts.prune_rel_tol)
                _, eta_slid = certificate(st, sw, sp)
                if c_desc <= crit and eta_slid <= stop_at:
                    thetas, weights, phis, crit = st, sw, sp, c_desc
                t_desc = time.perf_counter() - t0
            trace.records.append(IterationRecord(
                index=k, eta_max=eta_star, criterion_before=c_before, criterion_after_lasso=None,
                criterion_after_descent=crit if algorithm == BSFW else None,
                atom_count=len(thetas), t_certificate=t_cert, t_lasso=0.0, t_descent=t_desc))
            break
        duplicate = _is_duplicate(theta_star, thetas, opts.duplicate_tol)
        t0 = time.perf_counter()
        thetas.append(theta_star)
        phis.append(slab.phi(theta_star))
        w_init = np.append(weights, 0.0)
        g, b = gram.system(phis)
        weights = _lasso_on(g, b, lam, w_init, opts.lasso_tol, opts.lasso_max_iter, slab.dev)
        _, rr = resid(thetas, weights, phis)
        crit = 0.5 * rr + lam * float(weights.sum())
        c_lasso = crit
        t_lasso = time.perf_counter() - t0
        c_desc, t_desc = None, 0.0
        if algorithm == SFW:
            t0 = time.perf_counter()
            meas, c_desc, _ = _descent(slab, WeightedMeasure.from_pairs(thetas, weights), lam,
                                       bounds, opts.descent_gtol, opts.descent_ftol,
                                       opts.descent_max_iter)
            thetas, weights = list(meas.thetas), meas.weights
            phis = [slab.phi(th) for th in thetas]
            crit = c_desc
            t_desc = time.perf_counter() - t0
        thetas, weights, phis = prune(thetas, weights, phis, opts.prune_rel_tol)
        trace.records.append(IterationRecord(
            index=k, eta_max=eta_star, criterion_before=c_before, criterion_after_lasso=c_lasso,
            criterion_after_descent=c_desc, atom_count=len(thetas), t_certificate=t_cert,
            t_lasso=t_lasso, t_descent=t_desc))
        if duplicate and crit >= c_before * (1.0 - 1e-12):
            dup_streak += 1
            if dup_streak >= 2:
                termination = TERMINATED_STALLED
                break
        else:
            dup_streak = 0
    trace.t_total = time.perf_counter() - t_start
    measure = WeightedMeasure.from_pairs(thetas, weights)
    measure = prune_zero_weights(measure, default_prune_tol(measure, opts.prune_rel_tol))
    return SolveResult(measure=measure, criterion=crit, termination=termination, trace=trace)


__all__ = ["sharded_solve", "GRADIENT_COLUMNS"]
