"""CPU oracle for the boosted-SFW hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the arithmetic of the reference
package ``sfw3d`` 0.1.0 for the data-parallel path the B200 build replaces.
It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package (``paper_2009_05473_b200``) never imports it and has no
CPU fallback.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference (from
``/root/reference/pkg/src``, in the build container only) and stores
input/output vectors under ``tests/golden/*.npz``; ``tests/test_oracle.py``
checks this module against them.

Conventions (shared with the CUDA kernels):
  * volumes are float64 (nx, ny, nz) C-order, axis 2 contiguous
    (reference ``volumes.py:7-16``);
  * an atom row is ``(w, m_x, m_y, m_z, sigma, d)`` — the reference's
    gradient-column / ``_pack`` order (``forward.py:37``, ``solvers.py:183-186``);
  * the PSF is a centred kernel volume whose origin is voxel ``n//2`` per axis
    (``forward.py:40-58``).

Every function cites the reference lines whose arithmetic it restates.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.fft as sfft

# forward.py:31-34 — unit profile below 1e-12 is treated as exactly zero
TAIL_CUTOFF = 1e-12
TAIL_EXPONENT = 2.0 * np.log(1.0 / TAIL_CUTOFF)


# --------------------------------------------------------------------------
# atom geometry and profile                      (forward.py:97-152)
# --------------------------------------------------------------------------

def support_radius(sigma: float, d: float) -> int:
    """forward.py:97-99: ceil(sigma * (2 ln 1e12)^(1/d)) in float64."""
    return int(np.ceil(sigma * TAIL_EXPONENT ** (1.0 / d)))


def axis_box(n: int, centre: float, radius: int):
    """Wrapped voxel indices and signed offsets along one axis.

    forward.py:102-116: a full axis with minimum-image offsets when the box
    would cover the axis (2R+1 >= n), otherwise the span
    round_half_even(m) +- R wrapped modulo n, offsets taken *before* wrapping.
    """
    if 2 * radius + 1 >= n:
        idx = np.arange(n)
        off = np.remainder(idx - centre + n / 2.0, n) - n / 2.0
        return idx, off
    c = int(np.round(centre))
    span = np.arange(c - radius, c + radius + 1)
    return np.remainder(span, n), span - centre


def atom_profile(theta, dims, with_grads: bool):
    """Unit atom on its support box; theta = (m_x, m_y, m_z, sigma, d).

    forward.py:119-152. Returns (index triple, values, grads) where grads is
    (g_mx, g_my, g_mz, g_sigma, g_d) or None.
    """
    mx, my, mz, sigma, d = (float(v) for v in theta)
    if not (sigma > 0.0 and d > 0.0):
        raise ValueError("sigma and d must be positive")
    r = support_radius(sigma, d)
    boxes = [axis_box(n, c, r) for n, c in zip(dims, (mx, my, mz))]
    (ix, ox), (iy, oy), (iz, oz) = boxes
    u2 = ox[:, None, None] ** 2 + oy[None, :, None] ** 2 + oz[None, None, :] ** 2
    scale = 0.5 / sigma ** d
    t = scale * (u2 if d == 2.0 else u2 ** (0.5 * d))
    val = np.exp(-t)
    if not with_grads:
        return (ix, iy, iz), val, None
    inside = u2 > 0.0
    amp = np.zeros_like(u2)
    amp[inside] = d * val[inside] * t[inside] / u2[inside]
    g_sigma = val * t * (d / sigma)
    lr = np.zeros_like(u2)
    lr[inside] = 0.5 * np.log(u2[inside]) - np.log(sigma)
    g_d = -val * t * lr
    grads = (amp * ox[:, None, None], amp * oy[None, :, None], amp * oz[None, None, :],
             g_sigma, g_d)
    return (ix, iy, iz), val, grads


def render(params, dims) -> np.ndarray:
    """Sum of weighted atoms, summed in row order (forward.py:165-174)."""
    out = np.zeros(tuple(dims))
    for row in np.asarray(params, dtype=float).reshape(-1, 6):
        idx, val, _ = atom_profile(row[1:], dims, False)
        out[np.ix_(*idx)] += row[0] * val
    return out


# --------------------------------------------------------------------------
# PSF and circular convolution                    (forward.py:40-94)
# --------------------------------------------------------------------------

def psf_normalise(kernel: np.ndarray) -> np.ndarray:
    """forward.py:49-57: unit-sum normalisation with the ~0-sum guard."""
    k = np.asarray(kernel, dtype=float)
    s = float(k.sum())
    peak = float(np.abs(k).max()) if k.size else 0.0
    if abs(s) < 1e-12 * max(peak, 1.0):
        raise ValueError("kernel sum is ~0, cannot normalize to unit sum")
    return k / s


def psf_hat(kernel: np.ndarray) -> np.ndarray:
    """forward.py:58: transform of the kernel with its centre moved to 0."""
    return sfft.rfftn(sfft.ifftshift(kernel))


def conv(v: np.ndarray, khat: np.ndarray) -> np.ndarray:
    """forward.py:79-87: circular H * v."""
    return sfft.irfftn(sfft.rfftn(v) * khat, s=v.shape)


def corr(v: np.ndarray, khat: np.ndarray) -> np.ndarray:
    """forward.py:90-94: circular H^T * v (adjoint)."""
    return sfft.irfftn(sfft.rfftn(v) * np.conj(khat), s=v.shape)


def is_centrosymmetric(kernel: np.ndarray, tol: float = 1e-10) -> bool:
    """forward.py:71-76."""
    sh = sfft.ifftshift(kernel)
    mir = np.roll(sh[::-1, ::-1, ::-1], 1, axis=(0, 1, 2))
    scale = float(np.abs(sh).max()) or 1.0
    return bool(np.max(np.abs(sh - mir)) <= tol * scale)


# --------------------------------------------------------------------------
# criterion and gradient                          (forward.py:182-257)
# --------------------------------------------------------------------------

def criterion(y, params, khat, lam) -> float:
    """forward.py:182-190."""
    resid = conv(render(params, y.shape), khat) - y
    mass = float(np.sum(np.asarray(params, dtype=float).reshape(-1, 6)[:, 0]))
    return 0.5 * float(np.vdot(resid, resid).real) + lam * mass


def atom_rows(back: np.ndarray, params, lam: float) -> np.ndarray:
    """forward.py:209-229: per atom [<G,b>+lam, w<dG/dm_xyz,b>, w<dG/ds,b>, w<dG/dd,b>]."""
    p = np.asarray(params, dtype=float).reshape(-1, 6)
    rows = np.empty((p.shape[0], 6))
    for a, row in enumerate(p):
        idx, val, grads = atom_profile(row[1:], back.shape, True)
        sub = back[np.ix_(*idx)]
        rows[a, 0] = float(np.vdot(val, sub).real) + lam
        for c, g in enumerate(grads, start=1):
            rows[a, c] = row[0] * float(np.vdot(g, sub).real)
    if not np.isfinite(rows).all():
        raise FloatingPointError("non-finite criterion gradient")
    return rows


def criterion_and_gradient(y, params, khat, lam):
    """forward.py:232-257: (C, rows (k,6), back = H^T*(model - y))."""
    dims = y.shape
    acc_hat = sfft.rfftn(render(params, dims))
    model_hat = acc_hat * khat
    resid = sfft.irfftn(model_hat, s=dims) - y
    mass = float(np.sum(np.asarray(params, dtype=float).reshape(-1, 6)[:, 0]))
    value = 0.5 * float(np.vdot(resid, resid).real) + lam * mass
    back = sfft.irfftn(np.conj(khat) * (model_hat - sfft.rfftn(y)), s=dims)
    return value, atom_rows(back, params, lam), back


# --------------------------------------------------------------------------
# certificate                                     (certificate.py:37-236)
# --------------------------------------------------------------------------

def parameter_grids(sigma_min, sigma_max, shape_min, shape_max, n_sigma=8, n_shape=6):
    """certificate.py:37-49: geometric sigma samples, linear shape samples."""
    return (np.geomspace(sigma_min, sigma_max, n_sigma),
            np.linspace(shape_min, shape_max, n_shape))


def template_hats(kernel_hat, dims, sigma_grid, shape_grid) -> np.ndarray:
    """certificate.py:65-97: transform of H * G_unit(m=0; s_i, d_j), sigma-major."""
    out = []
    for s in np.sort(np.asarray(sigma_grid, dtype=float)):
        for d in np.sort(np.asarray(shape_grid, dtype=float)):
            idx, val, _ = atom_profile((0.0, 0.0, 0.0, s, d), dims, False)
            atom = np.zeros(dims)
            atom[np.ix_(*idx)] = val
            out.append(sfft.rfftn(atom) * kernel_hat)
    return np.stack(out)


def position_window(dims, pos_lower=None, pos_upper=None):
    """certificate.py:100-111: integer box [ceil(lo), floor(hi)] clipped to the grid."""
    if pos_lower is None:
        return tuple((0, n - 1) for n in dims)
    win = []
    for lo, hi, n in zip(pos_lower, pos_upper, dims):
        a, b = max(0, int(np.ceil(lo))), min(n - 1, int(np.floor(hi)))
        if a > b:
            raise ValueError("domain position bounds contain no integer grid point")
        win.append((a, b))
    return tuple(win)


def eta_field(residual, lam, hats, n_shape, window=None, keep_fields=False):
    """certificate.py:140-184.

    Returns (position, flat candidate index, eta_max, per-candidate list of
    (position, value), fields or None). Candidates are sigma-major; the global
    winner is the first candidate reaching the maximum (strict '>' scan) and
    within a candidate the first C-order maximum inside the window.
    """
    if lam <= 0.0:
        raise ValueError("lam must be > 0")
    dims = residual.shape
    if window is None:
        window = position_window(dims)
    reg = tuple(slice(a, b + 1) for a, b in window)
    rhat = sfft.rfftn(residual)
    best = (None, 0, -np.inf)
    per = []
    fields = [] if keep_fields else None
    for c in range(hats.shape[0]):
        vals = sfft.irfftn(rhat * np.conj(hats[c]), s=dims) / lam
        loc = vals[reg]
        p = np.unravel_index(int(np.argmax(loc)), loc.shape)
        p = tuple(int(q + a) for q, (a, _) in zip(p, window))
        v = float(vals[p])
        per.append((p, v))
        if v > best[2]:
            best = (p, c, v)
        if keep_fields:
            fields.append(vals)
    return best[0], best[1], best[2], per, fields


def eta_maxima(residual, lam, kernel_hat, sigma_grid, shape_grid, window=None, threads=1):
    """certificate.py:140-172 per candidate, memory-bounded for large grids:
    each worker builds one template spectrum (certificate.py:86-92), takes
    irfftn(r_hat conj(T_hat)) / lam and its first C-order maximum in the
    window. Returns [(position, eta)] in sigma-major order."""
    from concurrent.futures import ThreadPoolExecutor
    dims = residual.shape
    if window is None:
        window = position_window(dims)
    reg = tuple(slice(a, b + 1) for a, b in window)
    rhat = sfft.rfftn(np.asarray(residual, dtype=float))
    cands = [(s, d) for s in np.sort(np.asarray(sigma_grid, dtype=float))
             for d in np.sort(np.asarray(shape_grid, dtype=float))]

    def one(c):
        h = template_hats(kernel_hat, dims, [c[0]], [c[1]])[0]
        vals = sfft.irfftn(rhat * np.conj(h), s=dims) / lam
        loc = vals[reg]
        p = np.unravel_index(int(np.argmax(loc)), loc.shape)
        p = tuple(int(q + a) for q, (a, _) in zip(p, window))
        return p, float(vals[p])

    with ThreadPoolExecutor(max_workers=max(1, int(threads))) as pool:
        return list(pool.map(one, cands))


def eta_value_grad(back: np.ndarray, theta, lam: float):
    """certificate.py:201-209 (neg_eta, sign flipped): eta(theta) and its 5-gradient."""
    idx, val, grads = atom_profile(theta, back.shape, True)
    sub = back[np.ix_(*idx)]
    v = float(np.vdot(val, sub).real) / lam
    g = np.array([float(np.vdot(q, sub).real) for q in grads]) / lam
    return v, g


def clamp_theta(theta, box5):
    """measures.py:160-168: project (m_x, m_y, m_z, sigma, d) onto the box."""
    return np.array([min(max(float(x), lo), hi) for x, (lo, hi) in zip(theta, box5)])


def refine_eta_max(back, lam, start, box5, max_iter=200, gtol=1e-8):
    """certificate.py:187-224: L-BFGS-B ascent of eta from the grid seed with
    the analytic 5-gradient; keeps the start if not improved. `back` =
    H^T r; box5 = [(lo, hi)] for (m_x, m_y, m_z, sigma, d). Returns (theta, eta)."""
    from scipy.optimize import minimize
    start = clamp_theta(start, box5)

    def neg_eta(vec):
        v, g = eta_value_grad(back, vec, lam)
        if not (np.isfinite(v) and np.isfinite(g).all()):
            raise FloatingPointError("non-finite certificate value")
        return -v, -g

    start_val = -neg_eta(start)[0]
    res = minimize(neg_eta, start, jac=True, method="L-BFGS-B", bounds=list(box5),
                   options={"maxiter": max_iter, "gtol": gtol})
    if not np.isfinite(res.fun):
        raise FloatingPointError("certificate ascent diverged to a non-finite value")
    if -res.fun < start_val:
        return start, start_val
    return clamp_theta(res.x, box5), float(-res.fun)


def local_descent(y, rows, khat, lam, box5, gtol=1e-6, ftol=1e-10, max_iter=400):
    """solvers.py:197-240: joint L-BFGS-B slide of all (w, m, sigma, d) rows
    with w >= 0 (_unpack takes max(0, w)); keeps the start if not improved.
    Returns ((k, 6) rows, criterion)."""
    from scipy.optimize import minimize
    p = np.asarray(rows, dtype=float).reshape(-1, 6).copy()
    k = p.shape[0]
    for i in range(k):
        p[i, 1:] = clamp_theta(p[i, 1:], box5)

    def unpack(x):
        r = np.array(x, dtype=float).reshape(k, 6)
        r[:, 0] = np.maximum(r[:, 0], 0.0)
        return r

    def fun(x):
        value, g, _ = criterion_and_gradient(y, unpack(x), khat, lam)
        return value, g.ravel()

    box = []
    for _ in range(k):
        box.append((0.0, None))
        box.extend(box5)
    x0 = p.ravel()
    f0 = fun(x0)[0]
    res = minimize(fun, x0, jac=True, method="L-BFGS-B", bounds=box,
                   options={"maxiter": max_iter, "gtol": gtol, "ftol": ftol})
    if not np.isfinite(res.fun) or res.fun > f0:
        return p, float(f0)
    out = unpack(res.x)
    for i in range(k):
        out[i, 1:] = clamp_theta(out[i, 1:], box5)
    return out, float(res.fun)


# --------------------------------------------------------------------------
# non-negative LASSO weight step                  (solvers.py:111-180)
# --------------------------------------------------------------------------

def gram_system(phis: np.ndarray, y: np.ndarray):
    """solvers.py:141-143: Gram = Phi Phi^T, b = Phi y over flattened phis."""
    flat = np.asarray(phis, dtype=float).reshape(len(phis), -1)
    return flat @ flat.T, flat @ y.ravel()


def cd_solve(gram, b, lam, w_init=None, tol=1e-8, max_iter=5000):
    """solvers.py:145-180: cyclic coordinate descent, KKT / stall / cap stops.

    Returns (w, sweeps, reason) with reason in {"kkt", "stall", "cap"}.
    """
    k = len(b)
    w = np.zeros(k) if w_init is None else np.asarray(w_init, dtype=float).copy()
    if k == 0:
        return w, 0, "kkt"
    gw = gram @ w
    w_scale = max(1.0, float(np.max(w)))
    for sweep in range(1, max_iter + 1):
        step = 0.0
        for i in range(k):
            old = w[i]
            new = max(0.0, old + (b[i] - lam - gw[i]) / gram[i, i])
            if new != old:
                gw += (new - old) * gram[:, i]
                w[i] = new
                step = max(step, abs(new - old))
        slope = gw - b + lam
        act = w > 0.0
        kkt = 0.0
        if act.any():
            kkt = float(np.max(np.abs(slope[act])))
        if (~act).any():
            kkt = max(kkt, float(np.max(np.maximum(0.0, -slope[~act]))))
        if kkt <= tol:
            return w, sweep, "kkt"
        w_scale = max(w_scale, float(np.max(w)))
        if step <= 1e-14 * w_scale:
            return w, sweep, "stall"
    return w, max_iter, "cap"


def phi(theta, khat, dims) -> np.ndarray:
    """solvers.py:260-261: blurred unit atom."""
    return conv(render([[1.0, *theta]], dims), khat)


def residual(y, weights, phis) -> np.ndarray:
    """solvers.py:253-257: y - sum_i w_i phi_i in list order."""
    out = np.array(y, dtype=float, copy=True)
    for w, p in zip(weights, phis):
        out -= w * p
    return out


# --------------------------------------------------------------------------
# outer loop: SFW / boosted SFW                     (solvers.py:286-405)
# --------------------------------------------------------------------------

def solve(y, kernel_hat, lam, sigma_grid, shape_grid, box5, algorithm="bsfw",
          max_outer_iterations=50, eta_threshold=1.0, eta_slack=5e-3, lasso_tol=1e-6,
          lasso_max_iter=2000, descent_gtol=1e-6, descent_ftol=1e-10, descent_max_iter=400,
          prune_rel_tol=1e-10, duplicate_tol=1e-6):
    """solvers.py:286-395 restated on the oracle's numpy kernels: per outer
    iteration the certificate (FFT eta over the template spectra in the
    position window + L-BFGS-B refine), the duplicate guard, the weight step
    (Gram + cyclic CD with the warm start), the SFW descent after every atom
    or the BSFW final slide with its re-check, the relative prune and the
    stall rule. box5 = [(lo, hi)] for (m_x, m_y, m_z, sigma, d). Returns
    dict(rows (k, 6), criterion, termination, eta (per iteration), atoms
    (per iteration))."""
    dims = y.shape
    hats = template_hats(kernel_hat, dims, sigma_grid, shape_grid)
    sg, dg = np.sort(np.asarray(sigma_grid, float)), np.sort(np.asarray(shape_grid, float))
    window = position_window(dims, [b[0] for b in box5[:3]], [b[1] for b in box5[:3]])
    stop_at = eta_threshold + eta_slack
    thetas, weights, phis = [], np.zeros(0), []
    crit = 0.5 * float(np.vdot(y, y).real)
    term, dup_streak = "iteration_cap", 0
    etas, counts = [], []

    def cert(thetas_, weights_, phis_):
        r = residual(y, weights_, phis_)
        pos, flat, _, _, _ = eta_field(r, lam, hats, len(dg), window)
        i, j = divmod(flat, len(dg))
        return refine_eta_max(corr(r, kernel_hat), lam, np.array([*pos, sg[i], dg[j]], float), box5)

    def lasso_crit(weights_, phis_):
        r = residual(y, weights_, phis_)
        return 0.5 * float(np.vdot(r, r).real) + lam * float(np.sum(weights_))

    def prune(thetas_, weights_, phis_):
        tol = prune_rel_tol * float(np.max(weights_)) if len(weights_) else 0.0
        keep = [i for i, w in enumerate(weights_) if w > tol]
        return [thetas_[i] for i in keep], weights_[keep], [phis_[i] for i in keep]

    for k in range(1, max_outer_iterations + 1):
        c_before = crit
        theta, eta = cert(thetas, weights, phis)
        etas.append(eta)
        if eta <= stop_at:
            term = "certificate"
            if algorithm == "bsfw" and thetas:
                rows0 = np.column_stack([weights, np.array(thetas)])
                slid, c_desc = local_descent(y, rows0, kernel_hat, lam, box5, descent_gtol,
                                             descent_ftol, descent_max_iter)
                st = [list(r[1:]) for r in slid]
                sp = [phi(t, kernel_hat, dims) for t in st]
                st, sw, sp = prune(st, slid[:, 0].copy(), sp)
                _, eta_slid = cert(st, sw, sp)
                if c_desc <= crit and eta_slid <= stop_at:
                    thetas, weights, phis, crit = st, sw, sp, c_desc
            counts.append(len(thetas))
            break
        duplicate = any(np.max(np.abs(np.asarray(theta) - np.asarray(t))) <= duplicate_tol
                        for t in thetas)
        thetas.append(list(theta))
        phis.append(phi(theta, kernel_hat, dims))
        w_init = np.append(weights, 0.0)
        gram, b = gram_system(np.stack(phis), y)
        weights, _, _ = cd_solve(gram, b, lam, w_init, lasso_tol, lasso_max_iter)
        crit = lasso_crit(weights, phis)
        if algorithm == "sfw":
            rows0 = np.column_stack([weights, np.array(thetas)])
            slid, crit = local_descent(y, rows0, kernel_hat, lam, box5, descent_gtol,
                                       descent_ftol, descent_max_iter)
            thetas = [list(r[1:]) for r in slid]
            weights = slid[:, 0].copy()
            phis = [phi(t, kernel_hat, dims) for t in thetas]
        thetas, weights, phis = prune(thetas, weights, phis)
        counts.append(len(thetas))
        if duplicate and crit >= c_before * (1.0 - 1e-12):
            dup_streak += 1
            if dup_streak >= 2:
                term = "stalled_duplicate_atom"
                break
        else:
            dup_streak = 0
    rows = np.column_stack([weights, np.array(thetas).reshape(-1, 5)]) if thetas else np.zeros((0, 6))
    tol = prune_rel_tol * float(np.max(weights)) if len(weights) else 0.0
    rows = rows[rows[:, 0] > tol]
    return {"rows": rows, "criterion": crit, "termination": term, "eta": etas, "atoms": counts}


# --------------------------------------------------------------------------
# synthetic configs (BASELINE.json configs)
# --------------------------------------------------------------------------

def box_gaussian_psf(dims, sigmas, half):
    """Box-truncated sampled Gaussian exp(-1/2 sum (x_a/s_a)^2) over -h..h per
    axis, embedded centred at n//2 and normalised to unit sum."""
    k = np.zeros(tuple(dims))
    axes = []
    for n, s, h in zip(dims, sigmas, half):
        o = np.arange(-h, h + 1)
        axes.append(np.exp(-0.5 * (o / s) ** 2))
    box = axes[0][:, None, None] * axes[1][None, :, None] * axes[2][None, None, :]
    sl = tuple(slice(n // 2 - h, n // 2 + h + 1) for n, h in zip(dims, half))
    k[sl] = box
    return psf_normalise(k)


def power_snr_sigma(clean: np.ndarray, snr_db: float) -> float:
    return math.sqrt(float(np.mean(clean ** 2)) / 10.0 ** (snr_db / 10.0))
