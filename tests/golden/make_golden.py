"""Generate golden vectors by running the REAL reference (sfw3d 0.1.0).

Run in the build container only (the reference tree is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` fixtures next to this script. The fixtures pin both the
CPU oracle (``oracle/sfw3d_oracle.py``) and, in the GPU tests, the CUDA path.
Every case is seeded; the reference functions called are named per case.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("SFW3D_REFERENCE", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

import sfw3d  # noqa: E402  (the reference)
from sfw3d import (AtomParams, DomainBounds, Psf, SolverOptions, Volume,  # noqa: E402
                   WeightedMeasure)
from sfw3d import certificate as rcert  # noqa: E402
from sfw3d import solvers as rsolv  # noqa: E402

fwd = sys.modules["sfw3d.forward"]  # sfw3d.forward is shadowed by the function

OUT = Path(__file__).resolve().parent


def box_psf(dims, sigmas, half):
    k = np.zeros(dims)
    axes = [np.exp(-0.5 * (np.arange(-h, h + 1) / s) ** 2) for s, h in zip(sigmas, half)]
    box = axes[0][:, None, None] * axes[1][None, :, None] * axes[2][None, None, :]
    k[tuple(slice(n // 2 - h, n // 2 + h + 1) for n, h in zip(dims, half))] = box
    return k


def measure_from_rows(rows):
    return WeightedMeasure(tuple(
        (AtomParams(m=tuple(r[1:4]), sigma=r[4], d=r[5]), float(r[0])) for r in rows))


def rows_from_measure(m):
    return np.array([[w, *t.m, t.sigma, t.d] for t, w in m.atoms]).reshape(-1, 6)


def random_rows(rng, k, dims, sig=(1.0, 3.0), shp=(1.5, 2.5), w=(0.5, 2.0), edge=False):
    rows = []
    for _ in range(k):
        if edge:
            m = rng.uniform(-0.49, 1.0, size=3) * np.array(dims)  # some near / past faces
            m = np.mod(m, np.array(dims) - 1e-9)
        else:
            m = rng.uniform(2, np.array(dims) - 3)
        rows.append([rng.uniform(*w), *m, rng.uniform(*sig), rng.uniform(*shp)])
    return np.array(rows)


def case_kats():
    """SPEC.md:186-187 render KATs through the reference render_atom."""
    geom = sfw3d.GridGeometry((9, 9, 9))
    v1 = sfw3d.render_atom(AtomParams(m=(4.0, 4.0, 4.0), sigma=1.0, d=2.0), 1.0, geom).data
    v2 = sfw3d.render_atom(AtomParams(m=(4.0, 4.0, 3.0), sigma=1.7, d=1.6), 2.0, geom).data
    np.savez(OUT / "kat_render.npz", unit_d2=v1, w2=v2)


def case_convolution(rng):
    """forward.convolve / correlate_adjoint on a random and a box-Gaussian kernel."""
    out = {}
    for name, dims in (("cube", (12, 12, 12)), ("odd", (11, 14, 9))):
        v = rng.standard_normal(dims)
        k = box_psf(dims, (1.3, 1.1, 2.0), (2, 3, 3))
        psf = Psf(Volume(k))
        out[f"{name}_v"] = v
        out[f"{name}_kernel"] = psf.kernel.data
        out[f"{name}_conv"] = sfw3d.convolve(Volume(v), psf).data
        out[f"{name}_corr"] = sfw3d.correlate_adjoint(Volume(v), psf).data
        # general (non-separable, non-centrosymmetric) kernel
        kr = np.zeros(dims)
        kr[tuple(slice(n // 2 - 2, n // 2 + 3) for n in dims)] = rng.uniform(0.1, 1.0, (5, 5, 5))
        psfr = Psf(Volume(kr))
        out[f"{name}_rkernel"] = psfr.kernel.data
        out[f"{name}_rconv"] = sfw3d.convolve(Volume(v), psfr).data
        out[f"{name}_rcorr"] = sfw3d.correlate_adjoint(Volume(v), psfr).data
    np.savez(OUT / "convolution.npz", **out)


def case_forward(rng):
    """forward.forward / _accumulate_atoms incl. wrapped and full-axis boxes."""
    out = {}
    specs = (("interior", (16, 16, 16), False, (1.0, 2.0), (1.5, 2.5)),
             ("edge", (16, 16, 16), True, (1.0, 2.5), (1.5, 2.5)),
             ("fullaxis", (10, 12, 14), True, (2.0, 3.0), (1.2, 1.6)),
             ("odd", (13, 16, 11), True, (0.8, 1.5), (1.8, 2.8)))
    for name, dims, edge, sig, shp in specs:
        rows = random_rows(rng, 5, dims, sig=sig, shp=shp, edge=edge)
        rows[0, 5] = 2.0  # exercise the exact d == 2 branch
        rows[1, 1:4] = np.round(rows[1, 1:4]) + 0.5  # round-half-even ties
        k = box_psf(dims, (1.5, 1.5, 2.0), (2, 2, 3))
        psf = Psf(Volume(k))
        meas = measure_from_rows(rows)
        out[f"{name}_rows"] = rows
        out[f"{name}_kernel"] = psf.kernel.data
        out[f"{name}_acc"] = fwd._accumulate_atoms(meas, dims, None)
        out[f"{name}_forward"] = sfw3d.forward(meas, psf).data
    np.savez(OUT / "forward.npz", **out)


def case_cost_grad(rng):
    """forward.criterion_and_gradient on several instances."""
    out = {}
    specs = (("small", (16, 16, 16), 3, False), ("edge", (16, 18, 14), 4, True),
             ("fullaxis", (10, 12, 14), 3, True))
    for name, dims, k_atoms, edge in specs:
        truth = random_rows(rng, k_atoms, dims, edge=edge)
        k = box_psf(dims, (1.5, 1.5, 2.5), (2, 2, 3))
        psf = Psf(Volume(k))
        y = sfw3d.forward(measure_from_rows(truth), psf).data + 0.01 * rng.standard_normal(dims)
        est = truth.copy()
        est[:, 1:4] += 0.3 * rng.standard_normal((k_atoms, 3))
        est[:, 1:4] = np.mod(est[:, 1:4], np.array(dims) - 1e-9)
        est[:, 0] *= rng.uniform(0.7, 1.3, k_atoms)
        est[:, 4] = np.clip(est[:, 4] * rng.uniform(0.8, 1.2, k_atoms), 0.8, 3.2)
        est[:, 5] = np.clip(est[:, 5] + 0.1 * rng.standard_normal(k_atoms), 1.2, 2.8)
        est[0, 5] = 2.0
        lam = 0.1
        c, g = sfw3d.criterion_and_gradient(Volume(y), measure_from_rows(est), psf, lam)
        out[f"{name}_y"] = y
        out[f"{name}_kernel"] = psf.kernel.data
        out[f"{name}_rows"] = est
        out[f"{name}_lam"] = np.array(lam)
        out[f"{name}_C"] = np.array(c)
        out[f"{name}_grad"] = g.per_atom
        out[f"{name}_Conly"] = np.array(sfw3d.criterion(Volume(y), measure_from_rows(est), psf, lam))
    np.savez(OUT / "cost_grad.npz", **out)


def case_certificate(rng):
    """build_template_table + eta_field + refine_eta_max + neg_eta values."""
    out = {}
    dims = (16, 16, 16)
    k = box_psf(dims, (1.2, 1.2, 1.8), (2, 2, 3))
    psf = Psf(Volume(k))
    truth = np.array([[1.5, 5.2, 8.7, 9.1, 1.6, 1.9], [1.0, 11.0, 4.4, 6.0, 2.2, 1.6]])
    y = sfw3d.forward(measure_from_rows(truth), psf).data + 0.02 * rng.standard_normal(dims)
    bounds = DomainBounds(pos_lower=(2.5, 2.0, 2.0), pos_upper=(13.0, 13.5, 12.2),
                          sigma_min=1.0, sigma_max=2.5, shape_min=1.5, shape_max=2.5)
    sg, dg = rcert.make_parameter_grids(bounds, 3, 3)
    table = rcert.build_template_table(psf, sg, dg, bounds=bounds)
    lam = 0.3
    f = rcert.eta_field(Volume(y), lam, table, bounds=bounds, keep_fields=True)
    out.update(y=y, kernel=psf.kernel.data, lam=np.array(lam), sigma_grid=sg, shape_grid=dg,
               bounds=np.array([*bounds.pos_lower, *bounds.pos_upper, bounds.sigma_min,
                                bounds.sigma_max, bounds.shape_min, bounds.shape_max]),
               argmax_position=np.array(f.argmax_position),
               argmax_sigma_index=np.array(f.argmax_sigma_index),
               argmax_shape_index=np.array(f.argmax_shape_index),
               eta_max=np.array(f.eta_max),
               fields=np.stack([v.data for v in f.fields]))
    # no bounds: whole-grid window
    f2 = rcert.eta_field(Volume(y), 1.0, table, bounds=None, keep_fields=False)
    out.update(nb_argmax_position=np.array(f2.argmax_position),
               nb_argmax_flat=np.array(f2.argmax_sigma_index * dg.size + f2.argmax_shape_index),
               nb_eta_max=np.array(f2.eta_max))
    # neg_eta arithmetic at a few thetas (certificate.py:198-209)
    back = fwd.correlate_adjoint(Volume(y), psf).data
    thetas = np.array([[5.0, 9.0, 9.0, 1.6, 1.9], [10.7, 4.2, 6.3, 2.1, 1.55],
                       [8.0, 8.0, 8.0, 2.0, 2.0], [0.4, 15.6, 3.0, 1.3, 2.3]])
    vals, grads = [], []
    for th in thetas:
        idx, values, gr = fwd._unit_atom(AtomParams.from_array(th), dims, True)
        sub = back[np.ix_(*idx)]
        vals.append(float(np.vdot(values, sub).real) / lam)
        grads.append([float(np.vdot(g, sub).real) / lam for g in gr])
    out.update(theta=thetas, eta_vals=np.array(vals), eta_grads=np.array(grads), back=back)
    th, eta = rcert.refine_eta_max(Volume(y), lam, psf, f.argmax_params, bounds)
    out.update(refine_theta=th.to_array(), refine_eta=np.array(eta))
    np.savez(OUT / "certificate.npz", **out)


def case_lasso(rng):
    """solvers.nonneg_lasso with and without w_init."""
    dims = (14, 14, 14)
    k = box_psf(dims, (1.5, 1.5, 1.5), (2, 2, 2))
    psf = Psf(Volume(k))
    truth = random_rows(rng, 4, dims)
    y = sfw3d.forward(measure_from_rows(truth), psf).data + 0.01 * rng.standard_normal(dims)
    thetas = [AtomParams(m=tuple(r[1:4] + 0.2), sigma=r[4], d=r[5]) for r in truth]
    thetas.append(AtomParams(m=tuple(truth[0, 1:4] + 0.25), sigma=truth[0, 4], d=truth[0, 5]))
    lam = 0.05
    w1 = sfw3d.nonneg_lasso(Volume(y), thetas, psf, lam, tol=1e-6, max_iter=2000)
    w0 = np.array([0.5, 0.0, 1.0, 0.2, 0.0])
    w2 = sfw3d.nonneg_lasso(Volume(y), thetas, psf, lam, w_init=w0, tol=1e-6, max_iter=2000)
    phis = np.stack([rsolv._phi_for(t, psf) for t in thetas])
    np.savez(OUT / "lasso.npz", y=y, kernel=psf.kernel.data, lam=np.array(lam),
             thetas=np.array([t.to_array() for t in thetas]), w=w1, w_init=w0, w_warm=w2,
             phis=phis)


def case_solve(rng):
    """Tiny end-to-end sfw / bsfw solves (solvers.py:286-405)."""
    dims = (24, 24, 24)
    k = box_psf(dims, (1.2, 1.2, 1.6), (2, 2, 3))
    psf = Psf(Volume(k))
    truth = np.array([[1.6, 8.3, 9.1, 12.4, 1.8, 2.1], [1.2, 15.2, 14.6, 10.3, 1.5, 1.8]])
    y = sfw3d.forward(measure_from_rows(truth), psf).data + 0.01 * rng.standard_normal(dims)
    bounds = DomainBounds(pos_lower=(5.0,) * 3, pos_upper=(18.0,) * 3, sigma_min=1.2,
                          sigma_max=2.4, shape_min=1.6, shape_max=2.4)
    opts = SolverOptions(lam=0.5, max_outer_iterations=10, n_sigma=3, n_shape=3)
    out = dict(y=y, kernel=psf.kernel.data, truth=truth,
               bounds=np.array([*bounds.pos_lower, *bounds.pos_upper, bounds.sigma_min,
                                bounds.sigma_max, bounds.shape_min, bounds.shape_max]),
               lam=np.array(opts.lam), max_outer=np.array(opts.max_outer_iterations),
               n_sigma=np.array(opts.n_sigma), n_shape=np.array(opts.n_shape))
    for name, solver in (("bsfw", sfw3d.bsfw), ("sfw", sfw3d.sfw)):
        res = solver(Volume(y), psf, opts, bounds)
        out[f"{name}_rows"] = rows_from_measure(res.measure)
        out[f"{name}_C"] = np.array(res.criterion)
        out[f"{name}_eta"] = np.array([r.eta_max for r in res.trace.records])
        out[f"{name}_atoms"] = np.array([r.atom_count for r in res.trace.records])
        out[f"{name}_term"] = np.array(res.termination)
    np.savez(OUT / "solve.npz", **out)


def case_config1(seed=2):
    """BASELINE config 1 end to end: 64^3 f64, N=5 atoms (m ~ U[8,56]^3,
    sigma ~ U[1.5,3], d ~ U[1.5,2.5], w ~ U[1,2]), PSF sigma_h=2 on 15^3, white
    noise at 20 dB power SNR, lam = 0.1 max Phi*y over the certificate grid
    sigma {1.5,2,2.5,3} x d {1.5,2,2.5} (injected by rebinding
    solvers.make_parameter_grids), BSFW with 20 outer
    iterations. The truth is drawn exactly as paper_2009_05473_b200.configs
    .config1(seed) draws it."""
    rng = np.random.default_rng(seed)
    dims = (64, 64, 64)
    m = rng.uniform(8.0, 56.0, size=(5, 3))
    truth = np.column_stack([rng.uniform(1, 2, 5), m, rng.uniform(1.5, 3, 5),
                             rng.uniform(1.5, 2.5, 5)])
    psf = Psf(Volume(box_psf(dims, (2, 2, 2), (7, 7, 7))))
    clean = sfw3d.forward(measure_from_rows(truth), psf).data
    noise = np.sqrt(np.mean(clean ** 2) / 10 ** (20 / 10))
    y = clean + noise * np.random.default_rng(seed + 1000).standard_normal(dims)
    bounds = DomainBounds(pos_lower=(8.0,) * 3, pos_upper=(56.0,) * 3, sigma_min=1.5,
                          sigma_max=3.0, shape_min=1.5, shape_max=2.5)
    sg, dg = np.array([1.5, 2.0, 2.5, 3.0]), np.array([1.5, 2.0, 2.5])
    table = rcert.build_template_table(psf, sg, dg, bounds=bounds)
    lam = 0.1 * rcert.eta_field(Volume(y), 1.0, table, bounds=bounds, keep_fields=False).eta_max
    orig = rsolv.make_parameter_grids
    rsolv.make_parameter_grids = lambda b, ns, nd: (sg, dg)
    try:
        res = sfw3d.bsfw(Volume(y), psf, SolverOptions(lam=lam, max_outer_iterations=20), bounds)
    finally:
        rsolv.make_parameter_grids = orig
    np.savez_compressed(OUT / "config1.npz", y=y, truth=truth, lam=np.array(lam),
                        noise=np.array(noise), rows=rows_from_measure(res.measure),
                        C=np.array(res.criterion), term=np.array(res.termination),
                        eta=np.array([r.eta_max for r in res.trace.records]),
                        atoms=np.array([r.atom_count for r in res.trace.records]),
                        t_total=np.array(res.trace.t_total))


def main():
    rng = np.random.default_rng(20090547)
    case_kats()
    case_convolution(rng)
    case_forward(rng)
    case_cost_grad(rng)
    case_certificate(rng)
    case_lasso(rng)
    case_solve(rng)
    if "--with-config1" in sys.argv:
        case_config1()
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
