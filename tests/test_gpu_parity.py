"""GPU parity: the CUDA path through the C ABI against the reference's golden
vectors and the CPU oracle. Tolerances follow SURVEY §8(c):
  f64: C <= 1e-12 rel; gradient normwise per column <= 1e-11 of the column
       max; forward/phi <= 1e-12 of max; eta <= 1e-10 of eta_max (direct
       correlation in fp64);
  f32 storage (configs 3-5): eta <= 1e-5 of eta_max (north-star bar),
       C <= 1e-5 rel, gradient normwise per column <= 1e-4.
"""
import numpy as np
import pytest

import sfw3d_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2009_05473_b200 as pkg
    pkg.set_precision("f64")
    return pkg


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def colwise(g, ref):
    scale = np.maximum(np.max(np.abs(ref), axis=0), 1e-300)
    return float(np.max(np.max(np.abs(g - ref), axis=0) / scale))


def measure(P, rows):
    return P.WeightedMeasure(tuple((P.AtomParams(m=tuple(r[1:4]), sigma=r[4], d=r[5]), float(r[0]))
                                   for r in np.asarray(rows).reshape(-1, 6)))


# ---------------------------------------------------------------- K4
@pytest.mark.parametrize("name", ["cube", "odd"])
@pytest.mark.parametrize("kern", ["kernel", "rkernel"])
def test_psf_conv_corr_golden(P, golden, name, kern):
    g = golden("convolution")
    psf = P.Psf(P.Volume(g[f"{name}_{kern}"]), normalize=False)
    pre = "" if kern == "kernel" else "r"
    assert psf.separable() == (kern == "kernel")
    v = P.Volume(g[f"{name}_v"])
    assert rel(P.convolve(v, psf).data, g[f"{name}_{pre}conv"]) < 1e-12
    assert rel(P.correlate_adjoint(v, psf).data, g[f"{name}_{pre}corr"]) < 1e-12


def test_psf_delta_identity(P):
    rng = np.random.default_rng(3)
    v = P.Volume(rng.standard_normal((9, 10, 11)))
    psf = P.Psf.delta((9, 10, 11))
    np.testing.assert_array_equal(P.convolve(v, psf).data, v.data)
    np.testing.assert_array_equal(P.correlate_adjoint(v, psf).data, v.data)


# ---------------------------------------------------------------- K3
@pytest.mark.parametrize("name", ["interior", "edge", "fullaxis", "odd"])
def test_render_forward_golden(P, golden, name):
    g = golden("forward")
    rows = g[f"{name}_rows"]
    dims = g[f"{name}_acc"].shape
    from paper_2009_05473_b200.forward import render_dev
    acc = render_dev(rows, dims).cpu().numpy()
    assert rel(acc, g[f"{name}_acc"]) < 1e-14
    psf = P.Psf(P.Volume(g[f"{name}_kernel"]), normalize=False)
    assert rel(P.forward(measure(P, rows), psf).data, g[f"{name}_forward"]) < 1e-12


def test_render_kats(P, golden):
    g = golden("kat_render")
    v = P.render_atom(P.AtomParams(m=(4.0, 4.0, 4.0), sigma=1.0, d=2.0), 1.0, P.GridGeometry((9, 9, 9)))
    assert v.data[4, 4, 4] == 1.0
    assert v.data[5, 4, 4] == np.exp(-0.5)
    assert rel(v.data, g["unit_d2"]) < 1e-15  # CUDA exp vs numpy exp: ulp-level
    v2 = P.render_atom(P.AtomParams(m=(4.0, 4.0, 3.0), sigma=1.7, d=1.6), 2.0, P.GridGeometry((9, 9, 9)))
    assert rel(v2.data, g["w2"]) < 1e-15


# ---------------------------------------------------------------- K3-K6
@pytest.mark.parametrize("name", ["small", "edge", "fullaxis"])
def test_cost_grad_golden(P, golden, name):
    g = golden("cost_grad")
    psf = P.Psf(P.Volume(g[f"{name}_kernel"]), normalize=False)
    y = P.Volume(g[f"{name}_y"])
    lam = float(g[f"{name}_lam"])
    c, grad = P.criterion_and_gradient(y, measure(P, g[f"{name}_rows"]), psf, lam)
    assert abs(c - float(g[f"{name}_C"])) <= 1e-12 * abs(float(g[f"{name}_C"]))
    assert colwise(grad.per_atom, g[f"{name}_grad"]) < 1e-11
    c2 = P.criterion(y, measure(P, g[f"{name}_rows"]), psf, lam)
    assert abs(c2 - float(g[f"{name}_Conly"])) <= 1e-12 * abs(c2)


def test_cost_grad_kats(P):
    rng = np.random.default_rng(5)
    dims = (16, 16, 16)
    psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (1.5, 1.5, 2.0), (2, 2, 3))), normalize=False)
    y = P.Volume(rng.standard_normal(dims))
    # empty measure: C = 1/2 ||y||^2, no rows
    c, g = P.criterion_and_gradient(y, P.WeightedMeasure(()), psf, 0.3)
    assert abs(c - 0.5 * float(np.vdot(y.data, y.data))) <= 1e-13 * c
    assert g.per_atom.shape == (0, 6)
    # zero residual: dC/dw = lam, the rest 0
    rows = np.array([[1.3, 7.2, 8.1, 6.6, 1.7, 1.9]])
    yy = P.forward(measure(P, rows), psf)
    c, g = P.criterion_and_gradient(yy, measure(P, rows), psf, 0.25)
    assert abs(c - 0.25 * 1.3) < 1e-12
    assert abs(g.per_atom[0, 0] - 0.25) < 1e-12
    assert np.max(np.abs(g.per_atom[0, 1:])) < 1e-12
    with pytest.raises(ValueError):
        P.criterion_and_gradient(y, measure(P, rows), psf, 0.0)
    with pytest.raises(ValueError):
        P.criterion(P.Volume(np.zeros((8, 8, 8))), measure(P, rows), psf, 0.1)


def test_gradient_finite_differences(P):
    """every component vs central differences (h=1e-5)."""
    rng = np.random.default_rng(11)
    dims = (16, 16, 16)
    psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (1.3, 1.3, 1.8), (2, 2, 3))), normalize=False)
    y = P.Volume(rng.standard_normal(dims) * 0.1)
    rows = np.array([[1.2, 7.3, 8.6, 7.9, 1.6, 1.8], [0.8, 9.1, 6.2, 8.8, 2.1, 2.3]])
    lam = 0.2
    _, g = P.criterion_and_gradient(y, measure(P, rows), psf, lam)
    h = 1e-5
    num = np.zeros_like(rows)
    for i in range(rows.shape[0]):
        for c in range(6):
            rp, rm = rows.copy(), rows.copy()
            rp[i, c] += h
            rm[i, c] -= h
            num[i, c] = (P.criterion(y, measure(P, rp), psf, lam)
                         - P.criterion(y, measure(P, rm), psf, lam)) / (2 * h)
    assert np.max(np.abs(num - g.per_atom) / np.maximum(np.abs(num), 1e-3)) < 1e-4


def test_cost_grad_random_vs_oracle(P):
    rng = np.random.default_rng(21)
    dims = (20, 24, 18)
    kernel = O.box_gaussian_psf(dims, (1.4, 1.2, 2.2), (3, 2, 4))
    psf = P.Psf(P.Volume(kernel), normalize=False)
    rows = np.column_stack([rng.uniform(0.5, 2, 12), rng.uniform(0, 20, 12), rng.uniform(0, 24, 12),
                            rng.uniform(0, 18, 12), rng.uniform(0.8, 3, 12), rng.uniform(1.2, 2.8, 12)])
    y = rng.standard_normal(dims)
    c0, r0, _ = O.criterion_and_gradient(y, rows, O.psf_hat(kernel), 0.15)
    c, g = P.criterion_and_gradient(P.Volume(y), measure(P, rows), psf, 0.15)
    assert abs(c - c0) <= 1e-12 * abs(c0)
    assert colwise(g.per_atom, r0) < 1e-11


def test_cost_grad_f32(P):
    rng = np.random.default_rng(22)
    dims = (32, 32, 32)
    kernel = O.box_gaussian_psf(dims, (2.0, 2.0, 2.0), (7, 7, 7))
    psf = P.Psf(P.Volume(kernel), normalize=False)
    rows = np.column_stack([rng.uniform(0.5, 2, 30), rng.uniform(0, 32, (30, 3)),
                            rng.uniform(1, 3, 30), rng.uniform(1.5, 2.5, 30)])
    y = O.conv(O.render(rows, dims), O.psf_hat(kernel)).astype(np.float32).astype(np.float64)
    pert = rows.copy()
    pert[:, 1:] += 0.1 * rng.standard_normal((30, 5))
    pert[:, 0] = np.maximum(pert[:, 0], 0)
    c0, r0, _ = O.criterion_and_gradient(y, pert, O.psf_hat(kernel), 0.1)
    with P.precision("f32"):
        c, g = P.criterion_and_gradient(P.Volume(y), measure(P, pert), psf, 0.1)
    assert abs(c - c0) <= 1e-5 * abs(c0)     # measured 1.5e-6 on B200
    assert colwise(g.per_atom, r0) < 1e-4     # measured 1.5e-6 on B200


@pytest.mark.parametrize("dims", [(96, 80, 128), (48, 64, 96), (40, 40, 64)])
def test_cost_grad_f32_interval_kernels(P, dims):
    """The fp32 interval render / atom-sum kernels (boxes meeting every brick
    in one run per axis): atoms on the periodic seams, integer centres (u2 = 0
    voxels), d == 2 exactly, partial bricks; plus the forward render alone."""
    rng = np.random.default_rng(sum(dims))
    kernel = O.box_gaussian_psf(dims, (1.5, 1.5, 2.0), (4, 4, 6))
    psf = P.Psf(P.Volume(kernel), normalize=False)
    k = 60
    m = rng.uniform(0, 1, (k, 3)) * np.array(dims)
    m[:6] = [[0.2, 0.1, 0.3], [dims[0] - 0.4, 3.0, dims[2] - 0.2], [5.0, 7.0, 9.0],
             [dims[0] - 1.0, dims[1] - 1.0, 0.0], [12.5, 0.5, 31.5], [1.0, dims[1] / 2, 2.0]]
    rows = np.column_stack([rng.uniform(0.5, 2, k), m, rng.uniform(1, 2.2, k),
                            rng.uniform(1.9, 2.6, k)])
    rows[::7, 5] = 2.0
    y = (O.conv(O.render(rows, dims), O.psf_hat(kernel))
         + 0.01 * rng.standard_normal(dims)).astype(np.float32).astype(np.float64)
    pert = rows.copy()
    pert[6:, 1:4] += 0.1 * rng.standard_normal((k - 6, 3))  # rows 0-5 keep their centres
    pert[:, 1:4] %= np.array(dims)
    pert[2, 1:4] = [5.0, 7.0, 9.0]  # integer centre: a u2 = 0 voxel
    c0, r0, _ = O.criterion_and_gradient(y, pert, O.psf_hat(kernel), 0.1)
    with P.precision("f32"):
        c, g = P.criterion_and_gradient(P.Volume(y), measure(P, pert), psf, 0.1)
        fwd = P.forward(measure(P, pert), psf).data
    assert abs(c - c0) <= 1e-5 * abs(c0)
    assert colwise(g.per_atom, r0) < 1e-4
    ref = O.conv(O.render(pert, dims), O.psf_hat(kernel))
    assert np.max(np.abs(fwd - ref)) <= 2e-6 * np.max(np.abs(ref))


# ---------------------------------------------------------------- K1 / K7
def test_certificate_golden(P, golden):
    g = golden("certificate")
    psf = P.Psf(P.Volume(g["kernel"]), normalize=False)
    b = g["bounds"]
    bounds = P.DomainBounds(pos_lower=tuple(b[0:3]), pos_upper=tuple(b[3:6]), sigma_min=b[6],
                            sigma_max=b[7], shape_min=b[8], shape_max=b[9])
    table = P.build_template_table(psf, g["sigma_grid"], g["shape_grid"], bounds=bounds)
    y = P.Volume(g["y"])
    lam = float(g["lam"])
    f = P.eta_field(y, lam, table, bounds=bounds, keep_fields=True)
    assert f.argmax_position == tuple(g["argmax_position"])
    assert (f.argmax_sigma_index, f.argmax_shape_index) == (int(g["argmax_sigma_index"]),
                                                            int(g["argmax_shape_index"]))
    emax = float(g["eta_max"])
    assert abs(f.eta_max - emax) <= 1e-10 * abs(emax)
    assert np.max(np.abs(np.stack([v.data for v in f.fields]) - g["fields"])) <= 1e-10 * abs(emax)
    f2 = P.eta_field(y, 1.0, table, bounds=None, keep_fields=False)
    assert f2.fields is None
    assert f2.argmax_position == tuple(g["nb_argmax_position"])
    assert f2.argmax_sigma_index * len(g["shape_grid"]) + f2.argmax_shape_index == int(g["nb_argmax_flat"])
    # K7: eta value / gradient at fixed thetas (certificate.py:201-209)
    from paper_2009_05473_b200.forward import atom_sums_dev, to_dev
    back = to_dev(P.Volume(g["back"]))
    for th, v, gr in zip(g["theta"], g["eta_vals"], g["eta_grads"]):
        s = atom_sums_dev(back, np.array([[1.0, *th]]))[0]
        assert abs(s[0] / lam - v) <= 1e-12 * abs(v)
        assert np.max(np.abs(s[1:] / lam - gr)) <= 1e-11 * np.max(np.abs(gr))
    th, eta = P.refine_eta_max(y, lam, psf, f.argmax_params, bounds)
    assert abs(eta - float(g["refine_eta"])) <= 1e-9 * abs(eta)
    assert np.max(np.abs(th.to_array() - g["refine_theta"])) < 1e-4


@pytest.mark.parametrize("prec,tol", [("f64", 1e-10), ("f32", 1e-5)])
def test_eta_random_vs_oracle(P, prec, tol):
    rng = np.random.default_rng(31)
    dims = (24, 20, 28)
    kernel = O.box_gaussian_psf(dims, (1.2, 1.2, 2.0), (3, 3, 5))
    psf = P.Psf(P.Volume(kernel), normalize=False)
    sg, dg = np.array([1.0, 1.7, 2.5]), np.array([1.5, 2.0, 2.6])
    r = rng.standard_normal(dims)
    r += 5 * O.conv(O.render([[1.0, 11.3, 9.6, 14.2, 2.1, 1.7]], dims), O.psf_hat(kernel))
    if prec == "f32":
        r = r.astype(np.float32).astype(np.float64)
    hats = O.template_hats(O.psf_hat(kernel), dims, sg, dg)
    win = ((2, 21), (3, 17), (1, 26))
    pos, flat, val, per, fields = O.eta_field(r, 0.7, hats, 3, win, keep_fields=True)
    with P.precision(prec):
        table = P.build_template_table(psf, sg, dg)
        bounds = P.DomainBounds(pos_lower=(1.5, 2.2, 0.6), pos_upper=(21.0, 17.9, 26.4),
                                sigma_min=1.0, sigma_max=2.5, shape_min=1.5, shape_max=2.6)
        f = P.eta_field(P.Volume(r), 0.7, table, bounds=bounds, keep_fields=True)
    assert abs(f.eta_max - val) <= tol * abs(val)
    assert f.argmax_position == pos and f.argmax_sigma_index * 3 + f.argmax_shape_index == flat
    assert np.max(np.abs(np.stack([v.data for v in f.fields]) - np.stack(fields))) <= tol * abs(val)


def test_eta_edge_cases(P):
    dims = (12, 12, 12)
    psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (1, 1, 1), (2, 2, 2))), normalize=False)
    table = P.build_template_table(psf, [1.0, 2.0], [2.0])
    # zero residual -> eta == 0, argmax = first voxel of the window, first candidate
    f = P.eta_field(P.zero_volume(dims), 1.0, table, keep_fields=True)
    assert f.eta_max == 0.0 and f.argmax_position == (0, 0, 0)
    assert (f.argmax_sigma_index, f.argmax_shape_index) == (0, 0)
    # single-voxel window
    b = P.DomainBounds(pos_lower=(4.2, 5.0, 6.0), pos_upper=(5.9, 5.5, 6.9), sigma_min=0.5,
                       sigma_max=2.5, shape_min=1.0, shape_max=3.0)
    rng = np.random.default_rng(2)
    f = P.eta_field(P.Volume(rng.standard_normal(dims)), 1.0, table, bounds=b, keep_fields=False)
    assert f.argmax_position == (5, 5, 6)
    with pytest.raises(ValueError):
        P.eta_field(P.zero_volume(dims), 0.0, table)
    with pytest.raises(ValueError):
        P.eta_field(P.zero_volume((8, 8, 8)), 1.0, table)
    with pytest.raises(ValueError):
        P.build_template_table(psf, [], [2.0])


# ---------------------------------------------------------------- K8 / K9
def test_lasso_golden(P, golden):
    g = golden("lasso")
    psf = P.Psf(P.Volume(g["kernel"]), normalize=False)
    y = P.Volume(g["y"])
    thetas = [P.AtomParams.from_array(t) for t in g["thetas"]]
    from paper_2009_05473_b200.solvers import phi_dev
    phis = np.stack([phi_dev(t, psf).cpu().numpy() for t in thetas])
    assert rel(phis, g["phis"]) < 1e-12
    w = P.nonneg_lasso(y, thetas, psf, float(g["lam"]), tol=1e-6, max_iter=2000)
    np.testing.assert_allclose(w, g["w"], rtol=1e-8, atol=1e-12)
    w2 = P.nonneg_lasso(y, thetas, psf, float(g["lam"]), w_init=g["w_init"], tol=1e-6, max_iter=2000)
    np.testing.assert_allclose(w2, g["w_warm"], rtol=1e-8, atol=1e-12)
    # single atom closed form
    w1 = P.nonneg_lasso(y, thetas[:1], psf, float(g["lam"]), tol=1e-12, max_iter=10)
    phi = g["phis"][0]
    assert abs(w1[0] - max(0.0, (np.vdot(phi, g["y"]) - float(g["lam"])) / np.vdot(phi, phi))) < 1e-12


def test_cd_matches_oracle_sequence(P):
    """K9 alone: same Gram/b in -> same sweeps, stop reason and weights."""
    from paper_2009_05473_b200.solvers import cd_dev
    rng = np.random.default_rng(4)
    A = rng.standard_normal((40, 300))
    A[5] = A[4] + 1e-9 * rng.standard_normal(300)  # near-duplicate pair -> stall path
    gram = A @ A.T
    gram = 0.5 * (gram + gram.T)
    b = A @ rng.standard_normal(300)
    for tol, iters in ((1e-8, 5000), (1e-14, 3)):
        w0, s0, why0 = O.cd_solve(gram, b, 0.5, None, tol, iters)
        w, s, why, _ = cd_dev(gram, b, 0.5, np.zeros(40), tol, iters)
        assert (s, why) == (s0, why0)
        np.testing.assert_allclose(w, w0, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------- solves
@pytest.mark.parametrize("algo", ["bsfw", "sfw"])
def test_solve_golden(P, golden, algo):
    g = golden("solve")
    psf = P.Psf(P.Volume(g["kernel"]), normalize=False)
    b = g["bounds"]
    bounds = P.DomainBounds(pos_lower=tuple(b[0:3]), pos_upper=tuple(b[3:6]), sigma_min=b[6],
                            sigma_max=b[7], shape_min=b[8], shape_max=b[9])
    opts = P.SolverOptions(lam=float(g["lam"]), max_outer_iterations=int(g["max_outer"]),
                           n_sigma=int(g["n_sigma"]), n_shape=int(g["n_shape"]))
    res = getattr(P, algo)(P.Volume(g["y"]), psf, opts, bounds)
    ref_rows = g[f"{algo}_rows"]
    assert str(res.termination) == str(g[f"{algo}_term"])
    assert abs(res.criterion - float(g[f"{algo}_C"])) <= 1e-6 * abs(float(g[f"{algo}_C"]))
    etas = np.array([r.eta_max for r in res.trace.records])
    ref_eta = g[f"{algo}_eta"]
    assert len(etas) == len(ref_eta)
    np.testing.assert_allclose(etas, ref_eta, rtol=1e-5)
    assert len(res.measure) == ref_rows.shape[0]
    rows = res.measure.to_rows()
    assert np.max(np.abs(rows[:, 1:4] - ref_rows[:, 1:4])) < 1e-3
    np.testing.assert_allclose(rows[:, 0], ref_rows[:, 0], rtol=1e-4, atol=1e-8)
    assert P.audit_criterion_path(res.trace).ok


def test_qp_lasso_matches_converged_cd(P):
    """K9' (fp32-storage solves): the active-set QP reaches the LASSO optimum
    the reference's CD converges to — cold and warm starts, a sparse optimum
    (large lam), KKT residual within tol — and reports 'not applicable' for a
    near-singular free block (the caller then runs the CD)."""
    from paper_2009_05473_b200.solvers import cd_dev
    rng = np.random.default_rng(7)
    A = rng.standard_normal((60, 500))
    gram = A @ A.T
    gram = 0.5 * (gram + gram.T)
    b = A @ rng.standard_normal(500)
    for lam, w_init in ((0.5, np.zeros(60)), (0.5, np.abs(rng.standard_normal(60))),
                        (40.0, np.zeros(60))):
        w_ref, _, why = O.cd_solve(gram, b, lam, w_init.copy(), 1e-11, 200000)
        w, it, reason, kkt = cd_dev(gram, b, lam, w_init, 1e-9, 500, method="qp")
        assert reason == "kkt" and kkt <= 1e-9, (lam, reason, kkt)
        np.testing.assert_allclose(w, w_ref, rtol=1e-7, atol=1e-9)
        assert (w >= 0).all() and ((w > 0) == (w_ref > 0)).all()
    A[5] = A[4]  # exactly duplicated atom: singular free block -> not applicable
    gram = A @ A.T
    b = A @ rng.standard_normal(500)
    assert cd_dev(gram, b, 0.5, np.ones(60), 1e-9, 500, method="qp") is None
