"""The in-library L-BFGS-B drivers (sfw3d_refine_eta_max, sfw3d_local_descent;
SURVEY §8(f)1) against the reference's scipy loop over the same device
evaluations (N.OPTIMIZER = "scipy"), on BASELINE config 1: the certificate
ascent from the grid seed, the joint slide, and the whole BSFW solve."""
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


@pytest.fixture(scope="module")
def case(P, golden):
    g = golden("config1")
    dims = (64, 64, 64)
    psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (2, 2, 2), (7, 7, 7))), normalize=False)
    bounds = P.DomainBounds(pos_lower=(8.0,) * 3, pos_upper=(56.0,) * 3, sigma_min=1.5,
                            sigma_max=3.0, shape_min=1.5, shape_max=2.5)
    return {"y": g["y"], "lam": float(g["lam"]), "psf": psf, "bounds": bounds, "rows": g["rows"],
            "grids": (np.array([1.5, 2.0, 2.5, 3.0]), np.array([1.5, 2.0, 2.5]))}


def with_optimizer(name, fn):
    from paper_2009_05473_b200 import _native as N
    old, N.OPTIMIZER = N.OPTIMIZER, name
    try:
        return fn()
    finally:
        N.OPTIMIZER = old


def test_refine_native_equals_scipy(P, case):
    from paper_2009_05473_b200.certificate import certificate_max_dev
    from paper_2009_05473_b200.forward import to_dev
    table = P.build_template_table(case["psf"], *case["grids"])
    y = to_dev(P.Volume(case["y"]))
    info = {}
    th_n, eta_n = with_optimizer("native", lambda: certificate_max_dev(
        y, case["lam"], table, case["psf"], case["bounds"], info))
    th_s, eta_s = with_optimizer("scipy", lambda: certificate_max_dev(
        y, case["lam"], table, case["psf"], case["bounds"]))
    assert eta_n >= info["eta_grid"]  # the ascent starts from the grid argmax
    np.testing.assert_allclose(th_n.to_array(), th_s.to_array(), rtol=0, atol=1e-8)
    assert abs(eta_n - eta_s) <= 1e-12 * abs(eta_s)


def test_refine_seed_kept_and_errors(P, case):
    """certificate.py:195-196 (ValueError) and :221-222 (seed kept when not improved)."""
    from paper_2009_05473_b200.forward import to_dev
    y = P.Volume(case["y"])
    start = P.AtomParams(m=(30.0, 30.0, 30.0), sigma=2.0, d=2.0)
    with pytest.raises(ValueError):
        P.refine_eta_max(y, 0.0, case["psf"], start, case["bounds"])
    th, eta = P.refine_eta_max(y, case["lam"], case["psf"], start, case["bounds"], max_iter=0)
    th2, eta2 = with_optimizer("scipy", lambda: P.refine_eta_max(
        y, case["lam"], case["psf"], start, case["bounds"], max_iter=0))
    np.testing.assert_allclose(th.to_array(), th2.to_array(), atol=1e-12)
    assert abs(eta - eta2) <= 1e-12 * abs(eta2)


def test_descent_native_equals_scipy(P, case):
    from paper_2009_05473_b200 import solvers
    from paper_2009_05473_b200.forward import to_dev
    rng = np.random.default_rng(3)
    rows = case["rows"].copy()
    rows[:, 0] *= 1 + 0.05 * rng.standard_normal(len(rows))
    rows[:, 1:4] += 0.2 * rng.standard_normal((len(rows), 3))
    rows[:, 4:] = np.clip(rows[:, 4:] + 0.05 * rng.standard_normal((len(rows), 2)), 1.5, 2.5)
    start = P.WeightedMeasure(tuple((P.AtomParams(m=tuple(r[1:4]), sigma=r[4], d=r[5]), r[0])
                                    for r in rows))
    y = to_dev(P.Volume(case["y"]))
    run = lambda: solvers.local_descent_dev(y, start, case["psf"], case["lam"], case["bounds"])
    m_n, c_n, w_n = with_optimizer("native", run)
    m_s, c_s, w_s = with_optimizer("scipy", run)
    assert w_n == w_s
    assert abs(c_n - c_s) <= 1e-10 * abs(c_s)
    a, b = m_n.to_rows(), m_s.to_rows()
    np.testing.assert_allclose(a[:, 1:4], b[:, 1:4], rtol=0, atol=1e-5)
    np.testing.assert_allclose(a[:, [0, 4, 5]], b[:, [0, 4, 5]], rtol=1e-5)
    assert c_n < solvers.cost_grad_dev(case["psf"], y, rows, case["lam"], want_grad=False)[0]


def test_bsfw_native_equals_scipy(P, case):
    from paper_2009_05473_b200 import solvers
    orig = solvers.make_parameter_grids
    solvers.make_parameter_grids = lambda b, ns, nd: case["grids"]
    try:
        run = lambda: P.bsfw(P.Volume(case["y"]), case["psf"],
                             P.SolverOptions(lam=case["lam"], max_outer_iterations=20), case["bounds"])
        rn = with_optimizer("native", run)
        rs = with_optimizer("scipy", run)
    finally:
        solvers.make_parameter_grids = orig
    assert rn.termination == rs.termination
    assert [r.atom_count for r in rn.trace.records] == [r.atom_count for r in rs.trace.records]
    a, b = rn.measure.to_rows(), rs.measure.to_rows()
    assert a.shape == b.shape
    np.testing.assert_allclose(a[:, 1:4], b[:, 1:4], rtol=0, atol=1e-4)
    np.testing.assert_allclose(a[:, [0, 4, 5]], b[:, [0, 4, 5]], rtol=1e-5)
    assert abs(rn.criterion - rs.criterion) <= 1e-9 * abs(rs.criterion)
    print(f"bsfw cfg1: native {rn.trace.t_total:.3f} s, scipy loop {rs.trace.t_total:.3f} s")


@pytest.mark.parametrize("algorithm", ["bsfw", "sfw"])
def test_native_loop_equals_python_loop(P, case, algorithm):
    """sfw3d_solve (the outer loop inside the library) against
    the host loop of solvers._solve over the same device calls."""
    from paper_2009_05473_b200 import _native as N, solvers
    orig = solvers.make_parameter_grids
    solvers.make_parameter_grids = lambda b, ns, nd: case["grids"]
    try:
        def run(mode):
            old, N.SOLVER = N.SOLVER, mode
            try:
                return getattr(P, algorithm)(
                    P.Volume(case["y"]), case["psf"],
                    P.SolverOptions(lam=case["lam"], max_outer_iterations=20), case["bounds"])
            finally:
                N.SOLVER = old
        rn, rp = run("native"), run("python")
    finally:
        solvers.make_parameter_grids = orig
    assert rn.termination == rp.termination
    assert len(rn.trace.records) == len(rp.trace.records)
    for a, b in zip(rn.trace.records, rp.trace.records):
        assert a.index == b.index and a.atom_count == b.atom_count
        assert (a.criterion_after_lasso is None) == (b.criterion_after_lasso is None)
        assert (a.criterion_after_descent is None) == (b.criterion_after_descent is None)
        # (the library loop sums the Gram rows over each phi's x support only:
        # same inner products, another rounding order, amplified by the slides)
        np.testing.assert_allclose(a.eta_max, b.eta_max, rtol=1e-8)
        np.testing.assert_allclose(a.criterion_before, b.criterion_before, rtol=1e-10)
    np.testing.assert_allclose(rn.measure.to_rows(), rp.measure.to_rows(), rtol=1e-6, atol=1e-6)
    assert abs(rn.criterion - rp.criterion) <= 1e-10 * abs(rp.criterion)
    print(f"{algorithm} cfg1: library loop {rn.trace.t_total:.3f} s, host loop {rp.trace.t_total:.3f} s")


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_residual_with_supports_is_bit_identical(P, case, prec):
    """sfw3d_residual_ranged skips atoms on x planes where their phi is exactly
    zero: same volume and sum of squares as sfw3d_residual, bit for bit."""
    import ctypes as C
    import torch
    from paper_2009_05473_b200 import _native as N, solvers
    from paper_2009_05473_b200.forward import code_of, to_dev
    P.set_precision(prec)
    try:
        code = N.dtype_code()
        y = to_dev(P.Volume(case["y"]), code)
        thetas = [P.AtomParams(m=(30.2, 20.1, 40.7), sigma=2.0, d=2.0),
                  P.AtomParams(m=(8.0, 50.0, 12.0), sigma=3.0, d=1.5),     # wraps through x = 0
                  P.AtomParams(m=(55.5, 33.0, 30.0), sigma=2.5, d=2.5),    # wraps through x = n - 1
                  P.AtomParams(m=(40.0, 40.0, 40.0), sigma=1.5, d=1.8)]
        phis = [solvers.phi_dev(t, case["psf"], code) for t in thetas]
        w = np.array([1.3, 0.7, 2.1, 0.4])
        nx = y.shape[0]
        xr = np.zeros((len(phis), 2), dtype=np.int32)
        for i, p in enumerate(phis):
            on = torch.any(p.reshape(nx, -1) != 0, dim=1).cpu().numpy()
            idx = np.flatnonzero(on)
            if on.all():
                xr[i] = (0, nx - 1)
            elif on[0] and on[-1]:  # wrapped support: the gap is in the middle
                gap = np.flatnonzero(~on)
                xr[i] = (gap[-1] + 1, gap[0] - 1)
            else:
                xr[i] = (idx[0], idx[-1])
        assert (xr[:, 0] > xr[:, 1]).any() and (xr[:, 0] <= xr[:, 1]).any()
        ref, ss_ref = solvers.residual_dev(y, w, phis)
        out = torch.empty_like(y)
        ss = C.c_double()
        arr = (C.c_void_p * len(phis))(*[t.data_ptr() for t in phis])
        N.check(N.lib().sfw3d_residual_ranged(N.context(0).handle, code_of(y), N.dims_arg(y.shape),
                                              N.ptr(y), arr, N.f64_ptr(w),
                                              xr.ctypes.data_as(C.POINTER(C.c_int32)), len(phis),
                                              N.ptr(out), C.byref(ss)))
        assert torch.equal(out, ref)
        assert ss.value == ss_ref
    finally:
        P.set_precision("f64")


def test_multistart_refine_at_least_the_single_start(P, case):
    """Batched multi-start ascent: concurrent in-library L-BFGS-B runs (one
    stream / context per start) against one back-projection; the first start
    is the reference's grid argmax, so the result can only be >= its ascent."""
    from paper_2009_05473_b200.certificate import (certificate_max_dev,
                                                   certificate_max_multistart_dev)
    from paper_2009_05473_b200.forward import to_dev
    table = P.build_template_table(case["psf"], *case["grids"])
    y = to_dev(P.Volume(case["y"]))
    th1, eta1 = certificate_max_dev(y, case["lam"], table, case["psf"], case["bounds"])
    thm, etam = certificate_max_multistart_dev(y, case["lam"], table, case["psf"], case["bounds"], 6)
    assert etam >= eta1 * (1 - 1e-12)
    th_one, eta_one = certificate_max_multistart_dev(y, case["lam"], table, case["psf"],
                                                     case["bounds"], 1)
    np.testing.assert_allclose(th_one.to_array(), th1.to_array(), rtol=0, atol=1e-12)
    assert eta_one == eta1
