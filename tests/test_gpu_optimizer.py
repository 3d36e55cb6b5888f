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
        np.testing.assert_allclose(a.eta_max, b.eta_max, rtol=1e-12)
        np.testing.assert_allclose(a.criterion_before, b.criterion_before, rtol=1e-12)
    np.testing.assert_allclose(rn.measure.to_rows(), rp.measure.to_rows(), rtol=1e-10, atol=1e-10)
    assert abs(rn.criterion - rp.criterion) <= 1e-12 * abs(rp.criterion)
    print(f"{algorithm} cfg1: library loop {rn.trace.t_total:.3f} s, host loop {rp.trace.t_total:.3f} s")
