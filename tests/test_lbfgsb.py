"""The in-library L-BFGS-B (csrc/lbfgsb.cuh, sfw3d_lbfgsb_minimize) against
scipy.optimize.minimize(method="L-BFGS-B") — the optimiser the reference calls
at certificate.py:217-218 and solvers.py:231-232. Host-only (no GPU): every
EVALUATED point of the two runs is compared, i.e. the Cauchy points, subspace
steps, line-search trial steps and stopping decisions all follow scipy's."""

import numpy as np
import pytest
from scipy.optimize import minimize

from paper_2009_05473_b200 import optimize as O


def rosen(x):
    f = np.sum(100 * (x[1:] - x[:-1] ** 2) ** 2 + (1 - x[:-1]) ** 2)
    g = np.zeros_like(x)
    g[:-1] = -400 * x[:-1] * (x[1:] - x[:-1] ** 2) - 2 * (1 - x[:-1])
    g[1:] += 200 * (x[1:] - x[:-1] ** 2)
    return f, g


def quadratic(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    a = a @ a.T + 0.1 * np.eye(n)
    b = 3 * rng.standard_normal(n)
    return lambda x: (0.5 * x @ a @ x - b @ x, a @ x - b)


def gaussian_bump(x):
    """a 5-variable smooth ascent shaped like neg_eta (certificate.py:201-209)"""
    c = np.array([3.2, 4.1, 2.7, 2.2, 1.9])
    s = np.array([1.0, 1.5, 0.8, 0.6, 0.9])
    q = ((x - c) / s) ** 2
    f = -np.exp(-0.5 * q.sum())
    return f, -f * (x - c) / s ** 2


CASES = [
    ("rosen5_box", rosen, [-1.2, 1, -1.2, 1, 0.5], [(-5, 5)] * 5, {}),
    ("rosen5_tight", rosen, [-1.2, 1, -1.2, 1, 0.5],
     [(-1.5, 0.8), (-1, 2), (0.2, 0.9), (-3, 3), (0, 0.5)], {}),
    ("rosen10_lower", rosen, np.linspace(-1, 1, 10), [(0.3, None)] * 10, {}),
    ("rosen8_free", rosen, np.linspace(-1, 1, 8), [(None, None)] * 8, {}),
    ("rosen8_mixed", rosen, np.linspace(-1, 1, 8),
     [(None, None), (0, None), (None, 0.5), (-1, 1)] * 2, {}),
    ("quad30_box", quadratic(30, 0), np.zeros(30), [(-0.5, 0.5)] * 30, {"gtol": 1e-8}),
    ("quad30_lower", quadratic(30, 1), np.ones(30), [(0, None)] * 30,
     {"gtol": 1e-8, "ftol": 1e-12}),
    ("quad60_w_rows", quadratic(60, 2), np.full(60, 0.2),
     [(0.0, None), (-1, 1), (-1, 1), (-1, 1), (0.1, 3), (0.1, 3)] * 10,
     {"gtol": 1e-6, "ftol": 1e-10, "maxiter": 400}),
    ("bump_refine", gaussian_bump, [3.0, 4.0, 3.0, 2.0, 2.0],
     [(0, 7), (0, 7), (0, 7), (1.5, 3.0), (1.5, 2.5)], {"gtol": 1e-8, "maxiter": 200}),
    ("maxiter_cap", rosen, np.linspace(-1, 1, 8), [(-2, 2)] * 8, {"maxiter": 7}),
]


@pytest.mark.parametrize("name,fun,x0,bounds,kw", CASES, ids=[c[0] for c in CASES])
def test_same_evaluations_as_scipy(name, fun, x0, bounds, kw):
    kw = {"gtol": 1e-5, "ftol": 2.220446049250313e-09, "maxiter": 15000, **kw}
    ours, theirs = [], []

    def f_ours(x):
        ours.append(np.array(x))
        return fun(x)

    def f_theirs(x):
        theirs.append(np.array(x))
        return fun(x)

    got = O.minimize(f_ours, x0, bounds, **kw)
    ref = minimize(f_theirs, np.array(x0, dtype=float), jac=True, method="L-BFGS-B",
                   bounds=bounds, options=kw)
    assert got.nit == ref.nit and got.nfev == ref.nfev == len(ours) == len(theirs)
    assert got.success == ref.success
    for a, b in zip(ours, theirs):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-8 * (1 + np.max(np.abs(b))))
    np.testing.assert_allclose(got.x, ref.x, rtol=0, atol=1e-10 * (1 + np.max(np.abs(ref.x))))
    assert abs(got.fun - ref.fun) <= 1e-12 * max(1.0, abs(ref.fun))


def test_start_projected_and_converged_at_start():
    got = O.minimize(lambda x: (float(x @ x), 2 * x), [5.0, -5.0], [(1, 2), (-2, -1)])
    np.testing.assert_array_equal(got.x, [1.0, -1.0])
    assert got.success and got.nit <= 1


def test_objective_exception_propagates():
    def bad(x):
        raise FloatingPointError("non-finite certificate value")
    with pytest.raises(FloatingPointError):
        O.minimize(bad, [0.0, 0.0], [(-1, 1)] * 2)


def test_invalid_arguments_raise_value_error():
    f = lambda x: (float(x @ x), 2 * x)
    with pytest.raises(ValueError):
        O.minimize(f, [0.0, 0.0], [(1.0, -1.0), (0.0, 1.0)])  # lower bound above upper
    with pytest.raises(ValueError):
        O.minimize(f, [0.0], [(0.0, 1.0)], gtol=-1.0)
