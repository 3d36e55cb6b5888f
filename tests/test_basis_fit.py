"""CPU checks of the certificate's separable-basis fit (host-only C code):
exact for d = 2; for d < 2 within 1e-9 (the default basis_tol) on every
lattice value of the support box, with the reconstruction error it reports
matching an independent numpy evaluation."""
import numpy as np
import pytest

import sfw3d_oracle as O
from paper_2009_05473_b200 import _native as N


def lattice(lo, hi):
    sq = [np.arange(lo[a], hi[a] + 1) ** 2 for a in range(3)]
    return np.unique((sq[0][:, None, None] + sq[1][None, :, None] + sq[2][None, None, :]).ravel())


@pytest.mark.parametrize("sigma,d", [(1.0, 1.5), (1.5, 1.5), (2.0, 1.5), (3.0, 1.5), (2.5, 1.8),
                                     (1.2, 1.2), (3.0, 1.2), (1.0, 1.9), (3.0, 1.9), (1.7, 1.6)])
def test_fit_within_tolerance(sigma, d):
    R = O.support_radius(sigma, d)
    lo, hi = [-R] * 3, [R] * 3
    betas, w, w0, err = N.basis_fit(lo, hi, sigma, d)
    s = lattice(lo, hi).astype(float)
    g = np.exp(-0.5 * s ** (d / 2) / sigma ** d)
    approx = w0 * (s == 0) + np.exp(-np.outer(s, betas)) @ w
    assert np.all(w > 0) and w0 >= 0
    assert abs(np.max(np.abs(approx - g)) - err) <= 1e-13
    assert err <= 1e-9
    assert len(w) <= 40


def test_fit_exact_for_d2():
    betas, w, w0, err = N.basis_fit([-8, -8, -8], [8, 8, 8], 1.0, 2.0)
    assert err == 0.0 and w0 == 0.0 and list(w) == [1.0] and betas[0] == 0.5


def test_fit_full_axis_box():
    # asymmetric full-axis offsets (even n): [-n/2, n/2 - 1]
    betas, w, w0, err = N.basis_fit([-32, -32, -32], [31, 31, 31], 3.0, 1.5)
    assert err <= 1e-9


def test_fit_reports_failure_for_d_above_2():
    # not completely monotone in s: the non-negative basis cannot fit; the
    # table then keeps the direct evaluator for it
    R = O.support_radius(2.0, 2.5)
    _, _, _, err = N.basis_fit([-R] * 3, [R] * 3, 2.0, 2.5)
    assert err > 1e-3
