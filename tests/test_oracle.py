"""Pin the CPU oracle to golden vectors produced by the real reference.

The fixtures come from tests/golden/make_golden.py (reference sfw3d 0.1.0).
These run without a GPU.
"""
import numpy as np
import pytest

import sfw3d_oracle as O


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_render_kats(golden):
    g = golden("kat_render")
    v = O.render([[1.0, 4.0, 4.0, 4.0, 1.0, 2.0]], (9, 9, 9))
    assert v[4, 4, 4] == 1.0
    assert v[5, 4, 4] == np.exp(-0.5)
    np.testing.assert_array_equal(v, g["unit_d2"])
    v2 = O.render([[2.0, 4.0, 4.0, 3.0, 1.7, 1.6]], (9, 9, 9))
    assert rel(v2, g["w2"]) < 1e-15


@pytest.mark.parametrize("name", ["cube", "odd"])
def test_convolution(golden, name):
    g = golden("convolution")
    for kk, cv, cr in (("kernel", "conv", "corr"), ("rkernel", "rconv", "rcorr")):
        kh = O.psf_hat(g[f"{name}_{kk}"])
        assert rel(O.conv(g[f"{name}_v"], kh), g[f"{name}_{cv}"]) < 1e-13
        assert rel(O.corr(g[f"{name}_v"], kh), g[f"{name}_{cr}"]) < 1e-13


@pytest.mark.parametrize("name", ["interior", "edge", "fullaxis", "odd"])
def test_forward(golden, name):
    g = golden("forward")
    rows = g[f"{name}_rows"]
    acc = O.render(rows, g[f"{name}_acc"].shape)
    np.testing.assert_array_equal(acc, g[f"{name}_acc"])
    fw = O.conv(acc, O.psf_hat(g[f"{name}_kernel"]))
    assert rel(fw, g[f"{name}_forward"]) < 1e-13


@pytest.mark.parametrize("name", ["small", "edge", "fullaxis"])
def test_cost_grad(golden, name):
    g = golden("cost_grad")
    kh = O.psf_hat(g[f"{name}_kernel"])
    c, rows, _ = O.criterion_and_gradient(g[f"{name}_y"], g[f"{name}_rows"], kh, float(g[f"{name}_lam"]))
    assert abs(c - float(g[f"{name}_C"])) <= 1e-13 * abs(float(g[f"{name}_C"]))
    np.testing.assert_allclose(rows, g[f"{name}_grad"], rtol=1e-11, atol=1e-12)
    c2 = O.criterion(g[f"{name}_y"], g[f"{name}_rows"], kh, float(g[f"{name}_lam"]))
    assert abs(c2 - float(g[f"{name}_Conly"])) <= 1e-13 * abs(c2)


def test_certificate(golden):
    g = golden("certificate")
    kh = O.psf_hat(g["kernel"])
    y = g["y"]
    hats = O.template_hats(kh, y.shape, g["sigma_grid"], g["shape_grid"])
    b = g["bounds"]
    win = O.position_window(y.shape, b[0:3], b[3:6])
    pos, flat, val, per, fields = O.eta_field(y, float(g["lam"]), hats, len(g["shape_grid"]), win, True)
    ns = len(g["shape_grid"])
    assert pos == tuple(g["argmax_position"])
    assert divmod(flat, ns) == (int(g["argmax_sigma_index"]), int(g["argmax_shape_index"]))
    assert abs(val - float(g["eta_max"])) <= 1e-13 * abs(val)
    assert rel(np.stack(fields), g["fields"]) < 1e-13
    pos2, flat2, val2, _, _ = O.eta_field(y, 1.0, hats, ns, None)
    assert pos2 == tuple(g["nb_argmax_position"]) and flat2 == int(g["nb_argmax_flat"])
    back = O.corr(y, kh)
    assert rel(back, g["back"]) < 1e-13
    for th, v, gr in zip(g["theta"], g["eta_vals"], g["eta_grads"]):
        vv, gg = O.eta_value_grad(back, th, float(g["lam"]))
        assert abs(vv - v) <= 1e-12 * abs(v)
        np.testing.assert_allclose(gg, gr, rtol=1e-10, atol=1e-12 * np.max(np.abs(gr)))


def test_lasso(golden):
    g = golden("lasso")
    kh = O.psf_hat(g["kernel"])
    y = g["y"]
    phis = np.stack([O.phi(th, kh, y.shape) for th in g["thetas"]])
    assert rel(phis, g["phis"]) < 1e-13
    gram, b = O.gram_system(phis, y)
    w, _, _ = O.cd_solve(gram, b, float(g["lam"]), None, 1e-6, 2000)
    np.testing.assert_allclose(w, g["w"], rtol=1e-9, atol=1e-12)
    w2, _, _ = O.cd_solve(gram, b, float(g["lam"]), g["w_init"], 1e-6, 2000)
    np.testing.assert_allclose(w2, g["w_warm"], rtol=1e-9, atol=1e-12)


def test_support_and_axis_box():
    # round-half-even box centres, full-axis min-image offsets
    assert O.support_radius(1.0, 2.0) == 8
    idx, off = O.axis_box(64, 10.5, 3)
    assert idx[0] == 7 and off[0] == -3.5      # rint(10.5) = 10
    idx, off = O.axis_box(64, 11.5, 3)
    assert idx[0] == 9                          # rint(11.5) = 12
    idx, off = O.axis_box(8, 0.25, 10)
    assert list(idx) == list(range(8))
    assert off.min() >= -4.0 and off.max() < 4.0


def test_oracle_bsfw_matches_reference_config1(golden):
    """The oracle's outer loop (solve, solvers.py:286-405) reproduces the
    reference's own config-1 BSFW solve (tests/golden/config1.npz): same
    termination, atom count and criterion; atoms within 1e-6 voxel and 1e-6
    relative (measured ~1e-9)."""
    g = golden("config1")
    dims = (64, 64, 64)
    k = O.box_gaussian_psf(dims, (2, 2, 2), (7, 7, 7))
    box5 = [(8.0, 56.0)] * 3 + [(1.5, 3.0), (1.5, 2.5)]
    r = O.solve(g["y"], O.psf_hat(k), float(g["lam"]), [1.5, 2, 2.5, 3], [1.5, 2, 2.5], box5,
                "bsfw", max_outer_iterations=20)
    ref = g["rows"]
    assert r["termination"] == str(g["term"]) and r["rows"].shape == ref.shape
    assert abs(r["criterion"] - float(g["C"])) <= 1e-9 * abs(float(g["C"]))
    np.testing.assert_allclose(r["eta"], g["eta"], rtol=1e-6)
    for q in ref:
        j = int(np.argmin(np.linalg.norm(r["rows"][:, 1:4] - q[1:4], axis=1)))
        assert np.linalg.norm(r["rows"][j, 1:4] - q[1:4]) < 1e-6
        np.testing.assert_allclose(r["rows"][j, [0, 4, 5]], q[[0, 4, 5]], rtol=1e-6)
