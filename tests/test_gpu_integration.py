"""The INTEGRATION.md binding, executed verbatim on the GPU against
reference-shaped objects: a stand-in `sfw3d` package whose modules bind their
functions by name (as sfw3d 0.1.0 does) and whose value types
have the reference's attributes only (Volume.data, Psf.kernel/.kernel_hat,
AtomParams.m/.sigma/.d, WeightedMeasure.atoms, DomainBounds, SolverOptions).
After enable(), the reference-side call sites (sfw3d.cli.bsfw, sfw3d.forward.
criterion_and_gradient, sfw3d.certificate.eta_field, sfw3d.forward.Psf as the
CLI constructs it, cli.py:79-102) run the B200 path and match the oracle /
the reference's own config-1 solve."""
import sys
import types
from dataclasses import dataclass

import numpy as np
import pytest

import sfw3d_oracle as O
from integration_snippet import load_snippet

pytestmark = pytest.mark.gpu


@dataclass(frozen=True, eq=False)
class RefVolume:
    data: np.ndarray

    @property
    def dims(self):
        return self.data.shape


class RefPsf:
    def __init__(self, kernel, normalize=True):
        data = kernel.data / kernel.data.sum() if normalize else kernel.data
        self.kernel = RefVolume(data)
        self.kernel_hat = O.psf_hat(data)

    @property
    def dims(self):
        return self.kernel.dims

    def is_centrosymmetric(self, tol=1e-10):
        return O.is_centrosymmetric(self.kernel.data, tol)


@dataclass(frozen=True)
class RefAtomParams:
    m: tuple
    sigma: float
    d: float


@dataclass(frozen=True)
class RefWeightedMeasure:
    atoms: tuple = ()

    def __len__(self):
        return len(self.atoms)


@dataclass(frozen=True)
class RefDomainBounds:
    pos_lower: tuple
    pos_upper: tuple
    sigma_min: float
    sigma_max: float
    shape_min: float
    shape_max: float


@dataclass(frozen=True)
class RefSolverOptions:
    lam: float
    max_outer_iterations: int = 50
    eta_threshold: float = 1.0
    eta_slack: float = 5e-3
    lasso_tol: float = 1e-6
    lasso_max_iter: int = 2000
    descent_gtol: float = 1e-6
    descent_ftol: float = 1e-10
    descent_max_iter: int = 400
    prune_rel_tol: float = 1e-10
    n_sigma: int = 8
    n_shape: int = 6
    duplicate_tol: float = 1e-6
    workers: int | None = None


def _unreached(*a, **k):
    raise AssertionError("the reference's CPU implementation was called after enable()")


@pytest.fixture()
def ref_pkg(monkeypatch):
    """Stand-in sfw3d modules, each binding the hot names (the CPU bodies must
    never run once the binding is enabled)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    hot = ("convolve", "correlate_adjoint", "render_atom", "forward", "criterion",
           "criterion_and_gradient", "criterion_gradient", "build_template_table",
           "eta_field", "refine_eta_max", "certificate_max", "nonneg_lasso", "local_descent",
           "sfw", "bsfw")
    layout = {"sfw3d": hot + ("Psf",), "sfw3d.forward": ("Psf",) + hot[:7],
              "sfw3d.certificate": ("build_template_table", "eta_field", "refine_eta_max",
                                    "certificate_max"),
              "sfw3d.solvers": ("Psf", "nonneg_lasso", "local_descent", "sfw", "bsfw",
                                "build_template_table", "certificate_max", "criterion_and_gradient"),
              "sfw3d.experiment": ("Psf", "forward", "sfw", "bsfw"),
              "sfw3d.cli": ("sfw", "bsfw")}
    mods = {}
    for name, attrs in layout.items():
        m = types.ModuleType(name)
        for a in attrs:
            setattr(m, a, RefPsf if a == "Psf" else _unreached)
        monkeypatch.setitem(sys.modules, name, m)
        mods[name] = m
    return mods


def test_snippet_rebinds_reference_call_sites(ref_pkg):
    ns = load_snippet()
    done = ns["enable"]("f64")
    import paper_2009_05473_b200 as gpu
    for modname, m in ref_pkg.items():
        for a in vars(m):
            if not a.startswith("__"):
                assert getattr(m, a) is getattr(gpu, a), (modname, a)
    assert ("sfw3d.cli", "bsfw") in done and ("sfw3d.forward", "Psf") in done


def test_snippet_cost_grad_and_certificate_on_reference_objects(ref_pkg):
    load_snippet()["enable"]("f64")
    fwd, cert = sys.modules["sfw3d.forward"], sys.modules["sfw3d.certificate"]
    rng = np.random.default_rng(8)
    dims = (24, 28, 20)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.2, 2.0), (3, 3, 4))
    psf_ref = RefPsf(RefVolume(kernel), normalize=False)   # a reference Psf object
    rows = np.column_stack([rng.uniform(0.5, 2, 5), rng.uniform(4, 18, (5, 3)),
                            rng.uniform(1, 2.5, 5), rng.uniform(1.5, 2.5, 5)])
    meas = RefWeightedMeasure(tuple((RefAtomParams(tuple(r[1:4]), r[4], r[5]), r[0]) for r in rows))
    y = rng.standard_normal(dims)
    c, g = fwd.criterion_and_gradient(RefVolume(y), meas, psf_ref, 0.2)
    c0, g0, _ = O.criterion_and_gradient(y, rows, O.psf_hat(kernel), 0.2)
    assert abs(c - c0) <= 1e-12 * abs(c0)
    assert np.max(np.abs(g.per_atom - g0)) <= 1e-11 * np.max(np.abs(g0))
    # the CLI's Psf(...) (cli.py:85-86) now constructs the B200 Psf from a reference Volume
    psf_cli = fwd.Psf(RefVolume(kernel))
    sg, dg = np.array([1.0, 1.8]), np.array([1.6, 2.0])
    table = cert.build_template_table(psf_cli, sg, dg)
    bounds = RefDomainBounds((3.0, 3.0, 3.0), (20.0, 24.0, 16.0), 1.0, 1.8, 1.6, 2.0)
    f = cert.eta_field(RefVolume(y), 0.5, table, bounds=bounds, keep_fields=False)
    hats = O.template_hats(O.psf_hat(kernel / kernel.sum()), dims, sg, dg)
    win = O.position_window(dims, bounds.pos_lower, bounds.pos_upper)
    pos, flat, val, _, _ = O.eta_field(y, 0.5, hats, len(dg), win)
    assert f.argmax_position == pos and abs(f.eta_max - val) <= 1e-10 * abs(val)


def test_snippet_cli_bsfw_config1(ref_pkg, golden):
    """cli.py:79-102 with the binding on: Psf(read_volume(psf)) then
    bsfw(y, psf, SolverOptions, DomainBounds) on reference objects returns the
    reference's own config-1 result (tests/golden/config1.npz)."""
    load_snippet()["enable"]("f64")
    g = golden("config1")
    dims = (64, 64, 64)
    cli, fwd = sys.modules["sfw3d.cli"], sys.modules["sfw3d.forward"]
    psf = fwd.Psf(RefVolume(O.box_gaussian_psf(dims, (2, 2, 2), (7, 7, 7))))
    bounds = RefDomainBounds((8.0,) * 3, (56.0,) * 3, 1.5, 3.0, 1.5, 2.5)
    from paper_2009_05473_b200 import solvers
    orig = solvers.make_parameter_grids
    solvers.make_parameter_grids = lambda b, ns, nd: (np.array([1.5, 2.0, 2.5, 3.0]),
                                                       np.array([1.5, 2.0, 2.5]))
    try:
        res = cli.bsfw(RefVolume(g["y"]), psf, RefSolverOptions(lam=float(g["lam"]),
                                                                max_outer_iterations=20), bounds)
    finally:
        solvers.make_parameter_grids = orig
    ref = g["rows"]
    rows = np.array([[w, *th.m, th.sigma, th.d] for th, w in res.measure.atoms])
    assert rows.shape == ref.shape and str(res.termination) == str(g["term"])
    for r in ref:
        j = int(np.argmin(np.linalg.norm(rows[:, 1:4] - r[1:4], axis=1)))
        assert np.linalg.norm(rows[j, 1:4] - r[1:4]) < 1e-3
        np.testing.assert_allclose(rows[j, [0, 4, 5]], r[[0, 4, 5]], rtol=1e-4)
