"""Run-to-run determinism of the CUDA path (row a9: the reference's
map_ordered contract, _parallel.py:12-22, "fixed-order reductions,
reproducible"). Every reduction on the path is a fixed-order tree (no float
atomics), so two evaluations of the same inputs must agree BIT FOR BIT:
the certificate (basis + signed members with exact refinement, fields),
criterion_and_gradient (fp64 and fp32 storage) and a whole BSFW solve."""
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


def _recs(recs):
    return [(tuple(r.pos), int(r.cand), float(r.value).hex()) for r in recs]


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_certificate_bitwise_repeatable(P, prec):
    import torch
    from paper_2009_05473_b200 import configs
    inst = configs.config4(seed=2, n=96)
    r = configs.cfg4_residual_host(inst, seed=9)
    psf = P.Psf(P.Volume(inst.kernel), normalize=False)
    with P.precision(prec):
        table = P.build_template_table(psf, inst.sigma_grid, inst.shape_grid, tap_tol=1e-12,
                                       prune=True)
        rd = torch.from_numpy(r.astype(np.float32 if prec == "f32" else np.float64)).cuda()
        full = tuple((0, n - 1) for n in inst.dims)
        runs = [P.certificate.eta_argmax_dev(rd, 0.8, table, full) for _ in range(3)]
        f = [P.eta_field(P.Volume(r.astype(np.float64)), 0.8, table, keep_fields=True)
             for _ in range(2)]
    for b, recs, _ in runs[1:]:
        assert _recs([b]) == _recs([runs[0][0]]) and _recs(recs) == _recs(runs[0][1])
    for a, b in zip(f[0].fields, f[1].fields):
        assert np.array_equal(a.data, b.data)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_cost_grad_bitwise_repeatable(P, prec):
    dims = (48, 40, 56)
    rng = np.random.default_rng(3)
    kernel = O.box_gaussian_psf(dims, (1.5, 1.5, 2.5), (4, 4, 8))
    rows = np.column_stack([rng.uniform(0.5, 2, 40), rng.uniform(0, 48, (40, 3)),
                            rng.uniform(1, 3, 40), rng.uniform(1.5, 2.5, 40)])
    y = O.conv(O.render(rows, dims), O.psf_hat(kernel)) + 0.01 * rng.standard_normal(dims)
    psf = P.Psf(P.Volume(kernel), normalize=False)
    meas = P.WeightedMeasure(tuple((P.AtomParams(m=tuple(r[1:4]), sigma=r[4], d=r[5]), r[0])
                                   for r in rows + 0.05))
    with P.precision(prec):
        out = [P.criterion_and_gradient(P.Volume(y), meas, psf, 0.1) for _ in range(3)]
    for c, g in out[1:]:
        assert float(c).hex() == float(out[0][0]).hex()
        assert np.array_equal(g.per_atom, out[0][1].per_atom)


def test_bsfw_bitwise_repeatable(P, golden):
    g = golden("config1")
    dims = (64, 64, 64)
    psf = P.Psf(P.Volume(O.box_gaussian_psf(dims, (2, 2, 2), (7, 7, 7))), normalize=False)
    bounds = P.DomainBounds((8.0,) * 3, (56.0,) * 3, 1.5, 3.0, 1.5, 2.5)
    from paper_2009_05473_b200 import solvers
    orig = solvers.make_parameter_grids
    solvers.make_parameter_grids = lambda b, ns, nd: (np.array([1.5, 2.0, 2.5, 3.0]),
                                                       np.array([1.5, 2.0, 2.5]))
    try:
        opts = P.SolverOptions(lam=float(g["lam"]), max_outer_iterations=20)
        res = [P.bsfw(P.Volume(g["y"]), psf, opts, bounds) for _ in range(2)]
    finally:
        solvers.make_parameter_grids = orig
    assert np.array_equal(res[0].measure.to_rows(), res[1].measure.to_rows())
    assert float(res[0].criterion).hex() == float(res[1].criterion).hex()
    assert [r.eta_max for r in res[0].trace.records] == [r.eta_max for r in res[1].trace.records]
